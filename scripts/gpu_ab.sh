# product CTA shape: warps per CTA x parent n-tiles per warp
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/ab_c2_base.json 2>>gpurun_out/ab.err
for v in w8nt2 w8nt4 w2nt4; do
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/ab_c2_$v.json 2>>gpurun_out/ab.err
done
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c3_base.json 2>>gpurun_out/ab.err
for v in w8nt2 w2nt4; do
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c3_$v.json 2>>gpurun_out/ab.err
done
