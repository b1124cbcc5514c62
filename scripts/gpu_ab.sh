# DFT passes: m-tiles per warp iteration 2 (default) vs 3, 4 (variant libraries)
for c in 2 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_mt2.json 2>>gpurun_out/ab.err
  for v in mt3 mt4; do
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_$v.json 2>>gpurun_out/ab.err
  done
done
