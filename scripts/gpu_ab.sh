# pair kernel: 512 (default) vs 1024 threads per CTA
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_t512.json 2>>gpurun_out/ab.err
KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_t1024.so timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_t1024.json 2>>gpurun_out/ab.err
