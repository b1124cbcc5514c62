# per-pair product: 8 frequencies per target + conjugate-symmetric half table (default), 4 frequencies, 512 threads
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_fb8.json 2>>gpurun_out/ab.err
for v in fb4 fb8t512; do
KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_$v.json 2>>gpurun_out/ab.err
done
