# sparse-chunk product with 4 frequencies per target
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5.json 2>>gpurun_out/ab.err
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c4.json 2>>gpurun_out/ab.err
