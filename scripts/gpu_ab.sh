# sparse-chunk product: 16-B pair-list batches
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5.json 2>>gpurun_out/ab.err
