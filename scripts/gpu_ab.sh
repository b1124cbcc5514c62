timeout 1200 python -m pytest tests/test_gpu_m2l_modes.py -q > gpurun_out/modes.log 2>&1; echo pytest=$?; tail -3 gpurun_out/modes.log
