# forward transforms per CTA: default 2 everywhere; C5 (p = 8) with 4; parity at p = 12
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 3 > gpurun_out/ab_c4.json 2>>gpurun_out/ab.err
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_nb2.json 2>>gpurun_out/ab.err
KAFMM_FWD_NB=4 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_nb4.json 2>>gpurun_out/ab.err
