# StokesRegVelOmega functors in fused form (new) vs previous
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -x -q -k "omega or C7 or single or leaves or separate" > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 7 --no-cpu-baseline --steps 3 > gpurun_out/ab_c7_new.json 2>>gpurun_out/ab.err
KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_prev.so timeout 600 python bench.py --config 7 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c7_prev.json 2>>gpurun_out/ab.err
