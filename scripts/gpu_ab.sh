# LapQPGradGrad pair functor in fused form
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wall.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -x -q -k "qp or C9 or wall or single or leaves" > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 9 --no-cpu-baseline --steps 3 > gpurun_out/ab_c9_new.json 2>>gpurun_out/ab.err
