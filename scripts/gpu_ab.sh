# LapPGradGrad pair kernel in fused form (new) vs term by term (prev)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wall.py tests/test_gpu_edge.py -x -q -k "pgradgrad or C8 or wall or single or leaves" > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
timeout 600 python bench.py --config 8 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c8_new.json 2>>gpurun_out/ab.err
KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_prev.so timeout 600 python bench.py --config 8 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c8_prev.json 2>>gpurun_out/ab.err
