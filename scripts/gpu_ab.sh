# b^2 / eps^2 formed once per source in the gather (new) vs per pair (prev)
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wall.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
for c in 6 4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/ab_c${c}_new.json 2>>gpurun_out/ab.err
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_prev.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_prev.json 2>>gpurun_out/ab.err
done
