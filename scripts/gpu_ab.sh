# DFT passes: 2 m-tiles per warp iteration (default) vs 1 (variant library)
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_mt2.json 2>>gpurun_out/ab.err
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_mt1.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_mt1.json 2>>gpurun_out/ab.err
done
