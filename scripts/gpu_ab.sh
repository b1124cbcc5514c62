# forward DFT: densities + lattice map staged in SMEM (new) vs read through L1 (prev)
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_edge.py -x -q -k "modes or orders or single" > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_new.json 2>>gpurun_out/ab.err
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_prev.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_prev.json 2>>gpurun_out/ab.err
done
