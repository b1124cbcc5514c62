# forward DFT: twiddle fragments in registers per pass (default) vs from L1 (nort)
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
for c in 2 4 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_rt.json 2>>gpurun_out/ab.err
  KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_nort.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_nort.json 2>>gpurun_out/ab.err
done
