# single-matrix check->equivalent operators: tests, then C2 / C3 / C5 composed vs two-factor
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_one.json 2>>gpurun_out/ab.err
  KAFMM_C2E_FACTORS=2 timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c${c}_two.json 2>>gpurun_out/ab.err
done
