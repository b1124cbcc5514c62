# FFT transform rework: tests, then C2 / C3 / C5 with forward transforms-per-CTA 1, 2, 4
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
for nb in 1 2 4; do
  KAFMM_FWD_NB=$nb timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/ab_c2_nb$nb.json 2>>gpurun_out/ab.err
done
KAFMM_FWD_NB=2 timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c3_nb2.json 2>>gpurun_out/ab.err
KAFMM_FWD_NB=2 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ab_c5_nb2.json 2>>gpurun_out/ab.err
