# Round-end measurement recipe (run under gpurun from the repo root):
# full GPU tests, the default bench line, the per-launch list of one C2 evaluation,
# and a full ncu capture of the C2 M2L kernels (each ncu pass after its command ran plain).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/fin_pytest.log
timeout 900 python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err; echo bench=$?
timeout 300 python scripts/profile_eval.py 2 2 > gpurun_out/fin_prof.log 2>&1; echo prof=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c2.csv \
  python scripts/profile_eval.py 2 2 > gpurun_out/fin_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_m2l_dmma|k_fft_fwd|k_fft_inv|k_p2p|k_leaf_far' \
  -s 12 -c 10 -o gpurun_out/fin_c2 python scripts/profile_eval.py 2 2 > gpurun_out/fin_ncu_full.log 2>&1; echo ncu_full=$?
