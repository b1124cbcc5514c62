# Round-2 pass with the sparse-chunk product (k_m2l_sparse): M2L variant agreement and
# parity first, then the default (C5) bench, the launch list of the bench command, ncu
# summaries of the C5 product and GEMM kernels, and the full GPU suite last.
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo smoke=$?; tail -4 gpurun_out/b_smoke.log
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -q -x -k "modes or parity" > gpurun_out/b_pytest_modes.log 2>&1; echo pytest_modes=$?; tail -3 gpurun_out/b_pytest_modes.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/b_bench_c5.json 2> gpurun_out/b_bench_c5.err; echo bench=$?
for c in 3 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_c$c.json 2>> gpurun_out/b_bench_other.err; echo bench_c$c=$?
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/launch_summary.py gpurun_out/b_launches_c5.csv > gpurun_out/b_launches_c5_summary.txt 2>&1
python scripts/launch_summary.py gpurun_out/b_launches_c5.csv --last-eval > gpurun_out/b_launches_c5_lasteval.txt 2>&1
gzip -f gpurun_out/b_launches_c5.csv
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_ -c 18 -o /tmp/b_prod \
  python scripts/profile_eval.py 5 1 > gpurun_out/b_ncu_prod.log 2>&1; echo ncu_prod=$?
python scripts/ncu_summary.py /tmp/b_prod.ncu-rep > gpurun_out/b_c5_prod_ncu.txt 2>&1
ncu -i /tmp/b_prod.ncu-rep --page details --print-units base -c 1 > gpurun_out/b_c5_prod_details.txt 2>&1
timeout 1200 ncu -f --set full --clock-control none -k regex:k_gemm_dmma -c 14 -o /tmp/b_gemm \
  python scripts/profile_eval.py 5 1 > gpurun_out/b_ncu_gemm.log 2>&1; echo ncu_gemm=$?
python scripts/ncu_summary.py /tmp/b_gemm.ncu-rep > gpurun_out/b_c5_gemm_ncu.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/b_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/b_pytest.log
du -sh gpurun_out
