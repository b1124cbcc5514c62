# Round-2 re-entry pass: smoke, M2L variant agreement + small parity (stop on failure),
# the default (C5) bench line, C2..C4 lines, and the launch list of the C5 bench command.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c_smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo smoke=$?; tail -4 gpurun_out/c_smoke.log
timeout 1200 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -q -x > gpurun_out/c_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -15 gpurun_out/c_pytest_modes.log
[ $rc -ne 0 ] && exit 1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/c_bench_c5.json 2> gpurun_out/c_bench_c5.err; echo bench=$?; cat gpurun_out/c_bench_c5.json; tail -5 gpurun_out/c_bench_c5.err
for c in 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c_bench_c$c.json 2>> gpurun_out/c_bench_other.err; echo bench_c$c=$?
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c_ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/launch_summary.py gpurun_out/c_launches_c5.csv --last-eval > gpurun_out/c_launches_c5_lasteval.txt 2>&1
gzip -f gpurun_out/c_launches_c5.csv
cat gpurun_out/c_launches_c5_lasteval.txt | head -40
