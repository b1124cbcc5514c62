# Round-end measurement recipe (run under gpurun from the repo root):
# smoke, full GPU tests, the default bench line, bench lines of the other configs,
# the per-launch list of one C2 evaluation, and ncu captures of the C2 level-5 M2L
# kernels (each ncu pass after its command ran plain; reports summarised on the box).
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/fin_pytest.log
timeout 900 python bench.py > gpurun_out/fin_bench_c2.json 2> gpurun_out/fin_bench_c2.err; echo bench=$?
for c in 3 4 5 6 7 8 9; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > gpurun_out/fin_bench_c$c.json 2>> gpurun_out/fin_bench_other.err; echo bench_c$c=$?
done
timeout 300 python scripts/profile_eval.py 2 2 > gpurun_out/fin_prof.log 2>&1; echo prof=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c2.csv \
  python scripts/profile_eval.py 2 2 > gpurun_out/fin_ncu_launch.log 2>&1; echo ncu_launch=$?
for k in k_m2l_dmma k_fft_fwd k_fft_inv; do
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/fin_$k \
    python scripts/profile_eval.py 2 2 > gpurun_out/fin_ncu_$k.log 2>&1; echo ncu_$k=$?
  python scripts/ncu_summary.py /tmp/fin_$k.ncu-rep >> gpurun_out/fin_c2_l5_ncu.txt 2>&1
done
cp /tmp/fin_k_m2l_dmma.ncu-rep gpurun_out/ 2>/dev/null
