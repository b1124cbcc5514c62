# Round-end measurement recipe (run under gpurun from the repo root): smoke, the full GPU suite,
# the default bench line with the driver's flags (C5), the reference arm, C2..C4 lines,
# the launch list of one C5 evaluation (every kernel: time; product kernels: DRAM bytes)
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?; tail -4 gpurun_out/fin_smoke.log
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench_c5.json 2> gpurun_out/fin_bench_c5.err ) 2> gpurun_out/fin_bench_c5.time; echo bench=$?; tail -3 gpurun_out/fin_bench_c5.time
python -c "import json;d=json.load(open('gpurun_out/fin_bench_c5.json'));print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['frac'], d['e2e'], d['p2p']['frac'])"
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err ) 2> gpurun_out/fin_ref.time; echo ref=$?; tail -3 gpurun_out/fin_ref.time
for c in 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_c$c.json 2>> gpurun_out/fin_bench_other.err; echo bench_c$c=$?
  python -c "import json;d=json.load(open('gpurun_out/fin_bench_c$c.json'));print('C$c', d['value'], d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c5.csv \
    python scripts/profile_eval.py 5 1 > gpurun_out/fin_ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/launch_summary.py gpurun_out/fin_launches_c5.csv --last-eval > gpurun_out/fin_launches_c5_lasteval.txt 2>&1; cat gpurun_out/fin_launches_c5_lasteval.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/fin_prod_c5.csv python scripts/profile_eval.py 5 1 > gpurun_out/fin_ncu_prod.log 2>&1; echo ncu_prod=$?
python scripts/prod_launches.py gpurun_out/fin_prod_c5.csv > gpurun_out/fin_prod_c5.txt; tail -3 gpurun_out/fin_prod_c5.txt
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?; grep -E "FAILED|ERROR|passed|failed" gpurun_out/fin_pytest.log | tail -20
