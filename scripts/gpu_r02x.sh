# Round-2 re-entry checkpoint on HEAD: smoke, the default bench line (C5) with the driver's
# flags, the reference arm with the driver's flags (wall-clocked), the GPU suite, then
# ncu --set full (source page) of one large level-9 k_m2l_groups launch.
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.log 2>&1; echo smoke=$?
( time timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/x_bench.json 2> gpurun_out/x_bench.err ) 2> gpurun_out/x_bench.time; echo bench=$?; tail -3 gpurun_out/x_bench.time
python -c "import json;d=json.load(open('gpurun_out/x_bench.json'));print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline'], d['e2e'], d['cpu_baseline'])"
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/x_ref.json 2> gpurun_out/x_ref.err ) 2> gpurun_out/x_ref.time; echo ref=$?; tail -3 gpurun_out/x_ref.time; cat gpurun_out/x_ref.json
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_groups -s 7 -c 1 -o gpurun_out/x_groups_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/x_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/x_groups_big.ncu-rep > gpurun_out/x_groups_big.txt 2>&1; cat gpurun_out/x_groups_big.txt
ncu -i gpurun_out/x_groups_big.ncu-rep --page source --csv > gpurun_out/x_groups_big_source.csv 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/x_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/x_pytest.log
