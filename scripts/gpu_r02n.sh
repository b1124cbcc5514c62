# Round-2: k_m2l_items, per-item sign masks (one code path), half-parent units by default:
# variant agreement, C5 bench, product launch list, ncu --set full of a large launch
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/n_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -2 gpurun_out/n_pytest_modes.log
[ $rc -ne 0 ] && exit 1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/n_bench_c5.json 2>> gpurun_out/n_bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/n_bench_c5.json'));print('nb4', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/n_prod.csv python scripts/profile_eval.py 5 1 > gpurun_out/n_ncu.log 2>&1; echo ncu=$?
python scripts/prod_launches.py gpurun_out/n_prod.csv | tail -12
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_items -s 8 -c 1 -o gpurun_out/n_items_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/n_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/n_items_big.ncu-rep > gpurun_out/n_items_big.txt 2>&1; head -20 gpurun_out/n_items_big.txt
