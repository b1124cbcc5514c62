# Round-2: k_m2l_items with 32-bit shared addresses (no S2UR per b block), half vs whole parents
set -u
mkdir -p gpurun_out
for nb in 4 8; do
  KAFMM_ITEM_NB=$nb timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/k_pytest_modes_$nb.log 2>&1; rc=$?; echo pytest_modes_$nb=$rc; tail -2 gpurun_out/k_pytest_modes_$nb.log
  [ $rc -ne 0 ] && exit 1
done
for nb in 4 8; do
  KAFMM_ITEM_NB=$nb timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k_bench_c5_$nb.json 2>> gpurun_out/k_bench.err; echo bench_$nb=$?
  python -c "import json;d=json.load(open('gpurun_out/k_bench_c5_$nb.json'));print('nb$nb', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
done
for nb in 4 8; do
  KAFMM_ITEM_NB=$nb timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/k_prod_$nb.csv python scripts/profile_eval.py 5 1 > gpurun_out/k_ncu_$nb.log 2>&1; echo ncu_$nb=$?
  python scripts/prod_launches.py gpurun_out/k_prod_$nb.csv | tail -12
done
