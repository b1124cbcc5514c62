# Round-2: k_m2l_items with per-item sign patterns (8 code variants, signs folded into the
# multiply-adds): variant agreement, C5 bench (half / whole parents), product launch lists
set -u
mkdir -p gpurun_out
for nb in 4 8; do
  KAFMM_ITEM_NB=$nb timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/m_pytest_modes_$nb.log 2>&1; rc=$?; echo pytest_modes_$nb=$rc; tail -2 gpurun_out/m_pytest_modes_$nb.log
  [ $rc -ne 0 ] && exit 1
done
for nb in 4 8; do
  KAFMM_ITEM_NB=$nb timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/m_bench_c5_$nb.json 2>> gpurun_out/m_bench.err; echo bench_$nb=$?
  python -c "import json;d=json.load(open('gpurun_out/m_bench_c5_$nb.json'));print('nb$nb', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
done
KAFMM_ITEM_NB=4 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/m_prod_4.csv python scripts/profile_eval.py 5 1 > gpurun_out/m_ncu_4.log 2>&1; echo ncu_4=$?
python scripts/prod_launches.py gpurun_out/m_prod_4.csv | tail -12
KAFMM_ITEM_NB=4 timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_items -s 8 -c 1 -o gpurun_out/m_items_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/m_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/m_items_big.ncu-rep > gpurun_out/m_items_big.txt 2>&1; head -20 gpurun_out/m_items_big.txt
