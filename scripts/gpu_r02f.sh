# Round-2: the item-stream sparse product (k_m2l_items): M2L variant agreement and small
# parity first, then C5 bench lines (items vs the direction walk), ncu --set full of
# one k_m2l_items launch.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -q -x > gpurun_out/f_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -5 gpurun_out/f_pytest_modes.log
[ $rc -ne 0 ] && exit 1
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/f_bench_c5.json'));print('items', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
KAFMM_SPARSE_DIRS=1 timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_bench_c5_dirs.json 2>> gpurun_out/f_bench_c5.err; echo bench_dirs=$?
python -c "import json;d=json.load(open('gpurun_out/f_bench_c5_dirs.json'));print('dirs', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_items -s 2 -c 1 -o gpurun_out/f_items \
  python scripts/profile_eval.py 5 1 > gpurun_out/f_ncu_items.log 2>&1; echo ncu_items=$?
python scripts/ncu_summary.py gpurun_out/f_items.ncu-rep > gpurun_out/f_c5_items_ncu.txt 2>&1; head -30 gpurun_out/f_c5_items_ncu.txt
