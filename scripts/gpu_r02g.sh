# Round-2: k_m2l_items with balanced warp runs + L2 prefetch: variant agreement, then C5
# bench lines for the prefetch depth A/B (6 default, 2, 14) and the direction walk.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/g_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -3 gpurun_out/g_pytest_modes.log
[ $rc -ne 0 ] && exit 1
for v in default pf2 pf14; do
  if [ $v = default ]; then unset KAFMM_LIB; else export KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g_bench_c5_$v.json 2>> gpurun_out/g_bench.err; echo bench_$v=$?
  python -c "import json;d=json.load(open('gpurun_out/g_bench_c5_$v.json'));print('$v', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
done
unset KAFMM_LIB
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_items -s 2 -c 1 -o gpurun_out/g_items \
  python scripts/profile_eval.py 5 1 > gpurun_out/g_ncu_items.log 2>&1; echo ncu_items=$?
python scripts/ncu_summary.py gpurun_out/g_items.ncu-rep > gpurun_out/g_c5_items_ncu.txt 2>&1; head -30 gpurun_out/g_c5_items_ncu.txt
