# Round-2: k_m2l_items variants on C5 (default: half parents, paired blocks, 16 warps;
# np16: unpaired; w12: 12 warps) and the C2 line with the permuted spectra placement of
# k_m2l_dmma; agreement tests first
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/p_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -2 gpurun_out/p_pytest_modes.log
[ $rc -ne 0 ] && exit 1
for v in default np16 w12; do
  if [ $v = default ]; then unset KAFMM_LIB; else export KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_$v.so; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_bench_c5_$v.json 2>> gpurun_out/p_bench.err; echo bench_$v=$?
  python -c "import json;d=json.load(open('gpurun_out/p_bench_c5_$v.json'));print('$v', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
done
unset KAFMM_LIB
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_bench_c2.json 2>> gpurun_out/p_bench.err; echo bench_c2=$?
python -c "import json;d=json.load(open('gpurun_out/p_bench_c2.json'));print('C2', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_dmma -s 3 -c 1 -o gpurun_out/p_c2_dmma \
  python scripts/profile_eval.py 2 2 > gpurun_out/p_ncu_c2.log 2>&1; echo ncu_c2=$?
python scripts/ncu_summary.py gpurun_out/p_c2_dmma.ncu-rep > gpurun_out/p_c2_dmma.txt 2>&1; head -20 gpurun_out/p_c2_dmma.txt
