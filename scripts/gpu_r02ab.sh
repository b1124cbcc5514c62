# Round-2: k_m2l_groups with dynamically taken ranges (chunks of 8 / 4 / 16 unit positions)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -m gpu -q -x > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_bench_${name}.json 2>> gpurun_out/ab_bench.err
  python -c "import json;d=json.load(open('gpurun_out/ab_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3), 'setup', round(d['setup']['s'],2))"
}
run ck8 X=1
run ck4 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_ck4.so
run ck16 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_ck16.so
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_groups -s 7 -c 1 -o gpurun_out/ab_groups_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/ab_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/ab_groups_big.ncu-rep > gpurun_out/ab_groups_big.txt 2>&1; cat gpurun_out/ab_groups_big.txt
ncu -i gpurun_out/ab_groups_big.ncu-rep --page source --csv > gpurun_out/ab_groups_big_source.csv 2>/dev/null
