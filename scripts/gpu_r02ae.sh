# Round-2: k_m2l_groups with the next present offset's first operator half preloaded (KF_GPRE)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -m gpu -q -x > gpurun_out/ae_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ae_pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ae_bench_${name}.json 2>> gpurun_out/ae_bench.err
  python -c "import json;d=json.load(open('gpurun_out/ae_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3))"
}
run gpre X=1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_groups -s 7 -c 1 -o gpurun_out/ae_groups_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/ae_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/ae_groups_big.ncu-rep > gpurun_out/ae_groups_big.txt 2>&1; cat gpurun_out/ae_groups_big.txt
ncu -i gpurun_out/ae_groups_big.ncu-rep --page source --csv > gpurun_out/ae_groups_big_source.csv 2>/dev/null
