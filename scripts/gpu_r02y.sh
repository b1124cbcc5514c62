# Round-2: k_m2l_groups with warp-uniform group words (ballot), c_ginfo constant rows,
# prefetch distance 32: parity of the M2L variants, C5 line, DFMA latency microbenchmark
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/y_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/y_pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/y_bench_${name}.json 2>> gpurun_out/y_bench.err
  python -c "import json;d=json.load(open('gpurun_out/y_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3))"
}
run uni X=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_lat scripts/micro/dfma_lat.cu && /tmp/dfma_lat > gpurun_out/y_dfma_lat.txt 2>&1; cat gpurun_out/y_dfma_lat.txt
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_groups -s 7 -c 1 -o gpurun_out/y_groups_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/y_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/y_groups_big.ncu-rep > gpurun_out/y_groups_big.txt 2>&1; cat gpurun_out/y_groups_big.txt
ncu -i gpurun_out/y_groups_big.ncu-rep --page source --csv > gpurun_out/y_groups_big_source.csv 2>/dev/null
