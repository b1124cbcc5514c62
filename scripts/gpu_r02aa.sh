# Round-2: k_m2l_groups A/B -- cost-balanced dealing of units to warp slots (KAFMM_BALANCE),
# 16 warps at 128 registers (small spills) vs 12 warps at 156
set -u
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/aa_bench_${name}.json 2>> gpurun_out/aa_bench.err
  python -c "import json;d=json.load(open('gpurun_out/aa_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3), 'setup', round(d['setup']['s'],2))"
}
run bal0 KAFMM_BALANCE=0
run bal1 KAFMM_BALANCE=1
run w16bal1 KAFMM_BALANCE=1 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_w16.so
run w16bal0 KAFMM_BALANCE=0 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_w16.so
KAFMM_BALANCE=1 timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -m gpu -q -x > gpurun_out/aa_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/aa_pytest.log
