# Round-2: k_m2l_groups lane-parallel L2 prefetch per batch (default) vs per group (pf0);
# range chunk 2 vs 4 (KAFMM_GROUP_CHUNK, host-side layout)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -m gpu -q -x > gpurun_out/af_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/af_pytest.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/af_bench_${name}.json 2>> gpurun_out/af_bench.err
  python -c "import json;d=json.load(open('gpurun_out/af_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3))"
}
run lane X=1
run pf0 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_pf0.so
run lane_ck2 KAFMM_GROUP_CHUNK=2
run lane_ck3 KAFMM_GROUP_CHUNK=3
