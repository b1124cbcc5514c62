# Round-2: the dynamic-range test (KAFMM_GROUP_CHUNK=1), and the near field started with the
# M2L stage (KAFMM_NEAR_AT=m2l) vs right after the gather, C5 and C2
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -m gpu -q -x -k "dynamic or sparse" > gpurun_out/ac_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ac_pytest.log
run() {  # name, config, env...
  local name=$1; shift
  local c=$1; shift
  env "$@" timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ac_bench_${name}.json 2>> gpurun_out/ac_bench.err
  python -c "import json;d=json.load(open('gpurun_out/ac_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],3), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'graph', round(d['cuda_graph']['ms_per_step'],3))"
}
run c5_gather 5 X=1
run c5_m2l 5 KAFMM_NEAR_AT=m2l
run c2_gather 2 X=1
run c2_m2l 2 KAFMM_NEAR_AT=m2l
run c4_gather 4 X=1
run c4_m2l 4 KAFMM_NEAR_AT=m2l
