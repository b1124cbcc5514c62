# Round-2: sparse-chunk product with operator reuse (k_m2l_groups) -- agreement with
# k_m2l_items and the oracle, then C5 A/B lines (groups 16 warps, groups 12 warps, items)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -q -x > gpurun_out/v_pytest.log 2>&1; rc=$?; echo pytest=$rc; tail -3 gpurun_out/v_pytest.log
[ $rc -ne 0 ] && exit 1
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v_bench_${name}_c$C.json 2>> gpurun_out/v_bench.err
  python -c "import json;d=json.load(open('gpurun_out/v_bench_${name}_c$C.json'));s=d['stages_ms'];print('$name C$C', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3))"
}
for C in 5; do
  run groups X=1
  run g12 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_g12.so
  run items KAFMM_SPARSE=items
done
for C in 4 3; do run groups X=1; done
