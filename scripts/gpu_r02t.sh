# Round-2: forward DFT with staged density cubes, inverse with the bin map in shared memory,
# M2L overlapped with M2M: agreement + parity (small), then C5 / C2 A/B lines
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/t_pytest.log 2>&1; rc=$?; echo pytest=$rc; tail -3 gpurun_out/t_pytest.log
[ $rc -ne 0 ] && exit 1
run() {  # name, env..., config
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t_bench_${name}_c$C.json 2>> gpurun_out/t_bench.err
  python -c "import json;d=json.load(open('gpurun_out/t_bench_${name}_c$C.json'));s=d['stages_ms'];print('$name C$C', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'graph', d['cuda_graph'])"
}
for C in 5 2; do
  run default X=1
  run noovl KAFMM_M2L_OVERLAP=0
  run nostage KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_nostage.so
done
