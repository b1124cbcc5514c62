# Round-2: k_m2l_groups at 12 warps (default) vs L1 prefetch of the next group / unsplit
# operator loads; C5 lines, then ncu --set full of one large level-9 launch
set -u
mkdir -p gpurun_out
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/w_bench_${name}.json 2>> gpurun_out/w_bench.err
  python -c "import json;d=json.load(open('gpurun_out/w_bench_${name}.json'));s=d['stages_ms'];print('$name', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'frac', round(d['roofline']['frac'],3))"
}
run g12 X=1
run gpf1 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_gpf1.so
run ts0 KAFMM_LIB=$PWD/paper_2010_15155_b200/libkafmm_ts0.so
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_groups -s 7 -c 1 -o gpurun_out/w_groups_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/w_ncu_big.log 2>&1; echo ncu_big=$?
python scripts/ncu_summary.py gpurun_out/w_groups_big.ncu-rep > gpurun_out/w_groups_big.txt 2>&1; cat gpurun_out/w_groups_big.txt
