# Round-2: forward DFT x pass with fpos loaded before the DMMA loop: parity, C5 / C2 lines
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/ai_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ai_pytest.log
run() {  # name, config
  timeout 900 python bench.py --config $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ai_bench_$1.json 2>> gpurun_out/ai_bench.err
  python -c "import json;d=json.load(open('gpurun_out/ai_bench_$1.json'));s=d['stages_ms'];print('$1', round(d['ms_per_step'],2), 'm2l', s['m2l'], 'prod', s['m2l_product'], 'dft', round(s['m2l']-s['m2l_product'],2))"
}
run c5 5
run c2 2
