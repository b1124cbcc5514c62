# Round-2 last check on the final code: smoke, M2L variant + full-size parity, the default bench line
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ag_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -m gpu -q > gpurun_out/ag_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ag_pytest.log
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ag_bench_c5.json 2> gpurun_out/ag_bench_c5.err ) 2> gpurun_out/ag_bench_c5.time; echo bench=$?; tail -3 gpurun_out/ag_bench_c5.time
python -c "import json;d=json.load(open('gpurun_out/ag_bench_c5.json'));print(d['value'], d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])"
