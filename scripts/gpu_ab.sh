# round-end check on the final code: full GPU suite, smoke, default bench line
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin5_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/fin5_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/fin5_bench_c2.json 2> gpurun_out/fin5_bench_c2.err; echo bench=$?
timeout 900 python bench.py --config 6 --steps 3 --no-cpu-baseline > gpurun_out/fin5_bench_c6.json 2>> gpurun_out/fin5_bench_c2.err; echo bench6=$?
timeout 900 python bench.py --config 3 --steps 3 --no-cpu-baseline > gpurun_out/fin5_bench_c3.json 2>> gpurun_out/fin5_bench_c2.err; echo bench3=$?
