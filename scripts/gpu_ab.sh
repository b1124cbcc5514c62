# round-end check on the final code: full GPU suite, smoke, default bench line
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin3_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/fin3_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin3_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/fin3_bench_c2.json 2> gpurun_out/fin3_bench_c2.err; echo bench=$?
