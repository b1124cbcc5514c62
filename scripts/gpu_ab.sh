# final check after the LapPGradGrad functor change: full GPU suite, C2 default line, C9
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin2_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/fin2_pytest.log
timeout 900 python bench.py > gpurun_out/fin2_bench_c2.json 2> gpurun_out/fin2_bench_c2.err; echo bench=$?
timeout 900 python bench.py --config 9 --steps 3 --no-cpu-baseline > gpurun_out/fin2_bench_c9.json 2>> gpurun_out/fin2_bench_c2.err; echo bench9=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1; echo smoke=$?
