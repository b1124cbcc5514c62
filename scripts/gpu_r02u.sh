# Round-2 re-entry baseline on HEAD: smoke, the GPU suite, the default (C5) bench line
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/u_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/u_pytest.log
timeout 900 python bench.py > gpurun_out/u_bench_c5.json 2> gpurun_out/u_bench_c5.err; echo bench=$?
tail -c 600 gpurun_out/u_bench_c5.json
