# round-end check on the final code: full GPU suite, smoke, default bench line, partitioned path at world 1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin4_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/fin4_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/fin4_bench_c2.json 2> gpurun_out/fin4_bench_c2.err; echo bench=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 1 --dist --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin4_dist1.json 2> gpurun_out/fin4_dist1.err; echo dist=$?
