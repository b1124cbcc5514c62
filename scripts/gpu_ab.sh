# re-planning frees the previous lists; plan byte count after dfree
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_m2l_modes.py -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ab_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --dist --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dist1b.json 2> gpurun_out/dist1b.err; echo dist=$?
