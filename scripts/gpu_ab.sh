# the N-GPU bench path (torchrun + NCCL) at world size 1 on the final code
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --dist --steps 3 --warmup 3 > gpurun_out/dist1.json 2> gpurun_out/dist1.err; echo dist=$?
( time timeout 900 python bench.py --impl reference --steps 2 --warmup 1 ) > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref=$?
