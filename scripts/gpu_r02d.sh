# Round-2: the C-ABI multi-GPU path on one GPU (in-process ranks), and ncu --set full
# of one C5 sparse-chunk M2L product launch (k_m2l_sparse) with source correlation.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/d_pytest_dist.log 2>&1; echo pytest_dist=$?; tail -25 gpurun_out/d_pytest_dist.log
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_sparse -s 2 -c 1 -o gpurun_out/d_sparse \
  python scripts/profile_eval.py 5 1 > gpurun_out/d_ncu_sparse.log 2>&1; echo ncu_sparse=$?
python scripts/ncu_summary.py gpurun_out/d_sparse.ncu-rep > gpurun_out/d_c5_sparse_ncu.txt 2>&1; cat gpurun_out/d_c5_sparse_ncu.txt | head -40
ls -la gpurun_out/
