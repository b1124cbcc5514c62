# Round-2 re-entry: smoke, the full GPU suite (C-ABI multi-GPU path included), and
# ncu --set full of one C5 sparse-chunk M2L product launch (k_m2l_sparse).
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo smoke=$?; tail -4 gpurun_out/e_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo pytest=$?; grep -E "FAILED|ERROR|passed|failed" gpurun_out/e_pytest.log | tail -30
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_sparse -s 2 -c 1 -o gpurun_out/e_sparse \
  python scripts/profile_eval.py 5 1 > gpurun_out/e_ncu_sparse.log 2>&1; echo ncu_sparse=$?
python scripts/ncu_summary.py gpurun_out/e_sparse.ncu-rep > gpurun_out/e_c5_sparse_ncu.txt 2>&1; head -60 gpurun_out/e_c5_sparse_ncu.txt
