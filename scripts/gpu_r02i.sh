# Round-2: ncu --set full of one large (level-9) sparse-chunk product launch, items and direction walk
set -u
mkdir -p gpurun_out
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_items -s 8 -c 1 -o gpurun_out/i_items_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/i_ncu_items.log 2>&1; echo ncu_items=$?
KAFMM_SPARSE_DIRS=1 timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_sparse -s 8 -c 1 -o gpurun_out/i_dirs_big \
  python scripts/profile_eval.py 5 1 > gpurun_out/i_ncu_dirs.log 2>&1; echo ncu_dirs=$?
for v in items dirs; do python scripts/ncu_summary.py gpurun_out/i_${v}_big.ncu-rep > gpurun_out/i_${v}_big.txt 2>&1; head -20 gpurun_out/i_${v}_big.txt; done
