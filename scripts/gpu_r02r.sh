# Round-2: ncu --set full of the C5 DFT passes (one large forward / inverse launch) and of
# the leaf kernels (L2T+M2T, S2L, P2P) of the final code
set -u
mkdir -p gpurun_out
for k in k_fft_fwd k_fft_inv; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/r_$k \
    python scripts/profile_eval.py 5 1 > gpurun_out/r_ncu_$k.log 2>&1; echo ncu_$k=$?
done
for k in k_leaf_far k_points_to_surface k_p2p; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r_$k \
    python scripts/profile_eval.py 5 1 > gpurun_out/r_ncu_$k.log 2>&1; echo ncu_$k=$?
done
for k in k_fft_fwd k_fft_inv k_leaf_far k_points_to_surface k_p2p; do python scripts/ncu_summary.py gpurun_out/r_$k.ncu-rep; done > gpurun_out/r_c5_other_ncu.txt 2>&1
cat gpurun_out/r_c5_other_ncu.txt | grep -E "==|time|fp64_pipe|tensor_cycles|issue_active|warps_active|smem_bank|smem_wave"
