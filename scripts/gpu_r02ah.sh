# Round-2 evidence for the next steps: ncu --set full (source page) of one large C5 launch of each
# remaining kernel class: forward / inverse DFT, L2T+M2T, S2L, UC2UE GEMM
set -u
mkdir -p gpurun_out
cap() {  # name, regex, skip
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/ah_$1 \
    python scripts/profile_eval.py 5 1 > gpurun_out/ah_ncu_$1.log 2>&1; echo ncu_$1=$?
  python scripts/ncu_summary.py gpurun_out/ah_$1.ncu-rep > gpurun_out/ah_$1.txt 2>&1
  ncu -i gpurun_out/ah_$1.ncu-rep --page source --csv > gpurun_out/ah_$1_source.csv 2>/dev/null
  python scripts/ncu_opcodes.py gpurun_out/ah_$1_source.csv 12 >> gpurun_out/ah_$1.txt 2>&1
  cat gpurun_out/ah_$1.txt
}
cap fft_fwd k_fft_fwd 10
cap fft_inv k_fft_inv 10
cap leaf_far k_leaf_far 0
cap s2l "k_points_to_surface.*5, 1" 0
