# Round-2: padded shared-memory rows in the DFT passes + Stokeslet pair in 22 FP64 ops:
# parity (small cases, M2L variants, full size), C5 / C2 bench, ncu of the C5 DFT passes
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/s_pytest.log 2>&1; rc=$?; echo pytest=$rc; tail -3 gpurun_out/s_pytest.log
[ $rc -ne 0 ] && exit 1
for c in 5 2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s_bench_c$c.json 2>> gpurun_out/s_bench.err; echo bench_c$c=$?
  python -c "import json;d=json.load(open('gpurun_out/s_bench_c$c.json'));print('C$c', d['ms_per_step'], d['stages_ms'])"
done
for k in k_fft_fwd k_fft_inv; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/s_$k \
    python scripts/profile_eval.py 5 1 > gpurun_out/s_ncu_$k.log 2>&1; echo ncu_$k=$?
done
for k in k_fft_fwd k_fft_inv; do python scripts/ncu_summary.py gpurun_out/s_$k.ncu-rep; done > gpurun_out/s_c5_dft_ncu.txt 2>&1
grep -E "==|time|tensor_cycles|issue_active|warps_active|smem_bank|smem_wave" gpurun_out/s_c5_dft_ncu.txt
