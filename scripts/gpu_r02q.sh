# Round-2 checkpoint: smoke, the full GPU suite, the default (C5) bench line, C2..C4 lines,
# ncu counters of the translation GEMMs (C5, C2) and the C5 product launch list (traffic)
set -u
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo smoke=$?; tail -4 gpurun_out/q_smoke.log
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/q_pytest.log 2>&1; echo pytest=$?; grep -E "FAILED|ERROR|passed|failed" gpurun_out/q_pytest.log | tail -20
timeout 1500 python bench.py > gpurun_out/q_bench_c5.json 2> gpurun_out/q_bench_c5.err; echo bench=$?; cat gpurun_out/q_bench_c5.json | head -c 600; echo
for c in 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench_c$c.json 2>> gpurun_out/q_bench_other.err; echo bench_c$c=$?
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active
for c in 5 2; do
  timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:k_gemm_dmma --log-file gpurun_out/q_gemm_c$c.csv \
    python scripts/profile_eval.py $c 1 > gpurun_out/q_ncu_gemm_c$c.log 2>&1; echo ncu_gemm_c$c=$?
  python scripts/gemm_counters.py gpurun_out/q_gemm_c$c.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/q_prod_c5.csv python scripts/profile_eval.py 5 1 > gpurun_out/q_ncu_prod.log 2>&1; echo ncu_prod=$?
python scripts/prod_launches.py gpurun_out/q_prod_c5.csv | tail -3
