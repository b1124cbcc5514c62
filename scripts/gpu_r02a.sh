# Round-2 first GPU pass: smoke, full GPU suite, the default (C5) bench line, the
# launch list of the bench command, and ncu --set full of the C5 product and GEMM kernels.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo smoke=$?
timeout 2700 python -m pytest tests -m gpu -q -x > gpurun_out/a_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/a_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench_c5.json 2> gpurun_out/a_bench_c5.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a_launches_c5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/a_ncu_launch.log 2>&1; echo ncu_launch=$?
python scripts/launch_summary.py gpurun_out/a_launches_c5.csv > gpurun_out/a_launches_c5_summary.txt 2>&1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_m2l_ -c 18 -o /tmp/a_prod \
  python scripts/profile_eval.py 5 1 > gpurun_out/a_ncu_prod.log 2>&1; echo ncu_prod=$?
python scripts/ncu_summary.py /tmp/a_prod.ncu-rep > gpurun_out/a_c5_prod_ncu.txt 2>&1
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:k_gemm_dmma -c 14 -o /tmp/a_gemm \
  python scripts/profile_eval.py 5 1 > gpurun_out/a_ncu_gemm.log 2>&1; echo ncu_gemm=$?
python scripts/ncu_summary.py /tmp/a_gemm.ncu-rep > gpurun_out/a_c5_gemm_ncu.txt 2>&1
cp /tmp/a_prod.ncu-rep gpurun_out/ 2>/dev/null
