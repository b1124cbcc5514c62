set -x
timeout 600 python -m pytest tests/test_gpu_m2l_modes.py tests/test_gpu_parity.py -x -q > gpurun_out/k_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/k_pytest.log
for c in 2 3; do
 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/k_c$c.json 2>gpurun_out/k_c$c.err
 KAFMM_DMMA_NT=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/k_c${c}_half.json 2>>gpurun_out/k_c$c.err
done
timeout 400 python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/k_c4.json 2>gpurun_out/k_c4.err
