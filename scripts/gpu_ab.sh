# launch list of the bench command itself (C2), after it ran plain
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bl_plain.json 2>/dev/null; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bl_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bl_ncu.log 2>&1; echo ncu=$?
