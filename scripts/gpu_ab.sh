timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:'k_leaf_far' -c 1 -o /tmp/c5_lf python scripts/profile_eval.py 5 1 > gpurun_out/ncu_lf.log 2>&1; echo ncu=$?
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:'k_points_to_surface' -s 1 -c 1 -o /tmp/c5_s2l python scripts/profile_eval.py 5 1 > gpurun_out/ncu_s2l.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py /tmp/c5_lf.ncu-rep > gpurun_out/c5_lf_summary.txt 2>&1
python scripts/ncu_summary.py /tmp/c5_s2l.ncu-rep >> gpurun_out/c5_lf_summary.txt 2>&1
cp /tmp/c5_lf.ncu-rep /tmp/c5_s2l.ncu-rep gpurun_out/
