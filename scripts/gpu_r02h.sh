# Round-2: k_m2l_items with a round-robin (sweeping) parent order: variant agreement, C5
# bench (items vs the direction walk), per-launch time + DRAM bytes of the product kernels.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_m2l_modes.py -q -x > gpurun_out/h_pytest_modes.log 2>&1; rc=$?; echo pytest_modes=$rc; tail -3 gpurun_out/h_pytest_modes.log
[ $rc -ne 0 ] && exit 1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/h_bench_c5.json 2>> gpurun_out/h_bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/h_bench_c5.json'));print('items', d['ms_per_step'], d['stages_ms']['m2l_product'], d['roofline']['frac'])"
for v in items dirs; do
  if [ $v = dirs ]; then export KAFMM_SPARSE_DIRS=1; fi
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:k_m2l_ --log-file gpurun_out/h_prod_$v.csv python scripts/profile_eval.py 5 1 > gpurun_out/h_ncu_$v.log 2>&1; echo ncu_$v=$?
done
python - <<'PY'
import csv
for v in ("items","dirs"):
    rows=[r for r in csv.reader(open(f"gpurun_out/h_prod_{v}.csv")) if len(r)>10]
    h=rows[0]; data=rows[1:]
    iK=h.index("Kernel Name"); iM=h.index("Metric Name"); iV=h.index("Metric Value"); iU=h.index("Metric Unit"); iI=h.index("ID")
    per={}
    for r in data:
        d=per.setdefault(r[iI],{"k":r[iK][:30]}); val=float(r[iV].replace(",",""))
        u=r[iU]; 
        if u=="Gbyte": val*=1e3
        if u=="Kbyte": val*=1e-3
        if u=="byte": val*=1e-6
        if u in("usecond",): val*=1e-3
        if u=="nsecond": val*=1e-6
        d[r[iM]]=val
    tt=tr=tw=0
    for i,d in per.items():
        t=d.get("gpu__time_duration.sum",0); rd=d.get("dram__bytes_read.sum",0); wr=d.get("dram__bytes_write.sum",0)
        tt+=t; tr+=rd; tw+=wr
        print(v, d["k"], f"{t:8.3f} ms  rd {rd:9.1f} MB  wr {wr:9.1f} MB")
    print(v, "TOTAL", f"{tt:.1f} ms rd {tr/1e3:.2f} GB wr {tw/1e3:.2f} GB")
PY
