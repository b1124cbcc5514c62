"""Summarise an ncu --csv launch list of the translation GEMMs (k_gemm_dmma<mode>)
captured with the metrics of scripts/gpu_r02q.sh: per template (0 = store: UC2UE / DC2DE
factors, 1 = add: L2L, 2 = atomic: M2M) the launches, device time, DRAM bytes and GB/s,
the DMMA instruction count as FP64 TFLOP/s (one DMMA.8x8x4 = 512 flop) and the tensor
(DMMA sub-pipe) activity.  Usage: gemm_counters.py launches.csv"""
import csv
import re
import sys

SCALE = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, data = rows[0], rows[1:]
iK, iM, iV, iU, iI = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = {}
for r in data:
    d = per.setdefault(r[iI], {"k": r[iK]})
    d[r[iM]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
agg = {}
for d in per.values():
    m = re.search(r"k_gemm_dmma<(\d)>", d["k"])
    key = f"k_gemm_dmma<{m.group(1)}>" if m else d["k"][:40]
    a = agg.setdefault(key, {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0, "dmma": 0.0, "tc": 0.0})
    t = d.get("gpu__time_duration.sum", 0.0)
    a["n"] += 1
    a["t"] += t
    a["rd"] += d.get("dram__bytes_read.sum", 0.0)
    a["wr"] += d.get("dram__bytes_write.sum", 0.0)
    a["dmma"] += d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)
    a["tc"] += t * d.get("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
print(f"{'kernel':18s} {'launches':>8s} {'ms':>9s} {'DRAM GB':>9s} {'GB/s':>8s} {'TFLOP/s':>8s} {'dmma %':>7s}")
for k, a in sorted(agg.items()):
    t = max(a["t"], 1e-12)
    print(f"{k:18s} {a['n']:8d} {1e3 * a['t']:9.3f} {(a['rd'] + a['wr']) / 1e9:9.3f} "
          f"{(a['rd'] + a['wr']) / t / 1e9:8.1f} {a['dmma'] * 512 / t / 1e12:8.2f} {a['tc'] / t:7.1f}")
