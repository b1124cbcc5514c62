"""Summarise an ncu --csv launch list (gpu__time_duration + DRAM bytes per launch) of
the M2L product kernels: per-launch ms / GB and the totals.  Usage: prod_launches.py f.csv"""
import csv
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, data = rows[0], rows[1:]
iK, iM, iV, iU, iI = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = {}
for r in data:
    d = per.setdefault(r[iI], {"k": r[iK].split("(")[0]})
    d[r[iM]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
tt = tr = tw = 0.0
for d in per.values():
    t, rd, wr = (d.get(k, 0.0) for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"))
    tt, tr, tw = tt + t, tr + rd, tw + wr
    print(f"{d['k']:40s} {t:9.3f} ms  read {rd:7.2f} GB  write {wr:7.2f} GB")
print(f"{'TOTAL':40s} {tt:9.3f} ms  read {tr:7.2f} GB  write {tw:7.2f} GB")
