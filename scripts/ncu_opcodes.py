"""Per-opcode share of executed warp instructions and of warp-stall samples from an
ncu source-page export (ncu -i x.ncu-rep --page source --csv > x_source.csv).

    python scripts/ncu_opcodes.py gpurun_out/x_source.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
h, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}


def g(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0


COLS = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_branch_resolving", "stall_math", "stall_no_inst"]
tot = sum(g(r, "# Samples") for r in data)
inst = sum(g(r, "Instructions Executed") for r in data)
op = defaultdict(lambda: [0.0] * (2 + len(COLS)))
for r in data:
    t = r[ix["Source"]].strip().split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    a = op[o]
    a[0] += g(r, "Instructions Executed")
    a[1] += g(r, "# Samples")
    for j, c in enumerate(COLS):
        a[2 + j] += g(r, c)
print(f"# {rows[0][1][:90]}")
print(f"# warp instructions executed {inst:.4g}, stall samples {tot:.4g}; columns: % of instructions, % of samples,")
print("# then % of all samples by stall reason at that opcode")
print(f"{'opcode':10s} {'inst%':>7s} {'smpl%':>7s}  " + " ".join(f"{c[6:]:>10s}" for c in COLS))
for o, a in sorted(op.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{o:10s} {100 * a[0] / inst:7.2f} {100 * a[1] / tot:7.2f}  " + " ".join(f"{100 * v / tot:10.2f}" for v in a[2:]))
