"""Summarise an ncu --set full report (.ncu-rep) per kernel launch: time,
DRAM bytes, FP64 pipe and DMMA utilisation, issue/memory throughput, warps.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [> profiles/x.txt]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_cycles_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_cycles_%"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thr_inst"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul_thr_inst"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd_thr_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
ki = h.index("Kernel Name")
print(f"# {rep}")
for r in data:
    print(f"== {r[ki][:100]}")
    for k, name in KEYS:
        if k in h:
            i = h.index(k)
            print(f"   {name:22s} {r[i]:>18s} {units[i]}")
    # warp stall reasons (cycles per issued instruction), the largest first
    st = [(float(r[i] or 0), h[i]) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")]
    for v, k in sorted(st, reverse=True)[:8]:
        if v >= 0.05:
            print(f"   stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:16s} {v:10.3f}")
