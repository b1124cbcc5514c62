"""Minimal driver for ncu: set up config C and run `evals` evaluations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as WL
from paper_2010_15155_b200 import KAFMM
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
evals = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec, pts, vals = WL.make_config(cid)
plan = KAFMM(pts, spec.kernel, spec.p, spec.cap)
src = torch.from_numpy(vals).cuda()
for _ in range(evals):
    out = plan.eval(src)
torch.cuda.synchronize()
print("ok", plan.launch_count(), float(out.abs().sum()))
