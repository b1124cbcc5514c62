"""Tiny evaluations of every kernel, M2L variant, the partitioned path and the
wall path, for compute-sanitizer (one --tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as WL
from paper_2010_15155_b200 import KAFMM, KAFMMWall
from paper_2010_15155_b200 import dist as D

rng = np.random.default_rng(0)
c = rng.random((3, 3)) * 0.6 + 0.2
pts = np.clip(np.concatenate([c[i] + 0.05 * rng.standard_normal((500, 3)) for i in range(3)]
                             + [rng.random((500, 3))]), 0, np.nextafter(1.0, 0.0))
for kernel in WL.KERNELS:
    vals = torch.from_numpy(WL.random_values(kernel, pts.shape[0], 1)).cuda()
    plan = KAFMM(pts, kernel, 4, 20)
    for mode in ("fft", "fft_blocks", "fft_pairs", "dense"):
        plan.set_m2l(mode)
        plan.eval(vals)
    for t in (1, 2, 0):
        plan.set_timing(t)
        plan.eval(vals)
    torch.cuda.synchronize()
    plan.close()
    print("ok", kernel, flush=True)
offs = np.array([0, 700, 2000])
src = torch.from_numpy(WL.random_values("stokeslet", 2000, 2)).cuda()
ranks = [D.build_rank(torch.from_numpy(pts).cuda(), offs, r, 2, "stokeslet", 4, 20)[0] for r in range(2)]
D.spmd_eval(ranks, D.LocalTransport(), [src[offs[r]:offs[r + 1]] for r in range(2)])
torch.cuda.synchronize()
print("ok dist", flush=True)
wp = np.concatenate([rng.random((800, 2)), 0.5 + 0.5 * rng.random((800, 1))], axis=1)
w = KAFMMWall(wp, 4, 20)
w.eval(torch.from_numpy(np.concatenate([rng.standard_normal((800, 3)), 1e-3 * np.ones((800, 1))], 1)).cuda())
torch.cuda.synchronize()
print("ok wall", flush=True)
