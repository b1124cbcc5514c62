"""Shared helpers of the -m gpu parity tests (CUDA path vs oracle)."""
import numpy as np

from oracle import fmm as F


def run_gpu(pts, vals, kernel, p, cap):
    import torch

    from paper_2010_15155_b200 import KAFMM
    plan = KAFMM(pts, kernel, p, cap)
    src = torch.from_numpy(np.ascontiguousarray(vals)).cuda()
    out = plan.eval(src)
    torch.cuda.synchronize()
    return plan, out.cpu().numpy()


def block_errors(kernel, a, b):
    return [F.rel_l2(a[:, lo:hi], b[:, lo:hi]) for lo, hi in F.blocks(kernel)]


def tree_keyed(plan):
    """GPU tree as {(level, i, j, k): (is_leaf, sorted user point indices)}."""
    t = plan.tree()
    perm = plan.permutation()
    out = {}
    for b in range(t["level"].size):
        key = (int(t["level"][b]),) + tuple(int(v) for v in t["ijk"][b])
        out[key] = (bool(t["leaf"][b]), np.sort(perm[t["pbeg"][b]:t["pend"][b]]))
    return out, t


def oracle_tree_keyed(tree):
    return {(tree.level[b],) + tuple(tree.ijk[b]): (bool(tree.leaf[b]), np.sort(tree.pts[b]))
            for b in range(tree.nbox)}
