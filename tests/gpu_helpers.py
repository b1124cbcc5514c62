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


def block_max_errors(kernel, a, b):
    """Per output block: max over targets and components of |a - b| / max |b|.

    A fault confined to a few targets (one FFT chunk, one leaf pass, one
    level) is diluted by sqrt(N / N_bad) in the relative L2 norm; this bound
    is not."""
    out = []
    for lo, hi in F.blocks(kernel):
        d = np.abs(np.asarray(a)[:, lo:hi] - np.asarray(b)[:, lo:hi])
        s = float(np.abs(np.asarray(b)[:, lo:hi]).max()) if np.asarray(b).size else 0.0
        out.append(float(d.max()) / s if s > 0 else float(d.max()) if d.size else 0.0)
    return out


L2_TOL = 1e-10       # BASELINE.json north_star: relative L2 per output block (reading R11)
MAX_TOL = 1e-9       # per target, relative to the block's largest oracle value


def assert_parity(kernel, got, ref, l2_tol=L2_TOL, max_tol=MAX_TOL):
    """GPU vs oracle FMM: block relative L2 and per-target max bounds."""
    errs = block_errors(kernel, got, ref)
    assert max(errs) <= l2_tol, ("block rel L2", errs)
    merrs = block_max_errors(kernel, got, ref)
    assert max(merrs) <= max_tol, ("block max |d| / max |ref|", merrs)
    return errs, merrs


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
