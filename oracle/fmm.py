"""O2: plain KIFMM with the paper's kernel tables (oracle; test infrastructure).

Kernel tables (which kernel each of the 8 traversal stages uses):
  Table I the 8 slots S2M S2L S2T / M2M M2L M2T / L2L L2T
  Laplace   L on S-row and ML tree, L+gradL on the T column  (PAPER.md:207-244,
            Table XI LapPGrad, single layer only)
  Stokeslet G everywhere
  RPY       Table IV: S-row G_RPY, ML tree G,
            T column G+lapG, S2T G_RPY+lapG
  RegVel    Table V: S-row G_eps, ML tree and T column G
  LapPGradGrad Table III: S-row L (charges) and L^D (dipoles),
            ML tree L, T column L+gradL+gradgradL, S2T the same from [q, d]
  RegVelOmega Table VI: S-row G_eps+T_eps, ML tree G,
            T column G+Omega, S2T G_eps+Omega+T+W

Steps, in the paper's order (Fig. 1):
  S->M   leaf sources -> upward check surface -> UC2UE (two SVD factors)
  M->M   child upward equivalents -> parent, composed M2M, bottom-up
  M->L   V list, raw kernel matrix into the downward check surface
  S->L   X list, sources straight onto the downward check surface
         DC2DE (two SVD factors) + L->L from the parent (composed L2L)
  L->T   downward equivalent -> leaf targets
  M->T   W list, upward equivalents -> leaf targets
  S->T   U list, direct
Downward expansions start at level 2 (levels 0-1 have empty V lists), L2L
from level 3.  M2L pairs are grouped by offset only to call one matrix
product per offset on stacked vectors; the arithmetic is unchanged.
"""
from __future__ import annotations

import time

import numpy as np

from . import lists as L
from .kernels import DIMS, direct_sum
from .operators import (ALPHA_DC, ALPHA_DE, ALPHA_UC, ALPHA_UE, Operators, surface)
from .tree import Tree

TABLES = {
    "laplace_pgrad": dict(S="L", ML="L", T="L+gradL", ST="L+gradL"),
    "stokeslet": dict(S="G", ML="G", T="G", ST="G"),
    "rpy": dict(S="G_RPY", ML="G", T="G+lapG", ST="G_RPY+lapG"),
    "stokes_reg_vel": dict(S="G_eps", ML="G", T="G", ST="G_eps"),
    # Table VI: [f, t, eps] -> [u, omega]
    "stokes_reg_vel_omega": dict(S="G_eps+T_eps", ML="G", T="G+Omega", ST="G_eps+Omega+T+W"),
    # Table III: charges and dipoles [q, d] -> [phi, grad, grad grad]
    "laplace_pgradgrad": dict(S="L+LD", ML="L", T="L+gradL+gradgradL", ST="LD+gradLD+gradgradLD"),
    # LapQPGradGrad (Table XI; same pattern as Table III with quadrupoles)
    "laplace_qpgradgrad": dict(S="LQ", ML="L", T="L+gradL+gradgradL", ST="LQ+gradLQ+gradgradLQ"),
}

_OPS_CACHE: dict = {}


def operators(ml: str, p: int) -> Operators:
    key = (ml, p)
    if key not in _OPS_CACHE:
        _OPS_CACHE[key] = Operators(ml, p)
    return _OPS_CACHE[key]


def sample_leaves(tree: Tree, min_targets: int, seed: int) -> list[int]:
    """Seeded draw of whole leaves until at least min_targets points are covered."""
    rng = np.random.default_rng(seed)
    leaves = tree.leaves()
    order = rng.permutation(leaves.size)
    out, tot = [], 0
    for i in order:
        b = int(leaves[i])
        out.append(b)
        tot += tree.pts[b].size
        if tot >= min_targets:
            break
    return sorted(out)


def direct(kernel: str, points, values, trg_idx=None) -> np.ndarray:
    """O1 direct sum with the table's S->T kernel at all (or selected) targets."""
    name = TABLES[kernel]["ST"]
    trg = points if trg_idx is None else points[trg_idx]
    return direct_sum(name, trg, points, values)


def fmm(points, values, kernel: str, p: int, cap: int, target_leaves=None,
        tree: Tree | None = None, ops: Operators | None = None, keep_internals=False,
        timings: dict | None = None):
    """Evaluate the KAFMM sum.

    target_leaves=None: every target (returns out in user order, N x k_t).
    target_leaves=list: sampled mode -- full upward pass, downward pass only
    for the ancestors of those leaves; returns values at their points.
    Returns dict(out=..., idx=target point indices, tree=..., ops=...).
    timings (optional dict) receives wall seconds of the list building
    ('lists'), the upward pass ('upward') and the rest ('downward').
    """
    clock = time.perf_counter
    t_start = clock()
    tab = TABLES[kernel]
    points = np.asarray(points, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    t = tree if tree is not None else Tree(points, cap)
    op = ops if ops is not None else operators(tab["ML"], p)
    k, M, n = op.k, op.M, op.n
    k_t = DIMS[tab["ST"]][1]
    full = target_leaves is None
    tleaves = [int(b) for b in t.leaves()] if full else sorted(int(b) for b in target_leaves)

    # ---- which boxes take part ------------------------------------------------
    tboxes = set()
    for b in tleaves:
        for a in t.ancestors(b):
            if t.level[a] >= 2:
                tboxes.add(a)
    Vl = {b: L.v_list(t, b) for b in tboxes}
    Wl = {b: L.w_list(t, b) for b in tleaves}
    Ul = {b: L.u_list(t, b) for b in tleaves}
    if full:
        Wall = {b: L.w_list(t, b) for b in t.leaves()}
        Xinv = L.x_lists_by_inversion(t, Wall)
        Xl = {b: Xinv[b] for b in tboxes}
    else:
        Xl = {b: L.x_list_direct(t, b) for b in tboxes}
    needed = set()
    for b in tboxes:
        needed.update(Vl[b])
    for b in tleaves:
        needed.update(Wl[b])

    level_boxes = [np.nonzero(t.level_arr == l)[0] for l in range(t.depth + 1)]
    lstart = [int(ids[0]) for ids in level_boxes]

    # ---- upward pass: S->M at leaves, M->M bottom-up ---------------------------
    t_lists = clock()
    ue_store = {}
    ue_next = None
    for l in range(t.depth, -1, -1):
        ids = level_boxes[l]
        ue_l = np.zeros((ids.size, n))
        lf = [int(b) for b in ids if t.leaf[b]]
        if lf:
            chk = np.zeros((len(lf), n))
            for r, b in enumerate(lf):
                uc = surface(p, t.centre(b), t.half_width(b), ALPHA_UC)
                idx = t.pts[b]
                chk[r] = direct_sum(tab["S"], uc, points[idx], values[idx]).reshape(-1)
            ue_l[np.array(lf) - lstart[l]] = op.uc2ue(chk, l)
        if l < t.depth:
            for o in range(8):
                par, chi = [], []
                for b in ids:
                    c = t.child[b][o]
                    if c >= 0:
                        par.append(int(b) - lstart[l])
                        chi.append(c - lstart[l + 1])
                if par:
                    ue_l[par] += ue_next[chi] @ op.m2m[o].T
        for b in ids:
            if full or int(b) in needed:
                ue_store[int(b)] = ue_l[int(b) - lstart[l]]
        ue_next = ue_l

    # ---- downward pass: M->L (V), S->L (X), DC2DE, L->L -------------------------
    t_up = clock()
    de = {}
    for l in range(2, t.depth + 1):
        tb = sorted(b for b in tboxes if t.level[b] == l)
        if not tb:
            continue
        row = {b: r for r, b in enumerate(tb)}
        chk = np.zeros((len(tb), n))
        groups: dict = {}
        for b in tb:
            for c in Vl[b]:
                o = tuple(int(v) for v in (t.ijk_arr[c] - t.ijk_arr[b]))
                groups.setdefault(o, ([], []))
                groups[o][0].append(row[b])
                groups[o][1].append(c)
        for o, (rows, srcs) in groups.items():
            U = np.stack([ue_store[c] for c in srcs])
            chk[rows] += (U @ op.m2l[o].T) * 2.0 ** l
        for b in tb:
            if Xl[b]:
                dc = surface(p, t.centre(b), t.half_width(b), ALPHA_DC)
                for a in Xl[b]:
                    idx = t.pts[a]
                    chk[row[b]] += direct_sum(tab["S"], dc, points[idx], values[idx]).reshape(-1)
        de_l = op.dc2de(chk, l)
        if l >= 3:
            for b in tb:
                par = t.parent[b]
                de_l[row[b]] += op.l2l[t.octant(b)] @ de[par]
        for b in tb:
            de[b] = de_l[row[b]]

    # ---- leaves: L->T, M->T (W), S->T (U) ------------------------------------
    out_rows = []
    idx_all = []
    for b in tleaves:
        idx = t.pts[b]
        x = points[idx]
        g = np.zeros((idx.size, k_t))
        if t.level[b] >= 2:
            z = surface(p, t.centre(b), t.half_width(b), ALPHA_DE)
            g += direct_sum(tab["T"], x, z, de[b].reshape(M, k))
        for d in Wl[b]:
            z = surface(p, t.centre(d), t.half_width(d), ALPHA_UE)
            g += direct_sum(tab["T"], x, z, ue_store[d].reshape(M, k))
        for a in Ul[b]:
            ia = t.pts[a]
            g += direct_sum(tab["ST"], x, points[ia], values[ia])
        out_rows.append(g)
        idx_all.append(idx)
    idx_all = np.concatenate(idx_all) if idx_all else np.zeros(0, dtype=np.int64)
    g_all = np.concatenate(out_rows) if out_rows else np.zeros((0, k_t))
    if timings is not None:
        t_end = clock()
        timings.update(lists=t_lists - t_start, upward=t_up - t_lists, downward=t_end - t_up)
    res = dict(tree=t, ops=op, kept=(op.up_kept, op.dn_kept))
    if full:
        out = np.zeros((points.shape[0], k_t))
        out[idx_all] = g_all
        res.update(out=out, idx=np.arange(points.shape[0]))
    else:
        order = np.argsort(idx_all)
        res.update(out=g_all[order], idx=idx_all[order])
    if keep_internals:
        res.update(ue=ue_store, de=de, U=Ul, V=Vl, W=Wl, X=Xl)
    return res


def rel_l2(a, b) -> float:
    """epsilon_L2 of PAPER.md:635-637: ||a - b||_2 / ||b||_2."""
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def blocks(kernel: str):
    """Output blocks per reading R11 (phi | grad phi ; u | lap u)."""
    return {"laplace_pgrad": [(0, 1), (1, 4)], "stokeslet": [(0, 3)],
            "rpy": [(0, 3), (3, 6)], "stokes_reg_vel": [(0, 3)],
            "stokes_reg_vel_omega": [(0, 3), (3, 6)],
            "laplace_pgradgrad": [(0, 1), (1, 4), (4, 10)],
            "laplace_qpgradgrad": [(0, 1), (1, 4), (4, 10)]}[kernel]
