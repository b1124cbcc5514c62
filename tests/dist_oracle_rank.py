"""Test helper: one rank of the distributed evaluation with the ORACLE's
arithmetic in place of the GPU passes, so the product's host logic
(paper_2010_15155_b200.dist: partition, exchange lists, spmd_eval, the
torch.distributed transport) can run on CPU ranks over gloo.

The per-rank passes restate oracle/fmm.py restricted to the rank's work
(owned leaves; boxes whose subtree holds owned points), exactly as the
library's kafmm_restrict narrows the CUDA passes.  Test infrastructure only.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import fmm as F
from oracle import lists as OL
from oracle.kernels import direct_sum
from oracle.operators import ALPHA_DC, ALPHA_DE, ALPHA_UC, ALPHA_UE, surface
from oracle.tree import Tree
from paper_2010_15155_b200.dist import GlobalTree


def global_tree_from_oracle(points, cap, p, kml):
    """Oracle tree in the product's GlobalTree layout: points sorted by a
    depth-first walk in octant order, so every box owns a contiguous range."""
    t = Tree(points, cap)
    perm, pbeg, pend = [], np.zeros(t.nbox, np.int64), np.zeros(t.nbox, np.int64)

    def walk(b):
        pbeg[b] = len(perm)
        if t.leaf[b]:
            perm.extend(int(i) for i in t.pts[b])
        else:
            for c in t.child[b]:
                if c >= 0:
                    walk(c)
        pend[b] = len(perm)

    walk(0)
    U, V, W, X = OL.all_lists(t)

    def pairs(d):
        tg = [b for b, l in d.items() for _ in l]
        sr = [a for l in d.values() for a in l]
        return np.array(tg, np.int32), np.array(sr, np.int32)

    T = GlobalTree(level=t.level_arr.astype(np.int32), leaf=t.leaf_arr.copy(), pbeg=pbeg, pend=pend,
                   perm=np.array(perm, np.int64), lists={"U": pairs(U), "V": pairs(V), "W": pairs(W), "X": pairs(X)},
                   n_surf=6 * (p - 1) ** 2 + 2, kml=kml, n_freq=0)
    return t, T, dict(U=U, V=V, W=W, X=X)


class OracleRank:
    """Same interface as paper_2010_15155_b200.dist.RankPlan, CPU tensors."""

    def __init__(self, t, T, L, maps, points, kernel, p, n_local):
        self.t, self.T, self.L, self.m = t, T, L, maps
        self.points, self.kernel, self.p, self.n_local = points, kernel, p, n_local
        self.tab = F.TABLES[kernel]
        self.op = F.operators(self.tab["ML"], p)
        self.k_s, self.k_t = {"laplace_pgrad": (1, 4), "stokeslet": (3, 3), "rpy": (4, 6),
                              "stokes_reg_vel": (4, 3)}[kernel]
        n = T.n
        self.active = (T.pbeg < maps.phi) & (T.pend > maps.plo)
        self.gvals = np.zeros((n, self.k_s))
        self.gout = np.zeros((n, self.k_t))
        self.ue = np.zeros((t.nbox, self.op.n))

    # E1 ----------------------------------------------------------------------
    def pack_values(self, local_vals):
        v = np.asarray(local_vals)
        return [torch.from_numpy(np.ascontiguousarray(v[i])) for i in self.m.val_send]

    def values_rows(self):
        return [len(i) for i in self.m.val_recv]

    def unpack_values(self, recv):
        for buf, idx in zip(recv, self.m.val_recv):
            if len(idx):
                self.gvals[idx] = buf.numpy().reshape(len(idx), self.k_s)

    def up(self):
        t, op, p = self.t, self.op, self.p
        for l in range(t.depth, -1, -1):
            for b in t.boxes_at(l):
                b = int(b)
                if not self.active[b]:
                    continue
                if t.leaf[b] and l >= 2:
                    idx = t.pts[b]
                    uc = surface(p, t.centre(b), t.half_width(b), ALPHA_UC)
                    chk = direct_sum(self.tab["S"], uc, self.points[idx], self.gvals[idx]).reshape(1, -1)
                    self.ue[b] = op.uc2ue(chk, l)[0]
                for o in range(8):
                    c = t.child[b][o]
                    if c >= 0 and self.active[c]:
                        self.ue[b] += op.m2m[o] @ self.ue[c]

    # E2 / E3 -----------------------------------------------------------------
    def pack_shared(self):
        return torch.from_numpy(np.ascontiguousarray(self.ue[self.m.shared]))

    def unpack_shared(self, buf):
        if len(self.m.shared):
            self.ue[self.m.shared] = buf.numpy().reshape(len(self.m.shared), -1)

    def pack_ghost(self):
        return [torch.from_numpy(np.ascontiguousarray(self.ue[i])) for i in self.m.ue_send]

    def ghost_rows(self):
        return [len(i) for i in self.m.ue_recv]

    def unpack_ghost(self, recv):
        for buf, ids in zip(recv, self.m.ue_recv):
            if len(ids):
                self.ue[ids] = buf.numpy().reshape(len(ids), -1)

    def down(self):
        t, op, p, L = self.t, self.op, self.p, self.L
        M, k = op.M, op.k
        de = {}
        for l in range(2, t.depth + 1):
            for b in t.boxes_at(l):
                b = int(b)
                if not self.active[b]:
                    continue
                chk = np.zeros(op.n)
                for c in L["V"][b]:
                    o = tuple(int(v) for v in (t.ijk_arr[c] - t.ijk_arr[b]))
                    chk += (op.m2l[o] @ self.ue[c]) * 2.0 ** l
                if L["X"][b]:
                    dc = surface(p, t.centre(b), t.half_width(b), ALPHA_DC)
                    for a in L["X"][b]:
                        idx = t.pts[a]
                        chk += direct_sum(self.tab["S"], dc, self.points[idx], self.gvals[idx]).reshape(-1)
                d = op.dc2de(chk.reshape(1, -1), l)[0]
                if l >= 3:
                    d = d + op.l2l[t.octant(b)] @ de[t.parent[b]]
                de[b] = d
        pos = np.empty(self.T.n, np.int64)
        pos[self.T.perm] = np.arange(self.T.n)
        for b in t.leaves():
            b = int(b)
            if not self.active[b]:
                continue
            idx = t.pts[b]
            x = self.points[idx]
            g = np.zeros((idx.size, self.k_t))
            if t.level[b] >= 2:
                z = surface(p, t.centre(b), t.half_width(b), ALPHA_DE)
                g += direct_sum(self.tab["T"], x, z, de[b].reshape(M, k))
            for d in L["W"][b]:
                z = surface(p, t.centre(d), t.half_width(d), ALPHA_UE)
                g += direct_sum(self.tab["T"], x, z, self.ue[d].reshape(M, k))
            for a in L["U"][b]:
                ia = t.pts[a]
                g += direct_sum(self.tab["ST"], x, self.points[ia], self.gvals[ia])
            self.gout[idx] = g

    # E4 ----------------------------------------------------------------------
    def pack_out(self):
        return [torch.from_numpy(np.ascontiguousarray(self.gout[u])) for u in self.m.out_send]

    def out_rows(self):
        return [len(i) for i in self.m.out_recv]

    def unpack_out(self, recv, local_out):
        for buf, idx in zip(recv, self.m.out_recv):
            if len(idx):
                local_out[idx] = buf.numpy().reshape(len(idx), self.k_t)
        return local_out

    def new_out(self):
        return np.zeros((self.n_local, self.k_t))
