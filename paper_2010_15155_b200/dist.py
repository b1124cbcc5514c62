"""Multi-GPU evaluation of the KAFMM sum.

One process per GPU.  The octree is split into contiguous Morton ranges of
the sorted points (whole leaves), weighted by the work each point brings
(P2P pairs, W/X surface evaluations, S2M, M2L pairs).  Every rank builds the
same global tree and lists (kafmm_setup on the all-gathered points) and then
restricts its plan to its range (kafmm_restrict).  An evaluation is

    E1  all-to-all-v  source values, from the caller's rows to every rank that
                      needs them (its owned points and the remote leaves of
                      its U and X lists)
        kafmm_eval_up       S2M, UC2UE over owned leaves, M2M into active boxes
    E2  all-reduce    UE of the boxes that straddle ranks (partial sums)
    E3  all-to-all-v  ghost UE: remote boxes named by the V lists of this
                      rank's active boxes and the W lists of its leaves
        kafmm_eval_down     M2L, S2L, DC2DE, L2L, L2T, M2T, P2P, scatter
    E4  all-to-all-v  outputs, from the owning rank back to the caller's rows

The exchange maps are host logic here: deterministic numpy functions of the
global tree, so every rank derives the same send and receive lists without
communicating them.  The collectives go through a Transport:
TorchTransport (torch.distributed -- NCCL on GPUs, gloo in the CPU tests) or
LocalTransport (all ranks in one process, e.g. several restricted plans on
one GPU, run one after the other).  Packing and unpacking are library
kernels (kafmm_pack_ue, kafmm_gather_rows, ...); nothing here computes the
method's arithmetic.
"""
from __future__ import annotations

import dataclasses

import numpy as np

# ---------------------------------------------------------------------------
# global tree view and partition (host logic)
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class GlobalTree:
    """Box arrays (ids as in the plan), Morton permutation and the lists."""
    level: np.ndarray       # int32 per box
    leaf: np.ndarray        # bool per box
    pbeg: np.ndarray        # int64 per box: first sorted point
    pend: np.ndarray        # int64 per box: one past the last
    perm: np.ndarray        # int64 per sorted point: user row
    lists: dict             # 'U','V','W','X' -> (tgt int32, src int32)
    n_surf: int             # M points per surface
    kml: int                # ML-kernel dimension (1 Laplace, 3 Stokes family)
    n_freq: int = 0         # FFT M2L bins (0: dense M2L)

    @property
    def nbox(self) -> int:
        return int(self.level.size)

    @property
    def n(self) -> int:
        return int(self.perm.size)


def tree_from_plan(plan) -> GlobalTree:
    t = plan.tree()
    inf = plan.info()
    p = inf.p
    ng = 2 * p - 1
    return GlobalTree(level=t["level"], leaf=t["leaf"], pbeg=t["pbeg"], pend=t["pend"], perm=plan.permutation(),
                      lists={w: plan.lists(w) for w in "UVWX"}, n_surf=inf.n_surf,
                      kml=1 if inf.n_equiv == inf.n_surf else 3, n_freq=ng * ng * (ng // 2 + 1))


def point_weights(T: GlobalTree) -> np.ndarray:
    """Estimated work per sorted point (flop-like units), per SURVEY.md §8(a).

    Each box's work is spread evenly over its points: P2P pairs and W/X
    surface evaluations of leaves, S2M of leaves, and the FFT-M2L Hadamard
    work of the box's V pairs."""
    c_pair = 30.0
    npts = (T.pend - T.pbeg).astype(np.float64)
    cost = np.zeros(T.nbox)
    ut, us = T.lists["U"]
    np.add.at(cost, ut, npts[ut] * npts[us] * c_pair)
    wt, ws = T.lists["W"]
    np.add.at(cost, wt, npts[wt] * T.n_surf * c_pair)
    xt, xs = T.lists["X"]
    np.add.at(cost, xt, npts[xs] * T.n_surf * c_pair)
    leaf = T.leaf
    cost[leaf] += npts[leaf] * T.n_surf * c_pair * 2.0          # S2M + L2T
    vt, _ = T.lists["V"]
    c_v = 8.0 * T.kml * T.kml * max(T.n_freq, 1)
    np.add.at(cost, vt, c_v)
    dens = np.where(npts > 0, cost / np.maximum(npts, 1.0), 0.0)
    diff = np.zeros(T.n + 1)
    np.add.at(diff, T.pbeg, dens)
    np.add.at(diff, T.pend, -dens)
    return np.cumsum(diff[:-1])


def partition(T: GlobalTree, world: int, weights: np.ndarray | None = None) -> np.ndarray:
    """Cuts c_0 = 0 <= c_1 <= ... <= c_world = n at leaf boundaries: rank r owns
    the sorted points [c_r, c_{r+1}).  Balances the prefix sums of `weights`."""
    n = T.n
    if world == 1:
        return np.array([0, n], dtype=np.int64)
    w = point_weights(T) if weights is None else np.asarray(weights, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    bounds = np.unique(np.concatenate([T.pbeg[T.leaf], [n]])).astype(np.int64)  # leaf starts + n
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        j = int(np.searchsorted(cum[bounds], target))
        cand = [bounds[max(j - 1, 0)], bounds[min(j, bounds.size - 1)]]
        c = min(cand, key=lambda b: abs(cum[b] - target))
        cuts.append(max(int(c), cuts[-1]))
    cuts.append(n)
    return np.array(cuts, dtype=np.int64)


def _rank_of(cuts: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Rank owning sorted point idx (cuts as from partition)."""
    return np.searchsorted(cuts, idx, side="right") - 1


@dataclasses.dataclass
class RankMaps:
    rank: int
    world: int
    plo: int
    phi: int
    shared: np.ndarray          # int32 boxes straddling ranks (same on every rank)
    ue_send: list               # per destination rank: int32 box ids
    ue_recv: list               # per source rank: int32 box ids
    val_send: list              # per destination: int64 local caller rows
    val_recv: list              # per source: int64 global user rows
    out_send: list              # per destination: int64 global user rows
    out_recv: list              # per source: int64 local caller rows


def _needed(T: GlobalTree, cuts: np.ndarray, r: int, shared_mask: np.ndarray, owner: np.ndarray):
    """Ghost UE boxes and needed source points of rank r."""
    plo, phi = cuts[r], cuts[r + 1]
    active = (T.pbeg < phi) & (T.pend > plo)
    vt, vs = T.lists["V"]
    wt, ws = T.lists["W"]
    need = np.unique(np.concatenate([vs[active[vt]], ws[active[wt]]]))
    ghost = need[~active[need] & ~shared_mask[need]]
    ut, us = T.lists["U"]
    xt, xs = T.lists["X"]
    leaves = np.unique(np.concatenate([us[active[ut]], xs[active[xt]]]))
    leaves = leaves[(T.pbeg[leaves] < plo) | (T.pend[leaves] > phi)]  # remote leaves
    ranges = [np.arange(plo, phi, dtype=np.int64)] + [np.arange(T.pbeg[b], T.pend[b], dtype=np.int64)
                                                      for b in leaves]
    pts = np.unique(np.concatenate(ranges)) if ranges else np.zeros(0, np.int64)
    return ghost.astype(np.int32), owner[ghost], pts


def rank_maps(T: GlobalTree, cuts: np.ndarray, caller_offsets: np.ndarray, rank: int) -> RankMaps:
    """Exchange lists of `rank`.  caller_offsets[c] = first global user row of
    caller rank c (length world + 1): the rows each caller passes to eval."""
    world = cuts.size - 1
    lo = _rank_of(cuts, T.pbeg)
    hi = _rank_of(cuts, np.maximum(T.pend - 1, T.pbeg))
    shared_mask = lo != hi
    shared = np.nonzero(shared_mask)[0].astype(np.int32)
    caller_of = lambda u: np.searchsorted(caller_offsets, u, side="right") - 1  # noqa: E731
    per = [_needed(T, cuts, q, shared_mask, lo) for q in range(world)]
    ue_send, ue_recv, val_send, val_recv, out_send, out_recv = [], [], [], [], [], []
    g_r, o_r, pts_r = per[rank]
    u_r = np.sort(T.perm[pts_r])
    own_users = np.sort(T.perm[cuts[rank]:cuts[rank + 1]])
    for q in range(world):
        g_q, o_q, pts_q = per[q]
        ue_send.append(g_q[o_q == rank])           # sorted box ids (np.unique)
        ue_recv.append(g_r[o_r == q])
        u_q = np.sort(T.perm[pts_q])
        val_send.append(u_q[caller_of(u_q) == rank] - caller_offsets[rank])
        val_recv.append(u_r[caller_of(u_r) == q])
        out_send.append(own_users[caller_of(own_users) == q])
        users_q = np.sort(T.perm[cuts[q]:cuts[q + 1]])
        out_recv.append(users_q[caller_of(users_q) == rank] - caller_offsets[rank])
    return RankMaps(rank, world, int(cuts[rank]), int(cuts[rank + 1]), shared, ue_send, ue_recv, val_send, val_recv,
                    out_send, out_recv)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------
class LocalTransport:
    """All ranks in this process: lists over ranks in, lists over ranks out."""

    def all_to_all(self, sends, recv_rows):
        world = len(sends)
        return [[sends[s][r] for s in range(world)] for r in range(world)]

    def all_reduce(self, bufs):
        tot = bufs[0].clone()
        for b in bufs[1:]:
            tot += b
        return [tot.clone() for _ in bufs]


class TorchTransport:
    """torch.distributed collectives for the one local rank (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def all_to_all(self, sends, recv_rows):
        import torch
        (chunks,), (rrows,) = sends, recv_rows
        width = chunks[0].shape[1] if chunks[0].dim() == 2 else 1
        send = torch.cat([c.reshape(-1) for c in chunks])
        out = torch.empty(int(sum(rrows)) * width, dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send, [int(r) * width for r in rrows],
                                    [int(c.shape[0]) * width for c in chunks], group=self.group)
        parts = torch.split(out, [int(r) * width for r in rrows])
        return [[p.reshape(-1, width) if chunks[0].dim() == 2 else p for p in parts]]

    def all_reduce(self, bufs):
        (b,) = bufs
        self.dist.all_reduce(b, group=self.group)
        return [b]


# ---------------------------------------------------------------------------
# one rank's side of the exchange, on the GPU plan
# ---------------------------------------------------------------------------
class RankPlan:
    """A restricted plan plus its exchange lists as device index tensors."""

    def __init__(self, plan, maps: RankMaps, n_local: int):
        import torch
        self.plan, self.maps, self.n_local = plan, maps, n_local
        inf = plan.info()
        self.k_s, self.k_t, self.neq, self.n = inf.k_s, inf.k_t, inf.n_equiv, inf.n_points
        dev = torch.device("cuda", torch.cuda.current_device())
        i64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=dev)  # noqa: E731
        i32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)  # noqa: E731
        self.val_send = [i64(a) for a in maps.val_send]
        self.val_recv = [i64(a) for a in maps.val_recv]
        self.out_send = [i64(a) for a in maps.out_send]
        self.out_recv = [i64(a) for a in maps.out_recv]
        self.ue_send = [i32(a) for a in maps.ue_send]
        self.ue_recv = [i32(a) for a in maps.ue_recv]
        self.shared = i32(maps.shared)
        self.gvals = torch.zeros((self.n, self.k_s), dtype=torch.float64, device=dev)
        self.gout = torch.zeros((self.n, self.k_t), dtype=torch.float64, device=dev)
        self.dev = dev

    def _rows(self, src, idx, width):
        import torch
        dst = torch.empty((idx.numel(), width), dtype=torch.float64, device=self.dev)
        if idx.numel():
            self.plan.gather_rows(src, idx, dst)
        return dst

    def _boxes(self, ids):
        import torch
        buf = torch.empty((ids.numel(), self.neq), dtype=torch.float64, device=self.dev)
        if ids.numel():
            self.plan.pack_ue(ids, buf)
        return buf

    # E1
    def pack_values(self, local_vals):
        return [self._rows(local_vals, i, self.k_s) for i in self.val_send]

    def values_rows(self):
        return [int(i.numel()) for i in self.val_recv]

    def unpack_values(self, recv):
        for buf, idx in zip(recv, self.val_recv):
            if idx.numel():
                self.plan.scatter_rows(buf.contiguous(), idx, self.gvals)

    def up(self):
        self.plan.eval_up(self.gvals)

    # E2 / E3
    def pack_shared(self):
        return self._boxes(self.shared)

    def unpack_shared(self, buf):
        if self.shared.numel():
            self.plan.unpack_ue(self.shared, buf.contiguous())

    def pack_ghost(self):
        return [self._boxes(i) for i in self.ue_send]

    def ghost_rows(self):
        return [int(i.numel()) for i in self.ue_recv]

    def unpack_ghost(self, recv):
        for buf, ids in zip(recv, self.ue_recv):
            if ids.numel():
                self.plan.unpack_ue(ids, buf.contiguous())

    def down(self):
        self.plan.eval_down(self.gout)

    # E4
    def pack_out(self):
        return [self._rows(self.gout, i, self.k_t) for i in self.out_send]

    def out_rows(self):
        return [int(i.numel()) for i in self.out_recv]

    def unpack_out(self, recv, local_out):
        for buf, idx in zip(recv, self.out_recv):
            if idx.numel():
                self.plan.scatter_rows(buf.contiguous(), idx, local_out)
        return local_out

    def new_out(self):
        import torch
        return torch.empty((self.n_local, self.k_t), dtype=torch.float64, device=self.dev)


def spmd_eval(ranks, transport, local_vals):
    """One distributed evaluation over the ranks of this process (all of
    them for LocalTransport, one for TorchTransport)."""
    recv = transport.all_to_all([r.pack_values(v) for r, v in zip(ranks, local_vals)],
                                [r.values_rows() for r in ranks])
    for r, rv in zip(ranks, recv):
        r.unpack_values(rv)
        r.up()
    sums = transport.all_reduce([r.pack_shared() for r in ranks])
    ghosts = transport.all_to_all([r.pack_ghost() for r in ranks], [r.ghost_rows() for r in ranks])
    for r, s, g in zip(ranks, sums, ghosts):
        r.unpack_shared(s)
        r.unpack_ghost(g)
        r.down()
    outs = transport.all_to_all([r.pack_out() for r in ranks], [r.out_rows() for r in ranks])
    return [r.unpack_out(o, r.new_out()) for r, o in zip(ranks, outs)]


def build_rank(global_points, caller_offsets, rank, world, kernel, p, cap, stream=None, weights=None):
    """Set up rank `rank` of `world` on the current GPU."""
    from .kafmm import KAFMM
    plan = KAFMM(global_points, kernel, p, cap, stream=stream)
    T = tree_from_plan(plan)
    cuts = partition(T, world, weights)
    maps = rank_maps(T, cuts, np.asarray(caller_offsets, dtype=np.int64), rank)
    plan.restrict(maps.plo, maps.phi)
    n_local = int(caller_offsets[rank + 1] - caller_offsets[rank])
    rp = RankPlan(plan, maps, n_local)
    rp.work = local_work(T, maps.plo, maps.phi)
    return rp, cuts


def local_work(T: GlobalTree, plo: int, phi: int) -> dict:
    """V pairs and P2P pairs this rank's restricted plan evaluates."""
    active = (T.pbeg < phi) & (T.pend > plo)
    vt, _ = T.lists["V"]
    ut, us = T.lists["U"]
    npts = T.pend - T.pbeg
    m = active[ut]
    return {"n_v": int(active[vt].sum()), "n_p2p": int((npts[ut[m]] * npts[us[m]]).sum())}


class DistKAFMM:
    """The distributed evaluation for this process's rank (torch.distributed
    initialised, one GPU per process).  local_points: this rank's rows."""

    def __init__(self, local_points, kernel: str, p: int, cap: int, group=None, stream=None):
        import torch
        import torch.distributed as dist
        self.transport = TorchTransport(group)
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        pts = torch.as_tensor(np.ascontiguousarray(local_points, dtype=np.float64)).cuda() \
            if isinstance(local_points, np.ndarray) else local_points.to("cuda", torch.float64).contiguous()
        cnt = torch.tensor([pts.shape[0]], dtype=torch.int64, device="cuda")
        counts = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(counts, cnt, group=group)
        counts = [int(c.item()) for c in counts]
        mx = max(counts)
        pad = torch.zeros((mx, 3), dtype=torch.float64, device="cuda")
        pad[:pts.shape[0]] = pts
        allp = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(allp, pad, group=group)
        gpts = torch.cat([a[:c] for a, c in zip(allp, counts)])
        offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.rank, self.world = rank, world
        self.ctx, self.cuts = build_rank(gpts, offsets, rank, world, kernel, p, cap, stream=stream)

    def eval(self, local_vals):
        return spmd_eval([self.ctx], self.transport, [local_vals.contiguous()])[0]
