"""Multi-GPU evaluation of the KAFMM sum.

The product path is in libkafmm (csrc/kafmm_dist.cu, kafmm_comm.cu): the C ABI
kafmm_setup_dist / kafmm_eval with NCCL inside (``dist_plan`` below), or the
in-process test transport (``LocalDist``).  This module also holds the host
logic of the partition and exchange in plain numpy -- the specification the
C++ implementation follows and the GPU tests compare it with -- and the
transport-generic driver ``spmd_eval`` that tests/test_dist_host.py runs on gloo
process groups with the oracle's arithmetic per rank.

One process per GPU.  The octree is split into contiguous Morton ranges of
the sorted points (whole leaves), weighted by the work each point brings
(P2P pairs, W/X surface evaluations, S2M, M2L pairs).  Every rank builds the
same global tree and lists from the all-gathered points and keeps what its
range needs.  An evaluation is

    E1  all-to-all-v  source values, from the caller's rows to every rank that
                      needs them (its owned points and the remote leaves of
                      its U and X lists)
        up pass       S2M, UC2UE over owned leaves, M2M into active boxes
    E2  all-reduce    UE of the boxes that straddle ranks (partial sums)
    E3  all-to-all-v  ghost UE: remote boxes named by the V lists of this
                      rank's active boxes and the W lists of its leaves
        down pass     M2L, S2L, DC2DE, L2L, L2T, M2T, P2P, scatter
    E4  all-to-all-v  outputs, from the owning rank back to the caller's rows

The exchange maps are deterministic functions of the global tree, so every
rank derives the same send and receive lists without communicating them.
In ``spmd_eval`` the collectives go through a Transport: TorchTransport
(torch.distributed; gloo in the CPU tests) or LocalTransport (all ranks in one
process); nothing here computes the method's arithmetic.
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


def dist_plan(local_points, kernel: str, p: int, cap: int, group=None, stream=None):
    """This process's rank of a partitioned plan over torch.distributed's ranks
    (one GPU each): rank 0 makes the NCCL id, torch.distributed broadcasts it,
    and libkafmm sets up its own NCCL communicator (kafmm_setup_dist)."""
    import torch
    import torch.distributed as dist
    from .kafmm import DistKAFMM, unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = torch.zeros(128, dtype=torch.uint8, device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return DistKAFMM(local_points, kernel, p, cap, rank=rank, world=world, nccl_id=bytes(buf.cpu().numpy()),
                     stream=stream)


def _run_threads(fns):
    import threading
    res, err = [None] * len(fns), []

    def run(i):
        try:
            res[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return res


class LocalDist:
    """All ranks of a partitioned plan in this process, one host thread per rank
    on the current GPU (kafmm_comm_local_create): the test transport of the
    C-ABI multi-GPU path.  points[r] / values[r]: rank r's caller rows."""

    def __init__(self, points, kernel: str, p: int, cap: int):
        import torch
        from .kafmm import DistKAFMM, LocalComms
        self.world = len(points)
        self.comms = LocalComms(self.world)
        dev = torch.cuda.current_device()

        def mk(r):
            torch.cuda.set_device(dev)
            return DistKAFMM(points[r], kernel, p, cap, comm=self.comms.handles[r])

        self.plans = _run_threads([lambda r=r: mk(r) for r in range(self.world)])

    def eval(self, values):
        import torch
        dev = torch.cuda.current_device()

        def ev(r):
            torch.cuda.set_device(dev)
            out = self.plans[r].eval(values[r])
            self.plans[r].sync()
            return out

        return _run_threads([lambda r=r: ev(r) for r in range(self.world)])

    def close(self):
        for pl in self.plans:
            pl.close()
        self.plans = []
        self.comms.close()
