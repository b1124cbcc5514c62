"""Multi-GPU host logic on CPU: the Morton-range partition,
the exchange lists of every rank, and the distributed evaluation driver
(paper_2010_15155_b200.dist.spmd_eval) with the oracle's arithmetic standing
in for the GPU passes -- in one process (LocalTransport) and as world-size-2
gloo process groups (TorchTransport, the transport the GPUs use over NCCL).
The distributed result must equal the single-process oracle KIFMM to
rounding: the partition changes who computes what, not what is computed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fmm as F
from paper_2010_15155_b200 import dist as D

from .dist_oracle_rank import OracleRank, global_tree_from_oracle


def _cloud(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.random((3, 3)) * 0.6 + 0.2
    pts = np.concatenate([c[i] + 0.05 * rng.standard_normal((n // 3, 3)) for i in range(3)])
    pts = np.concatenate([pts, rng.random((n - pts.shape[0], 3))])
    return np.clip(pts, 0.0, np.nextafter(1.0, 0.0))


CASE = dict(kernel="stokeslet", n=900, cap=12, p=4, seed=3)


@pytest.fixture(scope="module")
def setup():
    pts = _cloud(CASE["n"], CASE["seed"])
    vals = np.random.default_rng(9).standard_normal((pts.shape[0], 3))
    t, T, L = global_tree_from_oracle(pts, CASE["cap"], CASE["p"], 3)
    ref = F.fmm(pts, vals, CASE["kernel"], CASE["p"], CASE["cap"], tree=t)["out"]
    return pts, vals, t, T, L, ref


def test_partition_cuts_whole_leaves_and_balances(setup):
    _, _, t, T, _, _ = setup
    w = D.point_weights(T)
    assert w.shape == (T.n,) and np.all(w > 0)
    for world in (1, 2, 3, 5, 8):
        cuts = D.partition(T, world)
        assert cuts[0] == 0 and cuts[-1] == T.n and np.all(np.diff(cuts) >= 0)
        leaf_starts = set(T.pbeg[T.leaf].tolist()) | {T.n}
        assert all(int(c) in leaf_starts for c in cuts)
        if world <= 3:  # coarse leaves limit the balance only for many ranks
            parts = [w[cuts[r]:cuts[r + 1]].sum() for r in range(world)]
            assert max(parts) <= 1.6 * w.sum() / world


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exchange_lists_agree_between_ranks(setup, world):
    _, _, t, T, _, _ = setup
    cuts = D.partition(T, world)
    n = T.n
    offs = np.linspace(0, n, world + 1).astype(np.int64)  # callers hold contiguous user rows
    maps = [D.rank_maps(T, cuts, offs, r) for r in range(world)]
    for r in range(world):
        assert np.array_equal(maps[r].shared, maps[0].shared)
        for q in range(world):
            assert np.array_equal(maps[r].ue_send[q], maps[q].ue_recv[r])
            assert np.array_equal(maps[r].val_send[q] + offs[r], maps[q].val_recv[r])
            assert np.array_equal(maps[r].out_send[q], maps[q].out_recv[r] + offs[q])
    # every point's output reaches its caller exactly once
    got = np.concatenate([m.out_recv[q] + offs[m.rank] for m in maps for q in range(world)])
    assert np.array_equal(np.sort(got), np.arange(n))
    # the shared boxes are exactly the boxes whose points span several ranks
    lo = np.searchsorted(cuts, T.pbeg, side="right") - 1
    hi = np.searchsorted(cuts, T.pend - 1, side="right") - 1
    assert set(maps[0].shared.tolist()) == set(np.nonzero(lo != hi)[0].tolist())
    # a ghost box is wholly owned by its sender and not active on the receiver
    for r in range(world):
        for q in range(world):
            for b in maps[r].ue_recv[q]:
                assert cuts[q] <= T.pbeg[b] and T.pend[b] <= cuts[q + 1]


@pytest.mark.parametrize("world", [2, 3])
def test_spmd_eval_local_transport_equals_oracle(setup, world):
    pts, vals, t, T, L, ref = setup
    n = T.n
    cuts = D.partition(T, world)
    offs = np.linspace(0, n, world + 1).astype(np.int64)
    ranks = []
    for r in range(world):
        m = D.rank_maps(T, cuts, offs, r)
        ranks.append(OracleRank(t, T, L, m, pts, CASE["kernel"], CASE["p"], int(offs[r + 1] - offs[r])))
    outs = D.spmd_eval(ranks, D.LocalTransport(), [vals[offs[r]:offs[r + 1]] for r in range(world)])
    got = np.concatenate(outs)
    assert F.rel_l2(got, ref) < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_rank(rank, world, port, pts, vals, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, T, L = global_tree_from_oracle(pts, CASE["cap"], CASE["p"], 3)
        cuts = D.partition(T, world)
        offs = np.linspace(0, T.n, world + 1).astype(np.int64)
        m = D.rank_maps(T, cuts, offs, rank)
        me = OracleRank(t, T, L, m, pts, CASE["kernel"], CASE["p"], int(offs[rank + 1] - offs[rank]))
        (out,) = D.spmd_eval([me], D.TorchTransport(), [vals[offs[rank]:offs[rank + 1]]])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_spmd_eval_gloo_equals_oracle(setup, world):
    pts, vals, _, _, _, ref = setup
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rank, args=(r, world, port, pts, vals, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r] for r in range(world)])
    assert F.rel_l2(got, ref) < 1e-12
