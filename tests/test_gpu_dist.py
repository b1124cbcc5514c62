"""The partitioned (multi-GPU) evaluation path of the C ABI on one GPU:
`world` ranks of kafmm_setup_dist_comm / kafmm_eval as host threads of this
process over the in-process transport (kafmm_comm_local_create) -- the same
library code as the NCCL ranks except the collective calls.  Ranks never wait
on each other on the device, only at host barriers.

Checks: the assembled result equals the single-GPU plan (1e-12) and the oracle
FMM; the library's Morton cuts and per-peer exchange counts equal the
reference host logic (paper_2010_15155_b200/dist.py, which the gloo tests run
with the oracle's arithmetic); per-rank plan memory falls with the rank count
on a C5-shaped cloud."""
import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM
from paper_2010_15155_b200 import dist as D

from .gpu_helpers import assert_parity

pytestmark = pytest.mark.gpu


def _clustered(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.random((4, 3)) * 0.8 + 0.1
    pts = np.concatenate([c[i] + 0.03 * rng.standard_normal((n // 4, 3)) for i in range(4)])
    return np.clip(pts, 0.0, np.nextafter(1.0, 0.0))


CASES = [("stokeslet", lambda: _clustered(8000, 11), 6, 40),
         ("laplace_pgrad", lambda: np.random.default_rng(12).random((12000, 3)), 8, 32),
         ("rpy", lambda: _clustered(6000, 13), 5, 30)]


def _reference_counts(single, world, offs, kernel):
    """Cuts and per-peer row counts from the reference host logic (dist.py)."""
    T = D.tree_from_plan(single)
    cuts = D.partition(T, world)
    maps = [D.rank_maps(T, cuts, offs, r) for r in range(world)]
    return cuts, maps


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_partitioned_equals_single_plan_and_oracle(case, world):
    import torch
    kernel, mk, p, cap = case
    pts = mk()
    n = pts.shape[0]
    vals = WL.random_values(kernel, n, 21)
    src = torch.from_numpy(vals).cuda()
    single = KAFMM(pts, kernel, p, cap)
    ref_gpu = single.eval(src).cpu().numpy()
    offs = np.linspace(0, n, world + 1).astype(np.int64)  # callers hold contiguous user rows
    cuts_ref, maps = _reference_counts(single, world, offs, kernel)
    single.close()
    ld = D.LocalDist([pts[offs[r]:offs[r + 1]] for r in range(world)], kernel, p, cap)
    try:
        outs = ld.eval([src[offs[r]:offs[r + 1]] for r in range(world)])
        got = torch.cat(outs).cpu().numpy()
        infos = [pl.dist_info() for pl in ld.plans]
        outs2 = ld.eval([src[offs[r]:offs[r + 1]] for r in range(world)])  # a second evaluation: same buffers
        got2 = torch.cat(outs2).cpu().numpy()
    finally:
        ld.close()
    errs = [F.rel_l2(got[:, lo:hi], ref_gpu[:, lo:hi]) for lo, hi in F.blocks(kernel)]
    assert max(errs) < 1e-12, errs
    assert np.max(np.abs(got2 - got)) <= 1e-12 * np.max(np.abs(got))
    ref = F.fmm(pts, vals, kernel, p, cap)["out"]
    assert_parity(kernel, got, ref)
    # the library's partition and exchange lists are the reference host logic's
    for r, inf in enumerate(infos):
        assert inf["rank"] == r and inf["world"] == world and inf["n_global"] == n
        assert np.array_equal(inf["cuts"], cuts_ref), (inf["cuts"], cuts_ref)
        m = maps[r]
        assert list(inf["ue_send"]) == [a.size for a in m.ue_send]
        assert list(inf["ue_recv"]) == [a.size for a in m.ue_recv]
        assert list(inf["out_send"]) == [a.size for a in m.out_send]
        assert list(inf["out_recv"]) == [a.size for a in m.out_recv]
        assert inf["n_owned"] == cuts_ref[r + 1] - cuts_ref[r]
        assert inf["n_shared"] == maps[0].shared.size > 0
        # values: the reference sends every needed row (owned + remote leaves)
        assert inf["val_recv"].sum() == inf["n_local"]
        assert list(inf["val_recv"]) == [a.size for a in m.val_recv]


def test_partitioned_world_one_and_empty_rank():
    """world 1 through the dist path, and a rank with no caller rows."""
    import torch
    pts = _clustered(5000, 17)
    vals = WL.random_values("stokeslet", 5000, 3)
    src = torch.from_numpy(vals).cuda()
    single = KAFMM(pts, "stokeslet", 5, 30)
    ref = single.eval(src).cpu().numpy()
    single.close()
    ld = D.LocalDist([pts], "stokeslet", 5, 30)
    try:
        got = ld.eval([src])[0].cpu().numpy()
    finally:
        ld.close()
    assert F.rel_l2(got, ref) < 1e-13
    ld = D.LocalDist([pts[:0], pts], "stokeslet", 5, 30)  # rank 0 passes no rows
    try:
        outs = ld.eval([src[:0], src])
    finally:
        ld.close()
    assert outs[0].shape == (0, 3)
    assert F.rel_l2(outs[1].cpu().numpy(), ref) < 1e-12


def test_plan_memory_falls_with_ranks_on_sphere_surfaces():
    """C5-shaped cloud (points on sphere surfaces, p = 8, cap 128), reduced N:
    the largest rank's plan at world 4 holds <= 0.4x the world-1 plan's bytes."""
    import torch
    spec, pts, vals = WL.make_config(5, n=1_000_000, n_spheres=1000)
    n = pts.shape[0]
    nb = {}
    for world in (1, 4):
        offs = np.linspace(0, n, world + 1).astype(np.int64)
        ld = D.LocalDist([pts[offs[r]:offs[r + 1]] for r in range(world)], spec.kernel, spec.p, spec.cap)
        try:
            infos = [pl.dist_info() for pl in ld.plans]
            if world == 4:
                src = torch.from_numpy(vals).cuda()
                outs = ld.eval([src[offs[r]:offs[r + 1]] for r in range(world)])
                assert all(bool(torch.isfinite(o).all()) for o in outs)
        finally:
            ld.close()
        nb[world] = max(i["plan_bytes"] for i in infos)
    assert nb[4] <= 0.4 * nb[1], nb
