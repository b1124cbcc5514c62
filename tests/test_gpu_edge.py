"""Edge cases of the CUDA path: degenerate trees, duplicates, boundaries,
invalid input, and properties that hold at any size."""
import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM, KafmmError

from .gpu_helpers import assert_parity, block_max_errors, run_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel", WL.KERNELS)
def test_single_point(kernel):
    pts = np.array([[0.3, 0.2, 0.9]])
    vals = WL.random_values(kernel, 1, 1)
    _, out = run_gpu(pts, vals, kernel, 4, 8)
    np.testing.assert_allclose(out, F.direct(kernel, pts, vals), rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("kernel", WL.KERNELS)
def test_single_leaf_equals_direct(kernel):
    pts = np.random.default_rng(2).random((300, 3))
    vals = WL.random_values(kernel, 300, 3)
    plan, out = run_gpu(pts, vals, kernel, 6, 300)
    assert plan.info().n_boxes == 1
    d = F.direct(kernel, pts, vals)
    assert F.rel_l2(out, d) < 1e-14


@pytest.mark.parametrize("kernel", ["laplace_pgrad", "stokes_reg_vel"])
def test_duplicate_points_and_zero_values(kernel):
    rng = np.random.default_rng(4)
    base = rng.random((700, 3))
    pts = np.concatenate([base, base[:300]])   # exact duplicates: r^2 == 0 pairs across indices
    vals = WL.random_values(kernel, 1000, 5)
    plan, out = run_gpu(pts, vals, kernel, 6, 24)
    ref = F.fmm(pts, vals, kernel, 6, 24)["out"]
    assert_parity(kernel, out, ref)
    z = np.zeros_like(vals)
    if z.shape[1] == 4:
        z[:, 3] = vals[:, 3]
    import torch
    assert float(plan.eval(torch.from_numpy(z).cuda()).abs().max()) == 0.0


def test_points_on_cell_boundaries_and_max_depth():
    # coordinates on dyadic planes (a point on a plane goes to the upper box) and a
    # tight cluster that forces the level-20 cap
    g = (np.arange(8) / 8.0)
    grid = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    tight = 0.5 + 1e-7 * np.random.default_rng(6).random((40, 3))
    pts = np.concatenate([grid, tight])
    vals = WL.random_values("stokeslet", pts.shape[0], 7)
    plan, out = run_gpu(pts, vals, "stokeslet", 5, 4)
    ref = F.fmm(pts, vals, "stokeslet", 5, 4)
    assert plan.info().depth == ref["tree"].depth == 20
    assert_parity("stokeslet", out, ref["out"])


def test_invalid_inputs_fail_loudly():
    pts = np.random.default_rng(8).random((100, 3))
    bad = pts.copy()
    bad[5, 1] = 1.0
    with pytest.raises(KafmmError) as e:
        KAFMM(bad, "stokeslet", 4, 10)
    assert e.value.status == 2   # KAFMM_EDOMAIN
    bad[5, 1] = np.nan
    with pytest.raises(KafmmError) as e:
        KAFMM(bad, "stokeslet", 4, 10)
    assert e.value.status == 3   # KAFMM_ENONFINITE
    import torch
    plan = KAFMM(pts, "rpy", 4, 10)
    v = torch.from_numpy(WL.random_values("rpy", 100, 9)).cuda()
    plan.check_values(v)
    v[3, 3] = -1.0
    with pytest.raises(KafmmError):
        plan.check_values(v)
    # the evaluation itself flags bad values without a host sync; kafmm_sync and
    # kafmm_eval_host report KAFMM_ENONFINITE once, then the flag is clear
    plan.eval(v)
    with pytest.raises(KafmmError) as e:
        plan.sync()
    assert e.value.status == 3
    plan.sync()
    good = WL.random_values("rpy", 100, 9)
    bad_v = good.copy()
    bad_v[7, 1] = np.inf
    with pytest.raises(KafmmError) as e:
        plan.eval_host(bad_v)
    assert e.value.status == 3
    plan.eval_host(good)
    plan.sync()


def test_superposition_and_scale_covariance_at_size():
    # linearity in the forces and exact power-of-two covariance hold at any size
    import torch
    spec, pts, vals = WL.make_config(1, n=20000)
    plan = KAFMM(pts, "stokeslet", 8, 50)
    v1 = torch.from_numpy(vals).cuda()
    v2 = torch.from_numpy(WL.random_values("stokeslet", 20000, 11)).cuda()
    a, b, c = plan.eval(v1), plan.eval(v2), plan.eval(v1 + 3 * v2)
    assert float((c - a - 3 * b).norm() / c.norm()) < 1e-11  # rounding x 1/sigma_min
    half = KAFMM(pts * 0.5, "stokeslet", 8, 50)
    h = half.eval(v1)
    assert float((h - 2 * a).norm() / h.norm()) < 1e-11


@pytest.mark.parametrize("kernel", WL.KERNELS)
def test_leaves_larger_than_one_thread_pass(kernel):
    # leaves of up to 1100 points: the leaf kernels run several target passes per
    # CTA (128 x TP targets each) over one shared source chunk; repeated evals agree
    import torch
    pts = np.concatenate([np.random.default_rng(8).random((1100, 3)) * 0.2 + 0.1,
                          np.random.default_rng(9).random((400, 3))])
    vals = WL.random_values(kernel, pts.shape[0], 10)
    plan, out = run_gpu(pts, vals, kernel, 5, 1100)
    src = torch.from_numpy(vals).cuda()
    for _ in range(3):
        again = plan.eval(src).cpu().numpy()
        assert F.rel_l2(again, out) < 1e-12
    ref = F.fmm(pts, vals, kernel, 5, 1100)["out"]
    assert_parity(kernel, out, ref)


@pytest.mark.parametrize("kernel", ["laplace_pgrad", "rpy"])
def test_overlapped_and_serialised_evaluations_agree(kernel):
    # timing mode 1 runs every stage on one stream; modes 0 and 2 overlap the near
    # field with the far field on a side stream (P2P stores, L2T/M2T add)
    import torch
    pts = np.random.default_rng(13).random((20000, 3))
    vals = WL.random_values(kernel, 20000, 14)
    plan, out0 = run_gpu(pts, vals, kernel, 6, 40)
    src = torch.from_numpy(vals).cuda()
    for mode in (1, 2, 0):
        plan.set_timing(mode)
        out = plan.eval(src).cpu().numpy()
        assert F.rel_l2(out, out0) < 1e-12
        if mode:
            st = plan.stage_times()
            assert st["total"] > 0 and st["m2l_product"] > 0
    plan.set_timing(0)


def test_cuda_graph_replay_matches_and_follows_inputs():
    import torch
    from paper_2010_15155_b200 import KAFMM
    pts = np.random.default_rng(15).random((6000, 3))
    v1 = WL.random_values("stokeslet", 6000, 16)
    v2 = WL.random_values("stokeslet", 6000, 17)
    plan = KAFMM(pts, "stokeslet", 6, 40)
    a = torch.from_numpy(v1).cuda()
    ref1 = plan.eval(a).cpu().numpy()
    plan.set_graph(True)
    out = torch.empty_like(a)
    for _ in range(3):                      # warm (uncaptured), capture, replay
        plan.eval(a, out)
        assert F.rel_l2(out.cpu().numpy(), ref1) < 1e-12
    a.copy_(torch.from_numpy(v2))           # same pointers, new values: the replay reads them
    plan.eval(a, out)
    ref2 = F.fmm(pts, v2, "stokeslet", 6, 40)["out"]
    assert_parity("stokeslet", out.cpu().numpy(), ref2)
    b = torch.from_numpy(v1).cuda()         # new pointer: re-captured
    assert F.rel_l2(plan.eval(b).cpu().numpy(), ref1) < 1e-12
    plan.set_graph(False)


@pytest.mark.parametrize("p", [2, 3, 9, 11])
def test_orders_outside_the_fft_set_and_tiny_orders(p):
    # p = 3 uses the FFT M2L (NG = 5); p = 2, 9, 11 fall back to the dense M2L
    import torch
    from paper_2010_15155_b200 import KAFMM
    pts = np.random.default_rng(20 + p).random((3000, 3))
    kernel = "stokeslet" if p <= 3 else "laplace_pgrad"   # dense Stokes operators at p = 11: 8 GB
    vals = WL.random_values(kernel, 3000, 21)
    plan = KAFMM(pts, kernel, p, 30)
    assert plan.m2l() == ("fft" if p == 3 else "dense")
    out = plan.eval(torch.from_numpy(vals).cuda()).cpu().numpy()
    ref = F.fmm(pts, vals, kernel, p, 30)["out"]
    assert_parity(kernel, out, ref)


@pytest.mark.parametrize("kernel", ["laplace_pgrad", "stokes_reg_vel_omega", "rpy"])
def test_separate_source_and_target_sets(kernel):
    import torch
    from paper_2010_15155_b200 import KAFMM2
    rng = np.random.default_rng(43)
    src = rng.random((4000, 3))
    trg = np.concatenate([0.2 + 0.5 * rng.random((2500, 3)), src[:100]])  # some targets on sources
    vals = WL.random_values(kernel, 4000, 44)
    plan = KAFMM2(src, trg, kernel, 6, 32)
    out = plan.eval(torch.from_numpy(vals).cuda()).cpu().numpy()
    assert out.shape == (trg.shape[0], WL.KERNEL_DIMS[kernel][1])
    union = np.concatenate([src, trg])
    uv = np.concatenate([vals, np.zeros((trg.shape[0], vals.shape[1]))])
    if kernel in WL.PARAM_COL and kernel != "rpy":
        uv[4000:, WL.PARAM_COL[kernel]] = 1.0   # reading R19: blob size of zero-strength target rows
    ref = F.fmm(union, uv, kernel, 6, 32)["out"][4000:]
    assert_parity(kernel, out, ref)
