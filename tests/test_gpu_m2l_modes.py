"""The M2L variants of the CUDA path (option b chosen by
measurement): dense per-offset GEMMs, and the FFT lattice convolution with
its frequency-space product as DMMA parent blocks or per V pair.  They apply
the same matrices, so they must agree to rounding and each match the oracle."""
import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM

from .gpu_helpers import assert_parity

pytestmark = pytest.mark.gpu


def _clustered(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.random((4, 3)) * 0.8 + 0.1
    pts = np.concatenate([c[i] + 0.02 * rng.standard_normal((n // 4, 3)) for i in range(4)])
    return np.clip(pts, 0.0, np.nextafter(1.0, 0.0))


CASES = [("stokeslet", lambda: _clustered(6000, 31), 6, 30),
         ("laplace_pgrad", lambda: np.random.default_rng(32).random((20000, 3)), 8, 40),
         ("rpy", lambda: WL.make_points(WL.CONFIGS[5], 9000, n_spheres=40), 5, 40),
         ("stokes_reg_vel", lambda: _clustered(5000, 33), 12, 40),
         ("laplace_pgradgrad", lambda: _clustered(6000, 34), 4, 30),
         ("stokes_reg_vel_omega", lambda: _clustered(5000, 35), 7, 40),
         ("laplace_qpgradgrad", lambda: np.random.default_rng(36).random((8000, 3)), 3, 30)]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_m2l_variants_agree(case):
    import torch
    kernel, mk, p, cap = case
    pts = mk()
    vals = WL.random_values(kernel, pts.shape[0], 41)
    plan = KAFMM(pts, kernel, p, cap)
    src = torch.from_numpy(vals).cuda()
    res = {}
    for mode in ("dense", "fft", "fft_blocks", "fft_pairs"):
        plan.set_m2l(mode)
        assert plan.m2l() == mode
        res[mode] = plan.eval(src).cpu().numpy()
    ref = F.fmm(pts, vals, kernel, p, cap)["out"]
    for mode, out in res.items():
        for lo, hi in F.blocks(kernel):
            assert F.rel_l2(out[:, lo:hi], res["dense"][:, lo:hi]) < 1e-12, mode
        assert_parity(kernel, out, ref)


@pytest.mark.parametrize("case", [CASES[0], CASES[2], CASES[5]], ids=["stokeslet", "rpy_spheres", "regvelomega"])
def test_sparse_products_agree(case, monkeypatch):
    """k_m2l_groups (operator loaded once per offset of a (unit, colleague, x half) group)
    and k_m2l_items (once per V pair) on every FFT chunk: same products, so rounding-level
    agreement, and both match the oracle (KAFMM_SPARSE is read at plan setup)."""
    import torch
    kernel, mk, p, cap = case
    pts = mk()
    vals = WL.random_values(kernel, pts.shape[0], 43)
    src = torch.from_numpy(vals).cuda()
    res = {}
    for mode in ("items", "groups"):
        monkeypatch.setenv("KAFMM_SPARSE", mode)
        plan = KAFMM(pts, kernel, p, cap)
        plan.set_m2l("fft_pairs")
        res[mode] = plan.eval(src).cpu().numpy()
        plan.close()
    ref = F.fmm(pts, vals, kernel, p, cap)["out"]
    for lo, hi in F.blocks(kernel):
        assert F.rel_l2(res["groups"][:, lo:hi], res["items"][:, lo:hi]) < 1e-12
    assert_parity(kernel, res["groups"], ref)


@pytest.mark.parametrize("kernel,p", [("stokeslet", 6), ("laplace_pgrad", 5)])
def test_groups_dynamic_ranges(kernel, p, monkeypatch):
    """k_m2l_groups takes ranges of unit positions from a per-CTA counter; at test sizes a
    warp slot has a single range, so KAFMM_GROUP_CHUNK=1 (one unit position per range)
    forces dozens of dynamically taken ranges per CTA.  Same arithmetic per unit, so the
    two layouts agree to rounding (M2M accumulates with atomics: not bitwise), and match
    the oracle."""
    import torch
    pts = WL.make_points(WL.CONFIGS[5], 30000, n_spheres=12)
    vals = WL.random_values(kernel, pts.shape[0], 47)
    src = torch.from_numpy(vals).cuda()
    res = {}
    for ck in ("1", "64"):
        monkeypatch.setenv("KAFMM_GROUP_CHUNK", ck)
        plan = KAFMM(pts, kernel, p, 40)
        plan.set_m2l("fft_pairs")
        res[ck] = plan.eval(src).cpu().numpy()
        st = plan.fft_stats()
        plan.close()
    assert st["items"] > 0
    for lo, hi in F.blocks(kernel):
        assert F.rel_l2(res["1"][:, lo:hi], res["64"][:, lo:hi]) < 1e-12
    ref = F.fmm(pts, vals, kernel, p, 40)["out"]
    assert_parity(kernel, res["1"], ref)
