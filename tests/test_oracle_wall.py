"""Pins for oracle/wall.py: RPY above a no-slip wall (Table X),
SURVEY.md §8(f) rank 4.  What the physics fixes: the velocity vanishes on the
wall; the RPY wall flow is (1 + b^2/6 lap_y) applied to the b = 0 wall
Stokeslet; the assembled lap u is the Laplacian of the assembled u; and the
FMM-evaluated image system converges to the direct one in p."""
import numpy as np
import pytest

from oracle import fmm as F
from oracle import wall as Wl


def _src(n, seed, bmax=0.05):
    rng = np.random.default_rng(seed)
    y = np.concatenate([rng.random((n, 2)) - 0.5, 0.05 + 0.4 * rng.random((n, 1))], axis=1)
    vals = np.concatenate([rng.standard_normal((n, 3)), bmax * rng.random((n, 1))], axis=1)
    return y, vals


def test_no_slip_on_the_wall():
    y, vals = _src(20, 1)
    rng = np.random.default_rng(2)
    xw = np.concatenate([rng.random((30, 2)) - 0.5, np.zeros((30, 1))], axis=1)
    u_wall = Wl.rpy_wall_direct(xw, y, vals)[:, :3]
    u_above = Wl.rpy_wall_direct(xw + np.array([0, 0, 0.2]), y, vals)[:, :3]
    assert np.abs(u_wall).max() < 1e-13 * np.abs(u_above).max()


def test_rpy_wall_is_laplacian_correction_of_wall_stokeslet():
    # u_RPY(x; y, b) = (1 + b^2/6 lap_y) u_G(x; y): finite differences in the source position
    rng = np.random.default_rng(3)
    x = np.array([[0.05, -0.1, 0.3]])
    for _ in range(3):
        y = np.array([rng.random(3) * np.array([0.4, 0.4, 0.3]) + np.array([-0.2, -0.2, 0.1])])
        f = rng.standard_normal(3)
        b = 0.04
        v0 = np.concatenate([f, [0.0]])[None]
        h = 3e-4
        lap = np.zeros(3)
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            lap += (Wl.rpy_wall_direct(x, y + e, v0)[0, :3] - 2 * Wl.rpy_wall_direct(x, y, v0)[0, :3]
                    + Wl.rpy_wall_direct(x, y - e, v0)[0, :3]) / h ** 2
        ref = Wl.rpy_wall_direct(x, y, v0)[0, :3] + b * b / 6 * lap
        got = Wl.rpy_wall_direct(x, y, np.concatenate([f, [b]])[None])[0, :3]
        # (with the Table X quadrupole at y instead of y^I the gap is ~5e-3: reading R18)
        assert np.abs(got - ref).max() < 1e-5 * np.abs(ref).max()


def test_assembled_laplacian_is_laplacian_of_u():
    y, vals = _src(6, 4)
    x = np.array([[0.1, 0.05, 0.25], [-0.2, 0.1, 0.4]])
    out = Wl.rpy_wall_direct(x, y, vals)

    def fd_lap(h):
        lap = np.zeros((2, 3))
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            lap += (Wl.rpy_wall_direct(x + e, y, vals)[:, :3] - 2 * out[:, :3]
                    + Wl.rpy_wall_direct(x - e, y, vals)[:, :3]) / h ** 2
        return lap

    lap = (4 * fd_lap(5e-4) - fd_lap(1e-3)) / 3  # Richardson: O(h^4)
    np.testing.assert_allclose(out[:, 3:], lap, rtol=1e-6, atol=1e-7 * np.abs(lap).max())


def test_wall_fmm_converges_to_direct():
    rng = np.random.default_rng(5)
    n = 800
    pts = np.concatenate([rng.random((n, 2)), 0.5 + 0.5 * rng.random((n, 1))], axis=1)
    vals = np.concatenate([rng.standard_normal((n, 3)), 1e-3 * rng.random((n, 1))], axis=1)
    y = pts - np.array([0, 0, 0.5])
    d = Wl.rpy_wall_direct(y, y, vals)
    errs = []
    for p in (4, 6, 8):
        out = Wl.rpy_wall_fmm(pts, vals, p, 40)
        errs.append(max(F.rel_l2(out[:, lo:hi], d[:, lo:hi]) for lo, hi in ((0, 3), (3, 6))))
    for e0, e1 in zip(errs, errs[1:]):
        assert e1 < e0 / 10.0, errs
