"""Pins for oracle/kernels.py (O1): closed forms, identities, special cases.

None of these re-types the oracle's formula: each checks it against a
different fact (a hand-worked value, a finite-difference derivative, the
defining equation of a derived kernel, a symmetry or a limit).
"""
import os

import numpy as np
import pytest

from oracle.kernels import DIMS, direct_sum, kernel_matrix, pair_values

GOLD = os.path.join(os.path.dirname(__file__), "golden", "kernel_values.txt")


def _golden_rows():
    rows = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, r, s, g, cite = [p.strip() for p in line.split("|")]
        rows.append((name, np.array(r.split(), float), np.array(s.split(), float),
                     np.array(g.split(), float), cite))
    return rows


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: f"{r[0]}@{r[4]}")
def test_golden_closed_form(row):
    name, r, s, g, _ = row
    out = pair_values(name, r, s)
    np.testing.assert_allclose(out, g, rtol=1e-15, atol=1e-17)


def _fd_grad(f, x, h):
    """4th-order central differences of a vector function along each axis."""
    cols = []
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        cols.append((-f(x + 2 * e) + 8 * f(x + e) - 8 * f(x - e) + f(x - 2 * e)) / (12 * h))
    return np.stack(cols, axis=-1)  # (..., comp, axis)


def _fd_lap(f, x, h):
    acc = 0.0
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        acc = acc + (-f(x + 2 * e) + 16 * f(x + e) - 30 * f(x) + 16 * f(x - e) - f(x - 2 * e)) / (12 * h * h)
    return acc


RNG = np.random.default_rng(7)
RS = [RNG.standard_normal(3) * s for s in (0.3, 1.0, 3.0)]


@pytest.mark.parametrize("r", RS)
def test_laplace_gradient_is_grad_of_potential(r):
    # grad_x phi with the sign rule d/dx = -d/dy
    q = np.array([1.7])
    phi = lambda x: pair_values("L", x, q)
    fd = _fd_grad(phi, r, 1e-4 * max(np.linalg.norm(r), 1))[0]
    an = pair_values("L+gradL", r, q)
    np.testing.assert_allclose(an[0], phi(r)[0], rtol=1e-15)
    np.testing.assert_allclose(an[1:], fd, rtol=1e-6)


@pytest.mark.parametrize("r", RS)
def test_stokeslet_divergence_free_and_symmetric(r):
    h = 1e-3 * np.linalg.norm(r)
    for b in range(3):
        f = np.zeros(3)
        f[b] = 1.0
        J = _fd_grad(lambda x: pair_values("G", x, f), r, h)
        assert abs(np.trace(J)) < 1e-7 * np.abs(J).max()
    K = kernel_matrix("G", r[None, :], np.zeros((1, 3)))
    np.testing.assert_allclose(K, K.T, rtol=0, atol=1e-16)
    K2 = kernel_matrix("G", -r[None, :], np.zeros((1, 3)))
    np.testing.assert_allclose(K, K2, rtol=1e-15)


@pytest.mark.parametrize("r", RS)
def test_lapG_is_laplacian_of_stokeslet_and_biharmonic(r):
    f = np.array([0.3, -1.1, 0.8])
    h = 1e-3 * np.linalg.norm(r)
    u = lambda x: pair_values("G", x, f)
    lap_fd = _fd_lap(u, r, h)
    lap = pair_values("G+lapG", r, f)[3:]
    np.testing.assert_allclose(lap, lap_fd, rtol=1e-6 * 1e3, atol=1e-6 * np.abs(lap).max())
    # lap lap G = 0: Laplacian of the analytic lap G vanishes
    bih = _fd_lap(lambda x: pair_values("G+lapG", x, f)[..., 3:], r, h)
    assert np.abs(bih).max() < 1e-5 * np.abs(lap).max() / np.dot(r, r)


@pytest.mark.parametrize("r", RS)
def test_rpy_is_one_plus_b2_over_6_lap_on_G(r):
    # Eq. (RPYkernel): G^RPY = (1 + b^2/6 lap) G, lap G by finite differences
    f = np.array([0.3, -1.1, 0.8])
    b = 0.2 * np.linalg.norm(r)
    u = lambda x: pair_values("G", x, f)
    expect = u(r) + b * b / 6.0 * _fd_lap(u, r, 1e-3 * np.linalg.norm(r))
    got = pair_values("G_RPY", r, np.r_[f, b])
    np.testing.assert_allclose(got, expect, rtol=1e-7)


def test_rpy_special_cases():
    rng = np.random.default_rng(3)
    r = rng.standard_normal((50, 3))
    f = rng.standard_normal((50, 3))
    g = pair_values("G", r, f)
    # b = 0 reduces exactly to the Stokeslet
    np.testing.assert_array_equal(pair_values("G_RPY", r, np.c_[f, np.zeros(50)]), g)
    # lap u is independent of b (lap lap G = 0)
    a1 = pair_values("G_RPY+lapG", r, np.c_[f, np.full(50, 0.01)])
    a2 = pair_values("G_RPY+lapG", r, np.c_[f, np.full(50, 0.3)])
    np.testing.assert_array_equal(a1[:, 3:], a2[:, 3:])
    np.testing.assert_array_equal(a1[:, 3:], pair_values("G+lapG", r, f)[:, 3:])
    # far field -> Stokeslet, difference O(b^2/r^2)
    rr = r * 100.0
    d = pair_values("G_RPY", rr, np.c_[f, np.full(50, 0.01)]) - pair_values("G", rr, f)
    assert np.abs(d).max() < 1e-7 * np.abs(pair_values("G", rr, f)).max()


def test_regularized_stokeslet_limits():
    rng = np.random.default_rng(4)
    r = rng.standard_normal((50, 3))
    f = rng.standard_normal((50, 3))
    # eps = 0 -> the singular Stokeslet (r != 0)
    np.testing.assert_allclose(pair_values("G_eps", r, np.c_[f, np.zeros(50)]),
                               pair_values("G", r, f), rtol=1e-14)
    # G^eps - G^RPY(b^2 = 1.5 eps^2) = O((eps/r)^4)
    rr = r / np.linalg.norm(r, axis=1, keepdims=True)
    errs = []
    for eps in (1e-1, 5e-2):
        d = pair_values("G_eps", rr, np.c_[f, np.full(50, eps)]) - pair_values(
            "G_RPY", rr, np.c_[f, np.full(50, np.sqrt(1.5) * eps)])
        errs.append(np.abs(d).max())
    assert 12.0 < errs[0] / errs[1] < 20.0  # fourth order: 2^4 = 16


def test_regularized_stokeslet_divergence_free_and_blob_mass():
    # incompressible regularized flow: div(G^eps f) = 0
    r = np.array([0.02, -0.01, 0.015])
    f = np.array([0.3, -1.1, 0.8])
    J = _fd_grad(lambda x: pair_values("G_eps", x, np.r_[f, 0.01]), r, 1e-4)
    assert abs(np.trace(J)) < 1e-7 * np.abs(J).max()
    # blob psi^eps integrates to 1: radial quadrature
    eps = 0.3
    from scipy.integrate import quad
    val, _ = quad(lambda s: 4 * np.pi * s * s * 15 * eps ** 4 / (8 * np.pi * (s * s + eps * eps) ** 3.5), 0, np.inf)
    assert abs(val - 1.0) < 1e-10


def test_self_pairs_skipped_for_singular_kept_for_regularized():
    z = np.zeros(3)
    for name in ("L", "L+gradL", "G", "G_RPY", "G_RPY+lapG", "G+lapG"):
        s = np.ones(DIMS[name][0])
        assert np.all(pair_values(name, z, s) == 0.0)
    assert np.all(pair_values("G_eps", z, np.array([1.0, 0, 0, 0.1]))[0] > 0)


def test_direct_sum_superposition_permutation_reciprocity():
    rng = np.random.default_rng(5)
    y = rng.random((300, 3))
    f1 = rng.standard_normal((300, 3))
    f2 = rng.standard_normal((300, 3))
    a = direct_sum("G", y, y, f1)
    b = direct_sum("G", y, y, f2)
    np.testing.assert_allclose(direct_sum("G", y, y, f1 + 2 * f2), a + 2 * b, rtol=1e-12, atol=1e-12)
    perm = rng.permutation(300)
    np.testing.assert_allclose(direct_sum("G", y[perm], y[perm], f1[perm]), a[perm], rtol=1e-12)
    # reciprocity of the symmetric mobility: f1 . (M f2) = f2 . (M f1)
    assert abs(np.sum(f1 * b) - np.sum(f2 * a)) < 1e-11 * abs(np.sum(f1 * b))
    # same for RPY (symmetric positive definite mobility)
    v1 = np.c_[f1, np.full(300, 1e-3)]
    v2 = np.c_[f2, np.full(300, 1e-3)]
    ra = direct_sum("G_RPY", y, y, v1)
    rb = direct_sum("G_RPY", y, y, v2)
    assert abs(np.sum(f1 * rb) - np.sum(f2 * ra)) < 1e-11 * abs(np.sum(f1 * rb))


def test_direct_sum_two_opposite_charges_and_scalar_loop():
    y = np.array([[0.2, 0.5, 0.5], [0.8, 0.5, 0.5]])
    q = np.array([[1.0], [-1.0]])
    x = np.array([[0.5, 0.1, 0.9], [0.5, 0.7, 0.3]])   # on the bisecting plane
    assert np.all(np.abs(direct_sum("L", x, y, q)) < 1e-16)
    # scalar double loop over pairs (no broadcasting) agrees with the vectorised sum
    rng = np.random.default_rng(8)
    X = rng.random((7, 3))
    Y = np.r_[rng.random((9, 3)), X[:2]]
    V = np.c_[rng.standard_normal((11, 3)), np.full(11, 0.05)]
    for name in ("G_RPY+lapG", "G_eps", "L+gradL"):
        vv = V[:, : DIMS[name][0]]
        ref = np.zeros((7, DIMS[name][1]))
        for i in range(7):
            for j in range(11):
                ref[i] += pair_values(name, X[i] - Y[j], vv[j])
        np.testing.assert_allclose(direct_sum(name, X, Y, vv), ref, rtol=1e-13, atol=1e-13)


# ---- StokesRegVelOmega, Table VI --------------------------
def _ft(rng):
    return rng.standard_normal(3), rng.standard_normal(3)


def _curl(fun, x, h=1e-5):
    J = np.zeros((3, 3))
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        J[:, k] = (fun(x + e) - fun(x - e)) / (2 * h)
    return np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])


@pytest.mark.parametrize("eps", [0.0, 0.3, 1.0])
def test_reg_vel_omega_is_half_curl_of_velocity(eps):
    # omega = (1/2) curl u for both the force and the torque parts (Omega = curl G / 2,
    # W = curl T / 2): a property of the blob-regularized flows, not of how they are coded
    rng = np.random.default_rng(21)
    for _ in range(3):
        r = rng.standard_normal(3)
        f, t = _ft(rng)
        for s in (np.concatenate([f, 0 * t, [eps]]), np.concatenate([0 * f, t, [eps]])):
            u = lambda x: pair_values("G_eps+Omega+T+W", x, s)[:3]  # noqa: E731
            w = pair_values("G_eps+Omega+T+W", r, s)[3:]
            np.testing.assert_allclose(w, 0.5 * _curl(u, r), rtol=1e-7, atol=1e-9)


def test_reg_vel_omega_limits_and_pieces():
    rng = np.random.default_rng(22)
    r = rng.standard_normal((50, 3))
    f = rng.standard_normal((50, 3))
    t = rng.standard_normal((50, 3))
    eps = 0.2 * rng.random(50)
    s7 = np.concatenate([f, t, eps[:, None]], axis=1)
    full = pair_values("G_eps+Omega+T+W", r, s7)
    # S-row kernel = the velocity block of the S->T kernel
    np.testing.assert_array_equal(pair_values("G_eps+T_eps", r, s7), full[:, :3])
    # no torque: the velocity is the regularized Stokeslet G_eps
    s0 = np.concatenate([f, 0 * t, eps[:, None]], axis=1)
    np.testing.assert_allclose(pair_values("G_eps+Omega+T+W", r, s0)[:, :3],
                               pair_values("G_eps", r, np.concatenate([f, eps[:, None]], axis=1)), rtol=1e-14)
    # eps -> 0 with no torque is the singular G (+) Omega of the T column
    z = np.concatenate([f, 0 * t, 0 * eps[:, None]], axis=1)
    np.testing.assert_allclose(pair_values("G_eps+Omega+T+W", r, z), pair_values("G+Omega", r, f), rtol=1e-13)


def test_reg_vel_omega_worked_values_and_self_term():
    # r = (1,0,0), eps = 0, torque t = (0,0,1): u = Q/2 (t x r), Q(1) = 2/(8 pi) -> u = (0, 1/(8 pi), 0)
    s = np.array([0, 0, 0, 0, 0, 1.0, 0.0])
    np.testing.assert_allclose(pair_values("G_eps+Omega+T+W", np.array([1.0, 0, 0]), s)[:3],
                               [0, 1 / (8 * np.pi), 0], atol=1e-17)
    # self term r = 0: H1(0) = 1/(4 pi eps), D1(0)/4 = 10/(32 pi eps^3), Q-terms vanish
    eps = 0.5
    f, t = np.array([1.0, 2, 3]), np.array([-1.0, 0.5, 2])
    got = pair_values("G_eps+Omega+T+W", np.zeros(3), np.concatenate([f, t, [eps]]))
    np.testing.assert_allclose(got[:3], f / (4 * np.pi * eps), rtol=1e-15)
    np.testing.assert_allclose(got[3:], 10 * t / (32 * np.pi * eps ** 3), rtol=1e-15)


def test_reg_vel_omega_mobility_is_symmetric():
    # two blobs with the same eps: the 12x12 mobility [u1, w1, u2, w2] <- [f1, t1, f2, t2] is symmetric
    rng = np.random.default_rng(23)
    x = rng.standard_normal((2, 3))
    eps = 0.3
    Mb = np.zeros((12, 12))
    for j in range(12):
        s = np.zeros((2, 7))
        s[:, 6] = eps
        s[j // 6, j % 6] = 1.0
        for a in range(2):
            Mb[6 * a:6 * a + 6, j] = sum(pair_values("G_eps+Omega+T+W", x[a] - x[b], s[b]) for b in range(2))
    np.testing.assert_allclose(Mb, Mb.T, rtol=0, atol=1e-14)


# ---- LapPGradGrad, Table III ------------------------------
def test_pgradgrad_derivatives_and_harmonicity():
    rng = np.random.default_rng(31)
    h = 1e-5
    for _ in range(4):
        r = rng.standard_normal(3)
        s = rng.standard_normal(4)
        v = pair_values("LD+gradLD+gradgradLD", r, s)
        # grad phi and grad grad phi are the target derivatives of phi and grad phi
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            dv = (pair_values("LD+gradLD+gradgradLD", r + e, s) - pair_values("LD+gradLD+gradgradLD", r - e, s)) / (2 * h)
            np.testing.assert_allclose(dv[0], v[1 + k], rtol=1e-7, atol=1e-9)
            H = {(0, 0): 4, (0, 1): 5, (0, 2): 6, (1, 1): 7, (1, 2): 8, (2, 2): 9}
            for j in range(3):
                np.testing.assert_allclose(dv[1 + j], v[H[tuple(sorted((j, k)))]], rtol=1e-6, atol=1e-8)
        # phi is harmonic away from the source: trace of grad grad phi = 0
        assert abs(v[4] + v[7] + v[9]) < 1e-12 * np.abs(v[4:]).max()


def test_dipole_is_limit_of_charge_pair():
    # L^D_j = -dL/dx_j: a dipole d at y is the limit of charges +1/h at
    # y + h d / 2 and -1/h at y - h d / 2
    rng = np.random.default_rng(32)
    r = rng.standard_normal(3)
    d = rng.standard_normal(3)
    h = 1e-5
    pair = (pair_values("L+gradL+gradgradL", r - 0.5 * h * d, np.array([1.0]))
            - pair_values("L+gradL+gradgradL", r + 0.5 * h * d, np.array([1.0]))) / h
    dip = pair_values("LD+gradLD+gradgradLD", r, np.concatenate([[0.0], d]))
    np.testing.assert_allclose(dip, pair, rtol=1e-5, atol=1e-7)
    # charges only: the S->T kernel reduces to the T-column kernel, and the S row to L + L^D's phi
    q = np.array([1.7, 0, 0, 0])
    np.testing.assert_allclose(pair_values("LD+gradLD+gradgradLD", r, q), pair_values("L+gradL+gradgradL", r, q[:1]),
                               rtol=1e-15)
    sd = np.concatenate([[0.3], d])
    np.testing.assert_allclose(pair_values("L+LD", r, sd), pair_values("LD+gradLD+gradgradLD", r, sd)[:1], rtol=1e-15)
    # worked value: dipole d = (0, 0, 4 pi) at r = (0, 0, 2): phi = d.r/(4 pi r^3) = 1/4
    np.testing.assert_allclose(pair_values("L+LD", np.array([0, 0, 2.0]), np.array([0, 0, 0, 4 * np.pi])), [0.25])


# ---- LapQPGradGrad (Table XI; L^Q_jk = d2 L / dx_j dx_k) ----
def test_qpgradgrad_derivatives_and_limits():
    rng = np.random.default_rng(41)
    h = 1e-5
    H = {(0, 0): 4, (0, 1): 5, (0, 2): 6, (1, 1): 7, (1, 2): 8, (2, 2): 9}
    for _ in range(4):
        r = rng.standard_normal(3) + 0.5
        Q = rng.standard_normal(9)
        v = pair_values("LQ+gradLQ+gradgradLQ", r, Q)
        np.testing.assert_allclose(pair_values("LQ", r, Q), v[:1], rtol=1e-15)
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            dv = (pair_values("LQ+gradLQ+gradgradLQ", r + e, Q) - pair_values("LQ+gradLQ+gradgradLQ", r - e, Q)) / (2 * h)
            np.testing.assert_allclose(dv[0], v[1 + k], rtol=1e-6, atol=1e-8)
            for j in range(3):
                np.testing.assert_allclose(dv[1 + j], v[H[tuple(sorted((j, k)))]], rtol=1e-6, atol=1e-8)
        assert abs(v[4] + v[7] + v[9]) < 1e-11 * np.abs(v[4:]).max()  # harmonic
        # the quadrupole Q = a b^T is the limit of dipoles +b/h at y + h a/2 and -b/h at
        # y - h a/2 (r = x - y, so the first sits at r - h a/2)
        a, b = rng.standard_normal(3), rng.standard_normal(3)
        lim = (pair_values("LD+gradLD+gradgradLD", r - 0.5 * h * a, np.concatenate([[0.0], b]))
               - pair_values("LD+gradLD+gradgradLD", r + 0.5 * h * a, np.concatenate([[0.0], b]))) / h
        np.testing.assert_allclose(pair_values("LQ+gradLQ+gradgradLQ", r, np.outer(a, b).ravel()), lim,
                                   rtol=1e-5, atol=1e-7)
    # an isotropic Q = I has phi = tr(d d L) = lap L = 0 away from the source
    assert abs(pair_values("LQ", np.array([0.3, -0.2, 0.7]), np.eye(3).ravel())[0]) < 1e-14
