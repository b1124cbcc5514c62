"""O1: pairwise kernel functions and the plain direct sum (oracle; test infrastructure).

Every kernel takes r = x - y (target minus source).
Constants: Laplace 1/(4 pi), Stokes 1/(8 pi) with mu = 1
(PAPER.md:251-253).

Kernel names follow the paper's notation:
  L          Laplace single layer, phi = q/(4 pi r)
  L+gradL    [phi, grad_x phi], grad_x L = -r/(4 pi r^3)           PAPER.md:102-117, Table XI LapPGrad
  G          Stokeslet (1/8pi)(delta/r + r r^T/r^3)
  G_RPY      (1 + b^2/6 lap) G, Eq. (RPYkernel)
  G_RPY+lapG [u, lap u]; lap G^RPY = lap G since lap lap G = 0
  G+lapG     [u, lap u] from point forces                          PAPER.md:106, Table IV
  G_eps      regularized Stokeslet
  L+LD       [q, d] -> phi = q L + d . L^D, L^D_j = -dL/dx_j = r_j/(4 pi r^3)   PAPER.md:215-221, Table III S row
  L+gradL+gradgradL    q -> [phi, grad phi, grad grad phi]         Table III T column (ML-tree charges)
  LD+gradLD+gradgradLD [q, d] -> [phi, grad phi, grad grad phi]  Table III S->T (charges and dipoles)
      grad grad phi as (xx, xy, xz, yy, yz, zz)
  LQ         Q -> phi = Q_jk L^Q_jk, L^Q_jk = d2 L/dx_j dx_k                  PAPER.md:218-221 (LapQPGradGrad S row)
  LQ+gradLQ+gradgradLQ  Q -> [phi, grad phi, grad grad phi]             LapQPGradGrad S->T (Table XI)
      Q a general 3x3 matrix, row-major (Q_xx, Q_xy, Q_xz, Q_yx, ...)
  G_eps+T_eps            [f, t, eps] -> u = G^eps f + T^eps t        Table VI S-row, PAPER.md:357-362
  G+Omega                f -> [u, omega] = [G f, Omega f] (eps = 0)  Table VI T column
  G_eps+Omega+T+W        [f, t, eps] -> [u, omega], the 7x6 S->T     PAPER.md:356-374, Table VI
with H1, H2, Q, D1, D2 of PAPER.md:363-369 (1/(8 pi) inside) and
Omega^eps_ij = T^eps_ij = Q eps_ijk r_k / 2, so Omega f = Q (f x r) / 2 and
T t = Q (t x r) / 2; W^eps = D1 delta / 4 + D2 r r^T / 4.
with lap G_ij = (1/8pi)(2 delta_ij / r^3 - 6 r_i r_j / r^5) (derived from
G_ij; checked by finite differences in tests/test_oracle_kernels.py).

Singular kernels skip pairs with r^2 == 0 exactly (self interaction,
DESIGN.md reading R5); G_eps is finite at r = 0 and keeps them.
"""
from __future__ import annotations

import numpy as np

FOUR_PI = 4.0 * np.pi
EIGHT_PI = 8.0 * np.pi

# (k_s, k_t) of each named kernel
DIMS = {
    "L": (1, 1),
    "L+gradL": (1, 4),
    "G": (3, 3),
    "G_RPY": (4, 3),
    "G_RPY+lapG": (4, 6),
    "G+lapG": (3, 6),
    "G_eps": (4, 3),
    "L+LD": (4, 1),
    "LQ": (9, 1),
    "LQ+gradLQ+gradgradLQ": (9, 10),
    "L+gradL+gradgradL": (1, 10),
    "LD+gradLD+gradgradLD": (4, 10),
    "G_eps+T_eps": (7, 3),
    "G+Omega": (3, 6),
    "G_eps+Omega+T+W": (7, 6),
}
SINGULAR = {"L": True, "L+gradL": True, "G": True, "G_RPY": True, "G_RPY+lapG": True,
            "G+lapG": True, "G_eps": False, "L+LD": True, "L+gradL+gradgradL": True,
            "LD+gradLD+gradgradLD": True, "LQ": True, "LQ+gradLQ+gradgradLQ": True, "G_eps+T_eps": False, "G+Omega": True,
            "G_eps+Omega+T+W": False}


def pair_values(name: str, r: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Kernel `name` applied to source values s at displacement r = x - y.

    r: (..., 3), s: (..., k_s) broadcastable -> (..., k_t).  Pairs with
    r^2 == 0 contribute zero for singular kernels.
    """
    r2 = np.sum(r * r, axis=-1)
    if name in ("G_eps+T_eps", "G_eps+Omega+T+W"):
        f, t, eps = s[..., 0:3], s[..., 3:6], s[..., 6]
        e2 = eps * eps
        d = e2 + r2
        sd = np.sqrt(d)
        d32 = d * sd
        d52 = d32 * d
        d72 = d52 * d
        H1 = (2.0 * e2 + r2) / (EIGHT_PI * d32)
        H2 = 1.0 / (EIGHT_PI * d32)
        Q = (5.0 * e2 + 2.0 * r2) / (EIGHT_PI * d52)
        rf = np.sum(r * f, axis=-1)
        u = H1[..., None] * f + (H2 * rf)[..., None] * r + 0.5 * Q[..., None] * np.cross(t, r)
        if name == "G_eps+T_eps":
            return u
        D1 = (10.0 * e2 * e2 - 7.0 * e2 * r2 - 2.0 * r2 * r2) / (EIGHT_PI * d72)
        D2 = (21.0 * e2 + 6.0 * r2) / (EIGHT_PI * d72)
        rt = np.sum(r * t, axis=-1)
        w = 0.5 * Q[..., None] * np.cross(f, r) + 0.25 * D1[..., None] * t + (0.25 * D2 * rt)[..., None] * r
        return np.concatenate([u, w], axis=-1)
    if name == "G_eps":
        eps = s[..., 3]
        f = s[..., :3]
        d = r2 + eps * eps
        d32 = d * np.sqrt(d)
        rf = np.sum(r * f, axis=-1)
        u = ((r2 + 2.0 * eps * eps)[..., None] * f + rf[..., None] * r) / d32[..., None]
        return u / EIGHT_PI
    zero = r2 == 0.0
    r2s = np.where(zero, 1.0, r2)
    rinv = 1.0 / np.sqrt(r2s)
    rinv = np.where(zero, 0.0, rinv)
    rinv3 = rinv * rinv * rinv
    if name == "L":
        return (s[..., 0] * rinv / FOUR_PI)[..., None]
    if name == "L+gradL":
        q = s[..., 0]
        phi = q * rinv / FOUR_PI
        grad = -(q * rinv3)[..., None] * r / FOUR_PI
        return np.concatenate([phi[..., None], grad], axis=-1)
    if name in ("LQ", "LQ+gradLQ+gradgradLQ"):
        # derivatives of 1/r contracted with Q_jk:
        #   d_j d_k     3 r_j r_k / r^5 - delta_jk / r^3
        #   d_i d_j d_k -15 r_i r_j r_k / r^7 + 3 (delta_ij r_k + delta_ik r_j + delta_jk r_i) / r^5
        #   d_i d_l d_j d_k  105 r_i r_j r_k r_l / r^9 - 15 (6 delta r r terms) / r^7 + 3 (3 delta delta) / r^5
        Q = s.reshape(s.shape[:-1] + (3, 3))
        rinv5 = rinv3 * rinv * rinv
        rinv7 = rinv5 * rinv * rinv
        rinv9 = rinv7 * rinv * rinv
        a = np.einsum("...j,...jk,...k->...", r, Q, r)
        tq = np.trace(Q, axis1=-2, axis2=-1)
        w = np.einsum("...ik,...k->...i", Q, r) + np.einsum("...ji,...j->...i", Q, r)
        phi = 3.0 * a * rinv5 - tq * rinv3
        if name == "LQ":
            return (phi / FOUR_PI)[..., None]
        grad = (-15.0 * a * rinv7)[..., None] * r + 3.0 * rinv5[..., None] * (w + tq[..., None] * r)
        I = np.eye(3)
        rr = r[..., :, None] * r[..., None, :]
        hess = ((105.0 * a * rinv9)[..., None, None] * rr
                - 15.0 * rinv7[..., None, None] * (a[..., None, None] * I + r[..., None, :] * w[..., :, None]
                                                   + r[..., :, None] * w[..., None, :] + tq[..., None, None] * rr)
                + 3.0 * rinv5[..., None, None] * (tq[..., None, None] * I + Q + np.swapaxes(Q, -1, -2)))
        iu = ([0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2])
        return np.concatenate([phi[..., None], grad, hess[..., iu[0], iu[1]]], axis=-1) / FOUR_PI
    if name in ("L+LD", "L+gradL+gradgradL", "LD+gradLD+gradgradLD"):
        q = s[..., 0]
        rinv5 = rinv3 * rinv * rinv
        # charge: phi = q/r, grad = -q r/r^3, grad grad_jk = q (3 r_j r_k/r^5 - delta_jk/r^3)
        phi = q * rinv
        grad = -(q * rinv3)[..., None] * r
        hess = q[..., None, None] * (3.0 * rinv5[..., None, None] * r[..., :, None] * r[..., None, :]
                                     - rinv3[..., None, None] * np.eye(3))
        if name != "L+gradL+gradgradL":
            # dipole: phi = d.r/r^3 (L^D_j = r_j/(4 pi r^3)), grad = d/r^3 - 3 (d.r) r/r^5,
            # grad grad_jk = -3 (d_j r_k + d_k r_j + (d.r) delta_jk)/r^5 + 15 (d.r) r_j r_k/r^7
            d = s[..., 1:4]
            dr = np.sum(d * r, axis=-1)
            rinv7 = rinv5 * rinv * rinv
            phi = phi + dr * rinv3
            if name == "L+LD":
                return (phi / FOUR_PI)[..., None]
            grad = grad + rinv3[..., None] * d - (3.0 * dr * rinv5)[..., None] * r
            hess = hess + (-3.0 * rinv5[..., None, None] * (d[..., :, None] * r[..., None, :]
                                                            + r[..., :, None] * d[..., None, :]
                                                            + dr[..., None, None] * np.eye(3))
                           + (15.0 * dr * rinv7)[..., None, None] * r[..., :, None] * r[..., None, :])
        iu = ([0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2])
        return np.concatenate([phi[..., None], grad, hess[..., iu[0], iu[1]]], axis=-1) / FOUR_PI
    f = s[..., :3]
    rf = np.sum(r * f, axis=-1)
    if name == "G":
        return (rinv[..., None] * f + (rf * rinv3)[..., None] * r) / EIGHT_PI
    if name == "G+Omega":  # Q(r) at eps = 0 is 2 / (8 pi r^3)
        u = (rinv[..., None] * f + (rf * rinv3)[..., None] * r) / EIGHT_PI
        w = rinv3[..., None] * np.cross(f, r) / EIGHT_PI
        return np.concatenate([u, w], axis=-1)
    rinv5 = rinv3 * rinv * rinv
    lap = (2.0 * rinv3[..., None] * f - 6.0 * (rf * rinv5)[..., None] * r) / EIGHT_PI
    if name == "G+lapG":
        u = (rinv[..., None] * f + (rf * rinv3)[..., None] * r) / EIGHT_PI
        return np.concatenate([u, lap], axis=-1)
    b2 = s[..., 3] * s[..., 3]
    u = ((rinv + b2 * rinv3 / 3.0)[..., None] * f + ((rinv3 - b2 * rinv5) * rf)[..., None] * r) / EIGHT_PI
    if name == "G_RPY":
        return u
    if name == "G_RPY+lapG":
        return np.concatenate([u, lap], axis=-1)
    raise ValueError(name)


def direct_sum(name: str, trg: np.ndarray, src: np.ndarray, vals: np.ndarray,
               chunk: int = 256) -> np.ndarray:
    """Eq. (1)/(2): g(x_a) = sum_b K(x_a, y_b, s_b).

    Plain all-pairs sum, chunked over targets only to bound memory.
    """
    k_t = DIMS[name][1]
    trg = np.asarray(trg, dtype=np.float64)
    src = np.asarray(src, dtype=np.float64)
    vals = np.asarray(vals, dtype=np.float64)
    out = np.zeros((trg.shape[0], k_t))
    if src.shape[0] == 0:
        return out
    step = max(1, min(chunk, (1 << 24) // max(1, src.shape[0])))
    for a in range(0, trg.shape[0], step):
        r = trg[a:a + step, None, :] - src[None, :, :]
        out[a:a + step] = pair_values(name, r, vals[None, :, :]).sum(axis=1)
    return out


def kernel_matrix(name: str, trg: np.ndarray, src: np.ndarray) -> np.ndarray:
    """Dense matrix of a LINEAR ML-tree kernel (L or G): rows (i, a), cols (j, b).

    Row index i*k + a (target point i, component a); column j*k + b.  Built by
    applying the kernel to unit source vectors, i.e. straight from
    pair_values, so the matrix and the pointwise kernel cannot disagree.
    """
    k = DIMS[name][0]
    assert DIMS[name] == (k, k) and name in ("L", "G")
    nt, ns = trg.shape[0], src.shape[0]
    r = trg[:, None, :] - src[None, :, :]
    K = np.empty((nt, k, ns, k))
    for b in range(k):
        e = np.zeros(k)
        e[b] = 1.0
        K[:, :, :, b] = np.moveaxis(pair_values(name, r, e), -1, 1)
    return K.reshape(nt * k, ns * k)
