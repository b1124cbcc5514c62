"""Seeded synthetic workloads shared by the oracle, the tests and bench.py.

This module holds ONLY input generation (random point clouds and source
values).  It contains none of the method's arithmetic: no kernels, no tree,
no operators.  Both sides of every parity check (``oracle/`` and the CUDA
path in ``paper_2010_15155_b200``) receive the arrays produced here.

Recipe:
  seeds   np.random.SeedSequence([201015155, c]) for config c, spawned into
          three independent streams: coordinates, values, centres.
  C1      2,000 iid U[0,1)^3, Stokeslet, f ~ N(0,1)^3, p=8, cap 50
  C2      10^6 iid U[0,1)^3, Laplace PGrad, q ~ N(0,1), p=10, cap 64
  C3      4x10^6 iid U[0,1)^3, RPY, f ~ N(0,1)^3, b = 1e-3, p=10, cap 64
  C4      64 cluster centres iid U[0,1)^3, 125,000 points each
          ~ centre + N(0, 0.01^2 I); points leaving [0,1)^3 are redrawn from
          the same cluster (reading R6); RegVel, eps = 1e-4, p=12,
          cap 64
  C5      10^4 sphere centres by random sequential addition in [r, 1-r]^3,
          r = 0.005, centre distance >= 2r; 6,400 points per sphere
          y = c + r v/|v|, v ~ N(0, I); Stokeslet, p=8, cap 128
  C6, C7 (not BASELINE configs) the paper's own
          benchmark cloud, Eq. (ptdist): x, y, z iid
          u - [u] with u log-normal (m = -1, s = 0.5), i.e. the paper's
          L (u - [u]) with L = 32 scaled to the unit cube; N = 10^6, leaf cap
          2000, values U[-1, 1], polydisperse
          b (C6, RPY [f, b] -> [u, lap u]) or eps (C7, StokesRegVelOmega
          [f, t, eps] -> [u, omega], Table VI) iid U[0, 1e-4] in the paper's units
          (PAPER.md:676), i.e. U[0, 1e-4 / 32] in the unit cube; p = 10
  C8      the same cloud and values for LapPGradGrad [q, d] -> [phi, grad phi,
          grad grad phi] (Table III; the paper's Fig. 3a case)
  C9      the same for LapQPGradGrad Q -> [phi, grad phi, grad grad phi]
          (Table XI; the paper's Fig. 3b case)
The BASELINE configs are the paper-shaped stand-ins for the paper's own
synthetic clouds (Eq. (ptdist)); no dataset is involved.
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED_ROOT = 201015155

KERNELS = ("laplace_pgrad", "stokeslet", "rpy", "stokes_reg_vel", "stokes_reg_vel_omega", "laplace_pgradgrad",
           "laplace_qpgradgrad")
# (k_s, k_t) per kernel: PAPER.md Table XI (lines 874-880)
KERNEL_DIMS = {"laplace_pgrad": (1, 4), "stokeslet": (3, 3), "rpy": (4, 6), "stokes_reg_vel": (4, 3),
               "stokes_reg_vel_omega": (7, 6), "laplace_pgradgrad": (4, 10), "laplace_qpgradgrad": (9, 10)}
# C-ABI enum values (include/kafmm.h)
KERNEL_ENUM = {"laplace_pgrad": 1, "stokeslet": 2, "rpy": 3, "stokes_reg_vel": 4, "stokes_reg_vel_omega": 5,
               "laplace_pgradgrad": 6, "laplace_qpgradgrad": 7}
# source column of the nonlinear per-source parameter (b or eps), if any
PARAM_COL = {"rpy": 3, "stokes_reg_vel": 3, "stokes_reg_vel_omega": 6}


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    cid: int
    kernel: str
    n: int
    p: int
    cap: int
    cloud: str          # "uniform" | "clusters" | "spheres" | "lognormal"
    extra: float = 0.0  # b (RPY) or eps (RegVel) carried as the 4th source column
    poly: bool = False  # 4th column iid U[0, extra] per source; values U[-1, 1] (paper's benchmarks)

    @property
    def name(self) -> str:
        return f"C{self.cid}"


CONFIGS = {
    1: ConfigSpec(1, "stokeslet", 2000, 8, 50, "uniform"),
    2: ConfigSpec(2, "laplace_pgrad", 1_000_000, 10, 64, "uniform"),
    3: ConfigSpec(3, "rpy", 4_000_000, 10, 64, "uniform", 1e-3),
    4: ConfigSpec(4, "stokes_reg_vel", 8_000_000, 12, 64, "clusters", 1e-4),
    5: ConfigSpec(5, "stokeslet", 64_000_000, 8, 128, "spheres"),
    6: ConfigSpec(6, "rpy", 1_000_000, 10, 2000, "lognormal", 1e-4 / 32, True),
    7: ConfigSpec(7, "stokes_reg_vel_omega", 1_000_000, 10, 2000, "lognormal", 1e-4 / 32, True),
    8: ConfigSpec(8, "laplace_pgradgrad", 1_000_000, 10, 2000, "lognormal", 0.0, True),
    9: ConfigSpec(9, "laplace_qpgradgrad", 1_000_000, 10, 2000, "lognormal", 0.0, True),
}
LOGNORMAL_M, LOGNORMAL_S = -1.0, 0.5


def _streams(cid: int):
    ss = np.random.SeedSequence([SEED_ROOT, cid])
    return [np.random.default_rng(s) for s in ss.spawn(3)]


def _uniform(rng, n):
    return rng.random((n, 3))


def _clusters(rng_pts, rng_ctr, n, n_clusters=64, sigma=0.01):
    centres = rng_ctr.random((n_clusters, 3))
    per = np.full(n_clusters, n // n_clusters, dtype=np.int64)
    per[: n - per.sum()] += 1
    pts = np.empty((n, 3))
    off = 0
    for c in range(n_clusters):
        m = int(per[c])
        blk = centres[c] + sigma * rng_pts.standard_normal((m, 3))
        bad = ~np.all((blk >= 0.0) & (blk < 1.0), axis=1)
        while bad.any():  # reading R6: redraw leakers from the same cluster
            blk[bad] = centres[c] + sigma * rng_pts.standard_normal((int(bad.sum()), 3))
            bad = ~np.all((blk >= 0.0) & (blk < 1.0), axis=1)
        pts[off:off + m] = blk
        off += m
    return pts


def sphere_centres(rng, n_spheres, r=0.005):
    """Random sequential addition of non-overlapping spheres in [r, 1-r]^3."""
    cell = 2.0 * r
    ncell = int(np.ceil(1.0 / cell))
    grid: dict = {}
    out = []
    tries = 0
    while len(out) < n_spheres:
        c = r + (1.0 - 2.0 * r) * rng.random(3)
        tries += 1
        g = tuple((c / cell).astype(int))
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    for o in grid.get((g[0] + dx, g[1] + dy, g[2] + dz), ()):
                        if np.sum((o - c) ** 2) < cell * cell:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            grid.setdefault(g, []).append(c)
            out.append(c)
    del ncell
    return np.array(out), tries


def _spheres(rng_pts, rng_ctr, n, n_spheres=10_000, r=0.005):
    centres, _ = sphere_centres(rng_ctr, n_spheres, r)
    per = np.full(n_spheres, n // n_spheres, dtype=np.int64)
    per[: n - per.sum()] += 1
    v = rng_pts.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    pts = np.repeat(centres, per, axis=0) + r * v
    return pts


def make_points(spec: ConfigSpec, n: int | None = None, n_spheres: int | None = None):
    n = spec.n if n is None else int(n)
    rp, _rv, rc = _streams(spec.cid)
    if spec.cloud == "uniform":
        pts = _uniform(rp, n)
    elif spec.cloud == "clusters":
        pts = _clusters(rp, rc, n)
    elif spec.cloud == "spheres":
        ns = 10_000 if n_spheres is None else int(n_spheres)
        pts = _spheres(rp, rc, n, n_spheres=min(ns, max(1, n)))
    elif spec.cloud == "lognormal":
        u = rp.lognormal(LOGNORMAL_M, LOGNORMAL_S, size=(n, 3))
        pts = u - np.floor(u)
    else:
        raise ValueError(spec.cloud)
    assert np.all((pts >= 0.0) & (pts < 1.0))
    return np.ascontiguousarray(pts, dtype=np.float64)


def make_values(spec: ConfigSpec, n: int | None = None):
    n = spec.n if n is None else int(n)
    _rp, rv, _rc = _streams(spec.cid)
    k_s = KERNEL_DIMS[spec.kernel][0]
    if spec.poly:
        vals = rv.uniform(-1.0, 1.0, size=(n, k_s))
        if spec.kernel in PARAM_COL:
            vals[:, PARAM_COL[spec.kernel]] = rv.uniform(0.0, spec.extra, size=n)
    elif spec.kernel == "laplace_pgrad":
        vals = rv.standard_normal((n, 1))
    elif spec.kernel == "stokeslet":
        vals = rv.standard_normal((n, 3))
    else:  # [f, b] or [f, eps]
        vals = np.empty((n, 4))
        vals[:, :3] = rv.standard_normal((n, 3))
        vals[:, 3] = spec.extra
    assert vals.shape[1] == k_s
    return np.ascontiguousarray(vals, dtype=np.float64)


def make_config(cid: int, n: int | None = None, n_spheres: int | None = None):
    """Return (spec, points N x 3, values N x k_s) for BASELINE config cid (1..5).

    ``n`` shrinks the cloud keeping its shape (parity tests at oracle-sized N).
    """
    spec = CONFIGS[cid]
    pts = make_points(spec, n, n_spheres)
    vals = make_values(spec, pts.shape[0])
    return spec, pts, vals


def random_values(kernel: str, n: int, seed: int, extra: float | None = None):
    """Seeded source values of the kernel's layout (tests)."""
    rng = np.random.default_rng(seed)
    k_s = KERNEL_DIMS[kernel][0]
    v = rng.standard_normal((n, k_s))
    if kernel in PARAM_COL:
        v[:, PARAM_COL[kernel]] = (1e-3 if kernel == "rpy" else 1e-4) if extra is None else extra
    return v
