"""Equivalent/check surfaces and translation operators (oracle; test infrastructure).

Surfaces (M = 6(m-1)^2 + 2 points per box
"placing a certain number of check points on a surface surrounding this
octree box"): the boundary points of an m x m x m lattice,
    c + alpha h (-1 + 2 i/(m-1)),  i in {0..m-1}^3 with some i_a in {0, m-1},
ordered lexicographically (i_x slowest).  Radii (reading R1):
    upward equivalent 1.05 h, upward check 2.95 h,
    downward check    1.05 h, downward equivalent 2.95 h.

Check -> equivalent ("backward stable SVD"): the SVD
K = U S V^T of the ML-kernel matrix from equivalent to check points,
truncated at sigma_i > tau sigma_max with tau = 1e-12 (reading R2), applied
as two factors  x = V_k (S_k^-1 U_k^T c)  -- never as an explicit
pseudo-inverse.

All operators are built once at the reference level 0 (h = 1/2).  The ML
kernels L and G are homogeneous of degree -1, so at
level l kernel matrices scale by 2^l and check->equivalent factors by 2^-l;
the composed M2M and L2L are level independent.
"""
from __future__ import annotations

import functools
import itertools

import numpy as np

from .kernels import kernel_matrix

ALPHA_UE = 1.05
ALPHA_UC = 2.95
ALPHA_DC = 1.05
ALPHA_DE = 2.95
TAU = 1e-12
H0 = 0.5
C0 = np.array([0.5, 0.5, 0.5])


@functools.lru_cache(maxsize=None)
def _lattice(m: int) -> np.ndarray:
    out = [(i, j, k) for i in range(m) for j in range(m) for k in range(m)
           if min(i, j, k) == 0 or max(i, j, k) == m - 1]
    a = np.array(out, dtype=np.float64)
    a.setflags(write=False)
    return a


def surface_lattice(m: int) -> np.ndarray:
    """Integer lattice indices of the boundary of an m^3 cube, lexicographic."""
    if m < 2:
        raise ValueError("m >= 2")
    return _lattice(m)


def surface(m: int, c, h: float, alpha: float) -> np.ndarray:
    lat = surface_lattice(m)
    return np.asarray(c, dtype=np.float64) + alpha * h * (-1.0 + 2.0 * lat / (m - 1))


def n_surface(m: int) -> int:
    return 6 * (m - 1) ** 2 + 2


def v_offsets() -> list[tuple]:
    """The 316 same-level offsets in {-3..3}^3 minus {-1..1}^3."""
    return [o for o in itertools.product(range(-3, 4), repeat=3) if max(abs(v) for v in o) >= 2]


def child_centre_offset(oct_: int) -> np.ndarray:
    bits = np.array([(oct_ >> 2) & 1, (oct_ >> 1) & 1, oct_ & 1], dtype=np.float64)
    return 2.0 * bits - 1.0  # in units of the child half-width


class _LazyM2L(dict):
    def __init__(self, ops):
        super().__init__()
        self._ops = ops

    def __missing__(self, o):
        mat = self._ops.m2l_matrix(o)
        self[o] = mat
        return mat


class Operators:
    """Translation operators of one ML kernel ('L' or 'G') at order m."""

    def __init__(self, ml: str, m: int, tau: float = TAU, build_m2l: bool = False):
        self.ml, self.m, self.tau = ml, m, tau
        self.k = 1 if ml == "L" else 3
        self.M = n_surface(m)
        self.n = self.M * self.k
        ue = surface(m, C0, H0, ALPHA_UE)
        uc = surface(m, C0, H0, ALPHA_UC)
        dc = surface(m, C0, H0, ALPHA_DC)
        de = surface(m, C0, H0, ALPHA_DE)
        # upward check <- upward equivalent
        U, s, Vt = np.linalg.svd(kernel_matrix(ml, uc, ue))
        keep = s > tau * s[0]
        self.up_sigma = s
        self.up_kept = int(keep.sum())
        self.uc2ue_1 = (U[:, keep] / s[keep]).T          # S_k^-1 U_k^T   (kept x n)
        self.uc2ue_2 = np.ascontiguousarray(Vt[keep].T)  # V_k            (n x kept)
        # downward check <- downward equivalent
        U, s, Vt = np.linalg.svd(kernel_matrix(ml, dc, de))
        keep = s > tau * s[0]
        self.dn_sigma = s
        self.dn_kept = int(keep.sum())
        self.dc2de_1 = (U[:, keep] / s[keep]).T
        self.dc2de_2 = np.ascontiguousarray(Vt[keep].T)
        # composed M2M[oct] = UC2UE_parent o K(uc_P <- ue_C)
        self.m2m = []
        self.l2l = []
        for o in range(8):
            cc = C0 + 0.5 * H0 * child_centre_offset(o)
            K = kernel_matrix(ml, uc, surface(m, cc, 0.5 * H0, ALPHA_UE))
            self.m2m.append(self.uc2ue_2 @ (self.uc2ue_1 @ K))
            # L2L[oct] = DC2DE_child o K(dc_C <- de_P); the child's
            # DC2DE is the level-1 one, i.e. the reference factors times 2^-1.
            K = kernel_matrix(ml, surface(m, cc, 0.5 * H0, ALPHA_DC), de)
            self.l2l.append(0.5 * (self.dc2de_2 @ (self.dc2de_1 @ K)))
        # raw M2L[o] = K(dc_B <- ue_C), C centre = B centre + 2h o  (M->L slot),
        # built on first use (316 offsets x n^2 doubles is 12 GB at p=12, k=3)
        self.m2l = _LazyM2L(self)
        if build_m2l:
            for o in v_offsets():
                self.m2l[o]

    def m2l_matrix(self, o) -> np.ndarray:
        m = self.m
        dc = surface(m, C0, H0, ALPHA_DC)
        ue = surface(m, C0 + 2.0 * H0 * np.asarray(o, dtype=np.float64), H0, ALPHA_UE)
        return kernel_matrix(self.ml, dc, ue)

    # applications at level l (reading: homogeneity)
    def uc2ue(self, chk: np.ndarray, level: int) -> np.ndarray:
        """chk: (..., n) -> upward equivalent densities, two factors."""
        t = chk @ self.uc2ue_1.T
        return (t @ self.uc2ue_2.T) * 2.0 ** (-level)

    def dc2de(self, chk: np.ndarray, level: int) -> np.ndarray:
        t = chk @ self.dc2de_1.T
        return (t @ self.dc2de_2.T) * 2.0 ** (-level)
