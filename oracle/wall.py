"""RPY above a no-slip wall by images (oracle; test infrastructure).

PAPER.md:729-779 (Sec. "No-slip Wall", Table X): the flow of polydisperse
RPY spheres above the wall x_3 = 0 is four free-space summations over the
sources y and their images y^I = (y_1, y_2, -y_3), assembled per target as

    u       = u^S + grad phi^SDZ + x_3 grad phi^SD + x_3 grad phi^Q - [0, 0, phi^SD + phi^Q]
    lap u   = lap u^S + 2 d/dx_3 grad (phi^SD + phi^Q)

with (Table X)
    RPY              [f_1, f_2, 0; b] at y,  [-f_1, -f_2, 0; b] at y^I      -> u^S, lap u^S
    Laplace SL + DL  charge f_3 at y;  charge -f_3, dipole y_3 (-f_1, -f_2, f_3) at y^I
                                                                              -> phi^SD and derivatives
    Laplace SL + DL  charge y_3 f_3 / 2, dipole b^2/6 (0, 0, f_3) at y;
                     charge -y_3 f_3 / 2, dipole b^2/6 (0, 0, f_3) at y^I     -> phi^SDZ, grad
    Laplace Q        Q = b^2/3 [[f_3, 0, 0], [0, f_3, 0], [f_1, f_2, 0]] at y^I  -> phi^Q and derivatives
The Laplace sums use L = 1/(4 pi r), the RPY sum 1/(8 pi) (mu = 1).

Reading R18: the extracted Table X prints the quadrupole in the
"source at y" column.  Placed at y it violates the no-slip condition at
O(b^2) (relative 2e-3 at b = 0.05, y_3 = 0.35); placed at y^I the assembled
velocity vanishes on the wall to rounding and equals (1 + b^2/6 lap_y)
applied to the b = 0 wall Stokeslet (tests/test_oracle_wall.py), as the
RPY construction requires.  The quadrupole is therefore placed at y^I.
(Q enters only through its symmetric part: d_j d_k L is symmetric.)

The oracle works in wall coordinates (heights above the wall); the unit-cube
embedding (wall at z = 1/2) is the product's concern.
"""
from __future__ import annotations

import numpy as np

from . import fmm as F
from .kernels import direct_sum


def image_sources(y: np.ndarray, vals: np.ndarray):
    """The four summations of Table X: (kernel name, source points, values)."""
    f, b = vals[:, :3], vals[:, 3]
    f1, f2, f3 = f[:, 0], f[:, 1], f[:, 2]
    y3 = y[:, 2]
    yI = y * np.array([1.0, 1.0, -1.0])
    n = y.shape[0]
    z = np.zeros(n)
    rpy = (np.concatenate([y, yI]), np.concatenate([np.stack([f1, f2, z, b], 1), np.stack([-f1, -f2, z, b], 1)]))
    sd = (np.concatenate([y, yI]),
          np.concatenate([np.stack([f3, z, z, z], 1), np.stack([-f3, -y3 * f1, -y3 * f2, y3 * f3], 1)]))
    b6 = b * b / 6.0
    sdz = (np.concatenate([y, yI]),
           np.concatenate([np.stack([0.5 * y3 * f3, z, z, b6 * f3], 1), np.stack([-0.5 * y3 * f3, z, z, b6 * f3], 1)]))
    b3 = b * b / 3.0
    Q = np.stack([b3 * f3, z, z, z, b3 * f3, z, b3 * f1, b3 * f2, z], 1)
    q = (yI, Q)
    return rpy, sd, sdz, q


def assemble(x3: np.ndarray, uS: np.ndarray, pSD: np.ndarray, pSDZ: np.ndarray, pQ: np.ndarray) -> np.ndarray:
    """Per-target assembly.  uS: [u, lap u]; pSD, pQ:
    [phi, grad, grad grad (xx, xy, xz, yy, yz, zz)]; pSDZ: [phi, grad, ...]."""
    u = uS[:, :3] + pSDZ[:, 1:4] + x3[:, None] * (pSD[:, 1:4] + pQ[:, 1:4])
    u[:, 2] -= pSD[:, 0] + pQ[:, 0]
    h = pSD + pQ
    lap = uS[:, 3:6] + 2.0 * h[:, [6, 8, 9]]   # d/dx_3 grad = (xz, yz, zz)
    return np.concatenate([u, lap], axis=1)


def rpy_wall_direct(x: np.ndarray, y: np.ndarray, vals: np.ndarray) -> np.ndarray:
    """[u, lap u] at targets x (heights x_3 >= 0) by direct sums (O1 of each summation)."""
    rpy, sd, sdz, q = image_sources(y, vals)
    uS = direct_sum("G_RPY+lapG", x, *rpy)
    pSD = direct_sum("LD+gradLD+gradgradLD", x, *sd)
    pSDZ = direct_sum("LD+gradLD+gradgradLD", x, *sdz)
    pQ = direct_sum("LQ+gradLQ+gradgradLQ", x, *q)
    return assemble(x[:, 2], uS, pSD, pSDZ, pQ)


def rpy_wall_fmm(points: np.ndarray, vals: np.ndarray, p: int, cap: int) -> np.ndarray:
    """The same with the oracle KIFMM for each summation, in the unit cube with
    the wall at z = 1/2: points (z >= 1/2) and their images share one point set
    of 2n points (images carry zero Q-free values where a summation has none),
    targets = the points.  Returns [u, lap u] at the points."""
    n = points.shape[0]
    y = points - np.array([0.0, 0.0, 0.5])
    rpy, sd, sdz, q = image_sources(y, vals)
    P2 = np.concatenate([points, points * np.array([1.0, 1.0, -1.0]) + np.array([0.0, 0.0, 1.0])])
    P2 = np.where(P2 >= 1.0, np.nextafter(1.0, 0.0), P2)
    qv = np.concatenate([np.zeros((n, 9)), q[1]])
    uS = F.fmm(P2, rpy[1], "rpy", p, cap)["out"][:n]
    pSD = F.fmm(P2, sd[1], "laplace_pgradgrad", p, cap)["out"][:n]
    pSDZ = F.fmm(P2, sdz[1], "laplace_pgradgrad", p, cap)["out"][:n]
    pQ = F.fmm(P2, qv, "laplace_qpgradgrad", p, cap)["out"][:n]
    return assemble(y[:, 2], uS, pSD, pSDZ, pQ)
