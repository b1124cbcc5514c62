"""RPY above a no-slip wall on the GPU (PAPER.md:729-779,
Table X) against the oracle's image-system FMM and direct sums."""
import numpy as np
import pytest

from oracle import fmm as F
from oracle import wall as Wl
from paper_2010_15155_b200 import KAFMMWall, KafmmError

from .gpu_helpers import assert_parity

pytestmark = pytest.mark.gpu


def _particles(n, seed, bmax):
    rng = np.random.default_rng(seed)
    pts = np.concatenate([rng.random((n, 2)), 0.5 + 0.5 * rng.random((n, 1))], axis=1)
    pts[:, 2] = np.clip(pts[:, 2], np.nextafter(0.5, 1.0), np.nextafter(1.0, 0.0))
    vals = np.concatenate([rng.standard_normal((n, 3)), bmax * rng.random((n, 1))], axis=1)
    return pts, vals


@pytest.mark.parametrize("n,p,cap", [(1500, 6, 40), (4000, 8, 60)])
def test_wall_matches_oracle_and_direct(n, p, cap):
    import torch
    pts, vals = _particles(n, 7 + n, 1e-3)
    w = KAFMMWall(pts, p, cap)
    out = w.eval(torch.from_numpy(vals).cuda()).cpu().numpy()
    ref = Wl.rpy_wall_fmm(pts, vals, p, cap)
    assert_parity("rpy", out, ref)   # blocks (u | lap u), as the RPY kernel
    y = pts - np.array([0, 0, 0.5])
    d = Wl.rpy_wall_direct(y, y, vals)
    for lo, hi in ((0, 3), (3, 6)):
        assert F.rel_l2(out[:, lo:hi], d[:, lo:hi]) <= 2.0 * F.rel_l2(ref[:, lo:hi], d[:, lo:hi]) + 1e-15


def test_wall_rejects_particles_below_the_wall():
    pts, _ = _particles(100, 3, 1e-3)
    pts[5, 2] = 0.4
    with pytest.raises(KafmmError):
        KAFMMWall(pts, 4, 20)
