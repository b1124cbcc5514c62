"""The partitioned (multi-GPU) evaluation path on one GPU: `world` restricted
plans in one process, the exchanges done by LocalTransport (the same
spmd_eval driver and exchange lists the NCCL ranks use; the ranks run one
after the other, nothing waits on another).  The assembled result must equal
the unpartitioned plan and the oracle FMM."""
import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM, KafmmError
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
    single.close()
    offs = np.linspace(0, n, world + 1).astype(np.int64)
    gp = torch.from_numpy(pts).cuda()
    ranks = [D.build_rank(gp, offs, r, world, kernel, p, cap)[0] for r in range(world)]
    outs = D.spmd_eval(ranks, D.LocalTransport(), [src[offs[r]:offs[r + 1]] for r in range(world)])
    got = torch.cat(outs).cpu().numpy()
    errs = [F.rel_l2(got[:, lo:hi], ref_gpu[:, lo:hi]) for lo, hi in F.blocks(kernel)]
    assert max(errs) < 1e-12, errs
    ref = F.fmm(pts, vals, kernel, p, cap)["out"]
    assert_parity(kernel, got, ref)
    # the ranks' owned ranges tile the points; shared boxes exist once world > 1
    assert ranks[0].maps.plo == 0 and ranks[-1].maps.phi == n
    assert ranks[0].maps.shared.size > 0


def test_restrict_rejects_bad_ranges():
    pts = np.random.default_rng(5).random((3000, 3))
    plan = KAFMM(pts, "stokeslet", 4, 20)
    t = plan.tree()
    leaf_starts = np.sort(t["pbeg"][t["leaf"]])
    inside = int(leaf_starts[5]) + 1  # strictly inside a leaf of >= 2 points
    assert t["pend"][t["leaf"]][np.argsort(t["pbeg"][t["leaf"]])][5] > inside
    with pytest.raises(KafmmError):
        plan.restrict(0, inside)
    with pytest.raises(KafmmError):
        plan.restrict(-1, 10)
    plan.restrict(0, 3000)
    with pytest.raises(KafmmError):
        plan.restrict(0, 3000)
