"""Full-size BASELINE configs on the GPU, in bench.py's launch configuration,
against oracle values at seeded sampled targets (tests/golden/oracle_C*.npz,
written by scripts/make_golden.py from oracle/ only) and against structural
facts that hold at any size."""
import os

import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F

from .gpu_helpers import assert_parity

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _run(cid):
    import torch

    from paper_2010_15155_b200 import KAFMM
    spec, pts, vals = WL.make_config(cid)
    plan = KAFMM(pts, spec.kernel, spec.p, spec.cap)
    out = plan.eval(torch.from_numpy(vals).cuda()).cpu().numpy()
    inf = plan.info()
    plan.close()
    del plan
    torch.cuda.empty_cache()
    return spec, out, inf


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_fullsize_parity_at_sampled_targets(cid):
    path = os.path.join(GOLD, f"oracle_C{cid}.npz")
    if cid == 1:
        spec, pts, vals = WL.make_config(1)
        ref = F.fmm(pts, vals, spec.kernel, spec.p, spec.cap)
        g = dict(idx=np.arange(spec.n), fmm=ref["out"], kept=np.array(ref["kept"]),
                 direct_idx=np.arange(spec.n), direct=F.direct(spec.kernel, pts, vals))
    else:
        if not os.path.exists(path):
            pytest.skip(f"{path} not generated yet (scripts/make_golden.py {cid})")
        g = dict(np.load(path))
    spec, out, inf = _run(cid)
    assert (inf.kept_up, inf.kept_dn) == tuple(int(v) for v in g["kept"])
    if "nleaf" in g:
        assert inf.n_leaves == int(g["nleaf"]) and inf.n_boxes == int(g["nbox"]) and inf.depth == int(g["depth"])
    got = out[g["idx"]]
    assert_parity(spec.kernel, got, g["fmm"])   # block rel L2 <= 1e-10 and per-target max <= 1e-9
    d_got = out[g["direct_idx"]]
    pos = np.searchsorted(g["idx"], g["direct_idx"])
    for lo, hi in F.blocks(spec.kernel):
        eg = F.rel_l2(d_got[:, lo:hi], g["direct"][:, lo:hi])
        eo = F.rel_l2(g["fmm"][pos, lo:hi], g["direct"][:, lo:hi])
        assert eg <= 2.0 * eo + 1e-15, (eg, eo)


def test_complete_grid_structure_c2_c3():
    # C2 is the complete level-5 grid and C3 the complete level-6 grid;
    # V pairs per level of a complete grid: 3096, 53352, 584136, 5398920, 46298376
    _, _, i2 = _run(2)
    assert i2.n_leaves == 32768 and i2.depth == 5
    assert i2.n_v_pairs == 3096 + 53352 + 584136 + 5398920 and i2.n_u_pairs == (3 * 32 - 2) ** 3
    _, _, i3 = _run(3)
    assert i3.n_leaves == 262144 and i3.depth == 6
    assert i3.n_v_pairs == 52337880 and i3.n_u_pairs == (3 * 64 - 2) ** 3
