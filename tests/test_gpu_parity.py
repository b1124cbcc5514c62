"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): relative L2 <= 1e-10 against the oracle FMM
per output block (reading R11), and error against the direct sum <= 2x the
oracle FMM's.  Tree, lists and SVD kept counts are compared exactly first.
Sizes: small enough for the oracle to finish in seconds, large enough for
several tree levels, many GEMM tiles and ragged tails.
"""
import numpy as np
import pytest

import workloads as WL
from oracle import fmm as F
from oracle import lists as OL
from oracle.tree import Tree

from .gpu_helpers import assert_parity, block_errors, oracle_tree_keyed, run_gpu, tree_keyed

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _clustered(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.random((4, 3)) * 0.8 + 0.1
    pts = np.concatenate([c[i] + 0.02 * rng.standard_normal((n // 4, 3)) for i in range(4)])
    return np.clip(pts, 0.0, np.nextafter(1.0, 0.0))


CASES = [
    # (name, kernel, points-factory, p, cap)
    ("C1", "stokeslet", lambda: WL.make_config(1)[1], 8, 50),
    ("lap_uniform", "laplace_pgrad", lambda: np.random.default_rng(3).random((6000, 3)), 6, 40),
    ("lap_clustered", "laplace_pgrad", lambda: _clustered(5000, 4), 8, 30),
    ("rpy_uniform", "rpy", lambda: np.random.default_rng(5).random((3000, 3)), 6, 40),
    ("regvel_clustered", "stokes_reg_vel", lambda: _clustered(4000, 6), 6, 32),
    ("stokeslet_spheres", "stokeslet", lambda: WL.make_points(WL.CONFIGS[5], 12000, n_spheres=60), 6, 64),
    # polydisperse b / eps on the paper's log-normal cloud (C6, C7 shapes)
    ("C6_poly_rpy", "rpy", lambda: WL.make_points(WL.CONFIGS[6], 12000), 8, 150),
    ("C7_poly_regvel_omega", "stokes_reg_vel_omega", lambda: WL.make_points(WL.CONFIGS[7], 12000), 8, 150),
    # StokesRegVelOmega (Table VI) on an adaptive tree
    ("regvel_omega_clustered", "stokes_reg_vel_omega", lambda: _clustered(4000, 7), 6, 32),
    # torque-free: omega = Omega^eps f has no self term, so the far field of the omega block is tested
    ("regvel_omega_forces", "stokes_reg_vel_omega", lambda: _clustered(4000, 9), 6, 32),
    # LapPGradGrad (Table III), charges + dipoles on the paper's cloud (C8 shape)
    ("C8_pgradgrad", "laplace_pgradgrad", lambda: WL.make_points(WL.CONFIGS[8], 12000), 8, 150),
    ("pgradgrad_clustered", "laplace_pgradgrad", lambda: _clustered(5000, 8), 7, 30),
    ("C9_qpgradgrad", "laplace_qpgradgrad", lambda: WL.make_points(WL.CONFIGS[9], 12000), 8, 150),
]
POLY = {"C6_poly_rpy": 6, "C7_poly_regvel_omega": 7, "C8_pgradgrad": 8, "C9_qpgradgrad": 9}


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def case(request):
    name, kernel, mk, p, cap = request.param
    pts = mk()
    if name in POLY:
        vals = WL.make_values(WL.CONFIGS[POLY[name]], pts.shape[0])
    else:
        vals = WL.random_values(kernel, pts.shape[0], 17)
    if name == "regvel_omega_forces":
        vals[:, 3:6] = 0.0
    plan, gpu = run_gpu(pts, vals, kernel, p, cap)
    ref = F.fmm(pts, vals, kernel, p, cap, keep_internals=True)
    return dict(name=name, kernel=kernel, pts=pts, vals=vals, p=p, cap=cap, plan=plan, gpu=gpu, ref=ref)


def test_tree_identical(case):
    g, _ = tree_keyed(case["plan"])
    o = oracle_tree_keyed(case["ref"]["tree"])
    assert g.keys() == o.keys()
    for k in o:
        assert g[k][0] == o[k][0], k
        assert np.array_equal(g[k][1], o[k][1]), k


def _pairs(plan, which, keyof):
    tgt, src = plan.lists(which)
    return sorted((keyof[t], keyof[s]) for t, s in zip(tgt, src))


def test_lists_identical(case):
    plan, ref = case["plan"], case["ref"]
    _, t = tree_keyed(plan)
    keyof = [(int(t["level"][b]),) + tuple(int(v) for v in t["ijk"][b]) for b in range(t["level"].size)]
    ot = ref["tree"]
    okey = [(ot.level[b],) + tuple(ot.ijk[b]) for b in range(ot.nbox)]
    U = sorted((okey[b], okey[a]) for b, l in ref["U"].items() for a in l)
    V = sorted((okey[b], okey[a]) for b, l in ref["V"].items() for a in l)
    W = sorted((okey[b], okey[a]) for b, l in ref["W"].items() for a in l)
    X = sorted((okey[b], okey[a]) for b, l in ref["X"].items() for a in l)
    assert _pairs(plan, "U", keyof) == U
    assert _pairs(plan, "V", keyof) == V
    assert _pairs(plan, "W", keyof) == W
    assert _pairs(plan, "X", keyof) == X


def test_kept_counts(case):
    inf = case["plan"].info()
    assert (inf.kept_up, inf.kept_dn) == case["ref"]["kept"]


def test_fmm_parity_with_oracle(case):
    assert_parity(case["kernel"], case["gpu"], case["ref"]["out"], l2_tol=TOL)


def test_error_vs_direct_within_2x_oracle(case):
    d = F.direct(case["kernel"], case["pts"], case["vals"])
    eg = block_errors(case["kernel"], case["gpu"], d)
    eo = block_errors(case["kernel"], case["ref"]["out"], d)
    for a, b in zip(eg, eo):
        assert a <= 2.0 * b + 1e-15, (eg, eo)


def test_eval_host_matches_eval(case):
    # same path with host buffers; fp64 atomics reorder sums (run-to-run ~1e-13
    # after the 1/sigma_min amplification of the check->equivalent solve)
    out = case["plan"].eval_host(np.ascontiguousarray(case["vals"]))
    assert F.rel_l2(out, case["gpu"]) < 1e-11
