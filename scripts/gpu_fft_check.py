"""M2L variants (dense / FFT blocks / FFT pairs / FFT auto) vs each other and
the oracle on small cases; per-variant timings on full configs (argv)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM

MODES = ("fft", "fft_blocks", "fft_pairs", "dense")


def errs(kernel, a, b):
    return [float(f"{F.rel_l2(a[:, lo:hi], b[:, lo:hi]):.2e}") for lo, hi in F.blocks(kernel)]


def small(name, kernel, pts, p, cap):
    vals = WL.random_values(kernel, pts.shape[0], 17)
    plan = KAFMM(pts, kernel, p, cap)
    src = torch.from_numpy(vals).cuda()
    res = {}
    for m in MODES:
        plan.set_m2l(m)
        res[m] = plan.eval(src).cpu().numpy()
    r = F.fmm(pts, vals, kernel, p, cap)["out"]
    print(name, {m: (errs(kernel, res[m], res["dense"]), errs(kernel, res[m], r)) for m in MODES}, flush=True)


rng = np.random.default_rng(4)
c = rng.random((4, 3)) * 0.8 + 0.1
cl = np.clip(np.concatenate([c[i] + 0.02 * rng.standard_normal((1000, 3)) for i in range(4)]), 0, 0.9999999)
if "--small" in sys.argv:
    small("C1", "stokeslet", WL.make_config(1)[1], 8, 50)
    small("lap10", "laplace_pgrad", np.random.default_rng(3).random((20000, 3)), 10, 40)
    small("rpy_sph", "rpy", WL.make_points(WL.CONFIGS[5], 9000, n_spheres=40), 6, 40)
    small("regvel_cl12", "stokes_reg_vel", cl, 12, 30)

for cid in [int(a) for a in sys.argv[1:] if a.isdigit()]:
    spec, pts, vals = WL.make_config(cid)
    t = time.time()
    plan = KAFMM(pts, spec.kernel, spec.p, spec.cap)
    torch.cuda.synchronize()
    ts = time.time() - t
    src = torch.from_numpy(vals).cuda()
    print(f"C{cid} fft stats", plan.fft_stats(), flush=True)
    res = {}
    for mode in MODES:
        if mode == "dense" and cid >= 3:
            continue
        plan.set_m2l(mode)
        out = plan.eval(src)
        torch.cuda.synchronize()
        plan.set_timing(True)
        out = plan.eval(src)
        torch.cuda.synchronize()
        st = plan.stage_times()
        plan.set_timing(False)
        res[mode] = out.cpu().numpy()
        print(f"C{cid} {mode}: setup {ts:.1f}s total {st['total']:.2f} ms -> {2*spec.n/st['total']*1e3:.3e} pts/s; "
              f"m2l {st['m2l']:.2f} product {st['m2l_product']:.2f}", flush=True)
    for mode in res:
        print(f"C{cid} {mode}-vs-fft_blocks", errs(spec.kernel, res[mode], res["fft_blocks"]), flush=True)
    del plan
    torch.cuda.empty_cache()
