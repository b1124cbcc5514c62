"""FFT M2L vs dense M2L vs oracle on small cases; timings on full configs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM

def errs(kernel, a, b): return [F.rel_l2(a[:, lo:hi], b[:, lo:hi]) for lo, hi in F.blocks(kernel)]

def small(name, kernel, pts, p, cap):
    vals = WL.random_values(kernel, pts.shape[0], 17)
    plan = KAFMM(pts, kernel, p, cap); src = torch.from_numpy(vals).cuda()
    plan.set_m2l("fft"); a = plan.eval(src).cpu().numpy()
    plan.set_m2l("dense"); b = plan.eval(src).cpu().numpy()
    r = F.fmm(pts, vals, kernel, p, cap)["out"]
    print(f"{name}: fft-vs-dense {errs(kernel, a, b)} fft-vs-oracle {errs(kernel, a, r)} dense-vs-oracle {errs(kernel, b, r)}", flush=True)

rng = np.random.default_rng(4); c = rng.random((4, 3)) * 0.8 + 0.1
cl = np.clip(np.concatenate([c[i] + 0.02 * rng.standard_normal((1000, 3)) for i in range(4)]), 0, 0.9999999)
small("C1", "stokeslet", WL.make_config(1)[1], 8, 50)
small("lap6", "laplace_pgrad", np.random.default_rng(3).random((6000, 3)), 6, 40)
small("lap10", "laplace_pgrad", np.random.default_rng(3).random((20000, 3)), 10, 40)
small("rpy", "rpy", np.random.default_rng(5).random((3000, 3)), 6, 40)
small("regvel_cl", "stokes_reg_vel", cl, 6, 32)
small("lap_cl12", "laplace_pgrad", cl, 12, 30)
small("stk_cl12", "stokeslet", cl, 12, 30)

for cid in [int(a) for a in sys.argv[1:]]:
    spec, pts, vals = WL.make_config(cid)
    t = time.time(); plan = KAFMM(pts, spec.kernel, spec.p, spec.cap); torch.cuda.synchronize(); ts = time.time() - t
    src = torch.from_numpy(vals).cuda()
    res = {}
    for mode in ("fft", "dense"):
        if mode == "dense" and cid >= 3: continue
        plan.set_m2l(mode)
        out = plan.eval(src); torch.cuda.synchronize()
        plan.set_timing(True); out = plan.eval(src); torch.cuda.synchronize()
        st = plan.stage_times(); plan.set_timing(False)
        res[mode] = out.cpu().numpy()
        print(f"C{cid} {mode}: setup {ts:.1f}s total {st['total']:.2f} ms -> {2*spec.n/st['total']*1e3:.3e} pts/s; stages", {k: round(v, 3) for k, v in st.items()}, flush=True)
    if "dense" in res: print(f"C{cid} fft-vs-dense", errs(spec.kernel, res["fft"], res["dense"]), flush=True)
    del plan; torch.cuda.empty_cache()
