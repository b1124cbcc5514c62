"""Quick GPU shakedown: run each small case, print parity errors and timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as WL
from oracle import fmm as F
from paper_2010_15155_b200 import KAFMM

def one(name, kernel, pts, p, cap, oracle=True):
    vals = WL.random_values(kernel, pts.shape[0], 17)
    t = time.time(); plan = KAFMM(pts, kernel, p, cap); torch.cuda.synchronize(); ts = time.time() - t
    src = torch.from_numpy(vals).cuda()
    out = plan.eval(src); torch.cuda.synchronize()
    plan.set_timing(True)
    out = plan.eval(src); torch.cuda.synchronize()
    st = plan.stage_times()
    g = out.cpu().numpy()
    inf = plan.info()
    print(f"== {name}: setup {ts:.2f}s info {inf.as_dict()}", flush=True)
    print("   stages", {k: round(v, 3) for k, v in st.items()}, flush=True)
    if oracle:
        r = F.fmm(pts, vals, kernel, p, cap)
        d = F.direct(kernel, pts, vals)
        print("   kept oracle", r["kept"], "gpu", (inf.kept_up, inf.kept_dn))
        print("   gpu-vs-oracle", [F.rel_l2(g[:, lo:hi], r["out"][:, lo:hi]) for lo, hi in F.blocks(kernel)])
        print("   gpu-vs-direct", [F.rel_l2(g[:, lo:hi], d[:, lo:hi]) for lo, hi in F.blocks(kernel)])
        print("   orc-vs-direct", [F.rel_l2(r["out"][:, lo:hi], d[:, lo:hi]) for lo, hi in F.blocks(kernel)], flush=True)

one("C1", "stokeslet", WL.make_config(1)[1], 8, 50)
one("lap", "laplace_pgrad", np.random.default_rng(3).random((6000, 3)), 6, 40)
one("rpy", "rpy", np.random.default_rng(5).random((3000, 3)), 6, 40)
rng = np.random.default_rng(4); c = rng.random((4, 3)) * 0.8 + 0.1
cl = np.clip(np.concatenate([c[i] + 0.02 * rng.standard_normal((1000, 3)) for i in range(4)]), 0, 0.9999999)
one("regvel_cl", "stokes_reg_vel", cl, 6, 32)
one("lap_cl", "laplace_pgrad", cl, 8, 30)
for cid in (2,):
    spec, pts, vals = WL.make_config(cid)
    one(f"C{cid}", spec.kernel, pts, spec.p, spec.cap, oracle=False)
