import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as WL
from paper_2010_15155_b200 import KAFMM
for cid in [int(a) for a in sys.argv[1:]] or [2]:
    spec, pts, vals = WL.make_config(cid)
    t = time.time(); plan = KAFMM(pts, spec.kernel, spec.p, spec.cap); torch.cuda.synchronize(); ts = time.time() - t
    src = torch.from_numpy(vals).cuda()
    for _ in range(2): out = plan.eval(src)
    torch.cuda.synchronize()
    plan.set_timing(True); out = plan.eval(src); torch.cuda.synchronize()
    print(f"== C{cid} setup {ts:.2f}s", plan.info().as_dict(), flush=True)
    print("   stages", {k: round(v, 3) for k, v in plan.stage_times().items()}, flush=True)
    plan.set_timing(False)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): plan.eval(src)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"   eval {ms:.2f} ms -> {2*spec.n/ms*1e3:.3e} points/s", flush=True)
    del plan; torch.cuda.empty_cache()
