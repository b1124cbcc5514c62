"""Write tests/golden/oracle_C{c}.npz: oracle KAFMM values at sampled targets of
the full-size BASELINE configs, plus the O1 direct sum at a subset of them.

Calls only oracle/ (and the seeded generators in workloads/).  Sampled mode
(SURVEY.md §8(c) step 10): full upward pass; downward pass and near field
only for the ancestors of a seeded draw of whole leaves.

    python scripts/make_golden.py 2 3 4 5
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as WL  # noqa: E402
from oracle import fmm as F  # noqa: E402
from oracle.kernels import direct_sum  # noqa: E402
from oracle.tree import Tree  # noqa: E402

SAMPLE_LEAVES = {2: 12, 3: 12, 4: 10, 5: 6, 6: 2, 7: 2, 8: 2, 9: 2}
DIRECT_TARGETS = {2: 400, 3: 300, 4: 200, 5: 96, 6: 200, 7: 200, 8: 200, 9: 200}


def main(cids):
    for cid in cids:
        t0 = time.time()
        spec, pts, vals = WL.make_config(cid)
        print(f"C{cid}: generated {pts.shape} in {time.time() - t0:.0f}s", flush=True)
        t = Tree(pts, spec.cap)
        print(f"C{cid}: tree nbox={t.nbox} leaves={t.leaves().size} depth={t.depth} ({time.time() - t0:.0f}s)",
              flush=True)
        rng = np.random.default_rng(cid + 7)
        leaves = t.leaves()
        smp = sorted(int(b) for b in rng.choice(leaves, size=SAMPLE_LEAVES[cid], replace=False))
        tm = {}
        r = F.fmm(pts, vals, spec.kernel, spec.p, spec.cap, target_leaves=smp, tree=t, timings=tm,
                  keep_internals=True)
        print(f"C{cid}: oracle sampled fmm {tm} kept={r['kept']} ({time.time() - t0:.0f}s)", flush=True)
        idx = r["idx"]
        sub = np.sort(rng.choice(idx, size=min(DIRECT_TARGETS[cid], idx.size), replace=False))
        d = direct_sum(F.TABLES[spec.kernel]["ST"], pts[sub], pts, vals, chunk=4)
        print(f"C{cid}: direct at {sub.size} targets ({time.time() - t0:.0f}s)", flush=True)
        pos = np.searchsorted(idx, sub)
        errs = [F.rel_l2(r["out"][pos, lo:hi], d[:, lo:hi]) for lo, hi in F.blocks(spec.kernel)]
        n_v_sample = sum(len(v) for v in r["V"].values())
        out = os.path.join(ROOT, "tests", "golden", f"oracle_C{cid}.npz")
        np.savez_compressed(
            out, cid=cid, kernel=spec.kernel, n=spec.n, p=spec.p, cap=spec.cap,
            leaf_keys=np.array([(t.level[b],) + tuple(t.ijk[b]) for b in smp], dtype=np.int64),
            idx=idx, fmm=r["out"], direct_idx=sub, direct=d, oracle_err_vs_direct=np.array(errs),
            kept=np.array(r["kept"]), nbox=t.nbox, nleaf=leaves.size, depth=t.depth,
            n_v_sampled_boxes=n_v_sample, timings=np.array([tm["lists"], tm["upward"], tm["downward"]]))
        print(f"C{cid}: wrote {out}; oracle err vs direct per block {errs} ({time.time() - t0:.0f}s)", flush=True)
        del t, r, pts, vals


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2, 3, 4, 5])
