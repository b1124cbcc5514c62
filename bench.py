#!/usr/bin/env python
"""Benchmark of the KAFMM evaluation pass (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Metric (BASELINE.json): FMM eval points/s = (N_S + N_T) / t_eval at fixed p.
A step is one kafmm_eval (gather, S2M, UC2UE, M2M, M2L, S2L, DC2DE, L2L,
L2T, M2T, P2P, scatter) over config C's synthetic cloud (default C5 =
BASELINE configs[4], 64M points on 10^4 sphere surfaces, Stokeslet p=8 cap
128: the largest config, which fits one GPU, and the 1-GPU point of the
BASELINE scaling curve), inputs resident in HBM.  L2 is flushed (256 MiB write) before every timed step, outside the
timed interval; each step is bracketed by CUDA events on the plan's stream.
"e2e" times kafmm_eval_host: pinned host values -> device, eval, -> host.

Multi-GPU (torchrun, N > 1): ONE problem split into contiguous Morton ranges
(paper_2010_15155_b200.dist): every rank holds a slice of the user rows,
the ranks exchange source values, shared and ghost multipoles and outputs
over NCCL (strong scaling).  Time = max over ranks.

--impl reference times the CPU oracle (oracle/, test infrastructure) on a
bounded sample of the same workload on the host cores (rank 0 only): each
step evaluates, with the unmodified oracle FMM, the points of a seeded set of
whole octree boxes of the workload (their subtrees are exactly the boxes'
subtrees of the full tree), and reports (N_S + N_T) / time of that sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as WL  # noqa: E402

# nominal flops per pair of the P2P kernels (rsqrt counted as 8)
P2P_FLOPS = {"laplace_pgrad": 27, "stokeslet": 36, "rpy": 56, "stokes_reg_vel": 39, "stokes_reg_vel_omega": 100,
             "laplace_pgradgrad": 90, "laplace_qpgradgrad": 120}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="kafmm", choices=["kafmm", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist", action="store_true", help="use the partitioned (NCCL) path even at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--sample-points", type=int, default=3000,
                    help="points per oracle sample (cpu_baseline / --impl reference step)")
    return ap.parse_args()


def workload_name(spec):
    return (f"C{spec.cid}: {spec.kernel}, N={spec.n}, {spec.cloud} cloud, p={spec.p}, "
            f"max {spec.cap} pts/leaf, open BC, fp64")


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        except Exception:
            rows = []
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def _oracle_ops(spec):
    """Oracle operators incl. all 316 M2L matrices: setup, not timed as eval."""
    from oracle import fmm as F
    from oracle.operators import v_offsets
    op = F.operators(F.TABLES[spec.kernel]["ML"], spec.p)
    for o in v_offsets():
        op.m2l[o]
    return op


def subbox_sample(spec, pts, target, seed):
    """Seeded sample of the workload: the points of whole octree boxes.

    Draw a point, take the deepest box of the full tree's quantisation that
    contains it and holds >= `target` points, and if that box holds more than
    4 x target, the Morton-consecutive run of its children (starting at the
    drawn point's child) until >= target points.  Every chosen box has more
    than `cap` points (target >= cap), so the oracle's tree over the sample
    reproduces those boxes' subtrees of the full tree exactly (same levels,
    same splits); what the sample lacks is the rest of the cloud, so its
    boundary leaves see fewer U/V/W/X neighbours than in the full problem and
    the oracle does less work per point than it would on the full workload.
    """
    target = max(int(target), spec.cap + 1)
    rng = np.random.default_rng(seed)
    q = np.clip(np.floor(pts * float(1 << 21)).astype(np.int64), 0, (1 << 21) - 1)
    i = int(rng.integers(pts.shape[0]))
    sel, level = np.arange(pts.shape[0]), 0
    for L in range(1, 21):
        sub = sel[np.all((q[sel] >> (21 - L)) == (q[i] >> (21 - L)), axis=1)]
        if sub.size < target:
            break
        sel, level = sub, L
    if sel.size > 4 * target and level < 20:
        sh = 20 - level
        octs = ((q[sel] >> sh) & 1) @ np.array([4, 2, 1])
        o0 = int(((q[i] >> sh) & 1) @ np.array([4, 2, 1]))
        keep = []
        for o in list(range(o0, 8)) + list(range(o0)):
            keep.append(sel[octs == o])
            if sum(k.size for k in keep) >= target:
                break
        sel = np.sort(np.concatenate(keep))
    return sel, level


def oracle_subbox_run(spec, pts, vals, target, seed, op):
    """One unmodified oracle FMM evaluation over a sub-box sample; returns
    (points in the sample, evaluation seconds = upward + downward pass, box level).
    The oracle's tree and interaction lists are setup (like the GPU plan)."""
    from oracle import fmm as F
    from oracle.tree import Tree
    sel, level = subbox_sample(spec, pts, target, seed)
    p_s, v_s = pts[sel], vals[sel]
    t = Tree(p_s, spec.cap)
    tm = {}
    F.fmm(p_s, v_s, spec.kernel, spec.p, spec.cap, tree=t, ops=op, timings=tm)
    return sel.size, tm["upward"] + tm["downward"], level


def oracle_sample_rate(spec, pts, vals, budget_s, target):
    """cpu_baseline: the oracle on seeded sub-box samples until budget_s of evaluation time."""
    op = _oracle_ops(spec)
    npts, secs, runs, levels = 0, 0.0, 0, []
    while secs < budget_s and runs < 64:
        n_s, t_s, lev = oracle_subbox_run(spec, pts, vals, target, 7919 + runs, op)
        npts += n_s
        secs += t_s
        levels.append(lev)
        runs += 1
    cores = len(os.sched_getaffinity(0))
    return dict(value=2 * npts / secs, unit="points/s", cores=cores, kind="oracle",
                sample=(f"oracle (numpy/scipy, {cores} host threads), full FMM evaluation (upward + downward "
                        f"pass, lists and operators as setup) of {runs} seeded samples of {spec.name}, each the "
                        f"points of whole boxes of its octree (box levels {sorted(set(levels))}, >= {target} "
                        f"points each, {npts} points in all) in {secs:.1f} s; a sample lacks the rest of the "
                        f"cloud, so its boundary leaves do less near/far work than in the full problem"))


def run_reference(args, spec, pts, vals, rank):
    if rank != 0:
        return
    op = _oracle_ops(spec)
    per, sizes = [], []
    for s in range(args.warmup + args.steps):
        # a step = one unmodified oracle evaluation of a seeded sub-box sample of the workload
        n_s, t_s, _ = oracle_subbox_run(spec, pts, vals, args.sample_points, 1000 + s, op)
        if s >= args.warmup:
            per.append(t_s)
            sizes.append(n_s)
    value = 2 * sum(sizes) / sum(per)
    ms = 1e3 * statistics.mean(per)
    cores = len(os.sched_getaffinity(0))
    sample = (f"per step: the unmodified oracle FMM (numpy/scipy, {cores} host threads) on a seeded sample of "
              f"whole octree boxes of {spec.name} (>= {args.sample_points} points; mean {statistics.mean(sizes):.0f} "
              f"points, upward + downward pass timed, lists and operators as setup); value = 2 x sampled points / "
              f"time summed over the {len(per)} timed steps")
    line = {"impl": "reference", "metric": "FMM eval points/sec (N_S+N_T) at fixed p", "value": value,
            "unit": "points/s", "n_gpus": args.gpus, "steps": len(per), "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(spec), "kernel": spec.kernel, "n": spec.n, "p": spec.p,
                       "max_pts_per_leaf": spec.cap},
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec = WL.CONFIGS[args.config]
    spec_pts = WL.make_points(spec)
    vals = WL.make_values(spec, spec_pts.shape[0])

    if args.impl == "reference":
        run_reference(args, spec, spec_pts, vals, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2010_15155_b200 import KAFMM
    from paper_2010_15155_b200.kafmm import fp64_peak

    torch.cuda.set_device(local)
    use_dist = world > 1 or args.dist
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    if not use_dist:
        # one GPU: the whole evaluation through kafmm_eval
        torch.cuda.synchronize()
        t_setup = time.perf_counter()
        plan = KAFMM(spec_pts, spec.kernel, spec.p, spec.cap, stream=stream)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t_setup
        info = plan.info()
        src = torch.from_numpy(vals).cuda()
        out = torch.empty((spec.n, info.k_t), dtype=torch.float64, device="cuda")
        run_step = lambda: plan.eval(src, out)  # noqa: E731
        n_v_local, n_p2p_local = info.n_v_pairs, info.n_p2p
        h_vals = vals
        def run_e2e(hsrc, hout):
            plan.eval_host(hsrc, hout)
    else:
        # N GPUs: ONE problem split by Morton ranges (strong scaling); every rank
        # holds a contiguous slice of the user rows and gets its rows' outputs back
        from paper_2010_15155_b200.dist import dist_plan
        offs = np.linspace(0, spec.n, world + 1).astype(np.int64)
        lo, hi = int(offs[rank]), int(offs[rank + 1])
        torch.cuda.synchronize()
        t_setup = time.perf_counter()
        plan = dist_plan(spec_pts[lo:hi], spec.kernel, spec.p, spec.cap, stream=stream)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t_setup
        info = plan.info()
        dinfo = plan.dist_info()
        h_vals = np.ascontiguousarray(vals[lo:hi])
        src = torch.from_numpy(h_vals).cuda()
        out = torch.empty((hi - lo, info.k_t), dtype=torch.float64, device="cuda")
        run_step = lambda: plan.eval(src, out)  # noqa: E731
        n_v_local, n_p2p_local = dinfo["n_v_local"], dinfo["n_p2p_local"]
        def run_e2e(hsrc, hout):
            plan.eval_host(hsrc, hout)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        run_step()
    barrier()

    # timed steps: total and M2L-product events only (mode 2), so the near field
    # still overlaps the far-field chain exactly as in an untimed evaluation
    plan.set_timing(2)
    step_ms, stages = [], []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            stages.append(plan.stage_times())
        barrier()
    clocks = clk.summary()
    # CUDA-graph replay of the same evaluation (launch overhead removed), timed
    # the same way but without per-kernel events: reported beside `value`
    graph_ms = None
    if world == 1 and not args.dist:
        plan.set_timing(0)
        plan.set_graph(True)
        run_step()
        run_step()
        gt = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            e1.synchronize()
            gt.append(e0.elapsed_time(e1))
        plan.set_graph(False)
        graph_ms = statistics.mean(gt)
    # one more evaluation with per-stage events (mode 1 serialises the near
    # field) for the breakdown and the P2P kernel time; not part of `value`
    plan.set_timing(1)
    run_step()
    torch.cuda.synchronize()
    breakdown = plan.stage_times()
    plan.set_timing(False)
    launches = plan.launch_count() * args.steps

    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / args.steps
    value = 2 * spec.n / (ms * 1e-3)   # the whole job: one problem of N_S + N_T = 2N points

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hsrc = torch.from_numpy(h_vals).pin_memory().numpy()
        hout = torch.empty((h_vals.shape[0], info.k_t), dtype=torch.float64).pin_memory().numpy()
        run_e2e(hsrc, hout)
        et = []
        for _ in range(args.steps):
            flush.fill_(1.0)   # same cold-L2 start as the device-timed steps
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            run_e2e(hsrc, hout)
            et.append(time.perf_counter() - t0)
        e = torch.tensor([sum(et)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        e_s = float(e.item()) / args.steps
        e2e = {"value": 2 * spec.n / e_s, "unit": "points/s", "ms_per_step": 1e3 * e_s,
               "h2d_bytes_per_step": int(hsrc.nbytes) * world, "d2h_bytes_per_step": int(hout.nbytes) * world}

    # roofline of the dominant kernel: the M2L product on the FP64 tensor cores
    # (DMMA.8x8x4): the frequency-space products of the FFT M2L, or the dense
    # per-offset GEMMs.  Algorithmic work per V pair:
    #   FFT:   8 kml^2 flop per frequency bin (kml x kml complex multiply-adds), NF bins
    #   dense: 2 n^2 flop, n = kml M
    mode = plan.m2l()
    m2l_ms = breakdown["m2l"]
    prod_ms = statistics.mean(s["m2l_product"] for s in stages)
    p2p_ms = breakdown["p2p"]
    n = info.n_equiv
    kml = n // info.n_surf
    ng = 2 * spec.p - 1
    nf = ng * ng * (ng // 2 + 1)
    if mode.startswith("fft"):
        m2l_flop = 8.0 * kml * kml * nf * n_v_local
        algo = (f"FFT M2L: 8 kml^2 flop per V pair per frequency bin, kml={kml}, NF={nf} (grid {ng}^3), "
                f"{n_v_local} V pairs = {m2l_flop:.3e} flop")
        kname = ("m2l product: k_m2l_dmma (dense chunks: per-frequency complex GEMM over parent blocks, "
                 "DMMA.8x8x4, 3 real products per complex multiply-add = 6 of the 8 algorithmic flops) + "
                 "k_m2l_groups (sparse chunks: per-warp stream of (half parent, colleague, source x half) "
                 "groups over 32 bins, each offset's operator loaded once for its valid pairs, absent child "
                 "pairs skipped, on the DFMA pipe; KAFMM_SPARSE=items selects the per-pair k_m2l_items)")
    else:
        m2l_flop = 2.0 * n * n * n_v_local
        algo = f"dense M2L: 2 n^2 flop per V pair, n={n}, {n_v_local} pairs = {m2l_flop:.3e} flop"
        kname = "m2l product (k_gemm_dmma: dense, grouped by V offset, DMMA.8x8x4)"
    peak_dmma = fp64_peak("dmma")
    # the dense chunks' product runs on the FP64 tensor pipe (DMMA), the sparse chunks' on
    # the FP64 ALU pipe (DFMA); both have the same nominal rate on B200 (37.2 TFLOP/s), and
    # the peak below is the higher measured one (the DMMA loop)
    fs0 = plan.fft_stats() if mode.startswith("fft") else None
    bound = "alu" if fs0 and 2 * fs0.get("pair_chunks", 0) > fs0.get("chunks", 0) else "tensor"
    peak_dfma = fp64_peak("dfma")
    achieved = m2l_flop / (prod_ms * 1e-3) / 1e12
    # DRAM traffic of the product kernels: device counters exist only under ncu, so it is
    # read from the committed `ncu --set full` capture of this config (named in
    # traffic_source), summed over the product launches of one evaluation, or null
    traffic, traffic_src = None, f"null: no ncu --set full capture of C{spec.cid}'s product kernels committed"
    tf = os.path.join(ROOT, "profiles", f"traffic_C{spec.cid}.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("m2l_mode") == mode:
                traffic = tj.get("m2l_dram_bytes_per_eval", tj.get("m2l_dram_bytes_per_launch"))
                traffic_src = tj.get("source")
        except Exception:
            traffic = None
    fs = plan.fft_stats() if mode.startswith("fft") else None
    algo_bytes = None
    if fs:
        # the spectra of every existing source child read once (ub) and of every target box
        # written once (cb), kml components x NF bins x 16 B, per evaluation
        algo_bytes = 16 * kml * nf * (fs["source_children"] + fs["targets"])
    p2p_flop = P2P_FLOPS[spec.kernel] * n_p2p_local
    stage_mean = {k: round(v, 4) for k, v in breakdown.items()}

    line = {
        "metric": "FMM eval points/sec (N_S+N_T) at fixed p", "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(spec), "kernel": spec.kernel, "n": spec.n, "p": spec.p,
                   "max_pts_per_leaf": spec.cap, "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": (f"{world} GPUs: one problem split into Morton ranges, NCCL exchanges "
                                   "(values, shared + ghost multipoles, outputs); roofline/stages of rank 0")
                   if use_dist else "1 GPU",
                   "m2l": mode},
        "roofline": {"kernel": kname, "bound": bound, "achieved": achieved, "peak": peak_dmma,
                     "unit": "TFLOP/s", "frac": achieved / peak_dmma, "traffic": traffic,
                     "traffic_source": traffic_src, "traffic_unit": "DRAM bytes per evaluation, product launches",
                     "algorithmic_bytes": algo_bytes,
                     "peak_source": "measured in this run: DMMA.8x8x4 loop (kafmm_fp64_peak); "
                                    "MEASURED_PEAKS.json has no FP64 entry",
                     "algorithmic": algo, "kernel_ms": prod_ms, "m2l_stage_ms": m2l_ms,
                     "m2l_stage_tflops": m2l_flop / (m2l_ms * 1e-3) / 1e12},
        "p2p": {"achieved_tflops": p2p_flop / (p2p_ms * 1e-3) / 1e12, "peak": peak_dmma,
                "frac": p2p_flop / (p2p_ms * 1e-3) / 1e12 / peak_dmma,
                "peak_note": "the chip's measured FP64 peak (DMMA loop); the DFMA loop reaches peak_dfma_loop",
                "peak_dfma_loop": peak_dfma, "pairs": n_p2p_local,
                "flop_per_pair": P2P_FLOPS[spec.kernel], "ms": p2p_ms},
        "stages_ms": stage_mean,
        "stages_note": ("per-stage events of one extra evaluation with the stages serialised (the timed steps run "
                        "the near field concurrently with the far field)"),
        "fft_m2l": fs,
        "cuda_graph": None if graph_ms is None else {"ms_per_step": graph_ms, "value": 2 * spec.n / (graph_ms * 1e-3)},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": e2e,
        "setup": {"s": t_setup, "plan_bytes": int(info.workspace_bytes), "n_boxes": int(info.n_boxes),
                  "note": "kafmm_setup (tree, lists, operators, FFT tables) wall clock, rank 0; not part of value"},
    }
    if use_dist:
        line["dist"] = {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in dinfo.items()}
        line["dist"]["note"] = ("rank 0's partition: kafmm_setup_dist (NCCL inside libkafmm); plan_bytes is this "
                                "rank's device memory, bytes_per_eval what it sends per evaluation")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in oracle_sample_rate(spec, spec_pts, vals, args.cpu_budget,
                                                                    args.sample_points).items()
                                if k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
