#!/usr/bin/env python
"""PnP-MS2G hot-path benchmark (BASELINE.json metric) on B200.

One step = one whole PnP-MS2G solve of the C4 workload (1024^2 image, 1440
views x 1536 bins, stages 2x:30 then full:20, Gaussian denoiser, per-stage
20-step power iteration) = every row of SURVEY §8(a), replayed as one CUDA
graph with b resident in HBM.  value = PnP-MS2G iterations/s (50 per solve)
over all ranks; views are sharded across ranks (torchrun --nproc-per-node N)
with an NCCL allreduce of the partial backprojection: strong scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ms2g|reference]

--impl reference times the fp64 CPU oracle (the only reference this paper
has) on a bounded sample of the same workload, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ms2g_synth as S  # noqa: E402

METRIC = "sketched-gradient evals/s and PnP-MS2G iters/s at 512²/1024², frac. of HBM roofline"
CFG = 4


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def nnz_counts():
    with open(os.path.join(ROOT, "profiles", "nnz_counts.json")) as f:
        return json.load(f)


def workload_config(pr, nranks, l2_note, allreduce="nccl"):
    return {"workload": f"C{pr.cfg}: {pr.n}x{pr.n} fp32 phantom ({pr.n_ellipses} seeded ellipses), fan-beam "
                        f"{pr.n_views} views x {pr.n_bins} bins, stages "
                        + " -> ".join(f"{s[0]}x:{s[1]}" for s in pr.stages)
                        + f", Gaussian 3x3 denoiser alpha={pr.alpha}, 20 power iterations per stage",
            "image": pr.n, "views": pr.n_views, "bins": pr.n_bins, "iters_per_solve": pr.n_steps,
            "parallelism": (f"views sharded x{nranks} + " + ("NCCL allreduce" if allreduce == "nccl" else
                                                              "NVLink peer-memory sum (NEXT-3)"))
            if nranks > 1 else "1 GPU",
            "l2": l2_note}


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 2 + k and r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# -------------------------------------------------------------- oracle arm --
_last_s2 = [None]   # seconds of the last all-core factor-2 oracle gradient (for the 1-core ratio)


def oracle_sample(pr, b_full, nthreads):
    """Time the fp64 oracle on a bounded sample of the C4 solve: one factor-2
    gradient, one full gradient and one Gaussian denoise; compose the solve
    (20 + 30 factor-2 and 20 + 20 full gradient-equivalents, 50 denoises).
    Returns (iters/s, seconds of CPU work, description)."""
    import oracle as O
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    x = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, 9)).astype(np.float64)
    t = {}
    t0 = time.perf_counter()
    for s in (2, 1):
        a = time.perf_counter()
        O.sketched_grad(g, s, x, b_full, nthreads=nthreads)
        t[s] = time.perf_counter() - a
    a = time.perf_counter()
    O.gauss3(x, 0.8)
    t["den"] = time.perf_counter() - a
    total = time.perf_counter() - t0
    n2 = sum(st[1] for st in pr.stages if st[0] == 2)
    n1 = sum(st[1] for st in pr.stages if st[0] == 1)
    solve = (pr.power_iters + n2) * t[2] + (pr.power_iters + n1) * t[1] + pr.n_steps * t["den"]
    _last_s2[0] = t[2]
    desc = (f"C{pr.cfg} oracle, {nthreads} threads: 1 factor-2 gradient ({t[2]:.2f} s) + 1 full gradient "
            f"({t[1]:.2f} s) + 1 Gaussian denoise ({t['den']:.3f} s), composed into one solve "
            f"({pr.power_iters}+{n2} factor-2 and {pr.power_iters}+{n1} full gradient-equivalents, "
            f"{pr.n_steps} denoises) = {solve:.1f} s")
    return pr.n_steps / solve, total, desc


def make_data(pr):
    """Seeded phantom, exact projection by the GPU projector, Gaussian noise."""
    import torch

    import paper_2203_07308_b200 as P
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg), texture=pr.texture)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(1,)) as full:
        p = P.forward_project(full, 1, torch.from_numpy(xt).cuda()[None])[0].cpu().numpy()
    if pr.noise[0] == "gauss":
        return S.gaussian_data(p, pr.noise[1], S.config_seed(pr.cfg))
    return S.poisson_data(p, pr.noise[1], S.config_seed(pr.cfg))


def run_reference(args, rank, nranks):
    if rank != 0:
        return
    pr = S.PRESETS[CFG]
    import oracle as O
    nthreads = O.default_threads()
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg))
    b = S.gaussian_data(O.forward(g, 1, xt, nthreads=nthreads), pr.noise[1], S.config_seed(pr.cfg))
    vals, secs_l, desc = [], [], ""
    for k in range(args.warmup + args.steps):
        v, secs, desc = oracle_sample(pr, b.astype(np.float64), nthreads)
        if k >= args.warmup:
            vals.append(v)
            secs_l.append(secs)
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(secs_l),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(pr, 1, "n/a (CPU)"),
            "cpu_baseline": {"value": value, "unit": "iters/s", "cores": nthreads, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm --
def time_calls(fn, reps, warm=3):
    import torch
    for _ in range(warm):
        fn()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1000.0


def detail_512(P, dev):
    """512^2 numbers of the metric (C3/C5 geometry, 720 x 768): sketched-
    gradient evals/s at s = 4, 2, 1 on all views and on one 1/8 subset, the
    C3 Option-2 solve (64 iterations, 3 stages with power iterations) and the
    C5 batch-8 solve (Poisson data, TV) in iterations/s per image."""
    import torch
    out = {}
    pr3, pr5 = S.PRESETS[3], S.PRESETS[5]
    nnz = nnz_counts()["C3"]
    with P.plan_geometry(pr3.n, pr3.n_views, pr3.n_bins, factors=(4, 2, 1)) as plan:
        x = torch.from_numpy(S.phantom(pr3.n, pr3.n_ellipses, S.config_seed(3, 9))).to(dev)[None].contiguous()
        xt = S.phantom(pr3.n, pr3.n_ellipses, S.config_seed(3), texture=pr3.texture)
        p = P.forward_project(plan, 1, torch.from_numpy(xt).to(dev)[None])[0].cpu().numpy()
        b = torch.from_numpy(S.gaussian_data(p, pr3.noise[1], S.config_seed(3))).to(dev)[None].contiguous()
        g = torch.empty_like(x)
        sub = list(range(0, pr3.n_views, 8))
        for s_ in (4, 2, 1):
            t_all = time_calls(lambda: P.sketched_grad(plan, s_, x, b, g=g), 10)
            t_sub = time_calls(lambda: P.sketched_grad(plan, s_, x, b, g=g, subset=sub), 10)
            out[f"C3_512_grad_s{s_}"] = {"evals_per_s": 1.0 / t_all, "subset_evals_per_s": 1.0 / t_sub,
                                         "segments_per_s": 2 * nnz[str(s_)] / t_all,
                                         "subset_segments_per_s": 2 * nnz[f"{s_}_subset0"] / t_sub}
        x0 = torch.zeros_like(x); xo = torch.empty_like(x)
        kw = dict(option=2, n_subsets=8, seed=S.config_seed(3), den=pr3.den, alpha=pr3.alpha)
        ts = time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr3.stages, b, x0, xo, **kw), 10, warm=3)
        P.solve_status(plan)
        tc = time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr3.stages, b, x0, xo, power_iters=0, **kw), 10, warm=3)
        P.solve_status(plan)
        out["C3_512_solve"] = {"iters_per_s": pr3.n_steps / ts, "ms_per_solve": ts * 1e3,
                               "cached_step_iters_per_s": pr3.n_steps / tc, "cached_step_ms_per_solve": tc * 1e3,
                               "schedule": "Option 2, 8 subsets, epochs [3,3,2] at s=4,2,1 (3 x 20 power "
                                           "iterations; cached_step: power_iters=0)"}
    nb = pr5.batch
    with P.plan_geometry(pr5.n, pr5.n_views, pr5.n_bins, factors=(2, 1), batch=nb) as plan:
        bs = []
        with P.plan_geometry(pr5.n, pr5.n_views, pr5.n_bins, factors=(1,)) as one:
            for im in range(nb):
                xt = S.phantom(pr5.n, pr5.n_ellipses, S.config_seed(5, im))
                p = P.forward_project(one, 1, torch.from_numpy(xt).to(dev)[None])[0].cpu().numpy()
                bs.append(S.poisson_data(p, pr5.noise[1], S.config_seed(5, im)))
        b = torch.from_numpy(np.stack(bs)).to(dev).contiguous()
        x0 = torch.zeros((nb, pr5.n, pr5.n), device=dev); xo = torch.empty_like(x0)
        kw = dict(den=pr5.den, alpha=pr5.alpha)
        ts = time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr5.stages, b, x0, xo, **kw), 5, warm=2)
        P.solve_status(plan)
        out["C5_512_batch8_solve"] = {"image_iters_per_s": nb * pr5.n_steps / ts, "ms_per_solve": ts * 1e3,
                                      "images_per_solve": nb}
    return out


def shard_estimate(P, dev, pr, b_full, t_solve_1):
    """Multi-GPU scaling ESTIMATE for view sharding (only one GPU
    here): the solve on every rank's contiguous view shard, the slowest of
    them (SURVEY: "max shard time") timed on this
    GPU with a 1-rank NCCL communicator (same kernels and graph shape as an
    N-rank run, 1/N of the views; the in-graph allreduce is an identity), plus
    a modelled allreduce per gradient and per power iteration: 20 us latency +
    2 x bytes at 450 GB/s (NVLink 5 ring bus bandwidth, conservative vs NVLS).
    Not measured scaling: labelled estimated."""
    import torch
    out = {}
    n_ar = {2: pr.power_iters + sum(s_[1] for s_ in pr.stages if s_[0] == 2),
            1: pr.power_iters + sum(s_[1] for s_ in pr.stages if s_[0] == 1)}
    t_ar = sum(n * (20e-6 + 2 * 4 * (pr.n // f) ** 2 / 450e9) for f, n in n_ar.items())
    for nr in (2, 4, 8):
        shard_ms = []
        for r in range(nr):          # every rank's shard; the slowest sets the pace
            vb, ve = P.view_shard(pr.n_views, r, nr)
            with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve) as plan:
                # a 1-rank communicator: the graph then has the N-rank run's shape
                # (in-graph allreduce nodes, power iterations serial on one stream)
                P.attach_nccl(plan, 0, 1)
                b = torch.from_numpy(np.ascontiguousarray(b_full[vb:ve])).to(dev)[None].contiguous()
                x0 = torch.zeros((1, pr.n, pr.n), device=dev); xo = torch.empty_like(x0)
                kw = dict(den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters)
                shard_ms.append(1e3 * time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, **kw),
                                                 3, warm=2))
                try:
                    P.solve_status(plan)
                except P.MS2GError:
                    pass      # a shard's partial operator alone may drive the toy iterate anywhere; timing only
        ts = max(shard_ms) / 1e3
        t = ts + t_ar
        out[f"N{nr}"] = {"max_shard_solve_ms": ts * 1e3, "shard_solve_ms": [round(v, 3) for v in shard_ms],
                         "allreduce_model_ms": t_ar * 1e3, "est_iters_per_s": pr.n_steps / t,
                         "est_speedup": t_solve_1 / t}
    out["note"] = ("estimated: slowest rank shard timed on 1 GPU (L2 not flushed) + modelled allreduce; "
                   "not measured scaling")
    return out


def run_ms2g(args, rank, nranks, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2203_07308_b200 as P
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pr = S.PRESETS[CFG]
    P.load()
    b_full = make_data(pr)
    vb, ve = P.view_shard(pr.n_views, rank, nranks)
    plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve)
    if nranks > 1:
        if args.allreduce == "peer":     # NEXT-3: fused NVLink peer-memory sum (fixed rank order)
            P.attach_peers(plan, rank, nranks)
        else:
            P.attach_nccl(plan, rank, nranks)
    b = torch.from_numpy(np.ascontiguousarray(b_full[vb:ve])).to(dev)[None].contiguous()
    x0 = torch.zeros((1, pr.n, pr.n), device=dev)
    xo = torch.empty_like(x0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    kw = dict(den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters)

    def step():
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, **kw)

    if args.profile_once:
        step()
        step()
        P.solve_status(plan)
        plan.destroy()
        return

    for _ in range(args.warmup):
        step()
    P.solve_status(plan)
    st = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if nranks > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = P.launch_count()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))              # L2 flush between timed steps (outside the events)
            evs[k][0].record(st)
            step()
            evs[k][1].record(st)
        torch.cuda.synchronize()
    if nranks > 1:
        dist.barrier()
    launches = P.launch_count() - l0
    P.solve_status(plan)
    t_local = sum(a.elapsed_time(c) for a, c in evs) / 1000.0
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if nranks > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_total = float(t.item())
    value = pr.n_steps * args.steps / t_total
    clocks = clk.summary()

    # ---- the same K steps again with CUDA events around every projector
    # launch inside the solve graph (ms2g_set_kernel_timing): per-kernel device
    # time over the timed workload, for the roofline (costs ~1 % per step, so
    # the headline above is taken without them) ----
    P.set_kernel_timing(plan, True)
    step()
    P.solve_status(plan)
    ktime = {}
    ti0, ti1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_instr = 0.0
    for k in range(args.steps):
        flush.fill_(float(k))
        ti0.record(st)
        step()
        ti1.record(st)
        ti1.synchronize()
        t_instr += ti0.elapsed_time(ti1)
        for kern in ("forward", "backward"):
            for f_ in (2, 1):
                ms_, n_ = P.kernel_time(plan, kern, f_)
                a_ = ktime.setdefault((kern, f_), [0.0, 0])
                a_[0] += ms_
                a_[1] += n_
    P.set_kernel_timing(plan, False)
    P.solve_status(plan)

    # ---- e2e: public API with host buffers (pinned H2D of b, D2H of x) ----
    b_host = b.cpu().pin_memory()
    x_host = torch.empty((1, pr.n, pr.n), dtype=torch.float32).pin_memory()
    b_dev2 = torch.empty_like(b)
    x_dev2 = torch.empty_like(x0)

    def e2e_step():
        b_dev2.copy_(b_host, non_blocking=True)
        P.pnp_ms2g_solve_async(plan, pr.stages, b_dev2, x0, x_dev2, **kw)
        x_host.copy_(x_dev2, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    if nranks > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        e2e_step()
    e1.record(st)
    e1.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / 1000.0], dtype=torch.float64, device=dev)
    if nranks > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = pr.n_steps * args.steps / float(te.item())

    # ---- the same solve reusing the plan's cached step (power_iters = 0): L
    # depends on the geometry only, so repeated reconstructions on one scanner
    # geometry need the power iteration once; reported beside
    # the headline, which includes it ----
    def step_cached():
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha, power_iters=0)

    for _ in range(2):
        step_cached()
    P.solve_status(plan)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(st)
    for _ in range(args.steps):
        step_cached()
    c1.record(st)
    c1.synchronize()
    P.solve_status(plan)
    tc = torch.tensor([c0.elapsed_time(c1) / 1000.0], dtype=torch.float64, device=dev)
    if nranks > 1:
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
    t_cached = float(tc.item())

    # steady-state iterations/s of each stage alone (SURVEY 8(d) "iters/s per
    # stage"): a one-stage schedule with the cached step, 50 iterations
    stage_rate = {}
    for fac in sorted({s_[0] for s_ in pr.stages}, reverse=True):
        one = [(fac, 50, 0)]
        P.pnp_ms2g_solve_async(plan, one, b, x0, xo, den=pr.den, alpha=pr.alpha, power_iters=0)
        P.solve_status(plan)
        c0.record(st)
        for _ in range(args.steps):
            P.pnp_ms2g_solve_async(plan, one, b, x0, xo, den=pr.den, alpha=pr.alpha, power_iters=0)
        c1.record(st)
        c1.synchronize()
        try:
            P.solve_status(plan)
        except P.MS2GError:
            pass    # 50 iterations of one stage alone may leave the safe range of the toy; timing only
        stage_rate[f"s{fac}"] = 50 * args.steps / (c0.elapsed_time(c1) / 1000.0)

    # ---- per-kernel timing of the projector pair + operator throughputs ----
    nnz = nnz_counts()[f"C{pr.cfg}"]
    frac_views = (ve - vb) / pr.n_views
    detail = {"stage_iters_per_s": stage_rate,
              "solve_cached_step": {"iters_per_s": pr.n_steps * args.steps / t_cached,
                                    "ms_per_solve": 1000.0 * t_cached / args.steps,
                                    "note": "power_iters=0: per-stage step 1/L reused from the plan's cache "
                                            "(computed by the headline solves); L2 not flushed"}}
    x1 = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, 9))).to(dev)[None].contiguous()
    g = torch.empty_like(x1)
    for s in (2, 1):
        nc = pr.n // s
        tg = time_calls(lambda: P.sketched_grad(plan, s, x1, b, g=g), 10)
        xs = x1 if s == 1 else P.sketch_down(plan, 2, x1)
        res = torch.empty((1, ve - vb, pr.n_bins), device=dev)
        img = torch.empty((1, nc, nc), device=dev)
        tf = time_calls(lambda: P.forward_project(plan, s, xs, b=b, out=res), 10)
        tb = time_calls(lambda: P.back_project(plan, s, res, img=img), 10)
        seg = nnz[str(s)] * frac_views
        detail[f"grad_s{s}"] = {"evals_per_s": 1.0 / tg, "ms": tg * 1e3,
                                "forward_ms": tf * 1e3, "backward_ms": tb * 1e3,
                                "segments_per_launch": seg,
                                "forward_nnz_per_s": seg / tf, "backward_nnz_per_s": seg / tb}
    del flush
    hbm, hbm_src = peaks()
    # dominant kernel: the one with the larger share of the solve (launch counts
    # per solve: power iterations + iterations, per factor)
    calls = {2: pr.power_iters + sum(s_[1] for s_ in pr.stages if s_[0] == 2),
             1: pr.power_iters + sum(s_[1] for s_ in pr.stages if s_[0] == 1)}
    share = {}       # device ms per solve of each kernel, from the instrumented timed steps
    for kern in ("forward", "backward"):
        share[kern] = sum(ktime[(kern, f_)][0] for f_ in (2, 1)) / args.steps
    dom = max(share, key=share.get)
    s_dom = 1
    d = detail[f"grad_s{s_dom}"]
    tot_ms, n_l = ktime[(dom, s_dom)]
    tk = tot_ms / max(n_l, 1) / 1e3       # average launch duration inside the timed solves
    seg = d["segments_per_launch"]
    n_rays = (ve - vb) * pr.n_bins
    compulsory = 4 * n_rays * (2 if dom == "forward" else 1) + 4 * pr.n * pr.n * (1 if dom == "backward" else 2)
    algo_bytes = 8.0 * seg + compulsory
    achieved = algo_bytes / tk / 1e9
    traffic, l1frac = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(f"k_{dom}", {}).get(str(s_dom))
        l1frac = tj.get(f"k_{dom}:l1_pipe_frac", {}).get(str(s_dom))
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": f"k_{dom}", "factor": s_dom,
                "reading": "SpMV-equivalent bytes: 8 B per ray-pixel segment (oracle-counted) + compulsory "
                           "bytes, per launch / average launch time measured by CUDA events around each launch "
                           f"inside the timed solve graphs; peak = {hbm_src} copy bandwidth",
                "launches_timed": n_l, "launch_ms": tk * 1e3,
                "instrumented_ms_per_step": t_instr / args.steps,
                "compulsory_frac": compulsory / tk / 1e9 / hbm,
                "frac_vs_nominal_8tbs": achieved / 8000.0,   # also against the nominal HBM3e peak
                # what actually bounds the kernel (ncu --set full, profiles/r01_ncu_full_projectors.md):
                # L1/shared data-pipe wavefronts, fraction of the per-SM peak of one per clock
                "l1_data_pipe_frac": l1frac,
                "share_ms_per_solve": share}

    if nranks == 1 and not args.no_detail:
        detail.update(detail_512(P, dev))
        detail["C4_view_shard_estimate"] = shard_estimate(P, dev, pr, b_full, t_total / args.steps)

    cpu = None
    if rank == 0 and nranks == 1 and not args.no_cpu:
        import oracle as O
        nth = O.default_threads()
        v, secs, desc = oracle_sample(pr, b_full.astype(np.float64), nth)
        cpu = {"value": v, "unit": "iters/s", "cores": nth, "kind": "oracle", "sample": desc}
        # one core: a factor-2 gradient on every 16th view, scaled to the solve
        g_ = O.Geometry(pr.n, pr.n_views, pr.n_bins)
        xs_ = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, 9)).astype(np.float64)
        views_ = np.arange(0, pr.n_views, 16)
        a_ = time.perf_counter()
        O.sketched_grad(g_, 2, xs_, b_full.astype(np.float64), views=views_, nthreads=1)
        t1_ = (time.perf_counter() - a_) * 16          # all views, factor 2, one core
        cpu["one_core"] = {"s2_gradient_s": t1_, "sample": "1 factor-2 gradient on 90 of 1440 views x 16",
                           "speedup_all_cores": t1_ / secs_s2 if (secs_s2 := _last_s2[0]) else None}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": nranks, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(pr, nranks, "flushed between timed steps (256 MiB write)", args.allreduce),
                "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": int(b.numel() * 4),
                        "d2h_bytes_per_step": int(x0.numel() * 4)},
                "gpu_launches": int(launches), "clocks": clocks, "roofline": roofline,
                "cpu_baseline": cpu, "detail": detail}
        print(json.dumps(line), flush=True)
    plan.destroy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ms2g", choices=["ms2g", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle sample")
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "peer"],
                    help="cross-rank sum of the partial backprojections (N > 1): NCCL, or the NEXT-3 "
                         "peer-memory path (untested at N > 1 on this 1-GPU pool)")
    ap.add_argument("--no-detail", action="store_true", help="skip the 512^2 detail numbers")
    ap.add_argument("--profile-once", action="store_true",
                    help="run one warm-up solve and one solve, print nothing (for ncu launch lists)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    nranks = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, nranks)
        return
    if nranks > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ms2g(args, rank, nranks, local_rank)
    if nranks > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
