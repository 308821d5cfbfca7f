#!/usr/bin/env python
"""PnP-MS2G hot-path benchmark (BASELINE.json metric) on B200.

--cfg 4 (default; the metric's 1024^2 configuration): one step = one whole
PnP-MS2G solve of C4 (1024^2 image, 1440 views x 1536 bins, stages 2x:30 then
full:20, Gaussian denoiser, per-stage 20-step power iteration) = every row of
SURVEY §8(a), replayed as one CUDA graph with b resident in HBM.  value =
PnP-MS2G iterations/s (50 per solve).  With N ranks the views are sharded
(rank r owns [rV/N, (r+1)V/N)) and the partial backprojections are summed by
an NCCL allreduce inside the graph: strong scaling.

--cfg 5: C5 data parallelism, 8 images per rank (images 8r .. 8r+7 of the
64), one batch-8 solve per step (stages 2x:20 then full:20, Poisson data, TV,
20 power iterations per stage), no collective in the data path; value =
image-iterations/s over all ranks: weak scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--cfg 4|5] [--impl ms2g|reference]

--gpus N > 1 without torchrun re-launches itself under
`torch.distributed.run --nproc-per-node N` (one process per GPU).
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
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from src_hash import src_hash  # noqa: E402

METRIC = "sketched-gradient evals/s and PnP-MS2G iters/s at 512²/1024², frac. of HBM roofline"


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
    den = ("Gaussian 3x3 denoiser" if pr.den[0] == "gauss"
           else f"TV-prox denoiser (lambda {pr.den[1]}, {pr.den[2]} Chambolle iterations)")
    data = "Gaussian noise" if pr.noise[0] == "gauss" else f"Poisson transmission data (I0 {pr.noise[1]:g})"
    cfg = {"workload": f"C{pr.cfg}: {pr.n}x{pr.n} fp32 phantom ({pr.n_ellipses} seeded ellipses), fan-beam "
                       f"{pr.n_views} views x {pr.n_bins} bins, {data}, stages "
                       + " -> ".join(f"{s[0]}x:{s[1]}" for s in pr.stages)
                       + f", {den} alpha={pr.alpha}, {pr.power_iters} power iterations per stage",
           "image": pr.n, "views": pr.n_views, "bins": pr.n_bins, "iters_per_solve": pr.n_steps,
           "l2": l2_note}
    if pr.batch > 1:
        cfg["images_per_rank"] = pr.batch
        cfg["images_total"] = pr.batch * nranks
        cfg["parallelism"] = f"images data-parallel x{nranks} (no collective in the data path)" if nranks > 1 \
            else "1 GPU"
    else:
        cfg["parallelism"] = (f"views sharded x{nranks} + " + ("NCCL allreduce" if allreduce == "nccl" else
                                                               "NVLink peer-memory sum (NEXT-3)")) \
            if nranks > 1 else "1 GPU"
    return cfg


def unit_of(pr):
    return "image-iters/s" if pr.batch > 1 else "iters/s"


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


def oracle_data(pr, image=0):
    """The workload's data for the oracle (seeded phantom, oracle projector)."""
    import oracle as O
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, image), texture=pr.texture)
    p = O.forward(g, 1, xt)
    if pr.noise[0] == "gauss":
        return S.gaussian_data(p, pr.noise[1], S.config_seed(pr.cfg, image))
    return S.poisson_data(p, pr.noise[1], S.config_seed(pr.cfg, image))


def oracle_composed(pr, b_full, nthreads):
    """Bounded sample of one solve of the workload (one image): one factor-2
    gradient, one full gradient and one denoise, timed, composed into the
    solve's counts (power iterations + steps per factor, one denoise per
    step).  Returns (iters/s of one image, seconds of CPU work, description)."""
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
    if pr.den[0] == "gauss":
        O.gauss3(x, pr.den[1])
    else:
        O.tv_chambolle(x, pr.den[1], pr.den[2])
    t["den"] = time.perf_counter() - a
    total = time.perf_counter() - t0
    n2 = sum(st[1] for st in pr.stages if st[0] == 2)
    n1 = sum(st[1] for st in pr.stages if st[0] == 1)
    solve = (pr.power_iters + n2) * t[2] + (pr.power_iters + n1) * t[1] + pr.n_steps * t["den"]
    _last_s2[0] = t[2]
    desc = (f"C{pr.cfg} oracle, one image, {nthreads} threads: 1 factor-2 gradient ({t[2]:.2f} s) + 1 full "
            f"gradient ({t[1]:.2f} s) + 1 denoise ({t['den']:.3f} s), composed into one solve "
            f"({pr.power_iters}+{n2} factor-2 and {pr.power_iters}+{n1} full gradient-equivalents, "
            f"{pr.n_steps} denoises) = {solve:.1f} s")
    return pr.n_steps / solve, total, desc


def oracle_solve(pr, b_full, nthreads):
    """One whole oracle solve of the workload (one image; Algorithm 1 with
    the configuration's schedule, denoiser and power iterations), timed.
    Returns (iters/s of one image, seconds)."""
    import oracle as O
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    a = time.perf_counter()
    O.pnp_ms2g(g, pr.stages, b_full, den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters, nthreads=nthreads)
    secs = time.perf_counter() - a
    return pr.n_steps / secs, secs


def run_reference(args, rank, nranks):
    if rank != 0:
        return
    pr = S.PRESETS[args.cfg]
    import oracle as O
    nthreads = O.default_threads()
    b = oracle_data(pr).astype(np.float64)
    vals, secs_l, desc = [], [], ""
    for k in range(args.warmup + args.steps):
        v, secs, desc = oracle_composed(pr, b, nthreads)
        if k >= args.warmup:
            vals.append(v)
            secs_l.append(secs)
    value = statistics.median(vals)
    unit = unit_of(pr)
    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(secs_l),
            "higher_is_better": True, "scaling": "weak" if pr.batch > 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(pr, 1, "n/a (CPU)"),
            "cpu_baseline": {"value": value, "unit": unit, "cores": nthreads, "kind": "oracle",
                             "sample": desc + "; each timed step is one such bounded sample (a whole oracle solve "
                                              "is timed by the GPU arm's cpu_baseline)"},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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
        rs = P.register_subset(plan, sub)         # uploaded once (the solve's own subset lists are too)
        for s_ in (4, 2, 1):
            t_all = time_calls(lambda: P.sketched_grad(plan, s_, x, b, g=g), 20)
            t_sub = time_calls(lambda: P.sketched_grad(plan, s_, x, b, g=g, subset=rs), 50)
            t_adhoc = time_calls(lambda: P.sketched_grad(plan, s_, x, b, g=g, subset=sub), 20)
            out[f"C3_512_grad_s{s_}"] = {"evals_per_s": 1.0 / t_all, "subset_evals_per_s": 1.0 / t_sub,
                                         "subset_adhoc_list_evals_per_s": 1.0 / t_adhoc,
                                         "segments_per_s": 2 * nnz[str(s_)] / t_all,
                                         "subset_segments_per_s": 2 * nnz[f"{s_}_subset0"] / t_sub}
        rs.release()
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
    # the same at 8 ranks with the NEXT-3 peer path's graph shape (publish
    # fused into the chunk sum, reduce-scatter, all-gather fused with the step;
    # at one rank the exchange kernels run but move nothing across NVLink),
    # plus a model of what they would move: 2 (P-1)/P of the image per rank at
    # 700 GB/s and 5 us for the two signal hops, per gradient and power step
    nr = 8
    shard_ms = []
    for r in range(nr):
        vb, ve = P.view_shard(pr.n_views, r, nr)
        with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve) as plan:
            P.attach_peers(plan, 0, 1)
            b = torch.from_numpy(np.ascontiguousarray(b_full[vb:ve])).to(dev)[None].contiguous()
            x0 = torch.zeros((1, pr.n, pr.n), device=dev); xo = torch.empty_like(x0)
            kw = dict(den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters)
            shard_ms.append(1e3 * time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, **kw), 3,
                                             warm=2))
            try:
                P.solve_status(plan)
            except P.MS2GError:
                pass
    t_pe = sum(n * (5e-6 + 2 * (nr - 1) / nr * 4 * (pr.n // f) ** 2 / 700e9) for f, n in n_ar.items())
    ts = max(shard_ms) / 1e3
    out["N8_peer"] = {"max_shard_solve_ms": ts * 1e3, "shard_solve_ms": [round(v, 3) for v in shard_ms],
                      "exchange_model_ms": t_pe * 1e3, "est_iters_per_s": pr.n_steps / (ts + t_pe),
                      "est_speedup": t_solve_1 / (ts + t_pe)}
    out["note"] = ("estimated: slowest rank shard timed on 1 GPU (L2 not flushed) + modelled allreduce (NCCL: 20 us + "
                   "2 x bytes at 450 GB/s; N8_peer: NEXT-3 reduce-scatter/all-gather, 5 us + 2 (P-1)/P x bytes at "
                   "700 GB/s -- at one rank its reduce-scatter still passes the whole image, P times its share at "
                   "P ranks, so N8_peer overstates the shard time); not measured scaling")
    return out


def make_data_images(P, pr, images, dev):
    """Seeded phantoms, exact projection by the GPU projector, noise (the
    bench times the solver; it is not a parity check)."""
    import torch
    bs = []
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(1,)) as full:
        for im in images:
            xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, im), texture=pr.texture)
            p = P.forward_project(full, 1, torch.from_numpy(xt).to(dev)[None])[0].cpu().numpy()
            bs.append(S.gaussian_data(p, pr.noise[1], S.config_seed(pr.cfg, im)) if pr.noise[0] == "gauss"
                      else S.poisson_data(p, pr.noise[1], S.config_seed(pr.cfg, im)))
    return np.stack(bs)


def roofline_entry(pr, ktime, steps, n_rays, hbm, hbm_src, nnz_seg):
    """Roofline of the dominant projector kernel (largest device time per
    solve), from the CUDA events around its launches inside the timed solves.

    bound "hbm": achieved = ALGORITHMIC (compulsory) bytes per launch / the
    average launch time -- adjoint: read the residual sinogram (4 B per ray)
    and write the image (4 B per pixel); forward: read the image and b, write
    the residual.  This is the honest HBM fraction of the method: it computes
    its matrix, so it is tiny.  Beside it:
      binding     -- the resource that actually bounds the kernel (ncu: the
                     L1/shared data pipe), stamped with the source hash of the
                     capture and marked stale if the kernels changed since;
      spmv_equivalent -- the north star's reading (8 B per ray-pixel segment
                     that an explicitly stored sparse A would stream), a
                     throughput figure in byte units, NOT a roofline fraction.
    """
    share = {k: sum(ktime[(k, f_)][0] for f_ in (2, 1)) / steps for k in ("forward", "backward")}
    dom = max(share, key=share.get)
    s_dom = 1
    tot_ms, n_l = ktime[(dom, s_dom)]
    tk = tot_ms / max(n_l, 1) / 1e3
    npix = pr.n * pr.n * pr.batch
    compulsory = (4 * n_rays + 4 * npix) if dom == "backward" else (4 * npix + 8 * n_rays)
    achieved = compulsory / tk / 1e9
    seg = nnz_seg * pr.batch
    spmv = (8.0 * seg + compulsory) / tk / 1e9
    traffic, binding = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        stamp = tj.get("source_hash")
        stale = stamp != src_hash()
        if pr.batch == 1:
            traffic = tj.get(f"k_{dom}", {}).get(str(s_dom))
        binding = {"resource": "L1/shared data pipe (l1tex__data_pipe_lsu_wavefronts, fraction of one wavefront "
                               "per SM clock)",
                   "frac": tj.get(f"k_{dom}:l1_pipe_frac", {}).get(str(s_dom)),
                   "source": "profiles/ncu_traffic.json (ncu --set full, C4 single image)",
                   "source_hash": stamp, "stale": stale}
        if stale:
            traffic = None
    except Exception:
        pass
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic, "kernel": f"k_{dom}", "factor": s_dom,
            "reading": "algorithmic = compulsory bytes per launch (residual sinogram read + image write for the "
                       "adjoint) / average launch time, CUDA events around each launch inside the timed solve "
                       f"graphs; peak = {hbm_src} copy bandwidth (MEASURED_PEAKS.json)",
            "launches_timed": n_l, "launch_ms": tk * 1e3, "share_ms_per_solve": share,
            "binding": binding,
            "spmv_equivalent": {"gbs": spmv, "segments_per_launch": seg, "segments_per_s": seg / tk,
                                "note": "north-star reading: 8 B per ray-pixel segment + compulsory bytes; a "
                                        "throughput in byte units (the matrix is computed, never streamed), "
                                        "not a fraction of HBM"}}


def run_ms2g(args, rank, nranks, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2203_07308_b200 as P
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pr = S.PRESETS[args.cfg]
    P.load()
    batched = pr.batch > 1
    if batched:          # C5: images 8r .. 8r+7 of this rank, every view
        images = list(range(rank * pr.batch, (rank + 1) * pr.batch))
        b_np = make_data_images(P, pr, images, dev)
        vb, ve = 0, pr.n_views
    else:                # C4: the rank's contiguous view shard of image 0
        b_full = make_data_images(P, pr, [0], dev)[0]
        vb, ve = P.view_shard(pr.n_views, rank, nranks)
        b_np = b_full[None, vb:ve]
    plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve,
                           batch=pr.batch)
    if nranks > 1 and not batched:
        if args.allreduce == "peer":     # NEXT-3: fused NVLink peer-memory sum (fixed rank order)
            P.attach_peers(plan, rank, nranks)
        else:
            P.attach_nccl(plan, rank, nranks)
    b = torch.from_numpy(np.ascontiguousarray(b_np)).to(dev).contiguous()
    x0 = torch.zeros((pr.batch, pr.n, pr.n), device=dev)
    xo = torch.empty_like(x0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    kw = dict(den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters)
    unit = unit_of(pr)
    per_step_units = pr.n_steps * pr.batch          # iterations (x images) per solve and rank

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
    # whole job: every rank's units (C4: the N ranks together do one solve per
    # step; C5: each rank solves its own 8 images per step)
    value = per_step_units * (nranks if batched else 1) * args.steps / t_total
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
    x_host = torch.empty(tuple(x0.shape), dtype=torch.float32).pin_memory()
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
    e2e_val = per_step_units * (nranks if batched else 1) * args.steps / float(te.item())

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
        stage_rate[f"s{fac}"] = 50 * pr.batch * args.steps / (c0.elapsed_time(c1) / 1000.0)

    # ---- per-kernel timing of the projector pair + operator throughputs ----
    nnz = nnz_counts()[f"C{3 if batched else pr.cfg}"]      # C5 has C3's geometry
    frac_views = (ve - vb) / pr.n_views
    detail = {"stage_iters_per_s": stage_rate,
              "solve_cached_step": {unit.replace("/s", "_per_s").replace("-", "_"):
                                    per_step_units * (nranks if batched else 1) * args.steps / t_cached,
                                    "ms_per_solve": 1000.0 * t_cached / args.steps,
                                    "note": "power_iters=0: per-stage step 1/L reused from the plan's cache "
                                            "(computed by the headline solves); L2 not flushed"}}
    x1 = torch.from_numpy(np.stack([S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, 9))] * pr.batch)).to(dev)
    g = torch.empty_like(x1)
    for s in (2, 1):
        nc = pr.n // s
        tg = time_calls(lambda: P.sketched_grad(plan, s, x1, b, g=g), 10)
        xs = x1 if s == 1 else P.sketch_down(plan, 2, x1)
        res = torch.empty((pr.batch, ve - vb, pr.n_bins), device=dev)
        img = torch.empty((pr.batch, nc, nc), device=dev)
        tf = time_calls(lambda: P.forward_project(plan, s, xs, b=b, out=res), 10)
        tb = time_calls(lambda: P.back_project(plan, s, res, img=img), 10)
        seg = nnz[str(s)] * frac_views * pr.batch
        detail[f"grad_s{s}"] = {"evals_per_s": pr.batch / tg, "ms": tg * 1e3,
                                "forward_ms": tf * 1e3, "backward_ms": tb * 1e3,
                                "segments_per_launch": seg,
                                "forward_nnz_per_s": seg / tf, "backward_nnz_per_s": seg / tb}
    del flush
    hbm, hbm_src = peaks()
    roofline = roofline_entry(pr, ktime, args.steps, (ve - vb) * pr.n_bins * pr.batch, hbm, hbm_src,
                              nnz["1"] * frac_views)
    roofline["instrumented_ms_per_step"] = t_instr / args.steps

    if nranks == 1 and not args.no_detail and not batched:
        detail.update(detail_512(P, dev))
        detail["C4_view_shard_estimate"] = shard_estimate(P, dev, pr, b_full, t_total / args.steps)

    cpu = None
    if rank == 0 and nranks == 1 and not args.no_cpu:
        import oracle as O
        nth = O.default_threads()
        b0 = b_np[0].astype(np.float64)
        vc, secs_c, desc_c = oracle_composed(pr, b0, nth)
        if args.cpu_sample == "solve":
            v, secs = oracle_solve(pr, b0, nth)
            cpu = {"value": v, "unit": "iters/s (one image)" if batched else "iters/s", "cores": nth,
                   "kind": "oracle",
                   "sample": f"one whole C{pr.cfg} oracle solve of image 0 (Algorithm 1, {pr.n_steps} steps, "
                             f"{pr.power_iters} power iterations per stage, fp64, {nth} threads): {secs:.1f} s",
                   "composed_estimate": {"value": vc, "sample": desc_c}}
        else:
            cpu = {"value": vc, "unit": "iters/s (one image)" if batched else "iters/s", "cores": nth,
                   "kind": "oracle", "sample": desc_c}
        # one core: a factor-2 gradient on every 16th view, scaled to all views
        g_ = O.Geometry(pr.n, pr.n_views, pr.n_bins)
        xs_ = S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, 9)).astype(np.float64)
        views_ = np.arange(0, pr.n_views, 16)
        a_ = time.perf_counter()
        O.sketched_grad(g_, 2, xs_, b0, views=views_, nthreads=1)
        t1_ = (time.perf_counter() - a_) * 16
        cpu["one_core"] = {"s2_gradient_s": t1_, "sample": f"1 factor-2 gradient on every 16th view x 16",
                           "speedup_all_cores": t1_ / secs_s2 if (secs_s2 := _last_s2[0]) else None}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": nranks, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / args.steps, "higher_is_better": True,
                "scaling": "weak" if batched else "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": workload_config(pr, nranks, "flushed between timed steps (256 MiB write)", args.allreduce),
                "e2e": {"value": e2e_val, "unit": unit, "h2d_bytes_per_step": int(b.numel() * 4),
                        "d2h_bytes_per_step": int(x0.numel() * 4)},
                "gpu_launches": int(launches), "clocks": clocks, "roofline": roofline,
                "cpu_baseline": cpu, "detail": detail}
        print(json.dumps(line), flush=True)
    plan.destroy()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def dry_run(args, rank, nranks):
    """--dry-run: the launcher and sharding plumbing without a GPU (gloo):
    every rank reports its shard; rank 0 prints them as one JSON line."""
    import torch.distributed as dist
    pr = S.PRESETS[args.cfg]
    if pr.batch > 1:
        mine = {"rank": rank, "images": list(range(rank * pr.batch, (rank + 1) * pr.batch))}
    else:
        import paper_2203_07308_b200 as P
        vb, ve = P.view_shard(pr.n_views, rank, nranks)
        mine = {"rank": rank, "views": [vb, ve]}
    out = [None] * nranks
    if nranks > 1:
        dist.all_gather_object(out, mine)
    else:
        out = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": nranks, "cfg": args.cfg, "shards": out}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cfg", type=int, default=4, choices=[4, 5],
                    help="4: C4 1024^2 view-sharded solve (the metric's configuration); 5: C5 8 images per rank")
    ap.add_argument("--impl", default="ms2g", choices=["ms2g", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle run")
    ap.add_argument("--cpu-sample", default="solve", choices=["solve", "composed"],
                    help="cpu_baseline: one whole timed oracle solve (default; ~200 s at C4 on 16 cores) or the "
                         "composed bounded sample")
    ap.add_argument("--allreduce", default="nccl", choices=["nccl", "peer"],
                    help="cross-rank sum of the partial backprojections (N > 1): NCCL, or the NEXT-3 "
                         "peer-memory path (untested at N > 1 on this 1-GPU pool)")
    ap.add_argument("--no-detail", action="store_true", help="skip the 512^2 detail numbers")
    ap.add_argument("--profile-once", action="store_true",
                    help="run one warm-up solve and one solve, print nothing (for ncu launch lists)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/sharding plumbing only (gloo, no GPU): print every rank's shard")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    nranks = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, nranks)
        return
    if args.dry_run:
        import torch.distributed as dist
        if nranks > 1:
            dist.init_process_group("gloo")
        dry_run(args, rank, nranks)
        if nranks > 1:
            dist.destroy_process_group()
        return
    if nranks > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.device_count() < nranks:
            raise SystemExit(f"bench.py: {nranks} ranks need {nranks} GPUs, found {torch.cuda.device_count()}")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ms2g(args, rank, nranks, local_rank)
    if nranks > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
