"""Overhead of the in-graph kernel-timing events on the C4 solve (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

pr = S.PRESETS[4]
plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1))
x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(4))).cuda()[None].contiguous()
b = P.forward_project(plan, 1, x)
x0 = torch.zeros_like(x); xo = torch.empty_like(x)
for timing in (False, True, False, True):
    P.set_kernel_timing(plan, timing)
    for _ in range(2):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha)
    e1.record(); e1.synchronize()
    msg = f"timing={timing}: {e0.elapsed_time(e1) / 5:.2f} ms/solve"
    if timing:
        for k in ("forward", "backward"):
            for s in (2, 1):
                t, n = P.kernel_time(plan, k, s)
                msg += f"  {k}@{s}: {n} x {t / max(n, 1):.3f} ms"
    print(msg, flush=True)
