"""Cost of a solve whose buffers change between calls (graph re-capture) vs a
replay (dev aid)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

for cfg in (4, 3):
    pr = S.PRESETS[cfg]
    factors = sorted({s[0] for s in pr.stages} | {1}, reverse=True)
    plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=tuple(factors))
    x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg))).cuda()[None].contiguous()
    b = P.forward_project(plan, 1, x)
    x0 = torch.zeros_like(x)
    outs = [torch.empty_like(x) for _ in range(2)]
    kw = dict(den=pr.den, alpha=pr.alpha)
    if cfg == 3:
        kw.update(option=2, n_subsets=8, seed=S.config_seed(3))
    for k in range(2):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, outs[0], **kw)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(4):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, outs[0], **kw)
    torch.cuda.synchronize()
    replay = (time.perf_counter() - t) / 4
    t = time.perf_counter()
    for k in range(4):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, outs[k % 2], **kw)   # new x_out every call
    torch.cuda.synchronize()
    recap = (time.perf_counter() - t) / 4
    print(f"C{cfg}: replay {1e3 * replay:.2f} ms, with re-capture {1e3 * recap:.2f} ms per solve", flush=True)
    plan.destroy()
