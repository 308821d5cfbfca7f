"""C3 Option-2 solve (512^2, 720 x 768, 8 subsets, TV) timed by CUDA events
under experiment switches: default, MS2G_PDL=0 (TV chain without
programmatic dependent launch), MS2G_TV_PERSIST=1 (persistent TV).  Also
C2 (256^2, TV).  Dev aid for DESIGN.md §7c."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for extra in ({}, {"MS2G_PDL": "0"}, {"MS2G_TV_PERSIST": "1"}):
        out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, **extra), capture_output=True,
                             text=True)
        print(json.dumps(extra), out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

res = {}
for cfg in (3, 2):
    pr = S.PRESETS[cfg]
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
        xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg), texture=pr.texture)
        p_ = P.forward_project(plan, 1, torch.from_numpy(xt).cuda()[None])[0].cpu().numpy()
        b = torch.from_numpy(S.gaussian_data(p_, pr.noise[1], S.config_seed(cfg))).cuda()[None].contiguous()
        x0 = torch.zeros((1, pr.n, pr.n), device="cuda"); xo = torch.empty_like(x0)
        kw = dict(option=pr.option, n_subsets=pr.n_subsets, seed=S.config_seed(cfg), den=pr.den, alpha=pr.alpha)
        t = bench.time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, **kw), 10, warm=3)
        tc = bench.time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, power_iters=0, **kw), 10,
                              warm=3)
        P.solve_status(plan)
        res[f"C{cfg}"] = {"solve_ms": round(t * 1e3, 3), "cached_step_ms": round(tc * 1e3, 3)}
print(json.dumps(res))
