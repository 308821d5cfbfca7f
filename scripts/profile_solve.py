"""ncu driver: one warm-up + one profiled solve of C3 (Option 2) or C5 (batch 8).
Run under gpurun; never report its timings."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
a = ap.parse_args()
pr = S.PRESETS[a.cfg]
nb = pr.batch if a.cfg == 5 else 1
factors = sorted({s[0] for s in pr.stages} | {1}, reverse=True)
plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=tuple(factors), batch=nb)
xs = np.stack([S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg, i), texture=pr.texture) for i in range(nb)])
b = P.forward_project(plan, 1, torch.from_numpy(xs).cuda().contiguous())
x0 = torch.zeros((nb, pr.n, pr.n), device="cuda"); xo = torch.empty_like(x0)
kw = dict(den=pr.den, alpha=pr.alpha)
if a.cfg == 3:
    kw.update(option=2, n_subsets=8, seed=S.config_seed(3))
for _ in range(2):
    P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, **kw)
P.solve_status(plan)
torch.cuda.synchronize()
print("ok")
