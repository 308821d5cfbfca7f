"""Small driver for ncu captures (run under gpurun; never report its timings).

  --mode solve    : one warm-up solve + one profiled C4 solve (launch list)
  --mode kernels  : C4 forward/backward at s = 2 and 1, called directly
"""
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
ap.add_argument("--mode", default="solve")
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--shard", type=int, default=1, help="rank 0's contiguous view shard of N (no communicator)")
a = ap.parse_args()
pr = S.PRESETS[a.cfg]
vb, ve = P.view_shard(pr.n_views, 0, a.shard)
plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), batch=1, view_begin=vb, view_end=ve)
x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg))).cuda()[None].contiguous()
b = P.forward_project(plan, 1, x)
if a.mode == "solve":
    x0 = torch.zeros_like(x); xo = torch.empty_like(x)
    for _ in range(2):
        P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha)
    try:
        P.solve_status(plan)
    except P.MS2GError:
        pass   # a shard's partial operator alone: timing/profiling only
else:
    for s in (2, 1):
        xs = x if s == 1 else P.sketch_down(plan, 2, x)
        r = P.forward_project(plan, s, xs, b=b)
        img = P.back_project(plan, s, r)
torch.cuda.synchronize()
print("ok")
