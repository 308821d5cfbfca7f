"""Short forward launches (dev aid): the single-image forward on a P = 8 view
shard of C4 (180 views) and on one registered 1/8 subset of C3 (90 views),
CUDA events, under the short-launch shapes of MS2G_FWD_SMALL (SPLIT x SEG:
44 default, 24, 48, 28); plus the C3 s=4 subset gradient rate."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for v in ("44", "24", "48", "28"):
        out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, MS2G_FWD_SMALL=v),
                             capture_output=True, text=True)
        print(v, out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

res = {}
pr = S.PRESETS[4]
vb, ve = P.view_shard(pr.n_views, 0, 8)
with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve) as plan:
    for s in (1, 2):
        x = torch.from_numpy(S.random_image(pr.n // s, 3)).cuda()[None].contiguous()
        out = torch.empty((1, ve - vb, pr.n_bins), device="cuda")
        res[f"C4_shard8_fwd_s{s}_us"] = round(1e6 * bench.time_calls(lambda: P.forward_project(plan, s, x, out=out), 50), 1)
pr = S.PRESETS[3]
with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
    rs = P.register_subset(plan, list(range(0, pr.n_views, 8)))
    x = torch.from_numpy(S.random_image(pr.n, 4)).cuda()[None].contiguous()
    b = torch.from_numpy(S.random_sinogram((pr.n_views, pr.n_bins), 5, zero_mean=False)).cuda()[None].contiguous()
    g = torch.empty_like(x)
    for s in (4, 2, 1):
        xs = torch.from_numpy(S.random_image(pr.n // s, 3)).cuda()[None].contiguous()
        out = torch.empty((1, rs.n_sel, pr.n_bins), device="cuda")
        res[f"C3_sub_fwd_s{s}_us"] = round(1e6 * bench.time_calls(lambda: P.forward_project(plan, s, xs, out=out,
                                                                                             subset=rs), 50), 1)
        res[f"C3_sub_grad_s{s}_evals"] = round(1.0 / bench.time_calls(lambda: P.sketched_grad(plan, s, x, b, g=g,
                                                                                              subset=rs), 100))
print(json.dumps(res))
