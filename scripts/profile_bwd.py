"""ncu driver: C4 back_project at s = 4, 2, 1 (one call each after warm-up)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

pr = S.PRESETS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1))
r = torch.from_numpy(S.random_sinogram((pr.n_views, pr.n_bins), 3)).cuda()[None].contiguous()
for s in (4, 2, 1):
    img = P.back_project(plan, s, r)
torch.cuda.synchronize()
for s in (4, 2, 1):
    img = P.back_project(plan, s, r)
torch.cuda.synchronize()
print("ok")
