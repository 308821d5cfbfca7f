"""Backprojector chunking (dev aid): the adjoint on C4's full view set and on
rank 0's 180-view shard of P = 8, CUDA events, under MS2G_BP_WAVES (blocks
per launch ~ waves x SMs, read at plan creation)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for w in ("24", "16", "12", "8", "6"):
        out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, MS2G_BP_WAVES=w),
                             capture_output=True, text=True)
        print(w, out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

pr = S.PRESETS[4]
res = {}
for shard in (1, 8):
    vb, ve = P.view_shard(pr.n_views, 0, shard)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve) as plan:
        r = torch.from_numpy(S.random_sinogram((ve - vb, pr.n_bins), 77)).cuda()[None].contiguous()
        for s in (1, 2):
            img = torch.empty((1, pr.n // s, pr.n // s), device="cuda")
            res[f"P{shard}_s{s}_us"] = round(1e6 * bench.time_calls(lambda: P.back_project(plan, s, r, img=img), 30), 1)
print(json.dumps(res))
