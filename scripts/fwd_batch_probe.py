"""Batched forward (C5 geometry, 512^2, 720 x 768): per-image segments/s of
k_forward_batch<8> with the separate pair layout (default) and the
interleaved one (MS2G_FWD_INTERLEAVE), against the single-image forward.
CUDA events over 20 calls of the pair prep + forward (forward_project)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for env in ({}, {"MS2G_FWD_INTERLEAVE": "1"}):
        out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, **env), capture_output=True,
                             text=True)
        print(("interleaved" if env else "separate   "), out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

nnz = bench.nnz_counts()["C3"]
res = {}
for batch in (1, 8):
    with P.plan_geometry(512, 720, 768, factors=(2, 1), batch=batch) as plan:
        for s in (1, 2):
            nc = 512 // s
            x = torch.from_numpy(np.stack([S.random_image(nc, 7 + i) for i in range(batch)])).cuda()
            out = torch.empty((batch, 720, 768), device="cuda")
            t = bench.time_calls(lambda: P.forward_project(plan, s, x, out=out), 20)
            res[f"b{batch}_s{s}"] = {"ms": round(t * 1e3, 4), "image_seg_per_s": batch * nnz[str(s)] / t}
for s in (1, 2):
    res[f"per_image_speedup_s{s}"] = res[f"b8_s{s}"]["image_seg_per_s"] / res[f"b1_s{s}"]["image_seg_per_s"]
print(json.dumps(res))
