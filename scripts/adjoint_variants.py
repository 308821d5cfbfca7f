"""Adjoint design comparison (north-star subsystem (2)): the tile-driven
scatter (default) against the pixel-driven gather (MS2G_BP_VARIANT=gather)
on the C4 (1024^2, 1440 x 1536) and C3 (512^2, 720 x 768) geometries:
CUDA-event time per launch, segments/s (oracle-counted nnz), and the
relative difference of the two results (both are the exact adjoint up to
fp32 rounding).  Run under gpurun; ncu evidence separately."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) == 1:
    res = {}
    for v in ("scatter", "gather"):
        env = dict(os.environ, MS2G_BP_VARIANT=v)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        if out.returncode:
            print(out.stderr[-3000:])
            sys.exit(1)
        res[v] = json.loads(out.stdout.strip().splitlines()[-1])
    import numpy as np
    for key in res["scatter"]:
        a, b = res["scatter"][key], res["gather"][key]
        print(f"{key:10s} scatter {a['ms']:.3f} ms ({a['seg_per_s']:.3e} seg/s)  gather {b['ms']:.3f} ms "
              f"({b['seg_per_s']:.3e} seg/s)  gather/scatter time {b['ms'] / a['ms']:.2f}x")
    diffs = {}
    for key in res["scatter"]:
        xa = np.load(f"/tmp/adj_scatter_{key}.npy"); xb = np.load(f"/tmp/adj_gather_{key}.npy")
        diffs[key] = float(np.linalg.norm(xa - xb) / np.linalg.norm(xa))
    print("relative L2 difference scatter vs gather:", diffs)
    print(json.dumps({"timings": res, "rel_diff": diffs}))
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

variant = os.environ.get("MS2G_BP_VARIANT", "scatter")
nnz = bench.nnz_counts()
out = {}
for cfg, n, V, B in ((4, 1024, 1440, 1536), (3, 512, 720, 768)):
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        r = torch.from_numpy(S.random_sinogram((V, B), 77)).cuda()[None].contiguous()
        for s in (1, 2):
            img = torch.empty((1, n // s, n // s), device="cuda")
            t = bench.time_calls(lambda: P.back_project(plan, s, r, img=img), 10)
            seg = nnz[f"C{cfg}"][str(s)]
            key = f"C{cfg}_s{s}"
            out[key] = {"ms": t * 1e3, "seg_per_s": seg / t}
            np.save(f"/tmp/adj_{variant}_{key}.npy", img.cpu().numpy())
print(json.dumps(out))
