"""Exact segment counts nnz(A_s) for the C1..C5 geometries, from the oracle only.

Writes profiles/nnz_counts.json: {"C<k>": {"geometry": [n, V, B], "<s>": nnz}}
(--study-only: adds "QS_<setting>" for the NEXT-2 quality-study geometries).
These are the algorithmic-work denominators of bench.py's roofline (8 B per
segment); the CUDA path never produces them.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ms2g_synth as S  # noqa: E402
import oracle as O  # noqa: E402

# geometries of the NEXT-2 quality study (scripts/quality_study.py): 256^2,
# 228 bins; sparse-view / low-dose over [0, 2 pi), limited-angle over [0, pi)
STUDY = {"sparse-view": (90, 2 * math.pi), "low-dose": (360, 2 * math.pi), "limited-angle": (90, math.pi)}

path = os.path.join(ROOT, "profiles", "nnz_counts.json")
out = json.load(open(path)) if os.path.exists(path) else {}
if "--study-only" in sys.argv:
    for name, (V, arc) in STUDY.items():
        g = O.Geometry(256, V, 228, arc=arc)
        out[f"QS_{name}"] = {"geometry": [256, V, 228, arc], **{str(s): O.count_nnz(g, s) for s in (4, 2, 1)}}
        print(name, out[f"QS_{name}"], flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    sys.exit(0)
for cfg, pr in S.PRESETS.items():
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    ent = {"geometry": [pr.n, pr.n_views, pr.n_bins]}
    for s in (4, 2, 1):
        ent[str(s)] = O.count_nnz(g, s)
    if pr.option == 2:
        for s in (4, 2, 1):
            ent[f"{s}_subset0"] = O.count_nnz(g, s, views=O.subset_views(pr.n_views, pr.n_subsets, 0))
    out[f"C{cfg}"] = ent
    print(cfg, ent, flush=True)
with open(path, "w") as f:
    json.dump(out, f, indent=1)
