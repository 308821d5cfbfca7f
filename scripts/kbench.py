"""Quick per-kernel timing of the projector pair at a config (CUDA events).

Development tool: the bench numbers of record come from bench.py."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--shard", type=int, default=1, help="time rank 0's contiguous view shard of N")
ap.add_argument("--lib", default=None, help="alternative libms2g build (kernel-variant experiments)")
a = ap.parse_args()
if a.lib:
    P._LIBPATH = a.lib
pr = S.PRESETS[a.cfg]
nnz = json.load(open(os.path.join(ROOT, "profiles", "nnz_counts.json")))[f"C{a.cfg}"]
vb, ve = P.view_shard(pr.n_views, 0, a.shard)
plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1), batch=a.batch, view_begin=vb, view_end=ve)
x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(pr.cfg))).cuda()[None].repeat(a.batch, 1, 1).contiguous()


def t(fn):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(a.reps):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / a.reps


res = {}
for s in (4, 2, 1):
    xs = x if s == 1 else P.sketch_down(plan, s, x)
    out = P.forward_project(plan, s, xs)
    img = P.back_project(plan, s, out)
    tf = t(lambda: P.forward_project(plan, s, xs, out=out))
    tb = t(lambda: P.back_project(plan, s, out, img=img))
    seg = nnz[str(s)] * a.batch * (ve - vb) / pr.n_views
    res[s] = dict(fwd_ms=round(tf, 4), bwd_ms=round(tb, 4), fwd_gnnz=round(seg / tf / 1e6, 1), bwd_gnnz=round(seg / tb / 1e6, 1))
print(json.dumps(res))
