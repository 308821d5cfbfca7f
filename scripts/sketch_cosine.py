"""Surrogate quality of the sketched gradient, logged per stage (SURVEY
§8(c): "cosine of g_s vs the full gradient at the same x ... Log it per
stage; do not gate on it").  For C2 (256^2, stages 4x:15 -> 2x:15 -> full:20,
TV) and C4 (1024^2, 2x:30 -> full:20, Gaussian): at the iterate where each
stage starts (the solve run through the preceding stages on the GPU), the
cosine between U_s A_s^T (A_s S_s y - b) and A^T (A y - b) for s = 2 and 4.
Writes gpurun_out/r02_sketch_cosine.md (copied to profiles/).  Run under gpurun."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

P.load()
lines = ["# Sketched vs full gradient: cosine at each stage start (round 2)", "",
         "`scripts/sketch_cosine.py` on one B200: at the iterate where each stage of the configuration's schedule "
         "starts (the GPU solve run through the preceding stages), cos(g_s, g_1) with g_s = U_s A_s^T (A_s S_s y - b). "
         "SURVEY §8(c) [calib] on a 32^2 toy: 0.998 (s=2) / 0.991 (s=4) at x = 0, falling as the iterate fits the "
         "data -- the reason the schedule moves coarse to full (P:102).  Logged, not gated.", "",
         "| config | stage start | iteration | cos(g_2, g_1) | cos(g_4, g_1) |", "|---|---|---|---|---|"]
for cfg in (2, 4):
    pr = S.PRESETS[cfg]
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg), texture=pr.texture)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
        p_ = P.forward_project(plan, 1, torch.from_numpy(xt).cuda()[None])[0].cpu().numpy()
        b = torch.from_numpy(S.gaussian_data(p_, pr.noise[1], S.config_seed(cfg))).cuda()[None].contiguous()
        it = 0
        for k in range(len(pr.stages) + 1):
            if k == 0:
                y = torch.zeros((1, pr.n, pr.n), device="cuda")
            else:
                y = P.pnp_ms2g_solve(plan, pr.stages[:k], b, den=pr.den, alpha=pr.alpha)
            g1 = P.sketched_grad(plan, 1, y, b).double()
            cos = []
            for s in (2, 4):
                gs = P.sketched_grad(plan, s, y, b).double()
                cos.append(float((gs * g1).sum() / (gs.norm() * g1.norm())))
            label = f"{pr.stages[k][0]}x" if k < len(pr.stages) else "end"
            lines.append(f"| C{cfg} | {label} | {it} | {cos[0]:.4f} | {cos[1]:.4f} |")
            if k < len(pr.stages):
                it += pr.stages[k][1]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
open(os.path.join(ROOT, "gpurun_out", "r02_sketch_cosine.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
