"""Small end-to-end exercise of every libms2g entry point for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

for (n, V, B, fac, batch) in [(64, 30, 96, (2, 1), 1), (40, 12, 62, (2, 1), 2)]:
    with P.plan_geometry(n, V, B, factors=fac, batch=batch) as plan:
        x = torch.from_numpy(np.stack([S.phantom(n, 5, i) for i in range(batch)])).cuda().contiguous()
        b = torch.from_numpy(np.stack([S.random_sinogram((V, B), i) for i in range(batch)])).cuda().contiguous()
        for s in fac:
            xs = x if s == 1 else P.sketch_down(plan, s, x)
            r = P.forward_project(plan, s, xs, b=b)
            P.back_project(plan, s, r)
            P.sketched_grad(plan, s, x, b)
            P.sketched_grad(plan, s, x, b, subset=list(range(1, V, 4)))
            P.sketch_up(plan, s, P.back_project(plan, s, r), y=x, eta=0.1)
            P.sketched_grad(plan, s, x, b, resampler="bicubic")
            P.power_iteration(plan, s, 3)
        for den in (("gauss", 0.8), ("tv", 0.02, 3), ("identity",)):
            P.denoise(plan, den, x)
        P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 2, 0)], b, den=("tv", 0.02, 2), alpha=1.0)
        P.pnp_ms2g_solve(plan, [(2, 1, 1), (1, 0, 1)], b, option=2, n_subsets=4, seed=3, den=("gauss", 0.8))
torch.cuda.synchronize()
print("sanitize run ok")
