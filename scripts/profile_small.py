"""ncu driver (dev aid): (a) 6 registered-subset s=4 gradients at C3 (the
standalone call the bench's subset rate times); (b) one C4 solve on rank 0's
shard of P=8 with a 1-rank NCCL communicator (the graph shape of the shard
estimate).  Run under gpurun with ncu; never report its timings."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "subset"
if mode == "subset":
    pr = S.PRESETS[3]
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
        x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(3, 9))).cuda()[None].contiguous()
        b = torch.from_numpy(S.random_sinogram((pr.n_views, pr.n_bins), 3, zero_mean=False)).cuda()[None].contiguous()
        g = torch.empty_like(x)
        rs = P.register_subset(plan, list(range(0, pr.n_views, 8)))
        for _ in range(6):
            P.sketched_grad(plan, 4, x, b, g=g, subset=rs)
        torch.cuda.synchronize()
else:
    pr = S.PRESETS[4]
    vb, ve = P.view_shard(pr.n_views, 0, 8)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), view_begin=vb, view_end=ve) as plan:
        P.attach_nccl(plan, 0, 1)
        b = torch.from_numpy(np.ascontiguousarray(S.random_sinogram((ve - vb, pr.n_bins), 3, zero_mean=False)))
        b = b.cuda()[None].contiguous()
        x0 = torch.zeros((1, pr.n, pr.n), device="cuda"); xo = torch.empty_like(x0)
        for _ in range(2):
            P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha)
        torch.cuda.synchronize()
print("ok")
