"""Cost of the NEXT-3 peer path and of the NCCL path at ONE rank against the
plain plan, C4 solve (dev aid): the machinery's fixed cost per allreduce."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

pr = S.PRESETS[4]
x = torch.from_numpy(S.phantom(pr.n, pr.n_ellipses, S.config_seed(4))).cuda()[None].contiguous()
res = {}
for mode in ("plain", "nccl", "peer", "plain"):
    plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1))
    if mode == "nccl":
        P.attach_nccl(plan, 0, 1)
    elif mode == "peer":
        P.attach_peers(plan, 0, 1)
    b = P.forward_project(plan, 1, x)
    x0 = torch.zeros_like(x); xo = torch.empty_like(x)
    t = bench.time_calls(lambda: P.pnp_ms2g_solve_async(plan, pr.stages, b, x0, xo, den=pr.den, alpha=pr.alpha),
                         5, warm=2)
    P.solve_status(plan)
    print(f"{mode}: {1e3 * t:.2f} ms per C4 solve (90 allreduces)", flush=True)
    plan.destroy()
