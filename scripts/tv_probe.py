"""Per-iteration cost of the TV-prox denoiser (dev aid): time denoise() with
K = 1 and K = 21 dual iterations at 512^2, batch 1 and 8."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2203_07308_b200 as P  # noqa: E402
import bench  # noqa: E402

for batch in (1, 8):
    plan = P.plan_geometry(512, 8, 16, factors=(1,), batch=batch)
    z = torch.rand((batch, 512, 512), device="cuda")
    out = torch.empty_like(z)
    t1 = bench.time_calls(lambda: P.denoise(plan, ("tv", 0.02, 1), z, out), 50)
    t21 = bench.time_calls(lambda: P.denoise(plan, ("tv", 0.02, 21), z, out), 50)
    print(f"batch {batch}: K=1 {1e6 * t1:.1f} us, K=21 {1e6 * t21:.1f} us -> {1e6 * (t21 - t1) / 20:.2f} us "
          f"per dual iteration", flush=True)
    plan.destroy()
