"""ncu driver: the TV-prox denoiser at 512^2, batch 8, K = 3 (dev aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2203_07308_b200 as P  # noqa: E402

plan = P.plan_geometry(512, 8, 16, factors=(1,), batch=8)
z = torch.rand((8, 512, 512), device="cuda")
out = torch.empty_like(z)
for _ in range(2):
    P.denoise(plan, ("tv", 0.02, 3), z, out)
torch.cuda.synchronize()
print("ok")
