"""Per-iteration cost of the TV-prox denoiser (dev aid): time denoise() with
K = 1, 10 and 21 dual iterations at 512^2 (batch 1 and 8), 1024^2 and 256^2,
for the default, the persistent kernel (MS2G_TV_PERSIST=1) and the K + 1 launches with and without programmatic
dependent launch (MS2G_PDL=0); per call from Python, and per call inside a
CUDA graph of 20 calls (no host overhead)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) == 1:
    for extra in ({"MS2G_TV_PERSIST": "1"}, {"MS2G_TV_PERSIST": "0"}, {"MS2G_TV_PERSIST": "0", "MS2G_PDL": "0"}):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, **extra), check=True)
    sys.exit(0)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

tag = {"0": "per-iteration", "1": "persistent"}.get(os.environ.get("MS2G_TV_PERSIST", ""), "default")
if tag == "per-iteration":
    tag += " (no PDL)" if os.environ.get("MS2G_PDL") == "0" else " (PDL)"
for n, batch in ((512, 1), (512, 8), (1024, 1), (256, 1)):
    plan = P.plan_geometry(n, 8, 16, factors=(1,), batch=batch)
    z = torch.rand((batch, n, n), device="cuda")
    out = torch.empty_like(z)
    t = {k: bench.time_calls(lambda: P.denoise(plan, ("tv", 0.02, k), z, out), 200) for k in (1, 10, 21)}
    print(f"{tag:26s} n={n} batch {batch}: K=1 {1e6 * t[1]:.1f} us, K=10 {1e6 * t[10]:.1f} us, "
          f"K=21 {1e6 * t[21]:.1f} us -> {1e6 * (t[21] - t[1]) / 20:.2f} us per dual iteration", flush=True)
    try:   # the same inside a CUDA graph of 20 calls
        tg = {}
        for k in (1, 10):
            P.denoise(plan, ("tv", 0.02, k), z, out)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    P.denoise(plan, ("tv", 0.02, k), z, out)
            g.replay()
            torch.cuda.synchronize()
            tg[k] = bench.time_calls(g.replay, 20) / 20
        print(f"{tag:26s} n={n} batch {batch}: in a graph K=1 {1e6 * tg[1]:.1f} us, K=10 {1e6 * tg[10]:.1f} us",
              flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{tag:26s} graph capture failed: {e}", flush=True)
    plan.destroy()
