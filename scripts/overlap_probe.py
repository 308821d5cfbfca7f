"""Does running two independent power iterations (factor 2 and factor 1 of the
C4 geometry, separate plans = separate workspaces) concurrently on two streams
beat running them back to back?  (dev aid; timings by CUDA events / wall)"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

pr = S.PRESETS[4]
pa = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2,))
pb = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(1,))
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def run(plan, f, st, out, k):
    with torch.cuda.stream(st):
        out[k] = P.power_iteration(plan, f, 20)


res = [None, None]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(pa, 2, sa, res, 0)
    run(pb, 1, sb, res, 1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ta = threading.Thread(target=run, args=(pa, 2, sa, res, 0))
    tb = threading.Thread(target=run, args=(pb, 1, sb, res, 1))
    t2 = time.perf_counter()
    ta.start(); tb.start(); ta.join(); tb.join()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"sequential {1e3 * (t1 - t0):.1f} ms, concurrent {1e3 * (t3 - t2):.1f} ms", flush=True)
