"""Does running independent power iterations (one per stage factor, separate
plans = separate workspaces) concurrently on separate streams beat running
them back to back?  (dev aid; wall-clock around synchronised regions)"""
import argparse
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
a = ap.parse_args()
pr = S.PRESETS[a.cfg]
facs = sorted({s[0] for s in pr.stages}, reverse=True)
plans = [P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(f,)) for f in facs]
streams = [torch.cuda.Stream() for _ in facs]


def run(plan, f, st):
    with torch.cuda.stream(st):
        P.power_iteration(plan, f, 20)


for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for pl, f, st in zip(plans, facs, streams):
        run(pl, f, st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    th = [threading.Thread(target=run, args=(pl, f, st)) for pl, f, st in zip(plans, facs, streams)]
    t2 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"C{a.cfg} factors {facs}: sequential {1e3 * (t1 - t0):.2f} ms, concurrent {1e3 * (t3 - t2):.2f} ms",
          flush=True)
