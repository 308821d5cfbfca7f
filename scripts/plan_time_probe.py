import sys, time
sys.path.insert(0, ".")
import torch
import ms2g_synth as S, paper_2203_07308_b200 as P
P.load(); torch.zeros(1, device="cuda")
pr = S.PRESETS[4]
for rep in range(2):
    t = time.perf_counter()
    plan = P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1))
    torch.cuda.synchronize()
    print("C4 plan", round(time.perf_counter() - t, 2), "s", flush=True)
    plan.destroy()
