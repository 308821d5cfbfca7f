"""NEXT-2: PnP-MS2G vs PnP-FISTA on the paper's three CT settings (GPU).

The paper's only claim: Option-1 PnP-MS2G "achieves almost the same
reconstruction accuracy in PSNR compared to its full counterpart PnP-FISTA,
while only requires a fraction of the computation".  Settings (P:111, P:139,
P:152): 256^2 image, 228 detector bins; sparse-view 90 views over
[0, 360) with I0 = 10^5.5, low-dose 360 views with I0 = 10^3.5, limited-angle
90 views over [0, 180) with I0 = 10^5.5; Poisson transmission data (Eq. 8).
Stand-ins: seeded ellipse phantom instead of the disk/head/chest
images, TV-prox (Chambolle, K=10) instead of BM3D, alpha = 1.
PnP-FISTA = one full-resolution stage (S:269 degeneracy); MS2G = the paper's
K=2 schedule (s=4 then s=2) and a coarse-to-full 3-stage variant.
Cost = ray-pixel segments processed (oracle-exact nnz per factor), including
the 20 power iterations per stage.  PSNR peak = max of the ground truth.

  python scripts/quality_study.py [--iters 40] [--out profiles/r01_quality_study.md]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ms2g_synth as S  # noqa: E402
import paper_2203_07308_b200 as P  # noqa: E402

SETTINGS = {
    "sparse-view": dict(n_views=90, arc=2 * math.pi, i0=10 ** 5.5),
    "low-dose": dict(n_views=360, arc=2 * math.pi, i0=10 ** 3.5),
    "limited-angle": dict(n_views=90, arc=math.pi, i0=10 ** 5.5),
}


def psnr(x, ref):
    mse = float(np.mean((x - ref) ** 2))
    return 300.0 if mse == 0 else 10 * math.log10(float(ref.max()) ** 2 / mse)




def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--bins", type=int, default=228)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--lam", type=float, default=0.01)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_quality_study.md"))
    a = ap.parse_args()
    dev = torch.device("cuda")
    # segment counts from the oracle-written table (scripts/count_nnz.py --study-only):
    # this script drives the product path only
    with open(os.path.join(ROOT, "profiles", "nnz_counts.json")) as f:
        nnz_all = json.load(f)
    n, B, N = a.n, a.bins, a.iters
    xt = S.phantom(n, 20, S.config_seed(2)).astype(np.float32)
    schedules = {
        "PnP-FISTA (s=1)": [(1, N, 0)],
        "MS2G paper K=2 (s=4,2)": [(4, N // 2, 0), (2, N - N // 2, 0)],
        "MS2G 3-stage (s=4,2,1)": [(4, N // 3, 0), (2, N // 3, 0), (1, N - 2 * (N // 3), 0)],
    }
    rows = []
    for name, st in SETTINGS.items():
        V = st["n_views"]
        ent = nnz_all[f"QS_{name}"]
        assert ent["geometry"][:3] == [n, V, B], "run scripts/count_nnz.py --study-only for this geometry"
        nnz = {s: ent[str(s)] for s in (4, 2, 1)}
        with P.plan_geometry(n, V, B, factors=(4, 2, 1), arc=st["arc"]) as plan:
            p = P.forward_project(plan, 1, torch.from_numpy(xt).to(dev)[None])[0].cpu().numpy()
            b = torch.from_numpy(S.poisson_data(p, st["i0"], S.config_seed(2))).to(dev)[None].contiguous()
            for sname, stages in schedules.items():
                for resampler in ("mean", "bicubic"):
                    if sname.startswith("PnP-FISTA") and resampler == "bicubic":
                        continue
                    # trajectory: PSNR after k iterations of the same schedule prefix
                    traj = []
                    total = sum(s_[1] for s_ in stages)
                    for frac in (0.25, 0.5, 0.75, 1.0):
                        k = max(1, int(round(total * frac)))
                        pre, left = [], k
                        for (s_, it, ep) in stages:
                            take = min(it, left)
                            if take > 0:
                                pre.append((s_, take, ep))
                            left -= take
                        x = P.pnp_ms2g_solve(plan, pre, b, den=("tv", a.lam, 10), alpha=1.0, resampler=resampler)
                        cost = sum((20 + it) * 2 * nnz[s_] for (s_, it, _) in pre)
                        traj.append((k, psnr(x[0].cpu().numpy(), xt), cost))
                    rows.append(dict(setting=name, schedule=sname, resampler=resampler, traj=traj))
                    print(name, sname, resampler, traj, flush=True)
    fista = {r["setting"]: r for r in rows if r["schedule"].startswith("PnP-FISTA")}
    lines = ["# NEXT-2: PnP-MS2G vs PnP-FISTA on the paper's CT settings (synthetic stand-ins)", "",
             f"256² seeded-ellipse phantom, {B} bins, Poisson data, TV-prox (λ={a.lam}, K=10), α=1, "
             f"{N} iterations; cost = segments processed incl. 20 power iterations per stage "
             "(scripts/quality_study.py, B200).", "",
             "| setting | schedule | S/U | PSNR @25% | @50% | @75% | final PSNR (dB) | final cost / FISTA cost | Δ PSNR vs FISTA |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        f = fista[r["setting"]]
        fin = r["traj"][-1]
        lines.append(f"| {r['setting']} | {r['schedule']} | {r['resampler']} | "
                     + " | ".join(f"{t[1]:.2f}" for t in r["traj"][:3])
                     + f" | {fin[1]:.2f} | {fin[2] / f['traj'][-1][2]:.2f} | {fin[1] - f['traj'][-1][1]:+.2f} |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(os.path.splitext(a.out)[0] + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
