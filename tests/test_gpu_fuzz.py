"""Randomised parity fuzz (GPU vs fp64 oracle) over the launch shapes: image
sides with ragged tiles, view counts from 1, detector widths, sketch factors,
batch sizes (single-image, batched and odd batches), view subsets.  Each case
checks the forward with residual, the adjoint and the sketched gradient at the
operator tolerance.  MS2G_FUZZ_CASES raises the case count for stress runs."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import ms2g_synth as S  # noqa: E402
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-5


def rel(a, b):
    """Error measure of every parity assertion: the larger of the relative L2
    error and one tenth of the largest element error over the reference's
    RMS.  `rel(...) <= tol` thus gates both ||d|| <= tol ||ref|| and
    max|d| <= 10 tol rms(ref) (a bad tile that the L2 norm dilutes fails)."""
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    d = a - b
    l2 = float(np.linalg.norm(d) / max(np.linalg.norm(b), 1e-300))
    if d.size == 0:
        return l2
    rms = float(np.sqrt(np.mean(b ** 2)))
    return max(l2, float(np.max(np.abs(d))) / max(rms, 1e-300) / 10.0)


def _case(rng):
    s_max = int(rng.choice([1, 2, 3, 4]))
    base = int(rng.integers(4, 60))
    n = base * s_max * (2 if s_max == 3 else 1)
    factors = sorted({1} | {f for f in (2, 3, 4) if n % f == 0 and rng.random() < 0.6}, reverse=True)
    V = int(rng.integers(1, 120))
    B = 2 * int(rng.integers(1, int(1.2 * n) + 2))       # even: no ray on a grid line (reading Z14)
    batch = int(rng.choice([1, 1, 2, 3, 8]))
    return n, V, B, tuple(factors), batch


def test_fuzz_operators():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2203_07308_b200 as P
    P.load()
    rng = np.random.default_rng(20261020)
    cases = int(os.environ.get("MS2G_FUZZ_CASES", "12"))
    for c in range(cases):
        n, V, B, factors, batch = _case(rng)
        g = O.Geometry(n, V, B)
        sub = sorted(rng.choice(V, size=int(rng.integers(1, V + 1)), replace=False).tolist())
        with P.plan_geometry(n, V, B, factors=factors, batch=batch) as plan:
            for s in factors:
                nc = n // s
                xs = np.stack([S.random_image(nc, 1000 * c + s + 10 * i) for i in range(batch)])
                bs = np.stack([S.random_sinogram((V, B), 1000 * c + s + 10 * i) for i in range(batch)])
                got = P.forward_project(plan, s, torch.from_numpy(xs).cuda(), b=torch.from_numpy(bs).cuda(),
                                        subset=sub).cpu().numpy()
                for i in (0, batch - 1):
                    ref = O.forward(g, s, xs[i], b=bs[i], views=sub)
                    assert rel(got[i], ref) <= TOL, ("fwd", c, n, V, B, factors, batch, s, rel(got[i], ref))
                r = np.stack([S.random_sinogram((len(sub), B), 2000 * c + s + 10 * i) for i in range(batch)])
                img = P.back_project(plan, s, torch.from_numpy(r).cuda(), subset=sub).cpu().numpy()
                for i in (0, batch - 1):
                    ref = O.backward(g, s, r[i], views=sub)
                    assert rel(img[i], ref) <= TOL, ("bwd", c, n, V, B, factors, batch, s, rel(img[i], ref))
            s = factors[0]
            x = np.stack([S.random_image(n, 3000 * c + i) for i in range(batch)])
            b = np.stack([S.random_sinogram((V, B), 3000 * c + i) for i in range(batch)])
            gg = P.sketched_grad(plan, s, torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda(),
                                 subset=sub).cpu().numpy()
            ref = O.sketched_grad(g, s, x[0], b[0], views=sub)
            assert rel(gg[0], ref) <= TOL, ("grad", c, n, V, B, factors, batch, s, rel(gg[0], ref))


def _solve_case(rng):
    n = int(rng.choice([16, 24, 32, 48, 64]))
    facs = [f for f in (4, 3, 2) if n % f == 0]
    V = int(rng.integers(8, 61))
    B = 2 * int(rng.integers(n // 2, n + 8))
    option = int(rng.choice([1, 2, 3, 4, 5]))
    k = int(rng.integers(1, 4))
    stage_f = sorted(rng.choice(facs + [1], size=k, replace=True).tolist(), reverse=True)
    if option in (2, 3, 5):
        n_sub = int(rng.integers(2, min(8, V) + 1))
        stages = [(int(f), 0, int(rng.integers(1, 3))) for f in stage_f]
    else:
        n_sub = int(rng.integers(2, V + 1)) if option == 4 else 1
        stages = [(int(f), int(rng.integers(1, 5)), 0) for f in stage_f]
    den = [("identity",), ("gauss", 0.8), ("tv", 0.02, 5)][int(rng.integers(0, 3))]
    alpha = 1.0 if den[0] != "gauss" else 0.5
    batch = int(rng.choice([1, 1, 2, 3]))
    return n, V, B, stages, option, n_sub, den, alpha, batch


def test_fuzz_solves():
    """Random schedules (1-3 stages, factors 1-4, repeated factors), all five
    options, the three denoisers, batches: the solve against the oracle's
    Algorithm 1 and the schedule bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2203_07308_b200 as P
    P.load()
    rng = np.random.default_rng(7)
    cases = int(os.environ.get("MS2G_FUZZ_SOLVES", "6"))
    for c in range(cases):
        n, V, B, stages, option, n_sub, den, alpha, batch = _solve_case(rng)
        g = O.Geometry(n, V, B)
        factors = sorted({s[0] for s in stages} | {1}, reverse=True)
        xt = [S.phantom(n, 5, 4000 * c + i) for i in range(batch)]
        bs = np.stack([O.forward(g, 1, x) for x in xt]).astype(np.float32)
        seed = int(rng.integers(0, 2 ** 31))
        with P.plan_geometry(n, V, B, factors=tuple(factors), batch=batch) as plan:
            xo, tr = P.pnp_ms2g_solve(plan, stages, torch.from_numpy(bs).cuda(), option=option, n_subsets=n_sub,
                                      seed=seed, den=den, alpha=alpha, trace=True)
            xo = xo.cpu().numpy()
        for i in (0, batch - 1):
            xr, trr, _ = O.pnp_ms2g(g, stages, bs[i], option=option, n_subsets=n_sub, seed=seed, den=den,
                                    alpha=alpha)
            assert [e[:4] for e in tr] == [e[:4] for e in trr], ("schedule", c)
            assert rel(xo[i], xr) <= 1e-3, ("solve", c, n, V, B, stages, option, n_sub, den, batch,
                                            rel(xo[i], xr))
