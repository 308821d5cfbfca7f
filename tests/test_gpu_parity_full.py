"""Full-size GPU vs fp64-oracle parity at the bench's own configuration.

C4 (1024^2, 1440 views x 1536 bins -- the workload `bench.py` times) element
by element: the forward projector with its fused residual and the exact
adjoint at s = 2 and s = 1 (zero-mean sinograms), the sketched
gradient at both factors from an x far from the data's solution (SURVEY
§8(c) "gradient parity inputs"), and the whole 50-step PnP-MS2G solve with
its 2 x 20 power iterations against the oracle's Algorithm 1.
C5 (batch of 8 512^2 images, Poisson data, TV) at full size: the batched
solve, images 0 and 7, against per-image oracle solves.

Every comparison checks BOTH the relative L2 error (north_star: <= 1e-5 per
operator call, <= 1e-3 per reconstruction) and the largest element error
relative to the reference's RMS, gated at 10x the same tolerance (a bad tile
or chunk that the L2 norm dilutes over a million pixels fails this one).
With MS2G_PARITY_LOG=<path> the achieved errors are written there as JSON
(profiles/parity_r02.md is made from it).
"""
import json
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import ms2g_synth as S  # noqa: E402
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_OP = 1e-5
TOL_SOLVE = 1e-3
LOG = {}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2203_07308_b200 as P
    P.load()
    yield P
    path = os.environ.get("MS2G_PARITY_LOG")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(LOG, f, indent=1, sort_keys=True)


def measure(name, got, ref, tol, **extra):
    got = np.asarray(got, np.float64); ref = np.asarray(ref, np.float64)
    d = got - ref
    rms = float(np.sqrt(np.mean(ref ** 2)))
    rl2 = float(np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-300))
    mx = float(np.max(np.abs(d)) / max(rms, 1e-300))
    LOG[name] = {"rel_l2": rl2, "max_abs_over_rms": mx, "tol": tol, "elements": int(d.size), **extra}
    assert rl2 <= tol, (name, rl2)
    assert mx <= 10 * tol, (name, mx)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def c4():
    """The C4 problem as bench.py builds it (seeded phantom, 1 % Gaussian
    noise), with b from the ORACLE's projector (tests never take inputs from
    the CUDA path), and an independent phantom far from the data."""
    pr = S.PRESETS[4]
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(4))
    b = S.gaussian_data(O.forward(g, 1, xt), pr.noise[1], S.config_seed(4))
    xfar = S.phantom(pr.n, pr.n_ellipses, S.config_seed(4, 9))
    return pr, g, b, xfar


@pytest.fixture(scope="module")
def c4plan(P, c4):
    pr = c4[0]
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as plan:
        yield plan


@pytest.mark.parametrize("s", [2, 1])
def test_c4_forward_residual_full(P, c4, c4plan, s):
    pr, g, b, xfar = c4
    xs = xfar if s == 1 else O.sketch_down(xfar, 2).astype(np.float32)
    got = host(P.forward_project(c4plan, s, dev(xs)[None], b=dev(b)[None]))[0]
    ref = O.forward(g, s, xs, b=b)
    measure(f"C4 forward+residual s={s}", got, ref, TOL_OP, shape=list(got.shape))


@pytest.mark.parametrize("s", [2, 1])
def test_c4_adjoint_zero_mean_full(P, c4, c4plan, s):
    pr, g, b, xfar = c4
    r = S.random_sinogram((pr.n_views, pr.n_bins), 440 + s)
    got = host(P.back_project(c4plan, s, dev(r)[None]))[0]
    ref = O.backward(g, s, r)
    measure(f"C4 adjoint (zero-mean sinogram) s={s}", got, ref, TOL_OP, shape=list(got.shape))


@pytest.mark.parametrize("s", [2, 1])
def test_c4_sketched_grad_full(P, c4, c4plan, s):
    pr, g, b, xfar = c4
    got = host(P.sketched_grad(c4plan, s, dev(xfar)[None], dev(b)[None]))[0]
    ref = O.sketched_grad(g, s, xfar, b)
    measure(f"C4 sketched_grad s={s}", got, ref, TOL_OP, shape=list(got.shape))


def test_c4_solve_full(P, c4, c4plan):
    """The bench's workload end to end: stages 2x:30 -> full:20, Gaussian
    3x3 (sigma 0.8) with alpha = 0.5, 20 power iterations per stage."""
    pr, g, b, xfar = c4
    t0 = time.perf_counter()
    xo, tr = P.pnp_ms2g_solve(c4plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha,
                              power_iters=pr.power_iters, trace=True)
    xo = host(xo)[0]
    t1 = time.perf_counter()
    xr, trr, etas = O.pnp_ms2g(g, pr.stages, b, den=pr.den, alpha=pr.alpha, power_iters=pr.power_iters)
    t2 = time.perf_counter()
    assert [e[:4] for e in tr] == [e[:4] for e in trr]
    eta_err = max(abs(e[4] - er[4]) / er[4] for e, er in zip(tr, trr))
    assert eta_err <= 1e-5
    measure("C4 PnP-MS2G solve (50 steps, 2x20 power iterations)", xo, xr, TOL_SOLVE, eta_rel_err=eta_err,
            gpu_s_incl_capture=t1 - t0, oracle_s=t2 - t1, oracle_threads=O.default_threads())


def test_c5_batch8_solve_full(P):
    """C5 at full size: one plan with batch 8 (Poisson transmission data,
    I0 = 1e5, Eq. 8; stages 2x:20 -> full:20; TV lambda 0.02, K 10,
    alpha 1), images 0 and 7 against their own oracle solves."""
    pr = S.PRESETS[5]
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    bs = []
    for im in range(pr.batch):
        xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(5, im))
        bs.append(S.poisson_data(O.forward(g, 1, xt), pr.noise[1], S.config_seed(5, im)))
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), batch=pr.batch) as plan:
        xb = host(P.pnp_ms2g_solve(plan, pr.stages, dev(np.stack(bs)), den=pr.den, alpha=pr.alpha))
    for im in (0, pr.batch - 1):
        xr, _, _ = O.pnp_ms2g(g, pr.stages, bs[im], den=pr.den, alpha=pr.alpha)
        measure(f"C5 batch-8 solve, image {im}", xb[im], xr, TOL_SOLVE)


def test_c5_ranks_spot_check(P):
    """C5 over 8 ranks x batch 8 (64 images, BASELINE configs[4]; SURVEY
    §8(d) "images {0, 21, 42, 63}"): rank r solves images 8r .. 8r+7 with no
    collective in the data path (bench.py --cfg 5), so the ranks owning
    images 21, 42 and 63 (ranks 2, 5, 7) are run one after another on one
    GPU, each as its full batch of 8, and those images are compared with
    their own oracle solves (image 0, rank 0: test_c5_batch8_solve_full)."""
    pr = S.PRESETS[5]
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1), batch=pr.batch) as plan:
        for im in (21, 42, 63):
            rank = im // pr.batch
            bs = []
            for j in range(rank * pr.batch, (rank + 1) * pr.batch):
                xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(5, j))
                bs.append(S.poisson_data(O.forward(g, 1, xt), pr.noise[1], S.config_seed(5, j)))
            xb = host(P.pnp_ms2g_solve(plan, pr.stages, dev(np.stack(bs)), den=pr.den, alpha=pr.alpha))
            xr, _, _ = O.pnp_ms2g(g, pr.stages, bs[im % pr.batch], den=pr.den, alpha=pr.alpha)
            measure(f"C5 rank {rank} of 8 (batch 8), image {im}", xb[im % pr.batch], xr, TOL_SOLVE)
