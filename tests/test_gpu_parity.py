"""GPU (libms2g, sm_100a) vs fp64 oracle parity, element by element.

Bar (BASELINE.json north_star): relative L2 <= 1e-5 per operator call,
<= 1e-3 on the reconstruction after the full schedule, bit-exact schedules.
Inputs are seeded (ms2g_synth) and shaped like C1..C5; sizes span several
32x32 tiles and ragged tails; backprojection inputs include zero-mean random
sinograms (consistent-sign inputs hide crossing-precision errors).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import ms2g_synth as S  # noqa: E402
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TOL_OP = 1e-5
TOL_SOLVE = 1e-3


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2203_07308_b200 as P
    P.load()
    return P


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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


# geometry cases: (n, V, B, factors); ragged n_c (20, 40, 48) leave partial tiles
GEOMS = [
    (64, 90, 96, (2, 1)),          # C1
    (256, 360, 384, (4, 2, 1)),    # C2
    (40, 20, 62, (2, 1)),          # ragged tiles (n_c = 20, 40)
    (96, 33, 150, (3, 1)),         # factor 3, wide detector
]


@pytest.mark.parametrize("n,V,B,factors", GEOMS)
def test_forward_parity(P, n, V, B, factors):
    g = O.Geometry(n, V, B)
    with P.plan_geometry(n, V, B, factors=factors) as plan:
        for s in factors:
            nc = n // s
            for x in (S.phantom(nc, 8, 11 + s), S.random_image(nc, 5 + s)):
                ref = O.forward(g, s, x)
                got = host(P.forward_project(plan, s, dev(x)[None]))[0]
                assert rel(got, ref) <= TOL_OP, (s, rel(got, ref))


@pytest.mark.parametrize("n,V,B,factors", GEOMS)
def test_forward_residual_and_subset(P, n, V, B, factors):
    g = O.Geometry(n, V, B)
    rng = np.random.default_rng(n)
    b = S.random_sinogram((V, B), 77, zero_mean=False) * 3
    sub = np.sort(rng.choice(V, size=max(1, V // 3), replace=False))
    with P.plan_geometry(n, V, B, factors=factors) as plan:
        s = factors[0]
        x = S.phantom(n // s, 6, 3)
        ref = O.forward(g, s, x, b=b, views=sub)
        got = host(P.forward_project(plan, s, dev(x)[None], b=dev(b)[None], subset=sub))[0]
        assert rel(got, ref) <= TOL_OP


@pytest.mark.parametrize("n,V,B,factors", GEOMS)
def test_backward_parity_zero_mean(P, n, V, B, factors):
    g = O.Geometry(n, V, B)
    with P.plan_geometry(n, V, B, factors=factors) as plan:
        for s in factors:
            for zm in (True, False):
                r = S.random_sinogram((V, B), 100 + s, zero_mean=zm)
                ref = O.backward(g, s, r)
                got = host(P.back_project(plan, s, dev(r)[None]))[0]
                assert rel(got, ref) <= TOL_OP, (s, zm, rel(got, ref))


def test_backward_subset_scale_accumulate(P):
    n, V, B = 128, 120, 192
    g = O.Geometry(n, V, B)
    sub = O.subset_views(V, 8, 3)
    r = S.random_sinogram((len(sub), B), 9)
    with P.plan_geometry(n, V, B, factors=(2,)) as plan:
        base = S.random_image(64, 4)
        ref = base + 8.0 * O.backward(g, 2, r, views=sub)
        img = dev(base)[None].clone()
        P.back_project(plan, 2, dev(r)[None], img=img, scale=8.0, accumulate=True, subset=sub)
        assert rel(host(img)[0], ref) <= TOL_OP


def test_adjoint_identity_fp32(P):
    """GPU-only invariant: <A x, y> = <x, A^T y> in fp32 (same weights)."""
    n, V, B = 256, 180, 384
    with P.plan_geometry(n, V, B, factors=(1, 2)) as plan:
        for s in (1, 2):
            nc = n // s
            for k in range(3):
                x = dev(S.random_image(nc, 30 + k) - 0.5)[None]
                y = dev(S.random_sinogram((V, B), 40 + k))[None]
                lhs = float((P.forward_project(plan, s, x).double() * y.double()).sum())
                rhs = float((x.double() * P.back_project(plan, s, y).double()).sum())
                assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_adjoint_fixed_point_scale(P):
    """The fixed-point adjoint (per-warp scale from per-view residual bounds):
    linear over 60 orders of magnitude of the residual (x 1e-30, x 1e+30),
    exact zeros for a zero sinogram, NaN for a non-finite residual (so the
    solve's divergence check sees it), and within 2e-6 of the fp32
    read-modify-write form (MS2G_BP_FP32=1, subprocess) on ragged grids, a
    subset and a batch."""
    import os
    import subprocess
    import sys
    n, V, B = 96, 60, 144
    g = O.Geometry(n, V, B)
    r = S.random_sinogram((V, B), 17)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        for s in (1, 2):
            ref = O.backward(g, s, r)
            base = host(P.back_project(plan, s, dev(r)[None]))[0]
            assert rel(base, ref) <= TOL_OP
            for k in (1e-30, 1e30):
                out = host(P.back_project(plan, s, dev(r * k)[None]))[0] / k
                assert rel(out, base) <= 1e-6, k
            assert not np.any(host(P.back_project(plan, s, dev(np.zeros((V, B)))[None])))
            rb = r.copy()
            rb[7, 70] = np.inf
            out = host(P.back_project(plan, s, dev(rb)[None]))[0]
            assert np.isnan(out).any()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import ms2g_synth as S, paper_2203_07308_b200 as P
P.load()
outs = []
for n, V, B, facs, batch, sub in ((62, 33, 94, (2, 1), 1, None), (128, 90, 192, (4, 1), 2, list(range(3, 90, 7)))):
    with P.plan_geometry(n, V, B, factors=facs, batch=batch) as plan:
        nv = len(sub) if sub else V
        for s in facs:
            r = np.stack([S.random_sinogram((nv, B), 70 + s + i) for i in range(batch)]).astype(np.float32)
            outs.append(P.back_project(plan, s, torch.from_numpy(r).cuda(), subset=sub).cpu().numpy().ravel())
sys.stdout.buffer.write(np.concatenate(outs).astype(np.float64).tobytes())
''' % root
    res = []
    for extra in ({}, {"MS2G_BP_FP32": "1"}):
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, env=dict(os.environ, **extra),
                             timeout=600)
        assert out.returncode == 0, out.stderr.decode()[-2000:]
        res.append(np.frombuffer(out.stdout, dtype=np.float64))
    assert res[0].size > 0 and rel(res[0], res[1]) <= 2e-6


def test_backward_deterministic(P):
    n, V, B = 256, 360, 384
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        r = dev(S.random_sinogram((V, B), 5))[None]
        for s in (2, 1):
            a = P.back_project(plan, s, r).clone(); b = P.back_project(plan, s, r)
            torch.cuda.synchronize()
            assert torch.equal(a, b)


@pytest.mark.parametrize("s", [1, 2, 4])
def test_sketch_down_up(P, s):
    n = 64
    x = S.random_image(n, 8)
    with P.plan_geometry(n, 10, 96, factors=(s,)) as plan:
        v = host(P.sketch_down(plan, s, dev(x)[None]))[0]
        ref = O.sketch_down(x, s)
        assert np.max(np.abs(v - ref)) <= 2e-7 * np.max(np.abs(ref))
        gc = S.random_image(n // s, 9)
        up = host(P.sketch_up(plan, s, dev(gc)[None]))[0]
        assert np.array_equal(up, O.sketch_up(gc.astype(np.float64), s).astype(np.float32).astype(np.float64))
        y = S.random_image(n, 10)
        z = host(P.sketch_up(plan, s, dev(gc)[None], y=dev(y)[None], eta=0.3))[0]
        zr = y - np.float32(0.3) * O.sketch_up(gc, s)
        assert np.max(np.abs(z - zr)) <= 1e-6


@pytest.mark.parametrize("cfg,factors", [(1, (2, 1)), (2, (4, 2, 1))])
def test_sketched_grad_option1(P, cfg, factors):
    pr = S.PRESETS[cfg]
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg))
    b = S.gaussian_data(O.forward(g, 1, xt), pr.noise[1], S.config_seed(cfg)).astype(np.float32)
    x = S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg, 9))   # independent image: ||r|| = O(||b||)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=factors) as plan:
        for s in factors:
            ref = O.sketched_grad(g, s, x, b)
            got = host(P.sketched_grad(plan, s, dev(x)[None], dev(b)[None]))[0]
            assert rel(got, ref) <= TOL_OP, (s, rel(got, ref))


def test_sketched_grad_option2_subsets(P):
    n, V, B = 128, 160, 192
    g = O.Geometry(n, V, B)
    b = S.random_sinogram((V, B), 3, zero_mean=False) * 2
    x = S.phantom(n, 12, 4)
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        for s in (4, 2, 1):
            for k in (0, 5):
                sub = O.subset_views(V, 8, k)
                ref = O.sketched_grad(g, s, x, b, views=sub)
                got = host(P.sketched_grad(plan, s, dev(x)[None], dev(b)[None], subset=sub))[0]
                assert rel(got, ref) <= TOL_OP, (s, k, rel(got, ref))


@pytest.mark.parametrize("n,V,B,s", [(64, 90, 96, 2), (64, 90, 96, 1), (256, 360, 384, 4), (128, 45, 200, 1)])
def test_power_iteration(P, n, V, B, s):
    g = O.Geometry(n, V, B)
    with P.plan_geometry(n, V, B, factors=(s,)) as plan:
        L = P.power_iteration(plan, s, 20)
    Lr = O.power_iteration(g, s, 20)
    assert abs(L - Lr) <= 1e-5 * Lr


def test_denoisers(P):
    n = 96
    z = S.phantom(n, 10, 21) + 0.05 * S.random_sinogram((n, n), 2)
    with P.plan_geometry(n, 8, 150, factors=(1,)) as plan:
        gz = host(P.denoise(plan, ("gauss", 0.8), dev(z)[None]))[0]
        assert rel(gz, O.gauss3(z, 0.8)) <= TOL_OP
        for lam in (0.02, 0.01):
            tz = host(P.denoise(plan, ("tv", lam, 10), dev(z)[None]))[0]
            assert rel(tz, O.tv_chambolle(z, lam, 10)) <= TOL_OP
        iz = host(P.denoise(plan, ("identity",), dev(z)[None]))[0]
        assert np.array_equal(iz, z.astype(np.float32))


@pytest.mark.parametrize("cfg", [3, 2])
def test_schedule_bit_exact(P, cfg):
    pr = S.PRESETS[cfg]
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(1,)) as plan:
        a = P.schedule(plan, pr.stages, pr.option, pr.n_subsets, S.config_seed(cfg))
    b = O.schedule(pr.stages, pr.option, pr.n_subsets, S.config_seed(cfg))
    assert [e[:4] for e in a] == [e[:4] for e in b]
    assert [e[5] for e in a] == [e[5] for e in b]


def _make_data(pr, cfg, image=0):
    g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
    xt = S.phantom(pr.n, pr.n_ellipses, S.config_seed(cfg, image), texture=pr.texture)
    p = O.forward(g, 1, xt)
    if pr.noise[0] == "gauss":
        b = S.gaussian_data(p, pr.noise[1], S.config_seed(cfg, image))
    else:
        b = S.poisson_data(p, pr.noise[1], S.config_seed(cfg, image))
    return g, xt, b


@pytest.mark.parametrize("cfg", [1, 2])
def test_solve_parity_option1(P, cfg):
    pr = S.PRESETS[cfg]
    g, xt, b = _make_data(pr, cfg)
    factors = sorted({s[0] for s in pr.stages} | {1}, reverse=True)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=factors) as plan:
        xo, tr = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha, trace=True)
        xo = host(xo)[0]
    xr, trr, etas = O.pnp_ms2g(g, pr.stages, b, den=pr.den, alpha=pr.alpha)
    assert rel(xo, xr) <= TOL_SOLVE, rel(xo, xr)
    assert [e[:4] for e in tr] == [e[:4] for e in trr]
    for e, er in zip(tr, trr):
        assert abs(e[4] - er[4]) <= 1e-5 * er[4]


@pytest.mark.slow
def test_solve_parity_option2_c3(P):
    pr = S.PRESETS[3]
    g, xt, b = _make_data(pr, 3)
    seed = S.config_seed(3)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
        xo, tr = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], option=2, n_subsets=8, seed=seed, den=pr.den,
                                  alpha=pr.alpha, trace=True)
        xo = host(xo)[0]
    xr, trr, _ = O.pnp_ms2g(g, pr.stages, b, option=2, n_subsets=8, seed=seed, den=pr.den, alpha=pr.alpha)
    assert [e[:4] for e in tr] == [e[:4] for e in trr]
    assert rel(xo, xr) <= TOL_SOLVE, rel(xo, xr)


def test_solve_batch_matches_single(P):
    """C5-style batch (Poisson data, TV): each batch image equals its own
    single-image solve and the oracle."""
    n, V, B = 128, 90, 192
    g = O.Geometry(n, V, B)
    stages = [(2, 4, 0), (1, 3, 0)]
    bs, xs = [], []
    for im in range(3):
        xt = S.phantom(n, 10, S.config_seed(5, im))
        bs.append(S.poisson_data(O.forward(g, 1, xt), 1e5, S.config_seed(5, im)))
    with P.plan_geometry(n, V, B, factors=(2, 1), batch=3) as plan:
        xb = host(P.pnp_ms2g_solve(plan, stages, dev(np.stack(bs)), den=("tv", 0.02, 10), alpha=1.0))
    for im in range(3):
        xr, _, _ = O.pnp_ms2g(g, stages, bs[im], den=("tv", 0.02, 10), alpha=1.0)
        assert rel(xb[im], xr) <= TOL_SOLVE


def test_emulated_view_sharding(P):
    """P view shards run one after another on one GPU: the sum of the partial
    backprojections equals the full one (the algebra the NCCL allreduce
    implements)."""
    n, V, B = 128, 90, 192
    r = S.random_sinogram((V, B), 12)
    x = S.phantom(n, 8, 2)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as full:
        ref = host(P.back_project(full, 1, dev(r)[None]))[0]
        fref = host(P.forward_project(full, 2, dev(x[::2, ::2])[None]))[0]
    for nr in (2, 3, 4):
        acc = np.zeros_like(ref)
        fwd = []
        for rk in range(nr):
            vb, ve = P.view_shard(V, rk, nr)
            with P.plan_geometry(n, V, B, factors=(2, 1), view_begin=vb, view_end=ve) as sh:
                acc += host(P.back_project(sh, 1, dev(r[vb:ve])[None]))[0]
                fwd.append(host(P.forward_project(sh, 2, dev(x[::2, ::2])[None]))[0])
        assert rel(acc, ref) <= 1e-6
        assert np.array_equal(np.concatenate(fwd, 0), fref)


def test_full_size_sampled_c4(P):
    """C4 full size (1024^2, 1440 x 1536) in the bench's launch configuration:
    sampled rays (forward) and pixels (adjoint) against the oracle, one by one."""
    pr = S.PRESETS[4]
    n, V, B = pr.n, pr.n_views, pr.n_bins
    g = O.Geometry(n, V, B)
    x = S.phantom(n, pr.n_ellipses, S.config_seed(4))
    rng = np.random.default_rng(4)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        for s in (2, 1):
            xs = x if s == 1 else O.sketch_down(x, 2).astype(np.float32)
            got = host(P.forward_project(plan, s, dev(xs)[None]))[0]
            vv, tt = rng.integers(0, V, 200), rng.integers(0, B, 200)
            ref = np.array([O.ray_sum(g, s, xs, int(v), int(t)) for v, t in zip(vv, tt)])
            assert rel(got[vv, tt], ref) <= TOL_OP
        r = S.random_sinogram((V, B), 44)
        # s = 2 (n_c = 512: 32x64 adjoint tiles) and s = 1 (n_c = 1024: 32x96 tiles)
        for s, pix in ((2, [(0, 0), (511, 511), (256, 100), (17, 400), (300, 301), (128, 0)]),
                       (1, [(0, 0), (1023, 1023), (512, 200), (95, 96), (96, 95), (700, 191), (191, 700),
                            (1000, 33)])):
            img = host(P.back_project(plan, s, dev(r)[None]))[0]
            ref = np.array([O.backward_pixel(g, s, r, i, j) for i, j in pix])
            gotp = np.array([img[i, j] for i, j in pix])
            assert np.max(np.abs(gotp - ref)) <= TOL_OP * np.sqrt(np.mean(img ** 2)) * 3, s
            # property at full size: <A_s x, r> = <x, A_s^T r> (fp64 dots of the fp32 results)
            xr = S.random_image(n // s, 45 + s)
            ax = host(P.forward_project(plan, s, dev(xr)[None]))[0]
            lhs, rhs = float(np.sum(ax * r)), float(np.sum(xr.astype(np.float64) * img))
            assert abs(lhs - rhs) <= TOL_OP * max(abs(lhs), abs(rhs)), (s, lhs, rhs)


def test_divergence_reported(P):
    """S:258 / SURVEY §8(b): a NaN planted in b is an INPUT error (code 7,
    checked on the device at the solve's start); iterates that overflow are
    a divergence (code 3) naming the stage and iteration."""
    n, V, B = 64, 30, 96
    b = np.ones((V, B), np.float32); b[3, 7] = np.nan
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        with pytest.raises(P.MS2GError, match="non-finite") as e:
            P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 1, 0)], dev(b)[None])
        assert e.value.code == 7
        x0 = torch.zeros((1, n, n), device="cuda"); x0[0, 5, 5] = float("inf")
        with pytest.raises(P.MS2GError) as e:
            P.pnp_ms2g_solve(plan, [(1, 1, 0)], dev(np.ones((V, B), np.float32))[None], x0=x0)
        assert e.value.code == 7
        big = np.full((V, B), 3e38, np.float32)    # finite data whose gradient overflows fp32
        with pytest.raises(P.DivergedError, match="non-finite iterate at stage"):
            P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 1, 0)], dev(big)[None])
        ok = P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 1, 0)], dev(np.ones((V, B), np.float32))[None])
        assert torch.isfinite(ok).all()          # the flags are reset for the next solve


def test_config_errors(P):
    with pytest.raises(P.MS2GError) as e:
        P.plan_geometry(64, 10, 96, factors=(3,))
    assert e.value.code == 2
    with pytest.raises(P.MS2GError):
        P.plan_geometry(64, 10, 96, factors=(1,), sod=1.0)
    with P.plan_geometry(64, 10, 96, factors=(2,)) as plan:
        x = torch.zeros((1, 32, 32), device="cuda")
        with pytest.raises(P.MS2GError) as e:
            P.forward_project(plan, 1, x)
        assert e.value.code == 2
        with pytest.raises(P.MS2GError) as e:
            P.forward_project(plan, 2, x, subset=[3, 1])
        assert e.value.code == 7
        with pytest.raises(P.MS2GError):
            P.pnp_ms2g_solve(plan, [(2, 1, 0)], torch.zeros((1, 10, 96), device="cuda"), alpha=0.0)


def test_launch_count_increases(P):
    before = P.launch_count()
    with P.plan_geometry(64, 10, 96, factors=(1,)) as plan:
        P.forward_project(plan, 1, torch.ones((1, 64, 64), device="cuda"))
    assert P.launch_count() > before


def test_emulated_sharding_with_subsets(P):
    """Option-2 subsets across view shards: each rank's compacted output covers
    shard ∩ subset in ascending order, and the partial adjoints sum to the
    full-plan adjoint; sketched_grad partials (scaled by V/|M| with the
    global |M|) sum to the single-plan gradient."""
    n, V, B = 96, 90, 144
    sub = O.subset_views(V, 8, 3)
    x = S.phantom(n, 8, 5)
    b = S.random_sinogram((V, B), 6, zero_mean=False)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as full:
        f_ref = host(P.forward_project(full, 2, dev(x[::2, ::2])[None], b=dev(b)[None], subset=sub))[0]
        r = S.random_sinogram((len(sub), B), 7)
        b_ref = host(P.back_project(full, 1, dev(r)[None], scale=8.0, subset=sub))[0]
        g_ref = host(P.sketched_grad(full, 2, dev(x)[None], dev(b)[None], subset=sub))[0]
    fwd, acc, gacc = [], np.zeros_like(b_ref), np.zeros_like(g_ref)
    pos = 0
    for rk in range(3):
        vb, ve = P.view_shard(V, rk, 3)
        mine = [v for v in sub if vb <= v < ve]
        with P.plan_geometry(n, V, B, factors=(2, 1), view_begin=vb, view_end=ve) as sh:
            fwd.append(host(P.forward_project(sh, 2, dev(x[::2, ::2])[None], b=dev(b[vb:ve])[None], subset=sub))[0])
            acc += host(P.back_project(sh, 1, dev(r[pos:pos + len(mine)])[None], scale=8.0, subset=sub))[0]
            gacc += host(P.sketched_grad(sh, 2, dev(x)[None], dev(b[vb:ve])[None], subset=sub))[0]
        pos += len(mine)
    assert np.array_equal(np.concatenate(fwd, 0), f_ref)
    assert rel(acc, b_ref) <= 1e-6
    assert rel(gacc, g_ref) <= 1e-6


@pytest.mark.parametrize("nb", [8, 4, 2, 6])
def test_batched_forward_shares_traversal(P, nb):
    """A batch-nb plan (one traversal applied to nb images) gives, per image,
    the single-image forward projection up to fp32 summation order (a batch
    sums each ray in 2 column segments, a single image in 4) and the oracle's."""
    n, V, B = 64, 45, 96
    g = O.Geometry(n, V, B)
    xs = np.stack([S.phantom(n, 6, 40 + i) for i in range(nb)]).astype(np.float32)
    bs = np.stack([S.random_sinogram((V, B), 50 + i) for i in range(nb)]).astype(np.float32)
    with P.plan_geometry(n, V, B, factors=(2, 1), batch=nb) as plan, \
            P.plan_geometry(n, V, B, factors=(2, 1), batch=1) as one:
        for s in (2, 1):
            xin = xs if s == 1 else xs[:, ::2, ::2].copy()
            got = host(P.forward_project(plan, s, dev(xin), b=dev(bs)))
            for i in range(nb):
                single = host(P.forward_project(one, s, dev(xin[i])[None], b=dev(bs[i])[None]))[0]
                assert rel(got[i], single) <= 1e-6
            i = nb - 1
            assert rel(got[i], O.forward(g, s, xin[i], b=bs[i])) <= TOL_OP


@pytest.mark.parametrize("s", [2, 4])
def test_bicubic_resampling_parity(P, s):
    """NEXT-1 bicubic S/U (P:156 imresize) against the oracle."""
    n = 96
    x = S.random_image(n, 60 + s)
    with P.plan_geometry(n, 10, 150, factors=(s,)) as plan:
        v = host(P.sketch_down(plan, s, dev(x)[None], resampler="bicubic"))[0]
        assert rel(v, O.bicubic_down(x, s)) <= 1e-6
        gc = S.random_image(n // s, 70 + s) - 0.5
        up = host(P.sketch_up(plan, s, dev(gc)[None], resampler="bicubic"))[0]
        assert rel(up, O.bicubic_up(gc, s)) <= 1e-6
        y = S.random_image(n, 80)
        z = host(P.sketch_up(plan, s, dev(gc)[None], y=dev(y)[None], eta=0.25, resampler="bicubic"))[0]
        assert rel(z, y - np.float32(0.25) * O.bicubic_up(gc, s)) <= 1e-6


def test_bicubic_sketched_grad_and_solve(P):
    """Sketched gradient and a 3-stage solve with the paper's bicubic S/U."""
    pr = S.PRESETS[2]
    g, xt, b = _make_data(pr, 2)
    x = S.phantom(pr.n, pr.n_ellipses, S.config_seed(2, 9))
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(4, 2, 1)) as plan:
        for s in (4, 2):
            got = host(P.sketched_grad(plan, s, dev(x)[None], dev(b)[None], resampler="bicubic"))[0]
            assert rel(got, O.sketched_grad(g, s, x, b, resampler=1)) <= TOL_OP
        stages = [(4, 6, 0), (2, 6, 0), (1, 4, 0)]
        xo = host(P.pnp_ms2g_solve(plan, stages, dev(b)[None], den=pr.den, alpha=pr.alpha, resampler="bicubic"))[0]
    xr, _, _ = O.pnp_ms2g(g, stages, b, den=pr.den, alpha=pr.alpha, resampler=1)
    assert rel(xo, xr) <= TOL_SOLVE


def test_nccl_attached_single_rank(P):
    """The NCCL path (ncclCommInitRank + in-graph ncclAllReduce of the partial
    adjoint) with a 1-rank communicator: results equal the unattached plan."""
    n, V, B = 64, 45, 96
    x = S.phantom(n, 6, 3)
    b = S.random_sinogram((V, B), 4, zero_mean=False)
    stages = [(2, 3, 0), (1, 2, 0)]
    with P.plan_geometry(n, V, B, factors=(2, 1)) as a, P.plan_geometry(n, V, B, factors=(2, 1)) as c:
        P.attach_nccl(c, 0, 1)
        ga = host(P.sketched_grad(a, 2, dev(x)[None], dev(b)[None]))
        gc = host(P.sketched_grad(c, 2, dev(x)[None], dev(b)[None]))
        assert np.array_equal(ga, gc)
        ra = host(P.back_project(a, 1, dev(b)[None]))
        rc = host(P.back_project(c, 1, dev(b)[None], allreduce=True))
        assert np.array_equal(ra, rc)
        xa = host(P.pnp_ms2g_solve(a, stages, dev(b)[None], den=("gauss", 0.8), alpha=0.5))
        xc = host(P.pnp_ms2g_solve(c, stages, dev(b)[None], den=("gauss", 0.8), alpha=0.5))
        assert np.array_equal(xa, xc)
        assert abs(P.power_iteration(a, 2, 5) - P.power_iteration(c, 2, 5)) == 0.0


def test_svrg_option3_solve(P):
    """NEXT-4 SVRG estimator (Option 3) on the C3-shaped subset schedule:
    GPU solve vs the oracle, bit-exact schedule."""
    n, V, B = 128, 160, 192
    g = O.Geometry(n, V, B)
    xt = S.phantom(n, 12, S.config_seed(3))
    b = S.gaussian_data(O.forward(g, 1, xt), 0.01, S.config_seed(3))
    stages = [(4, 0, 1), (2, 0, 1), (1, 0, 1)]
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        xo, tr = P.pnp_ms2g_solve(plan, stages, dev(b)[None], option=3, n_subsets=8, seed=7, den=("tv", 0.01, 10),
                                  alpha=1.0, trace=True)
        xo = host(xo)[0]
    xr, trr, _ = O.pnp_ms2g(g, stages, b, option=3, n_subsets=8, seed=7, den=("tv", 0.01, 10), alpha=1.0)
    assert [e[:4] for e in tr] == [e[:4] for e in trr]
    assert rel(xo, xr) <= TOL_SOLVE, rel(xo, xr)


@pytest.mark.parametrize("nb", [2, 4, 3])
def test_batched_backward_shares_traversal(P, nb):
    """Batch plans backproject each image like a single-image plan (pairs of
    images share one traversal) and match the oracle."""
    n, V, B = 96, 60, 144
    g = O.Geometry(n, V, B)
    rs = np.stack([S.random_sinogram((V, B), 90 + i) for i in range(nb)]).astype(np.float32)
    with P.plan_geometry(n, V, B, factors=(2, 1), batch=nb) as plan, \
            P.plan_geometry(n, V, B, factors=(2, 1), batch=1) as one:
        for s in (2, 1):
            got = host(P.back_project(plan, s, dev(rs)))
            for i in range(nb):
                single = host(P.back_project(one, s, dev(rs[i])[None]))[0]
                assert rel(got[i], single) <= 1e-6
            assert rel(got[nb - 1], O.backward(g, s, rs[nb - 1])) <= TOL_OP


def test_option4_uniform_minibatch_solve(P):
    """NEXT-4 uniform random view minibatches (Option 4): the per-step view
    lists are bit-exact with the oracle's and the solve matches it."""
    n, V, B = 128, 120, 192
    g = O.Geometry(n, V, B)
    xt = S.phantom(n, 12, 41)
    b = S.gaussian_data(O.forward(g, 1, xt), 0.01, 41)
    stages = [(4, 6, 0), (2, 6, 0), (1, 4, 0)]
    m, seed = 17, 99
    ref_views = O.minibatch_views(V, m, seed, 16)
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        for st in (0, 5, 15):
            assert P.schedule_views(plan, stages, st, option=4, n_subsets=m, seed=seed) == ref_views[st].tolist()
        xo = host(P.pnp_ms2g_solve(plan, stages, dev(b)[None], option=4, n_subsets=m, seed=seed,
                                   den=("gauss", 0.8), alpha=0.5))[0]
    xr, _, _ = O.pnp_ms2g(g, stages, b, option=4, n_subsets=m, seed=seed, den=("gauss", 0.8), alpha=0.5)
    assert rel(xo, xr) <= TOL_SOLVE, rel(xo, xr)


def test_saga_option5_solve(P):
    """NEXT-4 SAGA estimator (Option 5) on the interleaved-subset schedule:
    GPU solve vs the oracle."""
    n, V, B = 128, 160, 192
    g = O.Geometry(n, V, B)
    xt = S.phantom(n, 12, S.config_seed(3, 2))
    b = S.gaussian_data(O.forward(g, 1, xt), 0.01, S.config_seed(3, 2))
    stages = [(4, 0, 2), (2, 0, 1), (1, 0, 1)]
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        xo = host(P.pnp_ms2g_solve(plan, stages, dev(b)[None], option=5, n_subsets=8, seed=11,
                                   den=("tv", 0.01, 10), alpha=1.0))[0]
    xr, _, _ = O.pnp_ms2g(g, stages, b, option=5, n_subsets=8, seed=11, den=("tv", 0.01, 10), alpha=1.0)
    assert rel(xo, xr) <= TOL_SOLVE, rel(xo, xr)


def test_solve_reuses_cached_step(P):
    """power_iters = 0 reuses the plan's per-factor step (L depends on the
    geometry only): same iterates bit for bit as the solve that
    computed it, same trace; a plan with no power iteration yet refuses."""
    pr = S.PRESETS[1]
    g, xt, b = _make_data(pr, 1)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as plan:
        with pytest.raises(P.MS2GError) as e:
            P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha, power_iters=0)
        assert e.value.code == 2
        x1, tr1 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha, trace=True)
        x2, tr2 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha, trace=True,
                                   power_iters=0)
        assert torch.equal(x1, x2)
        assert tr1 == tr2
        L = P.power_iteration(plan, 2, 20)   # refreshes the cache with the same value
        x3 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha, power_iters=0)
        assert torch.equal(x1, x3)
        assert abs(L - tr1[0][4] ** -1) <= 1e-12 * L


def test_peer_allreduce_single_rank(P):
    """NEXT-3 peer-memory allreduce (fused chunk-reduce publish, signal-pad
    barrier, fixed-order peer sum) with one rank: results equal the plain
    plan bit for bit, across repeated calls (the two exchange slots alternate),
    the power iteration, every Option and a batch; the solve keeps its parity."""
    n, V, B = 64, 45, 96
    x = S.phantom(n, 6, 3)
    b = S.random_sinogram((V, B), 4, zero_mean=False)
    stages = [(2, 3, 0), (1, 2, 0)]
    with P.plan_geometry(n, V, B, factors=(2, 1)) as a, P.plan_geometry(n, V, B, factors=(2, 1)) as c:
        P.attach_peers(c, 0, 1)
        for _ in range(3):
            ga = host(P.sketched_grad(a, 2, dev(x)[None], dev(b)[None]))
            gc = host(P.sketched_grad(c, 2, dev(x)[None], dev(b)[None]))
            assert np.array_equal(ga, gc)
        ra = host(P.back_project(a, 1, dev(b)[None], scale=0.5))
        rc = host(P.back_project(c, 1, dev(b)[None], scale=0.5, allreduce=True))
        assert np.array_equal(ra, rc)
        assert P.power_iteration(a, 2, 7) == P.power_iteration(c, 2, 7)
        for opt in (1, 2, 3, 5):
            kw = dict(den=("gauss", 0.8), alpha=0.5, option=opt, n_subsets=3 if opt > 1 else 1, seed=11)
            xa = host(P.pnp_ms2g_solve(a, stages, dev(b)[None], **kw))
            xc = host(P.pnp_ms2g_solve(c, stages, dev(b)[None], **kw))
            assert np.array_equal(xa, xc), opt
    with P.plan_geometry(n, V, B, factors=(2, 1), batch=2) as a, \
            P.plan_geometry(n, V, B, factors=(2, 1), batch=2) as c:
        P.attach_peers(c, 0, 1)
        bb = dev(np.stack([b, b[::-1].copy()]))
        xa = host(P.pnp_ms2g_solve(a, stages, bb, den=("gauss", 0.8), alpha=0.5))
        xc = host(P.pnp_ms2g_solve(c, stages, bb, den=("gauss", 0.8), alpha=0.5))
        assert np.array_equal(xa, xc)
        with pytest.raises(P.MS2GError):
            P.attach_peers(c, 0, 1)     # already attached


def test_kernel_timing_events(P):
    """In-graph projector timing (measurement support): the instrumented solve
    counts every launch per (kind, factor) and gives the same iterate."""
    pr = S.PRESETS[1]
    g, xt, b = _make_data(pr, 1)
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as plan:
        x1 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha)
        P.set_kernel_timing(plan, True)
        x2 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha)
        assert torch.equal(x1, x2)
        for f, iters in ((2, 10), (1, 10)):      # C1: 10 + 10 steps, 20 power iterations per stage
            for kind in ("forward", "backward"):
                ms, n = P.kernel_time(plan, kind, f)
                assert n == 20 + iters and ms > 0.0, (kind, f, n, ms)
        P.set_kernel_timing(plan, False)
        x3 = P.pnp_ms2g_solve(plan, pr.stages, dev(b)[None], den=pr.den, alpha=pr.alpha)
        assert torch.equal(x1, x3)
        assert P.kernel_time(plan, "backward", 1) == (0.0, 0)


@pytest.mark.parametrize("n,V,B,factors", [
    (8, 1, 2, (2, 1)),          # one view, two bins: a single-tile, single-chunk launch
    (6, 5, 4, (3, 1)),          # n_c = 2: tiles far larger than the grid
    (32, 2, 64, (1,)),          # detector wider than the fan needs: most rays miss
    (1024, 3, 1536, (1,)),      # H = 96 tiles with only 3 views (tiny chunks, LPT order)
])
def test_degenerate_geometries(P, n, V, B, factors):
    """Edge cases of the launch shapes: tiny grids and view counts, mostly-
    missing rays; forward and adjoint against the oracle, plus the adjoint
    identity."""
    g = O.Geometry(n, V, B)
    with P.plan_geometry(n, V, B, factors=factors) as plan:
        for s in factors:
            nc = n // s
            x = S.random_image(nc, 70 + s)
            ref = O.forward(g, s, x)
            got = host(P.forward_project(plan, s, dev(x)[None]))[0]
            assert rel(got, ref) <= TOL_OP, (s, rel(got, ref))
            r = S.random_sinogram((V, B), 80 + s)
            refb = O.backward(g, s, r)
            gotb = host(P.back_project(plan, s, dev(r)[None]))[0]
            assert rel(gotb, refb) <= TOL_OP, (s, rel(gotb, refb))
            lhs, rhs = float(np.sum(got * r)), float(np.sum(x.astype(np.float64) * gotb))
            assert abs(lhs - rhs) <= TOL_OP * max(abs(lhs), abs(rhs), 1e-30)


def test_empty_subset_and_bad_views_rejected(P):
    """Boundary errors of the subset path: empty, unsorted,
    out-of-range view lists are input errors (code 7) and launch nothing."""
    n, V, B = 32, 10, 48
    with P.plan_geometry(n, V, B, factors=(1,)) as plan:
        x = torch.zeros((1, n, n), device="cuda")
        for bad in ([], [3, 3], [11], [-1, 2]):
            with pytest.raises(P.MS2GError) as e:
                P.forward_project(plan, 1, x, subset=bad)
            assert e.value.code == 7, bad


def test_plan_lifecycle_releases_memory(P):
    """Plans own every workspace (no allocation inside a solve) and release it:
    repeated plan / solve / destroy cycles leave device memory where it was."""
    n, V, B = 128, 60, 192
    b = torch.from_numpy(S.random_sinogram((V, B), 3, zero_mean=False)).cuda()[None].contiguous()

    def cycle():
        with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
            P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 1, 0)], b, den=("tv", 0.02, 5), alpha=1.0)
            P.set_kernel_timing(plan, True)
            P.pnp_ms2g_solve(plan, [(2, 2, 0), (1, 1, 0)], b, den=("tv", 0.02, 5), alpha=1.0)
            P.attach_peers(plan, 0, 1)
            P.sketched_grad(plan, 2, torch.zeros((1, n, n), device="cuda"), b)
        torch.cuda.synchronize()

    cycle()                                   # first-use allocations (libraries, module load)
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(10):
        cycle()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= 8 << 20, (free0 - free1) / 2**20


def test_full_size_sampled_c3_subset_and_c5_batch(P):
    """C3 (512^2, 720 x 768, one interleaved 90-view subset) and C5 (batch of
    8 images) at full size in the launch configurations the solves use:
    sampled rays and pixels against the oracle, one by one."""
    rng = np.random.default_rng(35)
    pr = S.PRESETS[3]
    n, V, B = pr.n, pr.n_views, pr.n_bins
    g = O.Geometry(n, V, B)
    sub = list(range(3, V, 8))
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        for s in (4, 1):
            nc = n // s
            x = S.random_image(nc, 90 + s)
            got = host(P.forward_project(plan, s, dev(x)[None], subset=sub))[0]
            kk, tt = rng.integers(0, len(sub), 100), rng.integers(0, B, 100)
            ref = np.array([O.ray_sum(g, s, x, sub[int(k)], int(t)) for k, t in zip(kk, tt)])
            assert rel(got[kk, tt], ref) <= TOL_OP, s
            r = S.random_sinogram((len(sub), B), 95 + s)
            img = host(P.back_project(plan, s, dev(r)[None], subset=sub))[0]
            pix = [(0, 0), (nc - 1, nc - 1), (nc // 2, nc // 3), (nc // 5, nc - 2)]
            refp = np.array([O.backward_pixel(g, s, r, i, j, views=sub) for i, j in pix])
            gotp = np.array([img[i, j] for i, j in pix])
            assert np.max(np.abs(gotp - refp)) <= TOL_OP * np.sqrt(np.mean(img ** 2)) * 3, s
    pr = S.PRESETS[5]
    nb = pr.batch
    with P.plan_geometry(n, V, B, factors=(2, 1), batch=nb) as plan:
        xs = np.stack([S.random_image(n, 200 + i) for i in range(nb)])
        got = host(P.forward_project(plan, 1, dev(xs)))
        for i in (0, nb - 1):
            vv, tt = rng.integers(0, V, 60), rng.integers(0, B, 60)
            ref = np.array([O.ray_sum(g, 1, xs[i], int(v), int(t)) for v, t in zip(vv, tt)])
            assert rel(got[i][vv, tt], ref) <= TOL_OP, i
        rs = np.stack([S.random_sinogram((V, B), 300 + i) for i in range(nb)])
        img = host(P.back_project(plan, 2, dev(rs)))
        for i in (0, nb - 1):
            pix = [(0, 0), (255, 255), (100, 17)]
            refp = np.array([O.backward_pixel(g, 2, rs[i], a, c) for a, c in pix])
            gotp = np.array([img[i][a, c] for a, c in pix])
            assert np.max(np.abs(gotp - refp)) <= TOL_OP * np.sqrt(np.mean(img[i] ** 2)) * 3, i


@pytest.mark.parametrize("kw", [
    dict(arc=np.pi),                                   # limited angle
    dict(fov=1.0, sod=1.3, sdd=3.1),                   # other FOV and distances
    dict(bin_pitch=0.03),                              # wider detector pitch
    dict(arc=np.pi / 3),                               # 60-degree arc
])
def test_geometry_variants(P, kw):
    """Forward, adjoint and a short solve on non-default geometries (limited
    angle, FOV / source distances, detector pitch) against the oracle."""
    n, V, B = 96, 48, 144
    g = O.Geometry(n, V, B, **{k: v for k, v in kw.items()})
    with P.plan_geometry(n, V, B, factors=(2, 1), **kw) as plan:
        for s in (2, 1):
            x = S.random_image(n // s, 60 + s)
            assert rel(host(P.forward_project(plan, s, dev(x)[None]))[0], O.forward(g, s, x)) <= TOL_OP, s
            r = S.random_sinogram((V, B), 61 + s)
            assert rel(host(P.back_project(plan, s, dev(r)[None]))[0], O.backward(g, s, r)) <= TOL_OP, s
        xt = S.phantom(n, 8, 62)
        b = O.forward(g, 1, xt).astype(np.float32)
        stages = [(2, 4, 0), (1, 3, 0)]
        xo = host(P.pnp_ms2g_solve(plan, stages, dev(b)[None], den=("tv", 0.02, 10), alpha=1.0))[0]
    xr, _, _ = O.pnp_ms2g(g, stages, b, den=("tv", 0.02, 10), alpha=1.0)
    assert rel(xo, xr) <= TOL_SOLVE


def test_solve_repeated_factors_and_serial_equivalence(P):
    """A schedule that returns to a factor (coarse -> full -> coarse): the
    concurrent power-iteration branches serve every stage of a factor, and the
    solve matches the oracle; a plan with a 1-rank communicator (serial power
    iterations on one stream) gives the same iterate bit for bit."""
    pr = S.PRESETS[1]
    g, xt, b = _make_data(pr, 1)
    stages = [(2, 3, 0), (1, 2, 0), (2, 2, 0), (1, 1, 0)]
    with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as a, \
            P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as c:
        P.attach_nccl(c, 0, 1)
        xa, ta = P.pnp_ms2g_solve(a, stages, dev(b)[None], den=pr.den, alpha=pr.alpha, trace=True)
        xc, tc = P.pnp_ms2g_solve(c, stages, dev(b)[None], den=pr.den, alpha=pr.alpha, trace=True)
        assert torch.equal(xa, xc)
        assert ta == tc
    xr, trr, _ = O.pnp_ms2g(g, stages, b, den=pr.den, alpha=pr.alpha)
    assert rel(host(xa)[0], xr) <= TOL_SOLVE
    for e, er in zip(ta, trr):
        assert e[:4] == er[:4] and abs(e[4] - er[4]) <= 1e-5 * er[4]


def test_registered_subsets_match_adhoc(P):
    """ms2g_register_subset: the registered list (with its own longest-first
    block orders) gives the same operators as the ad-hoc host list, against
    the oracle; released ids are rejected."""
    n, V, B = 128, 90, 192
    g = O.Geometry(n, V, B)
    sub = list(range(5, V, 8))
    x = S.random_image(n, 61)
    b = S.random_sinogram((V, B), 62)
    with P.plan_geometry(n, V, B, factors=(4, 2, 1)) as plan:
        rs = P.register_subset(plan, sub)
        for s in (4, 2, 1):
            xs = x if s == 1 else O.sketch_down(x, s).astype(np.float32)
            a = host(P.forward_project(plan, s, dev(xs)[None], b=dev(b)[None], subset=sub))[0]
            r_ = host(P.forward_project(plan, s, dev(xs)[None], b=dev(b)[None], subset=rs))[0]
            assert rel(r_, O.forward(g, s, xs, b=b, views=sub)) <= TOL_OP
            assert rel(a, r_) <= 1e-6
            ga = host(P.sketched_grad(plan, s, dev(x)[None], dev(b)[None], subset=sub))[0]
            gr = host(P.sketched_grad(plan, s, dev(x)[None], dev(b)[None], subset=rs))[0]
            assert rel(gr, O.sketched_grad(g, s, x, b, views=sub)) <= TOL_OP
            assert rel(ga, gr) <= 1e-6
            r = S.random_sinogram((len(sub), B), 63 + s)
            img = host(P.back_project(plan, s, dev(r)[None], subset=rs, scale=2.0))[0]
            assert rel(img, 2.0 * O.backward(g, s, r, views=sub)) <= TOL_OP
        rs.release()
        with pytest.raises(P.MS2GError) as e:
            P.sketched_grad(plan, 1, dev(x)[None], dev(b)[None], subset=rs)
        assert e.value.code == 7


def test_adhoc_subsets_on_two_streams(P):
    """The ad-hoc subset ring: back-to-back calls with different subsets on
    two streams (no host sync in between) each use their own list."""
    n, V, B = 96, 64, 144
    g = O.Geometry(n, V, B)
    x = S.random_image(n, 71)
    subs = [list(range(k, V, 4)) for k in range(4)] * 3
    with P.plan_geometry(n, V, B, factors=(1,)) as plan:
        xd = dev(x)[None]
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        outs = []
        for k, sub in enumerate(subs):
            with torch.cuda.stream(s1 if k % 2 == 0 else s2):
                outs.append(P.forward_project(plan, 1, xd, subset=sub))
        torch.cuda.synchronize()
        for k, sub in enumerate(subs[:4]):
            assert rel(host(outs[k])[0], O.forward(g, 1, x, views=sub)) <= TOL_OP, k


def test_solve_key_uses_exact_bits(P):
    """Two descriptors whose alpha differs only after the 6th digit must not
    share a cached solve graph: the second solve uses its own
    alpha, i.e. matches a fresh plan with that alpha bit for bit."""
    n, V, B = 64, 45, 96
    b = dev(S.random_sinogram((V, B), 5, zero_mean=False))[None].contiguous()
    a1, a2 = 1.0 / 3.0, 0.3333330
    assert np.float32(a1) != np.float32(a2)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        P.pnp_ms2g_solve(plan, [(2, 3, 0), (1, 2, 0)], b, den=("gauss", 0.8), alpha=a1)
        x2 = P.pnp_ms2g_solve(plan, [(2, 3, 0), (1, 2, 0)], b, den=("gauss", 0.8), alpha=a2)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as fresh:
        x2f = P.pnp_ms2g_solve(fresh, [(2, 3, 0), (1, 2, 0)], b, den=("gauss", 0.8), alpha=a2)
    assert torch.equal(x2, x2f)


def test_host_x_out_is_written(P):
    """pnp_ms2g_solve writes a host x_out whether b is on the host or the device."""
    n, V, B = 64, 45, 96
    bh = torch.from_numpy(S.random_sinogram((V, B), 6, zero_mean=False))[None].contiguous()
    with P.plan_geometry(n, V, B, factors=(1,)) as plan:
        ref = P.pnp_ms2g_solve(plan, [(1, 3, 0)], bh.cuda(), den=("gauss", 0.8), alpha=0.5).cpu()
        for b in (bh, bh.cuda()):
            xo = torch.full((1, n, n), -7.0)
            res = P.pnp_ms2g_solve(plan, [(1, 3, 0)], b, den=("gauss", 0.8), alpha=0.5, x_out=xo)
            assert res.data_ptr() == xo.data_ptr() and torch.equal(xo, ref)


@pytest.mark.parametrize("n,batch", [(37, 3), (512, 1), (512, 8), (1024, 1), (130, 2)])
def test_tv_persistent_kernel(P, n, batch):
    """The single-launch persistent TV-prox (row strips per CTA, neighbour
    flags) against the oracle's Chambolle iteration at several shapes (ragged
    strips, strips crossing image boundaries in a batch), repeated calls
    (launch generations) bit-identical, and bitwise equal to the K + 1-launch
    form (MS2G_TV_PERSIST=0 in a subprocess) and to the persistent form with
    short rounds (MS2G_TV_KROUND=3, =1: halo exchanges between rounds)."""
    import os
    import subprocess
    import sys
    zs = np.stack([S.random_image(n, 500 + i) for i in range(batch)]).astype(np.float32)
    with P.plan_geometry(n, 8, 2 * n, factors=(1,), batch=batch) as plan:
        zt = dev(zs)
        outs = [host(P.denoise(plan, ("tv", 0.05, 10), zt)) for _ in range(3)]
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    for i in {0, batch - 1}:
        assert rel(outs[0][i], O.tv_chambolle(zs[i], 0.05, 10)) <= TOL_OP
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); import ms2g_synth as S; "
            "import paper_2203_07308_b200 as P; P.load(); n, b = %d, %d; "
            "z = np.stack([S.random_image(n, 500 + i) for i in range(b)]).astype(np.float32); "
            "pl = P.plan_geometry(n, 8, 2 * n, factors=(1,), batch=b); "
            "o = P.denoise(pl, ('tv', 0.05, 10), torch.from_numpy(z).cuda()); torch.cuda.synchronize(); "
            "sys.stdout.buffer.write(o.cpu().numpy().tobytes())" % (root, n, batch))
    # the K + 1-launch form, and the persistent form forced to rounds of 3
    # iterations (halo exchanges through global memory between rounds)
    for extra in ({"MS2G_TV_PERSIST": "0"}, {"MS2G_TV_PERSIST": "1"}, {"MS2G_TV_PERSIST": "1", "MS2G_TV_KROUND": "3"},
                  {"MS2G_TV_PERSIST": "1", "MS2G_TV_KROUND": "1"}):
        env = dict(os.environ, **extra)
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, env=env, timeout=300)
        assert out.returncode == 0, out.stderr.decode()[-2000:]
        other = np.frombuffer(out.stdout, dtype=np.float32).reshape(outs[0].shape)
        assert np.array_equal(other.astype(np.float64), outs[0]), extra


def test_forward_fast_path_bitwise(P):
    """The forward's carry-chained element index (warps whose rays stay within
    kPairPad rows of the grid) against the clamped path for every warp
    (MS2G_FWD_NO_FAST=1, subprocess), and the 4-view warp tiling against 1
    and 2 views per warp (MS2G_FWD_TILE): bitwise equal on ragged grids,
    factors 2 and 3, a view subset, a 45-degree view shard, an odd batch and
    a tiny grid narrower than the pad."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import ms2g_synth as S, paper_2203_07308_b200 as P
P.load()
outs = []
for n, V, B, facs, batch, sub, vb, ve in ((64, 90, 96, (2, 1), 1, None, 0, None), (40, 20, 62, (2, 1), 3, [1, 4, 7, 9, 15], 0, None),
                                          (96, 33, 150, (3, 1), 1, list(range(0, 33, 3)), 0, None),
                                          (256, 360, 384, (2, 1), 1, None, 45, 90), (8, 12, 14, (1,), 1, None, 0, None)):
    with P.plan_geometry(n, V, B, factors=facs, batch=batch, view_begin=vb, view_end=ve) as plan:
        for s in facs:
            x = np.stack([S.random_image(n, 30 + s + i) for i in range(batch)]).astype(np.float32)
            outs.append(P.forward_project(plan, s, torch.from_numpy(x).cuda(), subset=sub).cpu().numpy().ravel())
sys.stdout.buffer.write(np.concatenate(outs).astype(np.float32).tobytes())
''' % root
    res = []
    # also the warp tilings (1, 2 or 4 views per warp): the same per-ray
    # arithmetic on other lanes, so bit for bit the same outputs
    for extra in ({}, {"MS2G_FWD_NO_FAST": "1"}, {"MS2G_FWD_TILE": "1"}, {"MS2G_FWD_TILE": "2"}):
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, env=dict(os.environ, **extra),
                             timeout=600)
        assert out.returncode == 0, out.stderr.decode()[-2000:]
        res.append(np.frombuffer(out.stdout, dtype=np.float32))
    assert res[0].size > 0 and all(np.array_equal(res[0], r) for r in res[1:])


def test_gather_adjoint_variant_parity(P):
    """The pixel-driven gather adjoint (MS2G_BP_VARIANT=gather, the measured
    alternative to the tile-driven scatter) against the oracle on zero-mean
    sinograms: ragged grids, factors, a view subset and a batch, plus a short
    solve -- run in a subprocess so the switch is read fresh."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import ms2g_synth as S, oracle as O, paper_2203_07308_b200 as P
P.load()
def rel(a, b):
    d = a - b
    return max(np.linalg.norm(d) / np.linalg.norm(b), np.abs(d).max() / np.sqrt(np.mean(b ** 2)) / 10)
worst = 0.0
for n, V, B, facs, batch, sub in ((64, 90, 96, (2, 1), 1, None), (40, 20, 62, (2, 1), 2, [1, 4, 7, 9, 15]),
                                  (96, 33, 150, (3, 1), 1, list(range(0, 33, 3))), (256, 360, 384, (4, 1), 1, None)):
    g = O.Geometry(n, V, B)
    views = sub if sub is not None else list(range(V))
    with P.plan_geometry(n, V, B, factors=facs, batch=batch) as plan:
        for s in facs:
            r = np.stack([S.random_sinogram((len(views), B), 90 + s + i) for i in range(batch)])
            img = P.back_project(plan, s, torch.from_numpy(r).cuda(), subset=sub).cpu().numpy()
            for i in range(batch):
                worst = max(worst, rel(img[i].astype(np.float64), O.backward(g, s, r[i], views=sub)))
pr = S.PRESETS[1]
g = O.Geometry(pr.n, pr.n_views, pr.n_bins)
b = S.gaussian_data(O.forward(g, 1, S.phantom(pr.n, pr.n_ellipses, S.config_seed(1))), 0.01, S.config_seed(1))
with P.plan_geometry(pr.n, pr.n_views, pr.n_bins, factors=(2, 1)) as plan:
    xo = P.pnp_ms2g_solve(plan, pr.stages, torch.from_numpy(b).cuda()[None], den=pr.den, alpha=pr.alpha)
xr, _, _ = O.pnp_ms2g(g, pr.stages, b, den=pr.den, alpha=pr.alpha)
print(worst, np.linalg.norm(xo[0].cpu().numpy() - xr) / np.linalg.norm(xr))
''' % root
    env = dict(os.environ, MS2G_BP_VARIANT="gather")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    op_err, solve_err = map(float, out.stdout.split()[-2:])
    assert op_err <= TOL_OP, op_err
    assert solve_err <= TOL_SOLVE, solve_err


def test_multicast_attach_fails_cleanly_on_one_gpu(P):
    """NEXT-3 NVLS path: on this pool's single-GPU boxes cuMulticastCreate is
    unavailable, so attach_multicast raises MS2G_ERR_CUDA naming the driver
    call, and the plan keeps working (same gradient as before the attempt)."""
    n, V, B = 64, 45, 96
    x = S.phantom(n, 6, 3)
    b = S.random_sinogram((V, B), 4, zero_mean=False)
    with P.plan_geometry(n, V, B, factors=(2, 1)) as plan:
        g0 = host(P.sketched_grad(plan, 2, dev(x)[None], dev(b)[None]))
        try:
            P.attach_multicast(plan, 0, 1)
            attached = True
        except P.MS2GError as e:
            attached = False
            assert e.code == 5 and "NVLS multicast" in str(e), str(e)
        g1 = host(P.sketched_grad(plan, 2, dev(x)[None], dev(b)[None]))
        if attached:      # a box with working multicast: the 1-rank in-switch sum is the identity
            assert rel(g1, g0) <= 1e-6
        else:
            assert np.array_equal(g0, g1)
