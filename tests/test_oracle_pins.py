"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each pin is chosen so that a plausible mistake in the oracle (dropped term,
wrong sign or index, transposed operand) fails one of them.  Citations:
P:NN = PAPER.md line, S:NN = SPEC.md line, O1..O13 / Z1..Z23 = readings in
DESIGN.md.
"""
import numpy as np
import pytest

import ms2g_synth as S
import oracle as O
from oracle import dense as D


def geom(n, V, B, **kw):
    return O.Geometry(n, V, B, **kw)


# ------------------------------------------------------------------ helpers
def chord_rect(p, q, x0, x1, y0, y1):
    """Length of the line through p,q inside the rectangle, by intersecting
    the line with each of the four edges (polygon clipping), an algorithm
    different from the oracle's parametric slab clip and Siddon merge."""
    pts = []
    dx, dy = q[0] - p[0], q[1] - p[1]
    for xe in (x0, x1):
        if dx != 0:
            t = (xe - p[0]) / dx
            y = p[1] + t * dy
            if y0 <= y <= y1:
                pts.append((xe, y))
    for ye in (y0, y1):
        if dy != 0:
            t = (ye - p[1]) / dy
            x = p[0] + t * dx
            if x0 <= x <= x1:
                pts.append((x, ye))
    if len(pts) < 2:
        return 0.0
    pts = np.array(pts)
    d = pts[:, None, :] - pts[None, :, :]
    return float(np.sqrt((d ** 2).sum(-1)).max())


def dist_point_line(c, p, q):
    d = np.asarray(q) - np.asarray(p)
    w = np.asarray(c) - np.asarray(p)
    return abs(d[0] * w[1] - d[1] * w[0]) / np.hypot(*d)


# ------------------------------------------------ O1/O2: known answers (C1)
def test_known_answer_rays_c1_geometry():
    """SURVEY §8(c) known-answer table, C1 geometry (N=64, V=90, B=96):
    x = 1 gives the chord of the FOV square; closed form 2 sqrt(1 + 2^-16) for
    the two central rays of view 0, 0 for the outermost bins (they miss)."""
    g = geom(64, 90, 96)
    one = np.ones((64, 64))
    exact = 2.0 * np.sqrt(1.0 + 2.0 ** -16)
    assert abs(O.ray_sum(g, 1, one, 0, 48) - exact) < 1e-13
    assert abs(O.ray_sum(g, 1, one, 0, 47) - exact) < 1e-13
    assert O.ray_sum(g, 1, one, 0, 0) == 0.0
    assert O.ray_sum(g, 1, one, 0, 95) == 0.0
    for (v, t), val in {(11, 30): 1.774487067086905, (45, 50): 2.000381433353712,
                        (22, 60): 2.017619550983414}.items():
        assert abs(O.ray_sum(g, 1, one, v, t) - val) < 1e-12


def test_known_answer_row_structure():
    """Ray (0,48) stays in row 32 (y in [0.0117, 0.0195]): exactly 64 segments
    of h sqrt(1+2^-16); on the 32^2 grid 32 segments of 2h sqrt(1+2^-16)."""
    g = geom(64, 90, 96)
    pix, ln = O.ray_segments(g, 1, 0, 48)
    assert len(pix) == 64
    assert np.all(pix // 64 == 32)
    assert sorted(pix % 64) == list(range(64))
    assert np.allclose(ln, (1 / 32) * np.sqrt(1 + 2.0 ** -16), rtol=0, atol=1e-15)
    pix, ln = O.ray_segments(g, 2, 0, 48)
    assert len(pix) == 32 and np.all(pix // 32 == 16)
    assert np.allclose(ln, (2 / 32) * np.sqrt(1 + 2.0 ** -16), rtol=0, atol=1e-15)


@pytest.mark.parametrize("n,V,B,arc", [(32, 36, 48, 2 * np.pi), (48, 20, 72, np.pi), (512, 7, 768, 2 * np.pi)])
def test_uniform_square_chord(n, V, B, arc):
    """x = 1 on the FOV: every ray sum is the chord of the square [-1,1]^2."""
    g = geom(n, V, B, arc=arc)
    one = np.ones((n, n))
    rng = np.random.default_rng(1)
    for _ in range(40):
        v, t = int(rng.integers(V)), int(rng.integers(B))
        p, q = O.ray_endpoints(g, v, t)
        ref = chord_rect(p, q, -1, 1, -1, 1)
        got = O.ray_sum(g, 1, one, v, t)
        assert abs(got - ref) <= 1e-13 * max(1.0, ref)


def test_pixel_aligned_rectangle_chord():
    """A pixel-aligned rectangle indicator projects to the rectangle chord."""
    n = 40
    g = geom(n, 24, 60)
    h = 2.0 / n
    i0, i1, j0, j1 = 7, 23, 11, 30           # rows [i0,i1), cols [j0,j1)
    x = np.zeros((n, n)); x[i0:i1, j0:j1] = 1.0
    for v in range(0, 24, 3):
        for t in range(0, 60, 7):
            p, q = O.ray_endpoints(g, v, t)
            ref = chord_rect(p, q, -1 + j0 * h, -1 + j1 * h, -1 + i0 * h, -1 + i1 * h)
            assert abs(O.ray_sum(g, 1, x, v, t) - ref) <= 1e-13 * max(1.0, ref)


def test_disk_ellipse_chord_convergence():
    """Pixel-centre rasterised disk r=0.5: ray sums converge to 2 sqrt(r^2-d^2)
    (north-star pin).  Not exact for pixelised shapes: gate 0.1 at N=64,
    0.015 at N=512 and decreasing."""
    errs = []
    for n in (64, 512):
        g = geom(n, 8, int(1.5 * n))
        c = -1 + (np.arange(n) + 0.5) * 2 / n
        X, Y = np.meshgrid(c, c, indexing="xy")
        disk = ((X ** 2 + Y ** 2) <= 0.25).astype(float)
        e = []
        for v in range(8):
            for t in range(int(0.5 * n), int(n), max(1, n // 16)):
                p, q = O.ray_endpoints(g, v, t)
                d = dist_point_line((0, 0), p, q)
                if d > 0.4:
                    continue
                ref = 2 * np.sqrt(0.25 - d * d)
                e.append(abs(O.ray_sum(g, 1, disk, v, t) - ref) / ref)
        errs.append(max(e))
    assert errs[0] < 0.1 and errs[1] < 0.015 and errs[1] < errs[0]


# ------------------------------------------------- O2/O3 vs brute force
@pytest.mark.parametrize("factor", [1, 2])
def test_dense_bruteforce_16(factor):
    """Dense A at 16x16 (C1 geometry ratios, independent per-pixel slab
    clipping) equals the oracle's Siddon rows entrywise <= 1e-13."""
    n, V, B = 16, 12, 24
    g = geom(n, V, B)
    A = D.dense_A(n, V, B, factor=factor)
    nc = n // factor
    for v in range(V):
        for t in range(B):
            row = np.zeros(nc * nc)
            pix, ln = O.ray_segments(g, factor, v, t)
            np.add.at(row, pix, ln)
            assert np.max(np.abs(row - A[v * B + t])) <= 1e-13
    x = np.random.default_rng(0).random((nc, nc))
    assert np.allclose(O.forward(g, factor, x).ravel(), A @ x.ravel(), rtol=0, atol=1e-12)
    r = np.random.default_rng(1).standard_normal((V, B))
    assert np.allclose(O.backward(g, factor, r).ravel(), A.T @ r.ravel(), rtol=0, atol=1e-12)


def test_single_ray_backprojection():
    """Single-ray sinogram -> image = that ray's intersection lengths."""
    n, V, B = 24, 10, 36
    g = geom(n, V, B)
    A = D.dense_A(n, V, B)
    for (v, t) in [(0, 18), (3, 5), (7, 30)]:
        r = np.zeros((V, B)); r[v, t] = 1.0
        img = O.backward(g, 1, r)
        assert np.max(np.abs(img.ravel() - A[v * B + t])) <= 1e-13


def test_backward_pixel_definition_matches_traversal():
    """Two algorithms for A^T (per-pixel slab clip vs Siddon scatter) agree."""
    n, V, B = 32, 18, 48
    g = geom(n, V, B)
    r = np.random.default_rng(3).standard_normal((V, B))
    img = O.backward(g, 1, r)
    for (i, j) in [(0, 0), (5, 17), (16, 16), (31, 2), (20, 31)]:
        assert abs(O.backward_pixel(g, 1, r, i, j) - img[i, j]) <= 1e-12 * max(1, np.abs(img).max())
    views = np.array([1, 4, 9, 15])
    rs = r[views]
    img = O.backward(g, 2, rs, views=views)
    assert abs(O.backward_pixel(g, 2, rs, 3, 7, views=views) - img[3, 7]) <= 1e-12


@pytest.mark.parametrize("n,V,B,factor", [(32, 30, 48, 1), (32, 30, 48, 2), (64, 16, 96, 4), (40, 9, 61, 1)])
def test_adjoint_identity_fp64(n, V, B, factor):
    """<A x, y> = <x, A^T y> to 1e-10 relative (north star), 20 random pairs."""
    g = geom(n, V, B)
    rng = np.random.default_rng(7)
    nc = n // factor
    for _ in range(20):
        x = rng.standard_normal((nc, nc)); y = rng.standard_normal((V, B))
        lhs = float(np.sum(O.forward(g, factor, x) * y))
        rhs = float(np.sum(x * O.backward(g, factor, y)))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1e-30) + 1e-12


def test_linearity_and_zero():
    """project(a x + c y) = a project(x) + c project(y); 0 -> 0."""
    g = geom(32, 12, 48)
    rng = np.random.default_rng(2)
    x, y = rng.random((32, 32)), rng.random((32, 32))
    a, c = 1.7, -0.3
    lhs = O.forward(g, 1, a * x + c * y)
    rhs = a * O.forward(g, 1, x) + c * O.forward(g, 1, y)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))
    assert np.all(O.forward(g, 1, np.zeros((32, 32))) == 0)
    assert np.all(O.backward(g, 1, np.zeros((12, 48))) == 0)


def test_coarse_operator_equals_fine_times_upsampler():
    """A_s = A U_s exactly (O5): coarse grid lines are fine grid lines and
    Siddon lengths are additive.  <= 1e-13 relative."""
    g = geom(48, 15, 72)
    rng = np.random.default_rng(4)
    for s in (2, 4, 3):
        v = rng.random((48 // s, 48 // s))
        a = O.forward(g, s, v)
        b = O.forward(g, 1, O.sketch_up(v, s))
        assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))


# ------------------------------------------------------------- O4 / O5
@pytest.mark.parametrize("s", [1, 2, 4])
def test_sketch_mass_and_identities(s):
    """Mass: sum(S_s x)(sh)^2 = sum(x) h^2; sum(U_s g) h^2 = sum(g)(sh)^2;
    S_s U_s = I; s^2 <S_s x, g> = <x, U_s g>; constants preserved."""
    n = 32
    rng = np.random.default_rng(s)
    x = rng.random((n, n)); gc = rng.random((n // s, n // s))
    h = 2.0 / n
    v = O.sketch_down(x, s)
    assert abs(v.sum() * (s * h) ** 2 - x.sum() * h ** 2) <= 1e-14 * x.sum() * h ** 2
    u = O.sketch_up(gc, s)
    assert abs(u.sum() * h ** 2 - gc.sum() * (s * h) ** 2) <= 1e-14 * u.sum() * h ** 2
    assert np.array_equal(O.sketch_down(u, s), gc) or np.max(np.abs(O.sketch_down(u, s) - gc)) <= 1e-15
    lhs = s * s * np.sum(v * gc); rhs = np.sum(x * u)
    assert abs(lhs - rhs) <= 1e-13 * abs(rhs)
    c = np.full((n, n), 0.37)
    assert np.allclose(O.sketch_down(c, s), 0.37, rtol=0, atol=1e-15)
    assert np.all(O.sketch_up(np.full((n // s, n // s), 0.37), s) == 0.37)
    # explicit value of one block
    assert abs(v[1, 0] - x[s:2 * s, 0:s].mean()) <= 1e-15


# ------------------------------------------------------------- O6 / O7
@pytest.mark.parametrize("s", [1, 2, 4])
def test_sketched_gradient_finite_difference(s):
    """g_s = s^2 grad_x 1/2||A_s S_s x - b||^2 ; central differences on the
    quadratic are exact up to rounding."""
    n, V, B = 32, 16, 48
    g = geom(n, V, B)
    rng = np.random.default_rng(10 + s)
    x = rng.random((n, n)); b = rng.random((V, B)) * 2
    gr = O.sketched_grad(g, s, x, b)

    def f(z):
        r = O.forward(g, s, O.sketch_down(z, s)) - b
        return 0.5 * np.sum(r * r)

    for _ in range(5):
        d = rng.standard_normal((n, n))
        eps = 1e-3
        fd = (f(x + eps * d) - f(x - eps * d)) / (2 * eps)
        assert abs(s * s * fd - np.sum(gr * d)) <= 1e-7 * abs(np.sum(gr * d))


def test_gradient_special_cases():
    """b = A_s S_s x => g = 0; s = 1 => A^T(Ax - b) via dense A."""
    n, V, B = 16, 12, 24
    g = geom(n, V, B)
    rng = np.random.default_rng(5)
    x = rng.random((n, n))
    b = O.forward(g, 2, O.sketch_down(x, 2))
    assert np.max(np.abs(O.sketched_grad(g, 2, x, b))) <= 1e-12
    A = D.dense_A(n, V, B)
    b = rng.random((V, B))
    ref = A.T @ (A @ x.ravel() - b.ravel())
    assert np.max(np.abs(O.sketched_grad(g, 1, x, b).ravel() - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("s", [1, 2])
def test_subset_partition_identity(s):
    """sum_k (|M_k|/V) g^{M_k} = g over the 8 interleaved subsets; M = all
    gives Option 1 (Z7, Z8)."""
    n, V, B = 32, 40, 48
    g = geom(n, V, B)
    rng = np.random.default_rng(6)
    x = rng.random((n, n)); b = rng.random((V, B))
    full = O.sketched_grad(g, s, x, b)
    acc = np.zeros_like(full)
    for k in range(8):
        m = O.subset_views(V, 8, k)
        assert np.array_equal(m, np.arange(k, V, 8))
        acc += (len(m) / V) * O.sketched_grad(g, s, x, b, views=m)
    assert np.max(np.abs(acc - full)) <= 1e-12 * np.max(np.abs(full))
    allv = np.arange(V)
    assert np.max(np.abs(O.sketched_grad(g, s, x, b, views=allv) - full)) <= 1e-12 * np.max(np.abs(full))


def test_exhaustive_pair_unbiasedness():
    """Average over all C(4,2) view pairs of the V/|M|-scaled gradient equals
    the full gradient to 1e-10 (acceptance 5)."""
    import itertools
    n, V, B = 16, 4, 24
    g = geom(n, V, B)
    rng = np.random.default_rng(8)
    x = rng.random((n, n)); b = rng.random((V, B))
    full = O.sketched_grad(g, 2, x, b)
    pairs = list(itertools.combinations(range(V), 2))
    acc = sum(O.sketched_grad(g, 2, x, b, views=np.array(p)) for p in pairs) / len(pairs)
    assert np.max(np.abs(acc - full)) <= 1e-10 * np.max(np.abs(full))


# ------------------------------------------------------------------ O8
@pytest.mark.parametrize("factor", [1, 2])
def test_power_iteration_vs_svd(factor):
    """L_20 equals sigma_max(A_s)^2 from numpy SVD of the dense A (16x16)."""
    n, V, B = 16, 12, 24
    g = geom(n, V, B)
    A = D.dense_A(n, V, B, factor=factor)
    smax = np.linalg.svd(A, compute_uv=False)[0]
    L = O.power_iteration(g, factor, 20)
    assert abs(L - smax ** 2) <= 1e-10 * smax ** 2


def test_power_iteration_single_ray_and_scaling():
    """One view, one bin: L = ||row||^2; L_s / L in [0.9 s^2, s^2]."""
    g = geom(32, 1, 1)
    pix, ln = O.ray_segments(g, 1, 0, 0)
    L = O.power_iteration(g, 1, 5)
    assert abs(L - np.sum(ln ** 2)) <= 1e-12 * L
    g = geom(32, 24, 48)
    L1 = O.power_iteration(g, 1, 20); L2 = O.power_iteration(g, 2, 20)
    assert 0.9 * 4 <= L2 / L1 <= 4.0 + 1e-9


# ------------------------------------------------------------------ O9
def test_gaussian_weights_and_delta_response():
    """3x3 sigma=0.8: centre 0.2724959735, edge 0.1247577476, corner
    0.0571182590 (outer product of [w1, w0, w1]); weights sum to 1;
    constants preserved; replicate boundary keeps mass at an edge delta."""
    w = O.gauss3_weights(0.8)
    assert abs(w[1] - 0.52201147) < 1e-8 and abs(w[0] - 0.23899427) < 1e-8
    assert abs(w.sum() - 1.0) <= 1e-15
    z = np.zeros((7, 7)); z[3, 3] = 1.0
    out = O.gauss3(z)
    assert abs(out[3, 3] - 0.2724959735) < 1e-10
    assert abs(out[3, 4] - 0.1247577476) < 1e-10 and abs(out[2, 3] - 0.1247577476) < 1e-10
    assert abs(out[2, 2] - 0.0571182590) < 1e-10 and abs(out[4, 4] - 0.0571182590) < 1e-10
    assert abs(out.sum() - 1.0) < 1e-14
    assert np.allclose(O.gauss3(np.full((9, 9), 0.3)), 0.3, rtol=0, atol=1e-15)
    z = np.zeros((5, 5)); z[0, 0] = 1.0
    out = O.gauss3(z)      # replicate: corner keeps (w0+w1)^2
    assert abs(out[0, 0] - (w[1] + w[0]) ** 2) < 1e-15


def test_tv_special_cases():
    """lambda = 0 -> identity; constant -> constant; adjointness of grad/div;
    dual feasibility |p| <= 1; non-expansive."""
    rng = np.random.default_rng(9)
    f = rng.random((12, 12))
    assert np.array_equal(O.tv_chambolle(f, 0.0, 10), f)
    c = np.full((10, 10), 0.42)
    assert np.allclose(O.tv_chambolle(c, 0.1, 50), 0.42, rtol=0, atol=1e-12)
    u = rng.standard_normal((11, 11)); p = rng.standard_normal((2, 11, 11))
    gx, gy = O.grad(u)
    lhs = np.sum(gx * p[0] + gy * p[1]); rhs = -np.sum(u * O.div(p[0], p[1]))
    assert abs(lhs - rhs) <= 1e-14 * max(1, abs(lhs))
    uu, pp = O.tv_chambolle(f, 0.05, 30, return_dual=True)
    assert np.max(np.hypot(pp[0], pp[1])) <= 1 + 1e-12
    g2 = f + 0.1 * rng.standard_normal(f.shape)
    d1 = np.linalg.norm(O.tv_chambolle(f, 0.05, 200) - O.tv_chambolle(g2, 0.05, 200))
    assert d1 <= np.linalg.norm(f - g2) + 1e-8


def _tv(u):
    gx, gy = O.grad(u)
    return np.sum(np.hypot(gx, gy))


def test_tv_duality_gap_certificate():
    """P(u_K) - D(p_K) >= 0 and decreases to ~0: P(u) = 1/2||u-f||^2 + lam
    TV(u), D(p) = 1/2||f||^2 - 1/2||f - lam div p||^2 (solver-independent)."""
    f = S.phantom(32, 6, 11).astype(np.float64)
    lam = 0.02
    gaps = []
    for K in (10, 100, 1000):
        u, p = O.tv_chambolle(f, lam, K, return_dual=True)
        P = 0.5 * np.sum((u - f) ** 2) + lam * _tv(u)
        Dd = 0.5 * np.sum(f ** 2) - 0.5 * np.sum((f - lam * O.div(p[0], p[1])) ** 2)
        gaps.append(P - Dd)
    assert all(gp >= -1e-12 for gp in gaps)
    assert gaps[2] < gaps[1] < gaps[0]
    assert gaps[2] < 1e-4 * (0.5 * np.sum(f ** 2))


def test_tv_two_by_two_closed_form():
    """f = [[1,0],[0,0]], lam = 0.1: converged prox is
    [[1 - lam sqrt2, lam sqrt2/3], [lam sqrt2/3, lam sqrt2/3]] (the
    symmetric ansatz with a subgradient check, valid for lam < 3/(4 sqrt2))."""
    lam = 0.1
    u = O.tv_chambolle(np.array([[1.0, 0.0], [0.0, 0.0]]), lam, 5000)
    a, b = 1 - lam * np.sqrt(2), lam * np.sqrt(2) / 3
    assert np.max(np.abs(u - np.array([[a, b], [b, b]]))) < 1e-7


def test_tv_one_iteration_closed_form():
    """K = 1 by hand (Z18; tau = 1/8, t = tau/lam): from p^0 = 0,
    p^1 = -t grad f / (1 + t |grad f|), u = f - lam div p^1.  For the 3x3
    unit impulse f (forward differences, zero last row / column) grad f is
    (1, 0) at (1,0), (0, 1) at (0,1), (-1, -1) at (1,1), so
      u(1,1) = 1 - lam (2t/(1+t) + 2t/(1+sqrt2 t)),
      u(1,0) = u(0,1) = lam t/(1+t),  u(1,2) = u(2,1) = lam t/(1+sqrt2 t),
    corners 0 (the left/top neighbours receive the 1-norm-1 fluxes, the
    right/bottom ones the diagonal flux)."""
    lam = 0.1
    t = 0.125 / lam
    f = np.zeros((3, 3)); f[1, 1] = 1.0
    u = O.tv_chambolle(f, lam, 1)
    a, d = t / (1 + t), t / (1 + np.sqrt(2) * t)
    want = np.array([[0.0, lam * a, 0.0], [lam * a, 1 - lam * (2 * a + 2 * d), lam * d], [0.0, lam * d, 0.0]])
    assert np.max(np.abs(u - want)) < 1e-15


def test_tv_finite_k_invariants():
    """Properties of Chambolle's iteration at every K (what K = 10 is
    pinned by): the mean is preserved (div has zero sum under the zero-flux
    boundary), translation and scale covariance u(f + c) = u(f) + c and
    u(c f; c lam) = c u(f; lam), transposition symmetry, |u - f| <= 4 lam
    (dual feasibility |p| <= 1), and the dual energy ||f - lam div p^n||^2
    non-increasing in n for tau <= 1/8 (Chambolle 2004, Thm 3.1)."""
    rng = np.random.default_rng(3)
    f = S.phantom(24, 5, 7).astype(np.float64) + 0.05 * rng.standard_normal((24, 24))
    lam = 0.05
    for K in (1, 2, 3, 10):
        u = O.tv_chambolle(f, lam, K)
        assert abs(u.sum() - f.sum()) <= 1e-12 * np.abs(f).sum()
        assert np.max(np.abs(O.tv_chambolle(f + 0.3, lam, K) - (u + 0.3))) < 1e-14
        assert np.max(np.abs(O.tv_chambolle(2.5 * f, 2.5 * lam, K) - 2.5 * u)) < 1e-14
        assert np.array_equal(O.tv_chambolle(np.ascontiguousarray(f.T), lam, K), u.T)
        assert np.max(np.abs(u - f)) <= 4 * lam * (1 + 1e-12)
    E = []
    for K in range(0, 25):
        _, p = O.tv_chambolle(f, lam, K, return_dual=True)
        E.append(np.sum((f - lam * O.div(p[0], p[1])) ** 2))
    assert all(E[k + 1] <= E[k] * (1 + 1e-14) for k in range(len(E) - 1)) and E[-1] < E[0]


# ------------------------------------------------------------- O11 / O13
def test_momentum_values():
    """a_i = (i-1)/(i+3): a1 = 0, a2 = 0.2, a5 = 0.5, a9 = 2/3."""
    assert O.momentum(1) == 0.0 and O.momentum(2) == 0.2 and O.momentum(5) == 0.5
    assert abs(O.momentum(9) - 2 / 3) < 1e-16
    assert all(O.momentum(i) < 1 for i in range(1, 10000, 97))


def test_splitmix64_known_answers():
    """SplitMix64 (seed 0) published first outputs."""
    assert O.splitmix64_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_schedule_known_answers_and_counts():
    """C3 (seed 220310308): subset order per epoch and [3,3,2] epochs; step
    counts C1..C5 = 20, 50, 64, 50, 40; continuous global i."""
    assert S.split_epochs(8, 3) == [3, 3, 2]
    pr = S.PRESETS[3]
    sch = O.schedule(pr.stages, 2, 8, S.config_seed(3, 0))
    subs = [e[3] for e in sch]
    expect = [[3, 5, 1, 2, 0, 4, 7, 6], [3, 4, 6, 0, 5, 7, 1, 2], [0, 7, 4, 1, 2, 3, 6, 5],
              [1, 2, 7, 0, 6, 3, 5, 4], [0, 6, 4, 5, 1, 7, 3, 2], [3, 7, 0, 5, 6, 2, 1, 4],
              [6, 3, 2, 1, 5, 7, 4, 0], [1, 2, 6, 7, 4, 3, 0, 5]]
    assert subs == sum(expect, [])
    assert [e[0] for e in sch] == list(range(1, 65))
    assert [e[2] for e in sch] == [4] * 24 + [2] * 24 + [1] * 16
    for cfg, steps in {1: 20, 2: 50, 3: 64, 4: 50, 5: 40}.items():
        p = S.PRESETS[cfg]
        assert len(O.schedule(p.stages, p.option, p.n_subsets, S.config_seed(cfg))) == steps == p.n_steps
    # same seed -> same subsets; different seed -> different order
    assert O.schedule(pr.stages, 2, 8, 5) == O.schedule(pr.stages, 2, 8, 5)
    assert O.schedule(pr.stages, 2, 8, 5) != O.schedule(pr.stages, 2, 8, 6)


def test_loop_reaches_least_squares_optimum():
    """Single stage s=1, identity denoiser, alpha=1, eta=1/L: after 200 steps
    the data fidelity is within 1e-3 relative of the least-squares optimum
    found by conjugate gradients on the normal equations.
    300 steps on a 32^2 / 90-view problem (condition number ~190)."""
    n, V, B = 32, 90, 48
    g = geom(n, V, B)
    A = D.dense_A(n, V, B)
    xt = S.phantom(n, 5, 3).astype(np.float64)
    b = A @ xt.ravel()
    b = b + 0.01 * b.max() * np.random.default_rng(0).standard_normal(b.shape)
    # CG on A^T A x = A^T b, tol 1e-10
    M = A.T @ A; rhs = A.T @ b
    x = np.zeros(n * n); r = rhs - M @ x; p = r.copy(); rs = r @ r
    for _ in range(5000):
        Mp = M @ p; al = rs / (p @ Mp); x += al * p; r -= al * Mp
        rn = r @ r
        if np.sqrt(rn) < 1e-10 * np.linalg.norm(rhs):
            break
        p = r + (rn / rs) * p; rs = rn
    fopt = 0.5 * np.sum((A @ x - b) ** 2)
    xo, trace, etas = O.pnp_ms2g(g, [(1, 300, 0)], b.reshape(V, B), den=("identity",), alpha=1.0)
    f = 0.5 * np.sum((A @ xo.ravel() - b) ** 2)
    assert fopt <= f <= fopt * (1 + 1e-3)
    assert abs(etas[0] - 1 / np.linalg.svd(A, compute_uv=False)[0] ** 2) <= 1e-9 * etas[0]
    assert [e[0] for e in trace] == list(range(1, 301))


def test_loop_first_step_has_no_momentum():
    """a_1 = 0: the first iterate is the plain PnP step x1 = mix(z1) with
    z1 = x0 - eta U G (Eq. 6); identity denoiser, s = 2."""
    n, V, B = 16, 12, 24
    g = geom(n, V, B)
    rng = np.random.default_rng(12)
    b = rng.random((V, B)); x0 = rng.random((n, n))
    x1, tr, etas = O.pnp_ms2g(g, [(2, 1, 0)], b, x0=x0, den=("identity",), alpha=1.0)
    ref = x0 - etas[0] * O.sketched_grad(g, 2, x0, b)
    assert np.max(np.abs(x1 - ref)) <= 1e-13


def test_divergence_is_reported():
    """A NaN planted in b makes the iterate non-finite -> DivergedError naming
    the iteration."""
    n, V, B = 16, 8, 24
    g = geom(n, V, B)
    b = np.ones((V, B)); b[2, 3] = np.nan
    with pytest.raises(O.DivergedError, match="iteration 1"):
        O.pnp_ms2g(g, [(1, 3, 0)], b)


def test_poisson_statistics():
    """x = 0, I0 = 1e6: mean of -ln(c/I0) within 3 standard errors of 0
    (delta-method variance 1/I0 per bin, acceptance 9)."""
    p = np.zeros((90, 228))
    b = S.poisson_data(p, 1e6, 123).astype(np.float64)
    se = np.sqrt(1e-6 / b.size)
    assert abs(b.mean()) < 3 * se
    assert np.all(np.isfinite(S.poisson_data(np.full((4, 4), 50.0), 1e3, 1)))


def test_phantom_determinism():
    a = S.phantom(64, 10, S.config_seed(1)); b = S.phantom(64, 10, S.config_seed(1))
    assert np.array_equal(a, b) and a.dtype == np.float32 and a.max() > 0
