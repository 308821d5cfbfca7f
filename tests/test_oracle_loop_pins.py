"""Pins of the oracle's Algorithm-1 wiring and of the ellipse chord (CPU only).

Round-2 additions (VERDICT r01 "oracle pins with holes"):
  * the RED-PRO mix x = (1 - alpha) z + alpha D(z) with a NON-identity
    denoiser and alpha < 1, against a step built by hand from independent
    pieces: the dense brute-force A of ``oracle/dense.py`` (per-pixel slab
    clipping, not the Siddon traversal), numpy S/U, and the Gaussian as
    ``scipy.ndimage.correlate`` with the cited golden taps;
  * the momentum wiring y_i = x_i + a_i (x_i - x_{i-1}), a_i = (i-1)/(i+3)
    (P:76): a three-step run whose third iterate depends on a_2 = 0.2,
    so using a_{i+1} or swapping x_i / x_{i-1} fails;
  * the analytic chord of a rotated, off-centre ellipse (north-star pin,
    SURVEY §8(c) "disk / ellipse ... vs analytic chord"): the pixel-centre
    rasterised ellipse's ray sums converge to it as N grows.
The step size eta = 1/L_20 comes back from the oracle; it is pinned on its
own against the SVD of the dense A (test_oracle_pins.test_power_iteration_vs_svd).
"""
import json
import os

import numpy as np
import pytest
from scipy import ndimage

import oracle as O
from oracle import dense as D

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold_gauss():
    with open(os.path.join(GOLD, "gauss3_sigma08.json")) as f:
        j = json.load(f)
    w = np.array([j["w1"], j["w0"], j["w1"]])
    return np.outer(w, w)


def _gauss_scipy(z):
    """3x3 Gaussian, replicate boundary = scipy 'nearest' mode."""
    return ndimage.correlate(z, _gold_gauss(), mode="nearest")


def _S(x, s):
    n = x.shape[-1]
    return x.reshape(n // s, s, n // s, s).mean(axis=(1, 3))


def _U(g, s):
    return np.repeat(np.repeat(g, s, axis=0), s, axis=1)


class Dense:
    """g_s(x) = U_s A_s^T (A_s S_s x - b) from the brute-force dense A_s."""

    def __init__(self, n, V, B):
        self.n = n
        self.A = {s: D.dense_A(n, V, B, factor=s) for s in (1, 2)}

    def grad(self, s, x, b):
        A = self.A[s]
        v = _S(x, s).ravel() if s > 1 else x.ravel()
        G = A.T @ (A @ v - b.ravel())
        nc = self.n // s
        return _U(G.reshape(nc, nc), s) if s > 1 else G.reshape(nc, nc)


N, V, B = 16, 12, 24


@pytest.fixture(scope="module")
def prob():
    rng = np.random.default_rng(2203)
    g = O.Geometry(N, V, B)
    return g, Dense(N, V, B), rng.random((V, B)), rng.random((N, N))


@pytest.mark.parametrize("alpha", [1.0, 0.5, 0.3])
def test_first_step_red_pro_mix_gaussian(prob, alpha):
    """x_1 = (1 - alpha) z_1 + alpha Gauss(z_1), z_1 = x_0 - eta U_2 A_2^T(A_2 S_2 x_0 - b)
    (Eq. 6; a_1 = 0 so y_1 = x_1).  alpha = 1 is the PnP step
    x_1 = D(z_1); alpha = 0.5 / 0.3 fail if alpha and 1 - alpha are
    swapped or if the mix is applied to anything but z."""
    g, Dn, b, x0 = prob
    x1, tr, etas = O.pnp_ms2g(g, [(2, 1, 0)], b, x0=x0, den=("gauss", 0.8), alpha=alpha)
    z1 = x0 - etas[0] * Dn.grad(2, x0, b)
    ref = (1 - alpha) * z1 + alpha * _gauss_scipy(z1)
    assert np.max(np.abs(x1 - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    # the mix is not the identity at this alpha: the pin has teeth
    assert np.max(np.abs(ref - z1)) > 1e-3


def test_momentum_wiring_three_steps(prob):
    """Three full-resolution steps with the identity denoiser, built by hand:
       x1 = y0 - eta g(y0), y1 = x1 + a1 (x1 - x0) = x1      (a1 = 0)
       x2 = y1 - eta g(y1), y2 = x2 + a2 (x2 - x1)           (a2 = 1/5)
       x3 = y2 - eta g(y2)
    (O11).  Also checks x3 is far from the a_{i+1} and
    swapped-difference variants, so those mistakes fail."""
    g, Dn, b, x0 = prob
    x3, tr, etas = O.pnp_ms2g(g, [(1, 3, 0)], b, x0=x0, den=("identity",), alpha=1.0)
    eta = etas[0]
    assert [e[5] for e in tr] == [0.0, 0.2, 1.0 / 3.0]

    def run(a_of, swap=False):
        x_prev, y = x0, x0
        for i in (1, 2, 3):
            x = y - eta * Dn.grad(1, y, b)
            a = a_of(i)
            y = x + a * ((x_prev - x) if swap else (x - x_prev))
            x_prev = x
        return x

    ref = run(lambda i: (i - 1) / (i + 3))
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(x3 - ref)) <= 1e-12 * scale
    wrong_next = run(lambda i: i / (i + 4))
    wrong_swap = run(lambda i: (i - 1) / (i + 3), swap=True)
    assert np.max(np.abs(wrong_next - ref)) > 1e-4 * scale
    assert np.max(np.abs(wrong_swap - ref)) > 1e-4 * scale


def test_two_stage_mix_and_momentum_tv(prob):
    """Stage change inside the loop: 2 steps at s = 2 then 1 step at s = 1,
    TV denoiser with alpha = 0.6.  The continuous counter carries a_2 into
    stage 2's first step (O11); each stage has its own eta (Z5).  The
    TV prox itself is the oracle's (pinned by its closed form, certificate and
    special cases); everything else is rebuilt from the dense A."""
    g, Dn, b, x0 = prob
    lam, K, alpha = 0.05, 10, 0.6
    x, tr, etas = O.pnp_ms2g(g, [(2, 2, 0), (1, 1, 0)], b, x0=x0, den=("tv", lam, K), alpha=alpha)
    x_prev, y = x0, x0
    for i, (s, eta) in enumerate([(2, etas[0]), (2, etas[0]), (1, etas[1])], start=1):
        z = y - eta * Dn.grad(s, y, b)
        xn = (1 - alpha) * z + alpha * O.tv_chambolle(z, lam, K)
        y = xn + (i - 1) / (i + 3) * (xn - x_prev)
        x_prev = xn
    assert np.max(np.abs(x - x_prev)) <= 1e-12 * np.max(np.abs(x_prev))
    assert etas[0] < etas[1]      # L(A_2) ~ 4 L(A) (Z2): the coarse stage takes the shorter step


# ------------------------------------------------------------ ellipse chord
def ellipse_chord(p, q, cx, cy, a, b, phi):
    """Length of the line p->q (infinite line) inside the ellipse
    ((X cos phi + Y sin phi)/a)^2 + ((-X sin phi + Y cos phi)/b)^2 <= 1,
    X = x - cx, Y = y - cy: roots of a quadratic in the line parameter."""
    p = np.asarray(p, float); d = np.asarray(q, float) - p
    c, s = np.cos(phi), np.sin(phi)
    R = np.array([[c, s], [-s, c]])
    P0 = R @ (p - np.array([cx, cy])); Dd = R @ d
    A2 = (Dd[0] / a) ** 2 + (Dd[1] / b) ** 2
    B2 = 2 * (P0[0] * Dd[0] / a ** 2 + P0[1] * Dd[1] / b ** 2)
    C2 = (P0[0] / a) ** 2 + (P0[1] / b) ** 2 - 1
    disc = B2 * B2 - 4 * A2 * C2
    if disc <= 0:
        return 0.0, 0.0
    # chord length and the depth of the line inside (for excluding grazing rays)
    return np.sqrt(disc) / A2 * np.linalg.norm(d), disc / (B2 * B2 + abs(4 * A2 * C2))


def test_ellipse_chord_convergence():
    """Pixel-centre rasterised ellipse (centre (0.12, -0.07), semi-axes 0.55 /
    0.3, angle 0.6 rad): ray sums converge to the analytic chord.  Not exact
    for a pixelised shape (SURVEY [calib]: 6.1e-2 at N=64 -> 7.5e-3 at N=512).
    Gates: the absolute error of every ray is at most 2 h (the staircase
    misplaces each of the two boundary crossings by under one pixel); for
    chords >= 0.4 the relative error is < 0.1 at N=64, < 0.015 at N=512 and
    decreasing; the RMS error decreases with N."""
    cx, cy, a, b, phi = 0.12, -0.07, 0.55, 0.3, 0.6
    rel_max, rms = [], []
    for n in (64, 512):
        g = O.Geometry(n, 10, int(1.5 * n))
        h = 2.0 / n
        c = -1 + (np.arange(n) + 0.5) * h
        X, Y = np.meshgrid(c, c, indexing="xy")
        Xr = (X - cx) * np.cos(phi) + (Y - cy) * np.sin(phi)
        Yr = -(X - cx) * np.sin(phi) + (Y - cy) * np.cos(phi)
        ell = ((Xr / a) ** 2 + (Yr / b) ** 2 <= 1.0).astype(float)
        ab, rl = [], []
        for v in range(10):
            for t in range(0, int(1.5 * n), max(1, n // 16)):
                p, q = O.ray_endpoints(g, v, t)
                ref, _ = ellipse_chord(p, q, cx, cy, a, b, phi)
                if ref <= 0:
                    continue
                e = abs(O.ray_sum(g, 1, ell, v, t) - ref)
                ab.append(e)
                if ref >= 0.4:
                    rl.append(e / ref)
        assert len(rl) > 50 and max(ab) <= 2 * h
        rel_max.append(max(rl))
        rms.append(float(np.sqrt(np.mean(np.square(ab)))))
    assert rel_max[0] < 0.1 and rel_max[1] < 0.015 and rel_max[1] < rel_max[0]
    assert rms[1] < 0.5 * rms[0]


def test_ellipse_chord_helper_against_disk():
    """The chord helper reduces to 2 sqrt(r^2 - d^2) for a = b = r (circle)."""
    p, q = (-3.0, 0.2), (3.0, 0.25)
    d = abs((q[0] - p[0]) * (0 - p[1]) - (q[1] - p[1]) * (0 - p[0])) / np.hypot(q[0] - p[0], q[1] - p[1])
    ch, _ = ellipse_chord(p, q, 0.0, 0.0, 0.5, 0.5, 0.3)
    assert abs(ch - 2 * np.sqrt(0.25 - d * d)) <= 1e-13
