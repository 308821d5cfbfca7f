"""Pins of the oracle's bicubic S/U (NEXT-1: the paper's "MATLAB imresize
with bicubic interpolation").  Keys kernel values,
constant preservation, linear-ramp reproduction away from the
boundary, factor-1 identity, linearity."""
import numpy as np
import pytest

import oracle as O


def test_keys_kernel_values():
    """Keys cubic convolution a = -0.5 evaluated by its piecewise formula:
    W(0)=1, W(0.5)=0.5625, W(1)=0, W(1.5)=-0.0625, W(2)=0, symmetric."""
    assert O.keys(0.0) == 1.0
    assert abs(O.keys(0.5) - 0.5625) < 1e-15
    assert O.keys(1.0) == 0.0 and O.keys(2.0) == 0.0 and O.keys(2.5) == 0.0
    assert abs(O.keys(1.5) + 0.0625) < 1e-15
    assert O.keys(-0.3) == O.keys(0.3)
    # interpolation partition of unity at any phase: sum_k W(u - k) = 1
    for u in np.linspace(0, 1, 7):
        assert abs(sum(O.keys(u - k) for k in range(-2, 4)) - 1.0) < 1e-14


@pytest.mark.parametrize("s", [2, 4])
def test_bicubic_constants_and_identity(s):
    c = np.full((32, 32), -0.37)
    assert np.max(np.abs(O.bicubic_down(c, s) + 0.37)) < 1e-14
    assert np.max(np.abs(O.bicubic_up(c[: 32 // s, : 32 // s], s) + 0.37)) < 1e-14
    x = np.random.default_rng(s).random((16, 16))
    assert np.array_equal(O.bicubic_down(x, 1), x) and np.array_equal(O.bicubic_up(x, 1), x)


@pytest.mark.parametrize("s", [2, 4])
def test_bicubic_ramp_reproduction(s):
    """A linear ramp is reproduced at the output sample positions away from
    the (clamped) boundary: up u = (i+0.5)/s - 0.5, down u = (i+0.5)s - 0.5."""
    nc = 16
    gi, gj = np.meshgrid(np.arange(nc, dtype=float), np.arange(nc, dtype=float), indexing="ij")
    ramp = 0.3 * gi - 0.7 * gj + 2.0
    up = O.bicubic_up(ramp, s)
    f = (np.arange(nc * s) + 0.5) / s - 0.5
    FI, FJ = np.meshgrid(f, f, indexing="ij")
    ref = 0.3 * FI - 0.7 * FJ + 2.0
    m = 2 * s + 2
    assert np.max(np.abs(up[m:-m, m:-m] - ref[m:-m, m:-m])) < 1e-12
    n = 64
    gi, gj = np.meshgrid(np.arange(n, dtype=float), np.arange(n, dtype=float), indexing="ij")
    down = O.bicubic_down(0.3 * gi - 0.7 * gj + 2.0, s)
    f = (np.arange(n // s) + 0.5) * s - 0.5
    FI, FJ = np.meshgrid(f, f, indexing="ij")
    ref = 0.3 * FI - 0.7 * FJ + 2.0
    m = 3
    assert np.max(np.abs(down[m:-m, m:-m] - ref[m:-m, m:-m])) < 1e-12


def test_bicubic_linearity_and_gradient_special_cases():
    rng = np.random.default_rng(3)
    x, y = rng.random((32, 32)), rng.random((32, 32))
    for f in (lambda z: O.bicubic_down(z, 2), lambda z: O.bicubic_up(z[:16, :16], 2)):
        assert np.max(np.abs(f(2 * x - 3 * y) - (2 * f(x) - 3 * f(y)))) < 1e-13
    g = O.Geometry(32, 12, 48)
    b = O.forward(g, 2, O.bicubic_down(x, 2))
    assert np.max(np.abs(O.sketched_grad(g, 2, x, b, resampler=1))) < 1e-12   # zero residual
    bb = rng.random((12, 48))
    assert np.array_equal(O.sketched_grad(g, 1, x, bb, resampler=1), O.sketched_grad(g, 1, x, bb))
