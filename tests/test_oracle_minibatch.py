"""Pins of Option 4 (NEXT-4; P:72 randomly sampled minibatch, P:98 uniformly
sampled): uniform view minibatches without replacement."""
import numpy as np

import oracle as O


def test_minibatch_determinism_and_shape():
    a = O.minibatch_views(90, 12, 7, 50)
    assert a.shape == (50, 12)
    assert np.array_equal(a, O.minibatch_views(90, 12, 7, 50))
    assert not np.array_equal(a, O.minibatch_views(90, 12, 8, 50))
    for row in a:
        assert np.all(np.diff(row) > 0) and row.min() >= 0 and row.max() < 90   # distinct, ascending
    assert np.array_equal(O.minibatch_views(9, 9, 3, 2), np.tile(np.arange(9), (2, 1)))   # m = V -> all views


def test_minibatch_inclusion_frequency():
    """n_views = 10, batch = 2, 10000 draws: each view's inclusion frequency
    within 3 standard errors of 0.2 (binomial statistics); pairs
    uniform too (45 pairs, each ~1/45)."""
    a = O.minibatch_views(10, 2, 2022, 10000)
    f = np.bincount(a.ravel(), minlength=10) / 10000
    se = np.sqrt(0.2 * 0.8 / 10000)
    assert np.all(np.abs(f - 0.2) < 3 * se)
    pairs = np.bincount(a[:, 0] * 10 + a[:, 1], minlength=100)
    nz = pairs[pairs > 0]
    assert len(nz) == 45
    assert np.all(np.abs(nz / 10000 - 1 / 45) < 4 * np.sqrt((1 / 45) * (44 / 45) / 10000))


def test_option4_full_batch_equals_option1():
    """m = V: every minibatch is the full view set, c = V/m = 1 -> Option 1
    iterates."""
    g = O.Geometry(32, 24, 48)
    b = np.random.default_rng(0).random((24, 48))
    st = [(2, 3, 0), (1, 2, 0)]
    x4, tr4, _ = O.pnp_ms2g(g, st, b, option=4, n_subsets=24, seed=3, den=("gauss", 0.8), alpha=0.5)
    x1, tr1, _ = O.pnp_ms2g(g, st, b, option=1, den=("gauss", 0.8), alpha=0.5)
    assert np.max(np.abs(x4 - x1)) <= 1e-12 * np.max(np.abs(x1))
    assert [t[3] for t in tr4] == list(range(5))
