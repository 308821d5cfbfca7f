"""Pins of the oracle's SVRG Option (NEXT-4; "stochastic variance-reduced
gradient estimator ... SVRG").  With a single subset (M = all views) the
SVRG step equals the Option-1 step; over one epoch the estimator averaged
over the subset partition equals the full gradient at the same point
(unbiasedness, exact for the quadratic fidelity)."""
import numpy as np

import oracle as O


def test_svrg_single_subset_equals_option1():
    n, V, B = 32, 24, 48
    g = O.Geometry(n, V, B)
    b = np.random.default_rng(0).random((V, B))
    st = [(2, 0, 2), (1, 0, 1)]
    x3, tr3, e3 = O.pnp_ms2g(g, st, b, option=3, n_subsets=1, seed=1, den=("gauss", 0.8), alpha=0.5)
    x1, tr1, e1 = O.pnp_ms2g(g, [(2, 2, 0), (1, 1, 0)], b, option=1, den=("gauss", 0.8), alpha=0.5)
    assert np.max(np.abs(x3 - x1)) <= 1e-12 * np.max(np.abs(x1))
    assert [t[0] for t in tr3] == [t[0] for t in tr1]


def test_svrg_estimator_unbiased_over_partition():
    """(1/K) sum_k [c U A_Mk^T A_Mk S (y - xs)] + mu = g(y) for K equal-size
    interleaved subsets (c = V/|M_k| = K): the variance-reduced estimator is
    unbiased for the full sketched gradient."""
    n, V, B, K = 32, 24, 48, 4
    g = O.Geometry(n, V, B)
    rng = np.random.default_rng(1)
    b = rng.random((V, B)); y = rng.random((n, n)); xs = rng.random((n, n))
    mu = O.sketched_grad(g, 2, xs, b)
    zero = np.zeros((V, B))
    est = sum(O.sketched_grad(g, 2, y - xs, zero, views=O.subset_views(V, K, k)) for k in range(K)) / K + mu
    full = O.sketched_grad(g, 2, y, b)
    assert np.max(np.abs(est - full)) <= 1e-12 * np.max(np.abs(full))


def test_saga_single_subset_equals_option1():
    """SAGA (Option 5) with one subset: new - phi + mean(phi) = new, the
    full gradient -> Option-1 iterates."""
    n, V, B = 32, 24, 48
    g = O.Geometry(n, V, B)
    b = np.random.default_rng(0).random((V, B))
    x5, _, _ = O.pnp_ms2g(g, [(2, 0, 2), (1, 0, 1)], b, option=5, n_subsets=1, seed=1, den=("gauss", 0.8),
                          alpha=0.5)
    x1, _, _ = O.pnp_ms2g(g, [(2, 2, 0), (1, 1, 0)], b, option=1, den=("gauss", 0.8), alpha=0.5)
    assert np.max(np.abs(x5 - x1)) <= 1e-12 * np.max(np.abs(x1))

