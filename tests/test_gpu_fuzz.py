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
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


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
