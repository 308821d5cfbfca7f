"""CPU checks of the C ABI: the library loads, exports every symbol the
header declares, fails loudly without a GPU, and its host-only schedule is
bit-exact with the oracle's."""
import ctypes
import os
import re

import pytest

import ms2g_synth as S
import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_2203_07308_b200 import build as B
    B.build()
    import paper_2203_07308_b200 as P
    P.load()
    return P


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ms2g.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ms2g_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(P):
    syms = declared_symbols()
    assert len(syms) >= 16
    lib = ctypes.CDLL(P.lib_path())
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.MS2GError) as e:
        P.plan_geometry(64, 90, 96, factors=(2, 1))
    assert e.value.code == 5


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_schedule_bit_exact_vs_oracle(P, cfg):
    pr = S.PRESETS[cfg]
    seed = S.config_seed(cfg)
    a = P.schedule(None, pr.stages, pr.option, pr.n_subsets, seed)
    b = O.schedule(pr.stages, pr.option, pr.n_subsets, seed)
    assert a == b
    assert len(a) == pr.n_steps


def test_schedule_random_descriptions(P):
    import numpy as np
    rng = np.random.default_rng(0)
    for _ in range(50):
        ns = int(rng.integers(1, 5))
        stages = [(int(rng.integers(1, 5)), int(rng.integers(0, 7)), int(rng.integers(0, 4))) for _ in range(ns)]
        opt = int(rng.integers(1, 6)); nsub = int(rng.integers(1, 12)); seed = int(rng.integers(0, 2**63))
        assert P.schedule(None, stages, opt, nsub, seed) == O.schedule(stages, opt, nsub, seed)


def test_schedule_config_errors(P):
    with pytest.raises(P.MS2GError) as e:
        P.schedule(None, [(2, 3, 0)], option=6)
    assert e.value.code == 2
    with pytest.raises(P.MS2GError):
        P.schedule(None, [(0, 3, 0)])
    with pytest.raises(P.MS2GError):
        P.schedule(None, [(2, 0, 1)], option=2, n_subsets=0)


def test_view_shards_partition(P):
    for V in (90, 720, 1440, 7):
        for nr in (1, 2, 3, 4, 8):
            shards = [P.view_shard(V, r, nr) for r in range(nr)]
            assert shards[0][0] == 0 and shards[-1][1] == V
            assert all(shards[k][1] == shards[k + 1][0] for k in range(nr - 1))
