"""The fp64 oracle against tests/golden/ (values fixed by definition: closed
forms of the paper's operators on the configs' geometry, the SplitMix64 test
vector, O13 schedule orders; each fixture states its source)."""
import json
import os

import numpy as np

import ms2g_synth as S
import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_golden_c1_rays():
    d = load("c1_known_rays.json")
    g = O.Geometry(64, 90, 96)
    one = np.ones((64, 64))
    for r in d["ray_sums_x_one"]:
        assert abs(O.ray_sum(g, 1, one, r["view"], r["bin"]) - r["value"]) <= d["tolerance"], r
    rs = d["row_structure"]
    for factor, key in ((1, "fine"), (2, "coarse_s2")):
        e = rs[key]
        nc = 64 // factor
        pix, ln = O.ray_segments(g, factor, rs["view"], rs["bin"])
        assert len(pix) == e["segments"] and np.all(pix // nc == e["row"])
        assert np.max(np.abs(ln - e["length"])) <= 1e-15


def test_golden_gauss3():
    d = load("gauss3_sigma08.json")
    w = O.gauss3_weights(d["sigma"])
    assert abs(w[1] - d["w0"]) <= d["tolerance"] and abs(w[0] - d["w1"]) <= d["tolerance"]
    z = np.zeros((7, 7)); z[3, 3] = 1.0
    out = O.gauss3(z, d["sigma"])
    r = d["delta_response"]
    assert abs(out[3, 3] - r["centre"]) <= d["tolerance"]
    assert abs(out[3, 4] - r["edge"]) <= d["tolerance"] and abs(out[2, 3] - r["edge"]) <= d["tolerance"]
    assert abs(out[2, 2] - r["corner"]) <= d["tolerance"]


def test_golden_tv_prox_2x2():
    d = load("tv_prox_2x2.json")
    u = O.tv_chambolle(np.array(d["f"]), d["lambda"], d["iterations"])
    assert np.max(np.abs(u - np.array(d["u"]))) <= d["tolerance"]


def test_golden_splitmix64():
    d = load("splitmix64_seed0.json")
    assert O.splitmix64_stream(d["seed"], len(d["outputs_hex"])) == [int(h, 16) for h in d["outputs_hex"]]


def test_golden_c3_schedule():
    d = load("c3_schedule.json")
    pr = S.PRESETS[3]
    assert S.config_seed(3, 0) == d["seed"] and S.split_epochs(8, 3) == d["epochs"]
    sch = O.schedule(pr.stages, 2, d["n_subsets"], d["seed"])
    assert [e[3] for e in sch] == sum(d["orders"], [])
    for i, a in d["momentum"].items():
        assert abs(O.momentum(int(i)) - a) <= 1e-16
