"""Pins for the roofline model oracle (oracle/ref_model.py) against numbers the paper
prints (tests/golden/paper_model_numbers.json), a brute-force grid search, and the
model's invariants (SURVEY.md P-M1 .. P-M5)."""
import json
import os

import numpy as np
import pytest

from oracle import ref_model as M


@pytest.fixture(scope="module")
def paper(golden_dir):
    return json.load(open(os.path.join(golden_dir, "paper_model_numbers.json")))


def conv5_cost(paper, **kw):
    g = paper["conv5"]
    return M.layer_cost(g["K"], g["C"], g["R"], g["S"], g["H"], g["W"], g["stride"], g["pad"],
                        g["groups"], **kw)


def test_conv5_cost_closed_form(paper):
    """C = 2*256*192*9*169, S_A = 4*(384+256)*169, S_W = 4*256*192*9 (grouped conv5)."""
    c = conv5_cost(paper)
    assert c["C"] == 149_520_384 and c["S_A"] == 432_640 and c["S_W"] == 1_769_472
    # ungrouped conv5 ~ 2.99e8 FLOP
    assert M.layer_cost(256, 384, 3, 3, 13, 13, 1, 1, 1)["C"] == pytest.approx(2.99e8, rel=2e-3)
    # batch doubles C and S_A and (per-image weights) S_W; amortised leaves S_W
    c2 = conv5_cost(paper, batch=2)
    assert c2["C"] == 2 * c["C"] and c2["S_A"] == 2 * c["S_A"] and c2["S_W"] == 2 * c["S_W"]
    assert conv5_cost(paper, batch=2, amortised=True)["S_W"] == c["S_W"]


def test_x_lo_matches_paper(paper):
    """P-M2: the bandwidth crossover reproduces the paper's x~0.02 (Xeon) and x~0.01 (Atom)
    for grouped conv5 within 15% (reading R3/R8)."""
    c = conv5_cost(paper)
    for e in paper["x_lo"]:
        p = paper["platforms"][e["platform"]]
        w = M.window(c, p["F"], p["B"], p["alpha"], p["beta"])
        assert w["x_lo"] == pytest.approx(e["value"], rel=0.15), (e, w)
        assert w["has_speedup_potential"]


def test_x_hi_matches_paper(paper):
    """P-M1: x_hi = 1/alpha = 0.333 vs the paper's measured x = 0.3."""
    for e in paper["x_hi"]:
        w = M.window(conv5_cost(paper), 2e12, 1e11, e["alpha"])
        assert w["x_hi"] == pytest.approx(1 / 3) and w["x_hi"] == pytest.approx(e["value"], abs=0.04)


def test_speedup_range_and_point(paper):
    """P-M3: compute-bound speedup = 1/(alpha x): 2.22..6.67 for x in (0.05,0.15) vs the
    paper's '2-7x'; 3.70 at x = 0.09 vs the measured 3.4x."""
    c = conv5_cost(paper)
    p = paper["platforms"]["BDW"]
    e = paper["speedup_range"][0]
    lo = M.project(c, e["x_range"][1], p["F"], p["B"], p["alpha"])["speedup"]
    hi = M.project(c, e["x_range"][0], p["F"], p["B"], p["alpha"])["speedup"]
    assert lo == pytest.approx(1 / (3 * 0.15)) and hi == pytest.approx(1 / (3 * 0.05))
    assert e["speedup_range"][0] - 0.5 <= lo and hi <= e["speedup_range"][1] + 0.5
    s = M.project(c, 0.09, p["F"], p["B"], p["alpha"])["speedup"]
    assert s == pytest.approx(3.7037, rel=1e-4)
    assert abs(s - paper["speedup_point"][0]["measured"]) / s < 0.1


def test_window_vs_grid_search(paper):
    """P-M4: closed-form window vs a brute-force scan of 10^4 densities in [1e-4, 1]."""
    c = conv5_cost(paper)
    for name, p in paper["platforms"].items():
        if name.startswith("_"):
            continue
        xs = np.geomspace(1e-4, 1.0, 10_000)
        sp = np.array([M.project(c, x, p["F"], p["B"], p["alpha"])["speedup"] for x in xs])
        w = M.window(c, p["F"], p["B"], p["alpha"])
        # (a) largest x with speedup > 1 ~ x_hi
        x_hi_grid = xs[np.nonzero(sp > 1.0)[0].max()]
        step = xs[1] / xs[0]
        assert w["x_hi"] / step <= x_hi_grid * step and x_hi_grid <= w["x_hi"] * step
        # (b) x_lo is where the bound switches from bandwidth to compute: below it the
        # speedup only creeps up through the beta*x*S_W term (near-plateau), above it it
        # falls as 1/(alpha x)
        pr = [M.project(c, x, p["F"], p["B"], p["alpha"]) for x in xs]
        comp = np.array([q["t_sparse_compute"] >= q["t_sparse_bw"] for q in pr])
        x_switch = xs[np.nonzero(comp)[0].min()]
        assert x_switch / step <= w["x_lo"] <= x_switch * step
        below = sp[xs < w["x_lo"] / step]
        assert below.max() / below.min() < 1.0 + 2 * w["x_lo"] * c["S_W"] / c["S_A"]


def test_invariants(paper):
    """P-M5: speedup(1/alpha) = 1 when compute bound; t_sparse non-decreasing in x;
    effective FLOP/s at x = 1 equals F/alpha when compute bound; no-potential case."""
    c = conv5_cost(paper)
    p = paper["platforms"]["BDW"]
    assert M.project(c, 1 / p["alpha"], p["F"], p["B"], p["alpha"])["speedup"] == pytest.approx(1.0)
    ts = [M.project(c, x, p["F"], p["B"], p["alpha"])["t_sparse"] for x in np.linspace(1e-3, 1, 200)]
    assert np.all(np.diff(ts) >= 0)
    assert M.project(c, 1.0, p["F"], p["B"], p["alpha"])["effective_flops"] == pytest.approx(p["F"] / p["alpha"])
    # a 1x1 reduce layer (GoogLeNet inception_4a/5x5_reduce-like) on a tiny-B platform
    c11 = M.layer_cost(16, 192, 1, 1, 14, 14)
    w = M.window(c11, 2.15e12, 1e9, 3.0)
    assert not w["has_speedup_potential"]
    with pytest.raises(ValueError):
        M.project(c, 0.0, 1, 1, 1)
