"""Row f4: the GSL controller -- its three rules, the SPEC.md:300-323
examples, property tests on random trajectories, and consistency with the model."""
import numpy as np
import pytest

from paper_1608_01409_b200 import gsl, skc

ALEX = {
    "conv1": dict(K=96, C=3, R=11, S=11, H=227, W=227, stride=4, pad=0, groups=1),
    "conv2": dict(K=256, C=96, R=5, S=5, H=27, W=27, stride=1, pad=2, groups=2),
    "conv3": dict(K=384, C=256, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=1),
    "conv4": dict(K=384, C=384, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=2),
    "conv5": dict(K=256, C=384, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=2),
}
REDUCE_1X1 = {"inception_4a/5x5_reduce": dict(K=16, C=480, R=1, S=1, H=14, W=14)}


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_1608_01409_b200 import build
    build.build()
    skc.lib()


def test_init_excludes_layers_without_potential():
    """'Exclude all Ls without speedup potential': a GoogLeNet 1x1 reduce
    layer is bandwidth bound on the Xeon profile, AlexNet conv2-5 are not;
    conv1 is excluded manually (not derivable from the model)."""
    c = gsl.GslController({**ALEX, **REDUCE_1X1}, gsl.BDW, gsl.GslConfig(exclude=("conv1",)))
    st = {n: L.status for n, L in c.layers.items()}
    assert st["inception_4a/5x5_reduce"] == gsl.EXCLUDED
    assert st["conv1"] == gsl.EXCLUDED
    assert all(st[f"conv{i}"] == gsl.ACTIVE for i in range(2, 6))
    with pytest.raises(ValueError):
        gsl.GslController({}, gsl.BDW)


def test_rules_spec_examples():
    """window (x_lo, x_hi); x below x_lo -> STOP_PRUNING; stabilized above
    1/alpha -> RESTORE_DENSE; inside the window and moving -> CONTINUE."""
    c = gsl.GslController(ALEX, gsl.BDW, gsl.GslConfig(window=3, eps=0.01))
    w5 = c.layers["conv5"].window
    assert w5["x_lo"] == pytest.approx(0.0197, rel=0.02) and w5["x_hi"] == pytest.approx(1 / 3)
    assert c.step(0, {"conv5": 0.015, "conv3": 0.30, "conv4": 0.45}) == {
        "conv5": gsl.STOP_PRUNING, "conv3": gsl.CONTINUE, "conv4": gsl.CONTINUE}
    assert c.step(1, {"conv4": 0.45, "conv3": 0.15}) == {"conv4": gsl.CONTINUE, "conv3": gsl.CONTINUE}
    assert c.step(2, {"conv4": 0.45, "conv3": 0.12}) == {"conv4": gsl.RESTORE_DENSE,
                                                          "conv3": gsl.CONTINUE}
    # no directives once a layer left ACTIVE
    assert c.step(3, {"conv5": 0.01, "conv4": 0.2}) == {}
    assert c.layers["conv5"].status == gsl.STOPPED_SATURATED
    assert c.layers["conv4"].status == gsl.RESTORED_DENSE
    with pytest.raises(KeyError):
        c.step(4, {"conv9": 0.1})


def test_random_trajectories_properties():
    """Transitions only ACTIVE -> {STOPPED_SATURATED, RESTORED_DENSE}; never a directive for a
    non-ACTIVE layer; RESTORE only after `window` stable checks at x >= x_hi; STOP exactly
    when x <= x_lo."""
    rng = np.random.default_rng(0)
    for trial in range(200):
        cfg = gsl.GslConfig(window=int(rng.integers(1, 5)), eps=float(rng.choice([0.005, 0.02])))
        c = gsl.GslController(ALEX, gsl.BDW, cfg)
        x = {n: float(rng.uniform(0.2, 1.0)) for n in ALEX}
        hist = {n: [] for n in ALEX}
        for it in range(40):
            for n in x:
                x[n] = float(np.clip(x[n] * rng.uniform(0.7, 1.02), 0.001, 1.0))
            before = {n: L.status for n, L in c.layers.items()}
            d = c.step(it, dict(x))
            for n, L in c.layers.items():
                if before[n] != gsl.ACTIVE:
                    assert n not in d and L.status == before[n]
                    continue
                hist[n].append(x[n])
                lo, hi = L.window["x_lo"], L.window["x_hi"]
                if x[n] <= lo:
                    assert d[n] == gsl.STOP_PRUNING and L.status == gsl.STOPPED_SATURATED
                elif d[n] == gsl.RESTORE_DENSE:
                    rec = hist[n][-cfg.window:]
                    assert len(rec) >= cfg.window and max(rec) - min(rec) < cfg.eps
                    assert x[n] >= hi
                else:
                    assert d[n] == gsl.CONTINUE and L.status == gsl.ACTIVE


def test_replay_and_report_consistency():
    """Replay: every ACTIVE layer decays to 0.001 -> all STOPPED_SATURATED at their first
    density <= x_lo; report speedups equal the model's projection at the final density;
    a constant x = 1 trajectory restores every layer; net speedup aggregates times."""
    c = gsl.GslController(ALEX, gsl.BDW, gsl.GslConfig(exclude=("conv1",)))
    traj = [(it, n, max(0.001, 0.8 * 0.7 ** it)) for it in range(30) for n in ALEX]
    rep = gsl.replay(c, traj)
    p = gsl.BDW
    t_d = t_s = 0.0
    for row in rep["layers"]:
        L = c.layers[row["layer"]]
        if row["layer"] == "conv1":
            assert row["status"] == gsl.EXCLUDED and row["projected_speedup"] == pytest.approx(1.0)
        else:
            assert row["status"] == gsl.STOPPED_SATURATED
            assert row["final_density"] <= row["x_lo"]
            pr = skc.skc_model_project(L.cost, row["final_density"], p.F, p.B, p.alpha)
            assert row["projected_speedup"] == pytest.approx(pr["speedup"])
        pr = skc.skc_model_project(L.cost, c.final_density(row["layer"]), p.F, p.B, p.alpha)
        t_d += pr["t_dense"]
        t_s += pr["t_sparse"] if row["status"] != gsl.EXCLUDED else pr["t_dense"]
    assert rep["net_speedup"] == pytest.approx(t_d / t_s)
    c2 = gsl.GslController(ALEX, gsl.BDW, gsl.GslConfig(window=3))
    rep2 = gsl.replay(c2, [(it, n, 1.0) for it in range(5) for n in ALEX])
    assert all(r["status"] in (gsl.RESTORED_DENSE, gsl.EXCLUDED) for r in rep2["layers"])
    assert rep2["net_speedup"] == pytest.approx(1.0)


def test_b200_profile_alpha():
    """The paper's alpha method on the config-3 measurement: F / actual sparse rate."""
    p = gsl.b200_platform(62.0e12, 6.545e12, 14.9e12)
    assert p.alpha == pytest.approx(62.0 / 14.9)
    c = gsl.GslController(ALEX, p)
    assert c.layers["conv3"].window["x_hi"] == pytest.approx(14.9 / 62.0)


def test_per_layer_platforms():
    """B200 windows are per layer (each layer's own measured F and alpha,
    tools/layer_windows.py): a layer with its own platform gets its own window and projected
    speedup; the others keep the default platform; unknown names are rejected."""
    own = gsl.Platform("B200-conv3", 60e12, 6.5e12, 1.8)
    c = gsl.GslController(ALEX, gsl.BDW, layer_platforms={"conv3": own})
    assert c.layers["conv3"].window["x_hi"] == pytest.approx(1 / 1.8)
    assert c.layers["conv4"].window["x_hi"] == pytest.approx(1 / gsl.BDW.alpha)
    rep = gsl.replay(c, [(it, n, 0.2) for it in range(4) for n in ALEX])
    row = {r["layer"]: r for r in rep["layers"]}
    pr = skc.skc_model_project(c.layers["conv3"].cost, 0.2, own.F, own.B, own.alpha)
    assert row["conv3"]["projected_speedup"] == pytest.approx(pr["speedup"])
    assert row["conv3"]["alpha"] == pytest.approx(1.8)
    with pytest.raises(KeyError):
        gsl.GslController(ALEX, gsl.BDW, layer_platforms={"nope": own})
