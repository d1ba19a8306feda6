#!/usr/bin/env python
"""Row f4: replay synthetic pruning trajectories through the GSL controller with B200 profiles
MEASURED on the shipped (JIT) kernel, next to the paper's Xeon profile:
  * per layer where measured (profiles/r02_layer_windows.jsonl, tools/layer_windows.py):
    F = the layer's FP32 SGEMM-proxy rate, alpha = F / the layer's sparse rate at x = 0.5;
  * the other layers: the config-3 sweep of the final kernel
    (profiles/r01_sparsity_sweep_cfg3_final.jsonl: alpha = 1.20);
  B = the measured HBM copy bandwidth.  Trajectories: each layer's density decays
geometrically from 1 to a per-layer floor (the layer's 'achievable' density, e.g. conv1
stalls at 0.7).

    python tools/gsl_replay.py > profiles/r02_gsl_replay.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1608_01409_b200 import gsl  # noqa: E402

LAYERS = {
    "conv1": dict(K=96, C=3, R=11, S=11, H=227, W=227, stride=4, pad=0, groups=1),
    "conv2": dict(K=256, C=96, R=5, S=5, H=27, W=27, stride=1, pad=2, groups=2),
    "conv3": dict(K=384, C=256, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=1),
    "conv4": dict(K=384, C=384, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=2),
    "conv5": dict(K=256, C=384, R=3, S=3, H=13, W=13, stride=1, pad=1, groups=2),
    "res128_3x3": dict(K=128, C=128, R=3, S=3, H=28, W=28, stride=1, pad=1, groups=1),
    "inception_4a/5x5_reduce": dict(K=16, C=480, R=1, S=1, H=14, W=14),
}
FLOOR = {"conv1": 0.7, "conv2": 0.15, "conv3": 0.07, "conv4": 0.09, "conv5": 0.12,
         "res128_3x3": 0.3, "inception_4a/5x5_reduce": 0.5}


def b200_from_profiles():
    path = os.path.join(ROOT, "profiles", "r01_sparsity_sweep_cfg3_final.jsonl")
    summ = json.loads(open(path).read().strip().splitlines()[-1])["summary"]
    return gsl.b200_platform(summ["F_sgemm_tflops"] * 1e12, summ["B_gbs"] * 1e9,
                             summ["actual_sparse_tflops_x_ge_0.4"] * 1e12)


def b200_per_layer():
    """name -> Platform from the per-layer windows of the shipped kernel."""
    path = os.path.join(ROOT, "profiles", "r02_layer_windows.jsonl")
    out = {}
    if not os.path.exists(path):
        return out
    alias = {"res128_28x28": "res128_3x3"}
    for line in open(path):
        d = json.loads(line)
        name = alias.get(d["layer"], d["layer"])
        if name in LAYERS:
            out[name] = gsl.Platform(f"B200 ({d['layer']})", d["F_sgemm_tflops"] * 1e12,
                                     d["B_gbs"] * 1e9, d["sgemm"]["alpha"])
    return out


def main():
    traj = [(it, n, max(FLOOR[n], 0.85 ** it)) for it in range(60) for n in LAYERS]
    out = {}
    b200 = b200_from_profiles()
    per = b200_per_layer()
    for plat, lp in ((b200, per), (gsl.BDW, None)):
        c = gsl.GslController(LAYERS, plat, gsl.GslConfig(window=3, eps=0.01), layer_platforms=lp)
        out[plat.name] = gsl.replay(c, traj)
        if lp:
            out[plat.name]["per_layer_platforms"] = {n: {"F_tflops": p.F / 1e12, "alpha": p.alpha}
                                                     for n, p in lp.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
