#!/usr/bin/env python
"""Row f4: replay synthetic pruning trajectories through the GSL controller with the B200
profile MEASURED in round 1 (profiles/r01_sparsity_sweep_cfg3.jsonl: F = FP32 SGEMM rate,
alpha = F / actual sparse rate at x >= 0.4, B = measured HBM copy bandwidth) next to the
paper's Xeon profile.  Trajectories: each layer's density decays geometrically from 1 to a
per-layer floor (the layer's 'achievable' density, e.g. conv1 stalls at 0.7)."""
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
    path = os.path.join(ROOT, "profiles", "r01_sparsity_sweep_cfg3.jsonl")
    summ = json.loads(open(path).read().strip().splitlines()[-1])["summary"]
    return gsl.b200_platform(summ["F_sgemm_tflops"] * 1e12, summ["B_gbs"] * 1e9,
                             summ["actual_sparse_tflops_x_ge_0.4"] * 1e12)


def main():
    traj = [(it, n, max(FLOOR[n], 0.85 ** it)) for it in range(60) for n in LAYERS]
    out = {}
    for plat in (b200_from_profiles(), gsl.BDW):
        c = gsl.GslController(LAYERS, plat, gsl.GslConfig(window=3, eps=0.01))
        out[plat.name] = gsl.replay(c, traj)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
