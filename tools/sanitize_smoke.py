#!/usr/bin/env python
"""Tiny layers through every kernel path (direct bulk / direct cp.async fallback / regtile,
pad) -- the target for compute-sanitizer (memcheck, racecheck, synccheck; one tool per run).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    rng = np.random.default_rng(7)
    cases = [
        (wl.Layer("rt3", 20, 8, 9, 9, 3, 3, 1, 1, 1, 0.8, 1.0), skc.SKC_KERNEL_REGTILE, 3),
        (wl.Layer("rt5", 12, 8, 11, 10, 5, 5, 1, 2, 2, 0.7, 1.0), skc.SKC_KERNEL_REGTILE, 2),
        (wl.Layer("d_bulk", 24, 16, 13, 13, 3, 3, 1, 1, 2, 0.9, 1.0), skc.SKC_KERNEL_DIRECT, 3),
        (wl.Layer("d_async", 10, 6, 7, 9, 3, 3, 1, 1, 1, 0.5, 1.0), skc.SKC_KERNEL_DIRECT, 2),
        (wl.Layer("d_band", 8, 4, 40, 12, 3, 3, 2, 1, 1, 0.5, 1.0), skc.SKC_KERNEL_DIRECT, 1),
    ]
    for L, kern, N in cases:
        w, x = wl.random_tensors(rng, L, N)
        conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern)
        out = conv.forward(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(w).double(),
                                         stride=L.stride, padding=L.pad, groups=L.groups)
        err = (out.double().cpu() - ref).abs().max().item()
        print(f"{L.name}: kernel {conv.geom['kernel']} max|err| {err:.2e}", flush=True)
        assert err < 1e-3
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
