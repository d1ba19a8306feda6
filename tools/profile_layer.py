#!/usr/bin/env python
"""Run one layer of a config (pad + conv) a few times -- a short target for ncu.

    python tools/profile_layer.py --config 2 --layer 1 --reps 3 [--kernel direct]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layer", type=int, default=1)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kernel", default="auto", choices=["auto", "direct", "regtile"])
    ap.add_argument("--batch-hint", type=int, default=0, help="plan configured for this batch")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    L = cfg.layers[a.layer]
    N = a.batch or cfg.batch
    kern = {"auto": 0, "direct": 1, "regtile": 2}[a.kernel]
    w = wl.gen_weights(a.config, a.layer, L)
    conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern,
                                       batch_hint=a.batch_hint or None)
    x = torch.from_numpy(wl.gen_input(a.config, a.layer, L, 0, N)).cuda()
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    out = torch.empty(conv.out_shape(N), device="cuda")
    for _ in range(a.reps):
        skc.skc_pad_input(conv.plan, x, xp, N)
        skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{L.name} N={N} nnz={conv.geom['nnz']} conv {ms:.3f} ms "
          f"{2 * conv.geom['nnz'] * L.Ho * L.Wo * N / ms / 1e9:.1f} nnz-GFLOP/s cfg={conv.geom}")


if __name__ == "__main__":
    main()
