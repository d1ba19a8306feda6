#!/usr/bin/env python
"""One config layer's pad pass (skc_pad_input, the plan's layout) as an ncu target: a warm-up
launch, an L2 flush, then ONE launch inside the NVTX range "prof".

    ncu --set full --nvtx --nvtx-include "prof/" -c 1 -o pad python tools/prof_pad.py --layer 1
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
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    L = cfg.layers[a.layer]
    N = cfg.batch
    conv = skc.SparseConv2d.from_dense(wl.gen_weights(a.config, a.layer, L), L.H, L.W, L.stride,
                                       L.pad, L.groups)
    x = torch.from_numpy(wl.gen_input(a.config, a.layer, L, 0, N)).cuda()
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    skc.skc_pad_input(conv.plan, x, xp, N)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("prof")
    e0.record()
    skc.skc_pad_input(conv.plan, x, xp, N)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    by = 4 * N * L.C * (L.H * L.W + (L.H + 2 * L.pad) * (L.W + 2 * L.pad))
    print(f"{L.name} pad {e0.elapsed_time(e1):.4f} ms {by / e0.elapsed_time(e1) / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
