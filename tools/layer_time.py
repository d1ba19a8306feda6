#!/usr/bin/env python
"""Time one config layer's conv kernel as bench.py runs it (AUTO plan tuned for the batch,
L2 flushed before every launch, median of --reps CUDA-event timings), under whatever SKC_JIT_*
knobs are set -- for configuration sweeps.  One JSON line.

    SKC_JIT_NW=12 SKC_JIT_TILE=1,1,64 python tools/layer_time.py --config 2 --layer 1
"""
import argparse
import json
import math
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tag", default="")
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between launches")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    L = cfg.layers[a.layer]
    N = cfg.batch
    conv = skc.SparseConv2d.from_dense(wl.gen_weights(a.config, a.layer, L), L.H, L.W, L.stride,
                                       L.pad, L.groups)
    conv.tune(N)
    x = torch.from_numpy(wl.gen_input(a.config, a.layer, L, 0, N)).cuda()
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    out = torch.empty(conv.out_shape(N), device="cuda")
    skc.skc_pad_input(conv.plan, x, xp, N)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for r in range(a.reps + 3):
        if not a.no_flush:
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    i = conv.plan.info()
    items = i["jit_blocks"] * math.ceil(N / max(1, i["images_per_cta"])) * max(1, i["bands"])
    print(json.dumps({"tag": a.tag, "layer": L.name, "ms": ms,
                      "nnz_tflops": 2 * i["nnz"] * L.Ho * L.Wo * N / (ms * 1e-3) / 1e12,
                      "warps": i["warps"], "M": i["channels_per_warp"], "NI": i["images_per_cta"],
                      "blocks": i["jit_blocks"], "bands": i["bands"], "CB": i["chunk_channels"],
                      "NS": i["stages"], "items": items, "rounds": items / 148.0,
                      "sched": i["jit_sched"], "whole": i["jit_whole"], "np": i["jit_np"]}), flush=True)


if __name__ == "__main__":
    main()
