#!/usr/bin/env python
"""Small-batch latency of one layer: pad + conv per forward call for plans configured for the
batch (skc_pack_csr_batch) -- AUTO, the direct kernel, the compiled-weights kernel -- and the
default 256-image plan, L2 flushed before every call, median of --reps CUDA-event timings;
every output compared bit for bit with the direct kernel's 256-image plan (every kernel and
configuration accumulates each output in CSR order; the GPU suite checks them against the
oracle).  One JSON line per (batch, plan).

    python tools/small_batch.py --config 1 --layer 0 --batches 1,2,4,8,16,32,64
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--batches", default="1,2,4,8,16,32,64")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--jit-hints", default="", help="extra JIT plans configured for these batches")
    a = ap.parse_args()
    a.jit_hints = [int(h) for h in a.jit_hints.split(",") if h]
    cfg = wl.CONFIGS[a.config]
    L = cfg.layers[a.layer]
    w = wl.gen_weights(a.config, a.layer, L)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for N in [int(b) for b in a.batches.split(",")]:
        xh = wl.gen_input(a.config, a.layer, L, 0, N)
        x = torch.from_numpy(xh).cuda()
        ref = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups,
                                          skc.SKC_KERNEL_DIRECT).forward(x).cpu().numpy()
        plans = [("auto", skc.SKC_KERNEL_AUTO, N), ("direct", skc.SKC_KERNEL_DIRECT, N),
                 ("jit", skc.SKC_KERNEL_JIT, N), ("auto_256", skc.SKC_KERNEL_AUTO, None)]
        plans += [("jit%d" % h, skc.SKC_KERNEL_JIT, h) for h in a.jit_hints if h != N and h < 256]
        for tag, kern, hint in plans:
            try:
                conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern,
                                                   batch_hint=hint)
            except skc.SkcError as e:
                print(json.dumps({"layer": L.name, "N": N, "plan": tag, "error": str(e)[:200]}), flush=True)
                continue
            if conv.geom["kernel"] == skc.SKC_KERNEL_JIT:
                conv.tune(N)
            xp = torch.empty(conv.padded_shape(N), device="cuda") \
                if conv.geom["layout"] != skc.SKC_LAYOUT_RAW else x
            out = torch.empty(conv.out_shape(N), device="cuda")
            ts = []
            for r in range(a.reps + 3):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                skc.skc_pad_input(conv.plan, x, xp, N)
                skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            ts.sort()
            ms = ts[len(ts) // 2]
            same = bool(np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32)))
            i = conv.plan.info()
            print(json.dumps({"layer": L.name, "N": N, "plan": tag, "ms": ms,
                              "nnz_tflops": 2 * i["nnz"] * L.Ho * L.Wo * N / (ms * 1e-3) / 1e12,
                              "kernel": i["kernel"], "warps": i["warps"], "M": i["channels_per_warp"],
                              "T": i["pixels_per_lane"], "NI": i["images_per_cta"],
                              "band_rows": i["band_rows"], "blocks": i["jit_blocks"], "bands": i["bands"],
                              "bitwise_equal_direct": same, "pass": same}), flush=True)
            del conv, xp, out


if __name__ == "__main__":
    main()
