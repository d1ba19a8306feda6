#!/usr/bin/env python
"""Row f3 measurement: direct sparse convolution vs sparse convolution WITH lowering
(im2col + SpMDM) on AlexNet conv2-5 at batch 256 -- the paper's direct-vs-lowered argument
(Fig. 3 "conv5 lowered") measured on B200, next to the roofline model's
projection for both (the lowered variant moves R*S times more activation bytes).

The direct side is the AUTO plan (the compiled-weights kernel, tuned); the lowered side runs
the 1x1 SpMDM over the im2col tensor with the data-driven direct kernel (default) or with the
AUTO plan too (--lowered-kernel auto: the compiled-weights kernel on the lowered matrix).

    python tools/lowered_bench.py [--lowered-kernel direct|auto] > profiles/r02_lowered_vs_direct.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from chain_bench import timed  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--lowered-kernel", default="direct", choices=["direct", "auto"])
    a = ap.parse_args()
    lk = skc.SKC_KERNEL_DIRECT if a.lowered_kernel == "direct" else skc.SKC_KERNEL_AUTO
    cfg = wl.CONFIGS[2]
    N = cfg.batch
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(2, li, L)
        x = torch.from_numpy(wl.gen_input(2, li, L, 0, N)).cuda()
        direct = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups)
        direct.tune(N)
        xp = torch.empty(direct.padded_shape(N), device="cuda")
        out = torch.empty(direct.out_shape(N), device="cuda")
        t_direct = timed(lambda: direct.forward(x, xp=xp, out=out))
        low = skc.LoweredSparseConv2d(w, L.H, L.W, L.stride, L.pad, L.groups, kernel=lk)
        if lk == skc.SKC_KERNEL_AUTO:
            low.conv.tune(N)
        lbuf = torch.empty(low.lowered_shape(N), device="cuda")
        out2 = torch.empty_like(out)
        t_low = timed(lambda: low.forward(x, lowered=lbuf, out=out2))
        t_im2col = timed(lambda: skc.skc_im2col_ex(low.geom_plan, x, lbuf, N, low._layout()))
        same = bool(torch.equal(out, out2))
        nnz = direct.geom["nnz"]
        flops = 2.0 * nnz * L.Ho * L.Wo * N
        print(json.dumps({"layer": L.name, "direct_kernel": direct.geom["kernel"],
                          "lowered_kernel": low.conv.geom["kernel"], "direct_ms": t_direct, "lowered_ms": t_low,
                          "im2col_ms": t_im2col, "direct_over_lowered": t_low / t_direct,
                          "direct_nnz_tflops": flops / (t_direct * 1e-3) / 1e12,
                          "lowered_nnz_tflops": flops / (t_low * 1e-3) / 1e12,
                          "lowered_bytes": lbuf.numel() * 4, "bitwise_equal": same}), flush=True)
        del lbuf, xp, out, out2


if __name__ == "__main__":
    main()
