#!/usr/bin/env python
"""Row f1 measurement: AlexNet conv3 -> conv4 -> conv5 at batch 256 with bias + ReLU between
layers, (a) unfused: skc_pad_input + skc_sparse_conv_forward + a bias/ReLU pass per layer,
(b) fused: skc_sparse_conv_forward_into writing each layer's activated output straight into
the next layer's zero-padded input, in that plan's layout (one pad pass for conv3's input
only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    cfg = wl.CONFIGS[2]
    N = cfg.batch
    layers = [cfg.layers[1], cfg.layers[2], cfg.layers[3]]
    convs = [skc.SparseConv2d.from_dense(wl.gen_weights(2, i + 1, L), L.H, L.W, L.stride, L.pad,
                                         L.groups) for i, L in enumerate(layers)]
    rng = np.random.default_rng(3)
    biases = [torch.from_numpy((0.1 * rng.standard_normal(L.K)).astype(np.float32)).cuda()
              for L in layers]
    x = torch.from_numpy(wl.gen_input(2, 1, layers[0], 0, N)).cuda()
    # unfused buffers
    xps = [torch.empty(c.padded_shape(N), device="cuda") for c in convs]
    outs = [torch.empty(c.out_shape(N), device="cuda") for c in convs]

    def unfused():
        h = x
        for conv, xp, out, b in zip(convs, xps, outs, biases):
            skc.skc_pad_input(conv.plan, h, xp, N)
            skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
            torch.relu_(out.add_(b.view(1, -1, 1, 1)))
            h = out

    # fused buffers: each layer writes the next layer's padded input (halo zeroed once)
    fbufs = [torch.zeros(c.padded_shape(N), device="cuda") for c in convs]
    fbufs.append(torch.zeros(convs[-1].out_shape(N), device="cuda"))

    def fused():
        skc.skc_pad_input(convs[0].plan, x, fbufs[0], N)
        for i, (conv, b) in enumerate(zip(convs, biases)):
            if i + 1 < len(convs):
                skc.skc_sparse_conv_forward_into(conv.plan, fbufs[i], convs[i + 1].plan,
                                                 fbufs[i + 1], N, b, True)
            else:
                skc.skc_sparse_conv_forward_ex(conv.plan, fbufs[i], fbufs[i + 1], N, b, True, 0)

    t_u = timed(unfused)
    t_f = timed(fused)
    unfused()
    fused()
    torch.cuda.synchronize()
    same = bool(torch.equal(outs[-1], fbufs[-1]))
    flops = sum(2.0 * c.geom["nnz"] * L.Ho * L.Wo * N for c, L in zip(convs, layers))
    print(json.dumps({"chain": "conv3->conv4->conv5 b256, bias+ReLU", "unfused_ms": t_u,
                      "fused_ms": t_f, "speedup": t_u / t_f,
                      "fused_nnz_tflops": flops / (t_f * 1e-3) / 1e12,
                      "bitwise_equal_outputs": same}))


if __name__ == "__main__":
    main()
