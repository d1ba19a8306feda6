#!/usr/bin/env python
"""Config 3 (BASELINE.json configs[2]): the conv3 shape at batch 256 across sparsities
0..98%, measured against dense FP32 convolution, next to the B200 roofline model's
predicted useful-sparsity window (Sec. 2.2, :381-459; skc_model_* in libskc).

Model parameters follow the paper's method: F = the measured dense FP32
rate (SGEMM proxy, the paper's baseline; cuDNN reported too), B = measured HBM copy
bandwidth, alpha = F / (measured sparse nnz-FLOP/s at the densest points, x >= 0.4),
beta = 2.  Prints one JSON line per sparsity and a summary line with the measured
crossover density x* (speedup = 1, log-linear interpolation) against the model's
x_hi = 1/alpha and x_lo.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def timed(fn, reps=10, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    cfg = wl.CONFIGS[3]
    N = cfg.batch
    peaks = {}
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    B = float(peaks.get("hbm_gbs", 6545.0)) * 1e9
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L0 = cfg.layers[0]
    x = torch.from_numpy(wl.gen_input(3, 0, L0, 0, N)).cuda()
    dense_flops = 2.0 * L0.K * (L0.C // L0.groups) * L0.R * L0.S * L0.Ho * L0.Wo * N
    # dense baselines (independent of sparsity)
    wd = torch.randn(L0.K, L0.C // L0.groups, L0.R, L0.S, device="cuda")
    t_cudnn = timed(lambda: torch.nn.functional.conv2d(x, wd, padding=L0.pad, groups=L0.groups),
                    flush=flush)
    A = torch.randn(L0.K, L0.C * L0.R * L0.S, device="cuda")
    Bm = torch.randn(L0.C * L0.R * L0.S, L0.Ho * L0.Wo * N, device="cuda")
    t_sgemm = timed(lambda: torch.matmul(A, Bm), flush=flush)
    del A, Bm, wd
    F_sgemm = dense_flops / (t_sgemm * 1e-3)
    F_cudnn = dense_flops / (t_cudnn * 1e-3)
    rows = []
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(3, li, L)
        conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups)
        conv.tune(N)
        xp = torch.empty(conv.padded_shape(N), device="cuda")
        out = torch.empty(conv.out_shape(N), device="cuda")
        t_pad = timed(lambda: skc.skc_pad_input(conv.plan, x, xp, N), flush=flush)
        t_conv = timed(lambda: skc.skc_sparse_conv_forward(conv.plan, xp, out, N), flush=flush)
        nnz = conv.geom["nnz"]
        density = nnz / (L.K * (L.C // L.groups) * L.R * L.S)
        t = t_pad + t_conv
        # rates on both time bases, named explicitly: conv = skc_sparse_conv_forward alone,
        # layer = skc_pad_input + skc_sparse_conv_forward (the speedups use the layer time)
        r = dict(sparsity=L.sparsity, density=density, nnz=nnz, kernel=conv.geom["kernel"],
                 t_pad_ms=t_pad, t_conv_ms=t_conv, t_layer_ms=t,
                 nnz_tflops=2 * nnz * L.Ho * L.Wo * N / (t_conv * 1e-3) / 1e12,
                 nnz_tflops_layer=2 * nnz * L.Ho * L.Wo * N / (t * 1e-3) / 1e12,
                 dense_equiv_tflops=dense_flops / (t * 1e-3) / 1e12,
                 dense_equiv_tflops_conv=dense_flops / (t_conv * 1e-3) / 1e12,
                 speedup_vs_sgemm_proxy=t_sgemm / t, speedup_vs_cudnn=t_cudnn / t)
        rows.append(r)
        print(json.dumps(r), flush=True)
        del conv, xp, out
    # alpha by the paper's method: F / actual sparse rate where compute bound (x >= 0.4)
    dense_pts = [r for r in rows if r["density"] >= 0.4]
    actual = np.mean([2 * r["nnz"] * L0.Ho * L0.Wo * N / (r["t_layer_ms"] * 1e-3) for r in dense_pts])
    cost = skc.skc_model_layer_cost(L0.K, L0.C, L0.R, L0.S, L0.H, L0.W, L0.stride, L0.pad,
                                    L0.groups, batch=N, amortised=True)
    summary = {"F_sgemm_tflops": F_sgemm / 1e12, "F_cudnn_dense_equiv_tflops": F_cudnn / 1e12,
               "t_sgemm_ms": t_sgemm, "t_cudnn_ms": t_cudnn, "B_gbs": B / 1e9,
               "actual_sparse_tflops_x_ge_0.4": actual / 1e12}
    for name, F in (("sgemm", F_sgemm), ("cudnn", F_cudnn)):
        alpha = F / actual
        win = skc.skc_model_window(cost, F, B, alpha)
        sp = [t_ref / r["t_layer_ms"] for r in rows
              for t_ref in [t_sgemm if name == "sgemm" else t_cudnn]]
        xs = [r["density"] for r in rows]
        # measured crossover: densest x with speedup >= 1 next to a point with speedup < 1
        xstar = None
        pts = sorted(zip(xs, sp))
        for (x1, s1), (x2, s2) in zip(pts, pts[1:]):
            if (s1 - 1) * (s2 - 1) <= 0 and s1 != s2:
                lx = math.log(x1) + (math.log(x2) - math.log(x1)) * (1 - s1) / (s2 - s1)
                xstar = math.exp(lx)
        pred = [skc.skc_model_project(cost, xx, F, B, alpha)["speedup"] for xx in xs]
        summary[name] = {"alpha": alpha, "model_x_hi": win["x_hi"], "model_x_lo": win["x_lo"],
                         "measured_crossover_x": xstar,
                         "measured_speedup": dict(zip([round(v, 4) for v in xs], sp)),
                         "model_speedup": dict(zip([round(v, 4) for v in xs], pred))}
    print(json.dumps({"summary": summary}), flush=True)


if __name__ == "__main__":
    main()
