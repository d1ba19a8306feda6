#!/usr/bin/env python
"""Row a7 on the shipped kernel: per-layer B200 sweet-spot windows (Sec. 2.2,
:381-459) for AlexNet conv2-5 (config 2) and the ResNet-50 3x3 layers (config 4), batch 256.

Per layer, by the paper's method: F = the measured dense FP32 rate of the
layer (the SGEMM proxy at its lowered shape, the paper's baseline; cuDNN FP32 beside it),
alpha = F / the measured sparse rate at density 0.5 (x >= 0.4: compute bound), B = the
measured HBM copy bandwidth, beta = 2; the model then gives x_hi = 1/alpha (sparse slower
than dense above it) and x_lo (bandwidth crossover).  The layer is also measured at its
config density: measured speedup vs the model's.  Sparse times are the whole layer
(skc_pad_input + skc_sparse_conv_forward, AUTO plan tuned for the batch), L2 flushed before
every timed launch.  One JSON line per layer.

    python tools/layer_windows.py > profiles/r02_layer_windows.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sparsity_sweep import timed  # noqa: E402


def sparse_layer_ms(cfg_id, li, L, w, x, N, flush):
    conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups)
    conv.tune(N)
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    out = torch.empty(conv.out_shape(N), device="cuda")
    t_pad = timed(lambda: skc.skc_pad_input(conv.plan, x, xp, N), flush=flush)
    t_conv = timed(lambda: skc.skc_sparse_conv_forward(conv.plan, xp, out, N), flush=flush)
    return t_pad, t_conv, conv.geom


def main():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    B = float(peaks.get("hbm_gbs", 6545.0)) * 1e9
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg_id in (2, 4):
        cfg = wl.CONFIGS[cfg_id]
        N = cfg.batch
        for li, L in enumerate(cfg.layers):
            x = torch.from_numpy(wl.gen_input(cfg_id, li, L, 0, N)).cuda()
            dflops = 2.0 * L.K * (L.C // L.groups) * L.R * L.S * L.Ho * L.Wo * N
            # dense baselines: the SGEMM proxy per group [K/g x C/g*R*S] x [C/g*R*S x Ho*Wo*N]
            A = torch.randn(L.K // L.groups, (L.C // L.groups) * L.R * L.S, device="cuda")
            Bm = torch.randn((L.C // L.groups) * L.R * L.S, L.Ho * L.Wo * N, device="cuda")
            t_sgemm = timed(lambda: torch.matmul(A, Bm), flush=flush) * L.groups
            del A, Bm
            wd = torch.randn(L.K, L.C // L.groups, L.R, L.S, device="cuda")
            t_cudnn = timed(lambda: torch.nn.functional.conv2d(x, wd, stride=L.stride, padding=L.pad,
                                                               groups=L.groups), flush=flush)
            del wd
            F_sgemm, F_cudnn = dflops / (t_sgemm * 1e-3), dflops / (t_cudnn * 1e-3)
            # sparse at density 0.5 (alpha) and at the config's density
            rows = {}
            for tag, Ls in (("x05", L.__class__(**{**L.__dict__, "sparsity": 0.5})), ("cfg", L)):
                w = wl.gen_weights(cfg_id, li, Ls)
                tp, tc, geom = sparse_layer_ms(cfg_id, li, Ls, w, x, N, flush)
                nnz = int(geom["nnz"])
                rows[tag] = dict(density=nnz / (L.K * (L.C // L.groups) * L.R * L.S), nnz=nnz,
                                 t_pad_ms=tp, t_conv_ms=tc,
                                 actual_tflops=2.0 * nnz * L.Ho * L.Wo * N / ((tp + tc) * 1e-3) / 1e12,
                                 conv_nnz_tflops=2.0 * nnz * L.Ho * L.Wo * N / (tc * 1e-3) / 1e12,
                                 kernel=geom["kernel"], jit_sched=geom.get("jit_sched"))
            cost = skc.skc_model_layer_cost(L.K, L.C, L.R, L.S, L.H, L.W, L.stride, L.pad, L.groups,
                                            batch=N, amortised=True)
            actual = rows["x05"]["actual_tflops"] * 1e12
            out = dict(config=cfg_id, layer=L.name, batch=N, B_gbs=B / 1e9,
                       F_sgemm_tflops=F_sgemm / 1e12, F_cudnn_dense_equiv_tflops=F_cudnn / 1e12,
                       t_sgemm_ms=t_sgemm, t_cudnn_ms=t_cudnn, sparse=rows)
            t_layer = rows["cfg"]["t_pad_ms"] + rows["cfg"]["t_conv_ms"]
            for name, F, t_ref in (("sgemm", F_sgemm, t_sgemm), ("cudnn", F_cudnn, t_cudnn)):
                alpha = F / actual
                win = skc.skc_model_window(cost, F, B, alpha)
                pred = skc.skc_model_project(cost, rows["cfg"]["density"], F, B, alpha)
                out[name] = dict(alpha=alpha, x_hi=win["x_hi"], x_lo=win["x_lo"],
                                 sparsity_window=[1 - win["x_hi"], 1 - win["x_lo"]],
                                 has_speedup_potential=win["has_speedup_potential"],
                                 speedup_at_cfg_measured=t_ref / t_layer,
                                 speedup_at_cfg_model=pred["speedup"])
            print(json.dumps(out), flush=True)
            del x


if __name__ == "__main__":
    main()
