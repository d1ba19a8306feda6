"""Roofline performance model, written from the paper -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md Sec. 2.2 "Analytical Performance Modeling" step by step, in fp64,
in the paper's notation:

    t_dense          = C / F
    t_sparse_compute = alpha * x * C / F
    t_sparse_bw      = (S_A + beta * x * S_W) / B
    speedup          = t_dense / max(t_sparse_compute, t_sparse_bw)

  * C   = FLOPs of the dense convolution, S_A = bytes of input+output activations,
    S_W = bytes of the weight tensor, "all without considering sparsity";
  * effective FLOP/s = C / t_sparse (dense-equivalent);
  * the density where t_sparse_compute = t_sparse_bw -- below it no
    further speedup ("upper bound of useful sparsity", called x_lo here, R9):
        x_lo = S_A / (alpha*C*B/F - beta*S_W)
  * "for x > 1/alpha ... sparse convolution becomes slower than dense":
        x_hi = 1/alpha.
Layer accounting (R8): per image, C = 2*K*(C_in/g)*R*S*Ho*Wo,
S_A = 4*(C_in*H*W + K*Ho*Wo) (input + output, unpadded), S_W = 4*K*(C_in/g)*R*S.
With amortised=True the weight bytes are divided by the batch (reported beside it).

Shares nothing with the product model in paper_1608_01409_b200/csrc/plan.cpp.
"""
from __future__ import annotations

import math


def layer_cost(K, C, R, S, H, W, stride=1, pad=0, groups=1, batch=1, amortised=False):
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (W + 2 * pad - S) // stride + 1
    flops = 2.0 * K * (C // groups) * R * S * Ho * Wo * batch
    s_a = 4.0 * batch * (C * H * W + K * Ho * Wo)
    s_w = 4.0 * K * (C // groups) * R * S
    if not amortised:
        s_w *= batch  # the paper's per-image shape: weights re-read for every image
    return dict(C=flops, S_A=s_a, S_W=s_w)


def project(cost, x, F, B, alpha, beta=2.0):
    if not (x > 0.0):
        raise ValueError("density x must be > 0")
    C, S_A, S_W = cost["C"], cost["S_A"], cost["S_W"]
    t_dense = C / F
    t_sc = alpha * x * C / F
    t_bw = (S_A + beta * x * S_W) / B
    t_sparse = max(t_sc, t_bw)
    return dict(t_dense=t_dense, t_sparse_compute=t_sc, t_sparse_bw=t_bw,
                t_sparse=t_sparse, speedup=t_dense / t_sparse,
                effective_flops=C / t_sparse, actual_flops=x * C / t_sparse)


def window(cost, F, B, alpha, beta=2.0):
    C, S_A, S_W = cost["C"], cost["S_A"], cost["S_W"]
    x_hi = 1.0 / alpha
    denom = alpha * C * B / F - beta * S_W
    if denom <= 0.0:
        return dict(x_lo=math.inf, x_hi=x_hi, has_speedup_potential=False)
    x_lo = S_A / denom
    # speedup at the crossover density (largest achievable); <= 1 means no benefit
    best = project(cost, min(x_lo, 1.0), F, B, alpha, beta)["speedup"]
    return dict(x_lo=x_lo, x_hi=x_hi, has_speedup_potential=bool(x_lo < x_hi and best > 1.0))
