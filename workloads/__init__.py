"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This module holds ONLY shapes and random-number generation -- none of the method's
arithmetic (no convolution, no CSR, no padding).  It is the one module both the tests'
oracle calls and the product path are fed from (the oracle and the CUDA path never
import each other).

Shapes follow BASELINE.json "configs" (configs[0..4]); distributions follow the same
entries and DESIGN.md "Input recipe":
  * weights: N(0, sigma) with sigma a STANDARD DEVIATION (Caffe Gaussian filler
    convention; reading R4), times an i.i.d. Bernoulli(keep = 1 - sparsity)
    mask from its own stream (reading R5);
  * inputs: ReLU(N(0,1)) -- about half exact zeros (activation sparsity is not exploited);
  * seeds: numpy PCG64(SeedSequence([1608, 1409, cfg, layer, role, block])), role
    0 = weight values, 1 = mask, 2 = input; inputs are drawn per 64-image block
    (block = image // 64) so any image range -- a GPU shard, an oracle sample --
    regenerates bit-identical images independent of how the batch is split.
These stand in for the paper's pruned AlexNet weights and ImageNet activations
(PAPER.md:724-727), which are not available; uniform masks are the benign case for
load balance (the paper warns random matrices are not representative).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

BLOCK = 64  # images per input-seed block


@dataclass(frozen=True)
class Layer:
    name: str
    K: int          # output channels (the paper's N, SURVEY.md trap 0.1)
    C: int          # input channels
    H: int
    W: int
    R: int
    S: int
    stride: int
    pad: int
    groups: int
    sparsity: float  # fraction of weights pruned (density x = 1 - sparsity)
    sigma: float     # weight std

    @property
    def density(self) -> float:
        return 1.0 - self.sparsity

    @property
    def Ho(self) -> int:
        return (self.H + 2 * self.pad - self.R) // self.stride + 1

    @property
    def Wo(self) -> int:
        return (self.W + 2 * self.pad - self.S) // self.stride + 1

    def geometry(self) -> dict:
        return dict(K=self.K, C=self.C, R=self.R, S=self.S, H=self.H, W=self.W,
                    stride=self.stride, pad=self.pad, groups=self.groups)


@dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    batch: int
    layers: tuple = field(default_factory=tuple)


def _alex(name, K, C, HW, RS, pad, g, sp):
    return Layer(name, K, C, HW, HW, RS, RS, 1, pad, g, sp, 0.01)


def _resnet(C, HW):
    return Layer(f"res{C}_{HW}x{HW}", C, C, HW, HW, 3, 3, 1, 1, 1, 0.70,
                 math.sqrt(2.0 / (9.0 * C)))


ALEXNET = (
    _alex("conv2", 256, 96, 27, 5, 2, 2, 0.85),
    _alex("conv3", 384, 256, 13, 3, 1, 1, 0.93),
    _alex("conv4", 384, 384, 13, 3, 1, 2, 0.91),
    _alex("conv5", 256, 384, 13, 3, 1, 2, 0.88),
)

SWEEP = (0.0, 0.50, 0.70, 0.80, 0.85, 0.90, 0.95, 0.98)

CONFIGS = {
    1: Config(1, "conv3_b1_s80", 1, (_alex("conv3", 384, 256, 13, 3, 1, 1, 0.80),)),
    2: Config(2, "alexnet_conv2-5_b256", 256, ALEXNET),
    3: Config(3, "conv3_sweep_b256", 256,
              tuple(_alex(f"conv3_s{int(round(s * 100)):02d}", 384, 256, 13, 3, 1, 1, s)
                    for s in SWEEP)),
    4: Config(4, "resnet50_3x3_b256_s70", 256,
              (_resnet(64, 56), _resnet(128, 28), _resnet(256, 14), _resnet(512, 7))),
    5: Config(5, "alexnet_conv2-5_b4096_sharded", 4096, ALEXNET),
}


@dataclass(frozen=True)
class FCLayer:
    name: str
    M: int          # outputs
    K: int          # inputs
    sparsity: float
    sigma: float

    @property
    def density(self) -> float:
        return 1.0 - self.sparsity


# Row f2 (not a BASELINE config): AlexNet's fully connected layers fc6-fc8 at batch 256,
# element-wise pruned to 90% (a round synthetic value; the paper gives no FC sparsities).
ALEXNET_FC = (FCLayer("fc6", 4096, 9216, 0.90, 0.005), FCLayer("fc7", 4096, 4096, 0.90, 0.005),
              FCLayer("fc8", 1000, 4096, 0.90, 0.01))
FC_BATCH = 256
FC_CFG_ID = 6


def gen_fc_weights(layer_idx: int, L: FCLayer) -> np.ndarray:
    w = _rng(FC_CFG_ID, layer_idx, 0).standard_normal((L.M, L.K), dtype=np.float32) * np.float32(L.sigma)
    keep = _rng(FC_CFG_ID, layer_idx, 1).random((L.M, L.K), dtype=np.float64) < L.density
    return np.where(keep, w, np.float32(0.0)).astype(np.float32)


def gen_fc_input(layer_idx: int, L: FCLayer, batch: int) -> np.ndarray:
    """X [K x B] (batch-minor), ReLU(N(0,1))."""
    x = _rng(FC_CFG_ID, layer_idx, 2).standard_normal((L.K, batch), dtype=np.float32)
    return np.maximum(x, np.float32(0.0))


def _rng(cfg_id: int, layer: int, role: int, block: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([1608, 1409, int(cfg_id), int(layer), int(role), int(block)])))


def gen_weights(cfg_id: int, layer_idx: int, L: Layer) -> np.ndarray:
    """Pruned dense weights, float32 [K, C/g, R, S]."""
    shape = (L.K, L.C // L.groups, L.R, L.S)
    w = (_rng(cfg_id, layer_idx, 0).standard_normal(shape, dtype=np.float32)
         * np.float32(L.sigma))
    keep = _rng(cfg_id, layer_idx, 1).random(shape, dtype=np.float64) < L.density
    return np.where(keep, w, np.float32(0.0)).astype(np.float32)


def gen_weights_skewed(cfg_id: int, layer_idx: int, L: Layer, spread: float = 1.0) -> np.ndarray:
    """Row f4 stress input: like gen_weights, but each output channel k keeps its weights with
    its own probability x_k = density * LogNormal(0, spread) / mean (clipped to [0, 1]), so
    per-channel nnz is heavily skewed at the same average density."""
    shape = (L.K, L.C // L.groups, L.R, L.S)
    w = (_rng(cfg_id, layer_idx, 0).standard_normal(shape, dtype=np.float32)
         * np.float32(L.sigma))
    z = _rng(cfg_id, layer_idx, 3).lognormal(0.0, spread, L.K)
    xk = np.clip(L.density * z / z.mean(), 0.0, 1.0)
    keep = _rng(cfg_id, layer_idx, 1).random(shape, dtype=np.float64) < xk[:, None, None, None]
    return np.where(keep, w, np.float32(0.0)).astype(np.float32)


def gen_input(cfg_id: int, layer_idx: int, L: Layer, n0: int, n1: int) -> np.ndarray:
    """Images [n0, n1) of the layer's input, float32 NCHW, ReLU(N(0,1))."""
    n0, n1 = int(n0), int(n1)
    out = np.empty((max(n1 - n0, 0), L.C, L.H, L.W), dtype=np.float32)
    if n1 <= n0:
        return out
    for b in range(n0 // BLOCK, (n1 - 1) // BLOCK + 1):
        blk = _rng(cfg_id, layer_idx, 2, b).standard_normal((BLOCK, L.C, L.H, L.W),
                                                            dtype=np.float32)
        np.maximum(blk, np.float32(0.0), out=blk)
        lo, hi = max(n0, b * BLOCK), min(n1, (b + 1) * BLOCK)
        out[lo - n0:hi - n0] = blk[lo - b * BLOCK:hi - b * BLOCK]
    return out


def random_layer(rng: np.random.Generator, max_c=8, max_hw=9, rs=(1, 2, 3, 5),
                 strides=(1, 2), pads=(0, 1, 2), groups=(1, 2), densities=(1.0, .5, .1, .01)):
    """A random small geometry for property / parity sweeps (SPEC.md:159-163 ranges)."""
    while True:
        g = int(rng.choice(groups))
        C = g * int(rng.integers(1, max_c // g + 1))
        K = g * int(rng.integers(1, max_c // g + 1))
        R = int(rng.choice(rs)); S = int(rng.choice(rs))
        H = int(rng.integers(1, max_hw + 1)); W = int(rng.integers(1, max_hw + 1))
        st = int(rng.choice(strides)); p = int(rng.choice(pads))
        if H + 2 * p >= R and W + 2 * p >= S:
            x = float(rng.choice(densities))
            return Layer("rand", K, C, H, W, R, S, st, p, g, 1.0 - x, 1.0)


def random_tensors(rng: np.random.Generator, L: Layer, N: int):
    """Weights N(0,1)*Bernoulli(density) and ReLU(N(0,1)) input for a random layer."""
    w = rng.standard_normal((L.K, L.C // L.groups, L.R, L.S), dtype=np.float32)
    w = np.where(rng.random(w.shape) < L.density, w, np.float32(0)).astype(np.float32)
    x = np.maximum(rng.standard_normal((N, L.C, L.H, L.W), dtype=np.float32), 0)
    return w, x.astype(np.float32)


def with_batch(cfg: Config, batch: int) -> Config:
    return replace(cfg, batch=int(batch))
