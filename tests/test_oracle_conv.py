"""Pins for the C oracle (oracle/oracle_conv.c) -- every check here compares it with
something OTHER than itself: a library routine (torch CPU float64 conv2d), a hand-derived
worked example, SPEC.md's printed examples, closed forms (delta kernel, all-ones input)
and invariants (linearity, sparse == zeroed-dense, bound properties).
SURVEY.md Sec. 8(c) pins P-O1 .. P-O7."""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workloads as wl


def torch_conv64(x, w, stride, pad, groups):
    """Library routine: PyTorch CPU conv2d in float64 (independent of oracle_conv.c)."""
    return F.conv2d(torch.from_numpy(x.astype(np.float64)), torch.from_numpy(w.astype(np.float64)),
                    stride=stride, padding=pad, groups=groups).numpy()


def test_worked_example(golden_dir):
    """P-O2: hand-derived 2x2 kernel [[1,0],[0,-1]] on 1..9 (tests/golden/worked_example_conv.json)."""
    g = json.load(open(os.path.join(golden_dir, "worked_example_conv.json")))
    x = np.array(g["input_1x1x3x3"], np.float32)
    w = np.array(g["weight_1x1x2x2"], np.float32)
    for case in g["cases"]:
        out, bound = oracle.conv2d_fp64(x, w, g["stride"], case["pad"], 1)
        np.testing.assert_array_equal(out, np.array(case["out"], np.float64))
        assert np.all(bound >= np.abs(out))


def test_spec_examples(golden_dir):
    """P-O3: SPEC.md:125-127 (1x1 w*v; 3x3 ones on ones = 9) and SPEC.md:134 (nnz=0 -> 0)."""
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for c in g["conv"]:
        w = np.ones((1, 1, 3, 3), np.float32) if c["w"] == "ones_1x1x3x3" else np.array(c["w"], np.float32)
        x = np.ones((1, 1, 3, 3), np.float32) if c["x"] == "ones_1x1x3x3" else np.array(c["x"], np.float32)
        out, _ = oracle.conv2d_fp64(x, w, c["stride"], c["pad"], 1)
        np.testing.assert_array_equal(out, np.array(c["out"], np.float64))
    x = np.random.default_rng(0).random((2, 3, 5, 5), dtype=np.float32)
    out, bound = oracle.conv2d_fp64(x, np.zeros((4, 3, 3, 3), np.float32), 1, 1, 1)
    assert not out.any() and not bound.any()


def test_identity_1x1():
    """identity 1x1 kernel (W(n,c)=delta_nc) reproduces the input exactly."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 5, 4, 6), dtype=np.float32)
    w = np.eye(5, dtype=np.float32).reshape(5, 5, 1, 1)
    out, _ = oracle.conv2d_fp64(x, w)
    np.testing.assert_array_equal(out, x.astype(np.float64))


@pytest.mark.parametrize("R,groups", [(3, 1), (5, 2), (1, 4), (3, 3)])
def test_delta_kernel(R, groups):
    """P-O4: K = C, odd R = S, p = (R-1)/2, W[k][cl][r][s] = [cl == k mod C/g][r==p][s==p]
    -> output equals input bitwise (one term times 1.0)."""
    rng = np.random.default_rng(R * 10 + groups)
    C = 12
    x = rng.standard_normal((2, C, 7, 9), dtype=np.float32)
    p = (R - 1) // 2
    w = np.zeros((C, C // groups, R, R), np.float32)
    for k in range(C):
        w[k, k % (C // groups), p, p] = 1.0
    out, _ = oracle.conv2d_fp64(x, w, 1, p, groups)
    np.testing.assert_array_equal(out, x.astype(np.float64))


def test_all_ones_interior_and_border():
    """P-O5 + reading R10: with an all-ones input, interior outputs equal the per-channel
    weight sum; border outputs equal the sum of only the in-bounds taps (hand-enumerated)."""
    rng = np.random.default_rng(2)
    K, C, H, W, R, S, p = 3, 4, 6, 7, 3, 3, 1
    w = rng.standard_normal((K, C, R, S)).astype(np.float32)
    x = np.ones((1, C, H, W), np.float32)
    out, _ = oracle.conv2d_fp64(x, w, 1, p, 1)
    wsum = w.astype(np.float64).sum(axis=(1, 2, 3))
    for k in range(K):
        np.testing.assert_allclose(out[0, k, 1:H - 1, 1:W - 1], wsum[k], rtol=1e-12)
        # top-left corner: taps r=0 and s=0 fall outside the image
        np.testing.assert_allclose(out[0, k, 0, 0], w[k, :, 1:, 1:].astype(np.float64).sum(), rtol=1e-12)
        # bottom edge (not a corner): taps r=2 fall outside
        np.testing.assert_allclose(out[0, k, H - 1, 3], w[k, :, :2, :].astype(np.float64).sum(), rtol=1e-12)


def test_linearity():
    """P-O6: conv(a*x + b*x') = a*conv(x) + b*conv(x')."""
    rng = np.random.default_rng(3)
    L = wl.Layer("t", 6, 4, 8, 8, 3, 3, 1, 1, 2, 0.5, 1.0)
    w, x = wl.random_tensors(rng, L, 2)
    _, x2 = wl.random_tensors(rng, L, 2)
    a, b = 0.75, -1.25
    lhs, _ = oracle.conv2d_fp64((a * x + b * x2).astype(np.float32), w, 1, 1, 2)
    o1, _ = oracle.conv2d_fp64(x, w, 1, 1, 2)
    o2, _ = oracle.conv2d_fp64(x2, w, 1, 1, 2)
    np.testing.assert_allclose(lhs, a * o1 + b * o2, rtol=1e-6, atol=1e-6)


def test_random_geometries_vs_torch_float64():
    """P-O1/P-O7: 300 random geometries (SPEC.md:159-163 ranges plus groups) against the
    library routine torch.nn.functional.conv2d in float64; also bound == conv(|w|,|x|)."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        L = wl.random_layer(rng, groups=(1, 2, 3))
        N = int(rng.integers(1, 3))
        w, x = wl.random_tensors(rng, L, N)
        out, bound = oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups)
        ref = torch_conv64(x, w, L.stride, L.pad, L.groups)
        assert out.shape == ref.shape, (L, out.shape, ref.shape)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
        refb = torch_conv64(np.abs(x), np.abs(w), L.stride, L.pad, L.groups)
        np.testing.assert_allclose(bound, refb, rtol=1e-12, atol=1e-12)


def test_config_shapes_vs_torch_sampled():
    """The oracle on real config geometries (groups = 2, 5x5, pad 2) for one image."""
    for cfg_id, li in [(2, 0), (2, 3), (4, 3)]:
        L = wl.CONFIGS[cfg_id].layers[li]
        w = wl.gen_weights(cfg_id, li, L)
        x = wl.gen_input(cfg_id, li, L, 0, 1)
        out, _ = oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups, want_bound=False)
        np.testing.assert_allclose(out, torch_conv64(x, w, L.stride, L.pad, L.groups),
                                   rtol=1e-11, atol=1e-12)


def test_pruning_equals_zeroing():
    """pruned weights == explicitly zeroed dense weights (same arithmetic)."""
    rng = np.random.default_rng(5)
    L = wl.Layer("t", 4, 4, 6, 6, 3, 3, 1, 1, 1, 0.0, 1.0)
    w, x = wl.random_tensors(rng, L, 1)
    mask = rng.random(w.shape) < 0.3
    wz = np.where(mask, w, 0).astype(np.float32)
    a, _ = oracle.conv2d_fp64(x, wz, 1, 1, 1)
    np.testing.assert_allclose(a, torch_conv64(x, wz, 1, 1, 1), rtol=1e-12, atol=1e-12)


def test_invalid_geometry():
    with pytest.raises(ValueError):
        oracle.conv2d_fp64(np.zeros((1, 2, 2, 2), np.float32), np.zeros((1, 2, 3, 3), np.float32))
