"""CPU tests of the compiled-weights (JIT) kernel's host side: configuration, the emitted
code and its compilation -- no GPU needed.

skc_plan_verify decodes the emitted PTX of every channel block back to (k, c, r, s, w)
per output pixel (window loads -> shared-memory offsets -> taps; FFMA2 / FFMA -> weight
bits and accumulators) and requires each pixel of each output channel to see EXACTLY its
canonical CSR row in CSR order (Fig. 2, the order that makes the result
bitwise equal to the direct kernel's), plus the lane table (every output pixel stored
exactly once, tiles inside the image) and the shared-memory layout."""
import os

import numpy as np
import pytest

import workloads as wl
from paper_1608_01409_b200 import skc


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_1608_01409_b200 import build
    build.build()
    return skc.lib()


def pack_jit(w, layer):
    return skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                            skc.SKC_KERNEL_JIT)


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4])
def test_jit_code_decodes_to_csr_configs(cfg_id):
    cfg = wl.CONFIGS[cfg_id]
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, layer)
        plan = pack_jit(w, layer)
        info = plan.info()
        assert info["kernel"] == skc.SKC_KERNEL_JIT
        assert info["jit_compiled"] == 0  # configuration only; code is generated lazily
        skc.skc_plan_verify(plan)


def test_jit_random_geometries_verify():
    """Random layers (R, S in {1,2,3,5}, stride 1/2, groups, ragged K and C/g, empty
    channels): either a verified JIT plan or SKC_ERR_UNSUPPORTED (TMA alignment)."""
    rng = np.random.default_rng(5)
    n_ok = 0
    for it in range(160):
        layer = wl.random_layer(rng, max_c=32, max_hw=20, rs=(1, 2, 3, 5), groups=(1, 2, 4))
        w, _ = wl.random_tensors(rng, layer, 1)
        if it % 7 == 0:
            w[rng.integers(0, layer.K)] = 0.0
        if it % 11 == 0:
            w[:] = 0.0
        try:
            plan = pack_jit(w, layer)
        except skc.SkcError as e:
            assert e.status == -5, e
            continue
        skc.skc_plan_verify(plan)
        n_ok += 1
    assert n_ok >= 60, n_ok


def test_jit_aligned_random_geometries_verify():
    """C % 4 == 0 layers are always supported (whole-channel TMA runs stay 16-B aligned)."""
    rng = np.random.default_rng(6)
    for it in range(60):
        R = int(rng.choice([1, 3, 5]))
        g = int(rng.choice([1, 2]))
        C = g * 4 * int(rng.integers(1, 9))
        K = g * int(rng.integers(1, 48))
        H = int(rng.integers(R, 30))
        W = int(rng.integers(R, 30))
        st = int(rng.choice([1, 2]))
        layer = wl.Layer("a", K, C, H, W, R, R, st, (R - 1) // 2, g, float(rng.choice([0.0, 0.7, 0.95])), 1.0)
        w, _ = wl.random_tensors(rng, layer, 1)
        plan = pack_jit(w, layer)
        skc.skc_plan_verify(plan)


def test_jit_compile_on_host_and_cache(tmp_path, monkeypatch):
    """The whole toolchain (PTX generation, PTX compiler library, nvJitLink) runs on the host;
    a second plan with the same code hits the on-disk cache."""
    monkeypatch.setenv("SKC_JIT_CACHE", str(tmp_path))
    monkeypatch.delenv("SKC_JIT_NOCACHE", raising=False)
    layer = wl.Layer("c", 24, 16, 9, 9, 3, 3, 1, 1, 2, 0.8, 0.05)
    rng = np.random.default_rng(7)
    w, _ = wl.random_tensors(rng, layer, 1)
    p1 = pack_jit(w, layer)
    skc.skc_plan_compile(p1)
    i1 = p1.info()
    assert i1["jit_compiled"] == 1 and i1["jit_cache_hit"] == 0 and i1["code_bytes"] > 0
    assert len(os.listdir(tmp_path)) == 1
    p2 = pack_jit(w, layer)
    skc.skc_plan_compile(p2)
    i2 = p2.info()
    assert i2["jit_compiled"] == 1 and i2["jit_cache_hit"] == 1
    assert i2["code_bytes"] == i1["code_bytes"]
    # different weights -> different code
    w2 = w.copy()
    w2[w2 != 0] *= 2.0
    p3 = pack_jit(w2, layer)
    skc.skc_plan_compile(p3)
    assert p3.info()["jit_cache_hit"] == 0


def test_jit_unsupported_alignment_is_reported():
    """Odd planes with C % 4 != 0 cannot be staged by 16-B TMA runs: an explicit JIT request
    fails with SKC_ERR_UNSUPPORTED; AUTO falls back to another kernel."""
    layer = wl.Layer("u", 8, 3, 5, 5, 3, 3, 1, 1, 1, 0.5, 1.0)  # plane 7x7 = 49, C = 3
    rng = np.random.default_rng(8)
    w, _ = wl.random_tensors(rng, layer, 1)
    with pytest.raises(skc.SkcError) as e:
        pack_jit(w, layer)
    assert e.value.status == -5
    plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups)
    assert plan.info()["kernel"] != skc.SKC_KERNEL_JIT


def test_forward_into_geometry_errors():
    """skc_sparse_conv_forward_into checks the next plan's geometry before anything else:
    next C must be this K and next H x W this Ho x Wo (SKC_ERR_GEOMETRY otherwise)."""
    rng = np.random.default_rng(9)
    a = wl.Layer("a", 16, 8, 13, 13, 3, 3, 1, 1, 1, 0.5, 1.0)
    b_ok = wl.Layer("b", 8, 16, 13, 13, 3, 3, 1, 1, 1, 0.5, 1.0)
    b_bad_c = wl.Layer("c", 8, 12, 13, 13, 3, 3, 1, 1, 1, 0.5, 1.0)
    b_bad_hw = wl.Layer("d", 8, 16, 12, 13, 3, 3, 1, 1, 1, 0.5, 1.0)
    pa = skc.skc_pack_csr(wl.random_tensors(rng, a, 1)[0], 13, 13, 1, 1, 1)
    for bad in (b_bad_c, b_bad_hw):
        pb = skc.skc_pack_csr(wl.random_tensors(rng, bad, 1)[0], bad.H, bad.W, 1, 1, 1)
        st = skc.lib().skc_sparse_conv_forward_into(pa.handle, 16, pb.handle, 16, 2, None, 0, None)
        assert st == -2, st
    pb = skc.skc_pack_csr(wl.random_tensors(rng, b_ok, 1)[0], 13, 13, 1, 1, 1)
    # geometry fine, plan not uploaded -> SKC_ERR_STATE (no device work attempted)
    st = skc.lib().skc_sparse_conv_forward_into(pa.handle, 16, pb.handle, 16, 2, None, 0, None)
    assert st == -7, st


def test_padded_shape_per_layout():
    """The padded-input buffer shape follows the plan's layout: NCHW for direct plans,
    [ceil(N/2)][C][Hp][Wp][2] for pair-layout JIT plans (odd N rounds up)."""
    rng = np.random.default_rng(10)
    layer = wl.Layer("p", 8, 16, 13, 13, 3, 3, 1, 1, 1, 0.5, 1.0)
    w, _ = wl.random_tensors(rng, layer, 1)
    d = skc.skc_pack_csr(w, 13, 13, 1, 1, 1, skc.SKC_KERNEL_DIRECT).info()
    assert d["layout"] == skc.SKC_LAYOUT_NCHW and skc.padded_shape(d, 5) == (5, 16, 15, 15)
    j = skc.skc_pack_csr(w, 13, 13, 1, 1, 1, skc.SKC_KERNEL_JIT).info()
    if j["layout"] == skc.SKC_LAYOUT_PAIRS:
        assert skc.padded_shape(j, 5) == (3, 16, 15, 15, 2)
        assert skc.padded_shape(j, 6) == (3, 16, 15, 15, 2)


@pytest.mark.parametrize("knobs", [
    {"SKC_JIT_DYN": "1", "SKC_JIT_SPLIT": "2"},
    {"SKC_JIT_DYN": "1", "SKC_JIT_SPLIT": "9"},
    {"SKC_JIT_XPF": "1"},
    {"SKC_JIT_PMAJOR": "0"},
    {"SKC_JIT_PAIR": "0"},
])
def test_jit_scheduling_variants_verify(knobs, monkeypatch):
    """Tail split (halved blocks at the end of the queue), cross-item staging, code order and
    layout variants: every plan still decodes to exactly the CSR (skc_plan_verify checks that
    each output channel sits in exactly one block of its own group, and every block's code
    against its channels' CSR rows), and the split count is reported."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(8)
    n_ok = 0
    for it in range(40):
        layer = wl.random_layer(rng, max_c=32, max_hw=20, rs=(1, 3, 5), groups=(1, 2))
        w, _ = wl.random_tensors(rng, layer, 1)
        try:
            plan = pack_jit(w, layer)
        except skc.SkcError as e:
            assert e.status == -5, e
            continue
        skc.skc_plan_verify(plan)
        info = plan.info()
        if "SKC_JIT_SPLIT" in knobs:
            nbg = -(-layer.K // layer.groups // info["channels_per_warp"])  # even blocks per group
            assert 0 <= info["jit_split"] <= nbg
            assert info["jit_blocks"] >= layer.groups * nbg
        n_ok += 1
    assert n_ok >= 15, n_ok
