"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every symbol
include/skc.h declares, its host packer is BIT-EXACT against the independent NumPy packer
(oracle/ref_pack.py) on every config and on random geometries, its model agrees with the
oracle model, and its argument/geometry errors come back as the documented statuses."""
import os
import re

import numpy as np
import pytest

import workloads as wl
from oracle import ref_model
from oracle.ref_pack import ref_pack
from paper_1608_01409_b200 import skc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1608_01409_b200 import build
    build.build()
    return skc.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "skc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//.*", "", src)
    return sorted(set(re.findall(r"\b(skc_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), f"libskc.so does not export {s}"
    assert sorted(skc.EXPORTS) == syms


def assert_pack_equal(plan, ref):
    rp, ci, va = plan.csr()
    np.testing.assert_array_equal(rp, ref["rowptr"])
    np.testing.assert_array_equal(ci, ref["colidx"])
    np.testing.assert_array_equal(va.view(np.uint32), ref["values"].view(np.uint32))
    np.testing.assert_array_equal(plan.perm(), ref["perm"])


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4])
def test_pack_bit_exact_configs(L, cfg_id):
    """P-P6 on every BASELINE config layer (config 5 uses config 2's layers)."""
    cfg = wl.CONFIGS[cfg_id]
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, layer)
        plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups)
        assert_pack_equal(plan, ref_pack(w, layer.H, layer.W, layer.pad, layer.groups))
        info = plan.info()
        assert info["nnz"] == np.count_nonzero(w)
        assert (info["Ho"], info["Wo"]) == (layer.Ho, layer.Wo)


def test_pack_bit_exact_random(L):
    """P-P6: 1000 random geometries incl. groups, empty rows, signed zeros, strides."""
    rng = np.random.default_rng(7)
    for it in range(1000):
        layer = wl.random_layer(rng, max_c=12, groups=(1, 2, 3, 4))
        w, _ = wl.random_tensors(rng, layer, 1)
        if it % 7 == 0:
            w[rng.random(w.shape) < 0.5] = -0.0
        plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups)
        assert_pack_equal(plan, ref_pack(w, layer.H, layer.W, layer.pad, layer.groups))


def test_layout_offset_hook(L):
    """SPEC.md:49-51 through the C-ABI test hook, plus out-of-range = -1."""
    plan = skc.skc_pack_csr(np.ones((1, 2, 1, 1), np.float32), 3, 3, 1, 0, 1)
    assert skc.skc_layout_offset(plan, 1, 2, 1) == 16
    assert skc.skc_layout_offset(plan, 0, 0, 0) == 0
    assert skc.skc_layout_offset(plan, 2, 0, 0) == -1
    plan = skc.skc_pack_csr(np.ones((1, 2, 1, 1), np.float32), 3, 3, 1, 1, 1)  # Hp=Wp=5
    assert skc.skc_layout_offset(plan, 1, 4, 4) == (1 * 5 + 4) * 5 + 4
    assert skc.skc_layout_offset(plan, 0, 5, 0) == -1


def test_errors(L):
    w = np.ones((4, 2, 3, 3), np.float32)
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pack_csr(w, 5, 5, 1, 1, groups=3)       # K, C not divisible by 3
    assert e.value.status == -2
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pack_csr(w, 1, 1, 1, 0, 1)              # 3x3 kernel on 1x1 input, no pad
    assert e.value.status == -2
    bad = w.copy(); bad[1, 0, 2, 2] = np.nan
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pack_csr(bad, 5, 5, 1, 1, 1)
    assert e.value.status == -3
    bad[1, 0, 2, 2] = np.inf
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pack_csr(bad, 5, 5, 1, 1, 1)
    assert e.value.status == -3
    with pytest.raises(skc.SkcError) as e:                # C*Hp*Wp >= 2^31
        skc.skc_pack_csr(np.ones((1, 1, 1, 1), np.float32), 50000, 50000, 1, 0, 1)
    assert e.value.status == -4
    plan = skc.skc_pack_csr(w, 5, 5, 1, 1, 1)
    # forward before upload -> STATE; negative N -> ARG (both before any CUDA call)
    with pytest.raises(skc.SkcError) as e:
        skc.skc_sparse_conv_forward(plan, 16, 16, 1, 0)
    assert e.value.status == -7
    with pytest.raises(skc.SkcError) as e:
        skc.skc_sparse_conv_forward(plan, 16, 16, -1, 0)
    assert e.value.status == -1
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pad_input(plan, 16, 16, -2, 0)
    assert e.value.status == -1
    skc.skc_pad_input(plan, 0, 0, 0, 0)                  # N = 0 is a no-op
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pad_input(plan, 8, 16, 1, 0)             # misaligned device pointer
    assert e.value.status == -6


def test_plan_info_configuration(L):
    """Kernel configurations for the AlexNet layers: the direct kernel's tiling covers every
    output pixel with full-image slabs; AUTO picks the compiled-weights (JIT) kernel, whose
    lanes x images cover the CTA's images and whose staging fits shared memory."""
    for li, layer in enumerate(wl.ALEXNET):
        w = wl.gen_weights(2, li, layer)
        info = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                skc.SKC_KERNEL_DIRECT).info()
        assert info["kernel"] == skc.SKC_KERNEL_DIRECT
        assert info["smem_bytes"] <= 227 * 1024
        assert info["pixels_per_lane"] * 32 * -(-layer.Ho // info["band_rows"]) >= layer.Ho * layer.Wo
        info = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups).info()
        assert info["kernel"] == skc.SKC_KERNEL_JIT
        assert info["smem_bytes"] <= 227 * 1024
        ty = -(-layer.Ho // info["tile_h"])
        band_rows = -(-ty // info["bands"])  # tile rows of the largest row band
        tiles = band_rows * -(-layer.Wo // info["tile_w"])
        per_lane = 2 if info["layout"] == skc.SKC_LAYOUT_PAIRS else 1  # images per lane tile
        assert tiles * info["images_per_cta"] <= info["warps"] * 32 * per_lane
        assert info["jit_blocks"] * info["channels_per_warp"] >= layer.K


@pytest.mark.parametrize("li", range(4))
def test_model_matches_oracle_model(L, li):
    """a7: the C++ model equals the oracle model (both written from PAPER.md Sec. 2.2)."""
    layer = wl.ALEXNET[li]
    g = layer.geometry()
    for batch, am in [(1, False), (256, False), (256, True)]:
        c = skc.skc_model_layer_cost(**g, batch=batch, amortised=am)
        r = ref_model.layer_cost(**g, batch=batch, amortised=am)
        assert c == pytest.approx(r, rel=1e-15)
        for F, B, a in [(2.15e12, 1.22e11, 3.0), (6.2e10, 1.5e10, 1.2), (6e13, 6.5e12, 4.0)]:
            for x in (0.01, 0.07, 0.3, 1.0):
                p = skc.skc_model_project(c, x, F, B, a)
                q = ref_model.project(r, x, F, B, a)
                for key in q:
                    assert p[key] == pytest.approx(q[key], rel=1e-13), key
            wc, wr = skc.skc_model_window(c, F, B, a), ref_model.window(r, F, B, a)
            assert wc["x_hi"] == pytest.approx(wr["x_hi"]) and wc["x_lo"] == pytest.approx(wr["x_lo"])
            assert wc["has_speedup_potential"] == wr["has_speedup_potential"]


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4])
def test_plan_verify_configs(L, cfg_id):
    """Every config layer, both kernels: kernel-private indices in bounds, the kernel streams
    decode exactly to the canonical CSR, every output written exactly once."""
    cfg = wl.CONFIGS[cfg_id]
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, layer)
        for kern in (skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT, skc.SKC_KERNEL_REGTILE):
            try:
                plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad,
                                        layer.groups, kern)
            except skc.SkcError as e:
                assert kern == skc.SKC_KERNEL_REGTILE and e.status == -5
                continue
            skc.skc_plan_verify(plan)


def test_plan_verify_random(L):
    """400 random geometries (strides, groups, ragged sizes, empty rows), both kernels."""
    rng = np.random.default_rng(21)
    n_rt = 0
    for it in range(400):
        if it % 2:
            layer = wl.random_layer(rng, max_c=24, max_hw=30, rs=(1, 2, 3, 5), groups=(1, 2, 4))
        else:  # register-tile friendly: 3x3 / 5x5, stride 1, TMA-aligned planes
            R = int(rng.choice([3, 5]))
            g = int(rng.choice([1, 2]))
            layer = wl.Layer("rt", g * int(rng.integers(1, 30)), g * 4 * int(rng.integers(1, 7)),
                             int(rng.integers(1, 40)), int(rng.integers(1, 40)), R, R, 1,
                             (R - 1) // 2, g, float(rng.choice([0.0, 0.5, 0.9, 0.98])), 1.0)
        w, _ = wl.random_tensors(rng, layer, 1)
        if it % 9 == 0:
            w[rng.integers(0, layer.K)] = 0.0
        for kern in (skc.SKC_KERNEL_DIRECT, skc.SKC_KERNEL_REGTILE):
            try:
                plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad,
                                        layer.groups, kern)
            except skc.SkcError as e:
                assert kern == skc.SKC_KERNEL_REGTILE and e.status == -5, e
                continue
            n_rt += kern == skc.SKC_KERNEL_REGTILE
            skc.skc_plan_verify(plan)
    assert n_rt >= 20


def test_batch_hint_configurations(L):
    """skc_pack_csr_batch: the configuration follows the batch the plan is packed for (DESIGN.md
    Sec. 7.5): AUTO takes the direct kernel below 16 images per call and the compiled-weights
    kernel from 16 up; a batch hint never changes the canonical CSR (bit-exact against the
    independent packer for every hint); small-batch direct configurations stage no more images
    per CTA than the batch has and pass the plan's static self-check on random geometries."""
    cfg = wl.CONFIGS[2]
    L = cfg.layers[1]
    w = wl.gen_weights(2, 1, L)
    with pytest.raises(skc.SkcError) as e:
        skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_AUTO, 0)
    assert e.value.status == -1
    ref = ref_pack(w, L.H, L.W, L.pad, L.groups)
    for hint, kern in ((1, skc.SKC_KERNEL_DIRECT), (2, skc.SKC_KERNEL_DIRECT), (15, skc.SKC_KERNEL_DIRECT),
                       (16, skc.SKC_KERNEL_JIT), (256, skc.SKC_KERNEL_JIT), (4096, skc.SKC_KERNEL_JIT)):
        plan = skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_AUTO, hint)
        info = plan.info()
        assert info["kernel"] == kern, (hint, info["kernel"])
        assert info["images_per_cta"] <= max(2, hint) or kern == skc.SKC_KERNEL_JIT
        assert_pack_equal(plan, ref)
        skc.skc_plan_verify(plan)
    rng = np.random.default_rng(23)
    for it in range(60):
        layer = wl.random_layer(rng, max_c=24, max_hw=30, rs=(1, 3, 5), groups=(1, 2))
        w, _ = wl.random_tensors(rng, layer, 1)
        for hint in (1, 3):
            plan = skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                    skc.SKC_KERNEL_AUTO, hint)
            assert plan.info()["kernel"] == skc.SKC_KERNEL_DIRECT
            assert plan.info()["images_per_cta"] <= hint + (hint % 2)
            skc.skc_plan_verify(plan)


def test_library_never_allocates_device_memory():
    """skc.h: libskc never allocates device memory -- PyTorch owns every buffer (workspace,
    activations, tuning scratch).  No allocation call may appear in the library's sources."""
    import glob
    import re
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_1608_01409_b200", "csrc")
    bad = re.compile(r"\b(cudaMalloc\w*|cuMemAlloc\w*|cudaMallocAsync|cudaHostAlloc|cudaMallocManaged)\s*\(")
    hits = []
    for path in glob.glob(os.path.join(root, "*")):
        for n, line in enumerate(open(path, errors="replace"), 1):
            if bad.search(line):
                hits.append(f"{os.path.basename(path)}:{n}: {line.strip()}")
    assert not hits, hits
