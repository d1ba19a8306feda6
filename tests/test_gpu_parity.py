"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs.  Tolerance (BASELINE.json north_star): per output element
|gpu - oracle| <= 1e-4 * sum|w*x|, and exactly 0 where that sum is 0.  Packing is bit-exact
(tests/test_abi.py); the pad kernel is bitwise equal to numpy.pad."""
import os
import numpy as np
import pytest

import oracle
import workloads as wl
from paper_1608_01409_b200 import skc

pytestmark = pytest.mark.gpu
TOL = 1e-4

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1608_01409_b200 import build
    build.build()
    skc.lib()
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False


def run_gpu(w, x, layer, kernel=skc.SKC_KERNEL_AUTO, xp_out=False):
    conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                       layer.groups, kernel)
    skc.skc_plan_verify(conv.plan)
    xd = torch.from_numpy(x).cuda()
    xp = torch.empty(conv.padded_shape(x.shape[0]), device="cuda")
    out = conv.forward(xd, xp=xp)
    torch.cuda.synchronize()
    if xp_out:
        return out.cpu().numpy(), xp.cpu().numpy(), conv
    return out.cpu().numpy(), conv


def check(out, ref, bound, what=""):
    assert out.shape == ref.shape, (what, out.shape, ref.shape)
    err = np.abs(out.astype(np.float64) - ref)
    zero = bound == 0
    assert np.all(out[zero] == 0), f"{what}: nonzero where sum|wx| = 0"
    ratio = np.where(zero, 0.0, err / np.where(zero, 1.0, bound))
    worst = float(ratio.max()) if ratio.size else 0.0
    assert worst <= TOL, f"{what}: max err/sum|wx| = {worst:.3e}"
    return worst


@pytest.mark.parametrize("layout", ["nchw", "pairs", "pairs_flat"])
def test_pad_bitwise_numpy(layout, monkeypatch):
    """a2 vs the library routine numpy.pad, ragged sizes and pads; for the
    image-pair layout of JIT plans, de-interleaving must give numpy.pad bit for bit and an
    odd batch's missing second image must be zeros.  (The JIT configuration may pick either
    layout for a tiny layer; the pair cases force the pair layout; both pair-pad kernels --
    the per-pair grid (default) and the flat one -- are checked.)"""
    if layout.startswith("pairs"):
        monkeypatch.setenv("SKC_JIT_PAIR", "1")
        monkeypatch.setenv("SKC_PAD_FLAT", "1" if layout == "pairs_flat" else "0")
        layout = "pairs"
    rng = np.random.default_rng(0)
    kern = skc.SKC_KERNEL_DIRECT if layout == "nchw" else skc.SKC_KERNEL_JIT
    for (N, C, H, W, p) in [(1, 4, 1, 1, 1), (3, 8, 7, 9, 2), (2, 96, 27, 27, 2), (4, 256, 13, 13, 1),
                            (2, 4, 5, 4, 0), (1, 64, 56, 56, 1), (65, 4, 3, 3, 3), (5, 2, 3, 3, 1),
                            (7, 12, 40, 40, 2), (3, 4, 14, 14, 1)]:
        x = rng.standard_normal((N, C, H, W), dtype=np.float32)
        x[0, 0, 0, 0] = -0.0
        try:
            plan = skc.skc_pack_csr(np.ones((1, C, 1, 1), np.float32), H, W, 1, p, 1, kern)
        except skc.SkcError as e:
            assert e.status == -5
            continue
        info = plan.info()
        assert info["layout"] == (skc.SKC_LAYOUT_NCHW if layout == "nchw" else skc.SKC_LAYOUT_PAIRS)
        xd = torch.from_numpy(x).cuda()
        xp = torch.full(skc.padded_shape(info, N), float("nan"), device="cuda")
        skc.skc_pad_input(plan, xd, xp, N)
        torch.cuda.synchronize()
        if layout == "pairs":
            full = xp.movedim(-1, 1).reshape(-1, C, H + 2 * p, W + 2 * p).cpu().numpy()
            if N % 2:
                assert not full[N].any(), "missing second image must be zero"
            got = full[:N]
        else:
            got = xp.cpu().numpy()
        np.testing.assert_array_equal(got.view(np.uint32), oracle.pad_ref(x, p).view(np.uint32))


def test_worked_example_gpu(golden_dir):
    import json, os
    g = json.load(open(os.path.join(golden_dir, "worked_example_conv.json")))
    x = np.array(g["input_1x1x3x3"], np.float32)
    w = np.array(g["weight_1x1x2x2"], np.float32)
    for case in g["cases"]:
        layer = wl.Layer("we", 1, 1, 3, 3, 2, 2, 1, case["pad"], 1, 0.0, 1.0)
        out, _ = run_gpu(w, x, layer)
        np.testing.assert_array_equal(out, np.array(case["out"], np.float32))


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_random_geometries(kernel):
    """SPEC.md:159-163 property suite ranges (+ groups, stride 2): >= 200 random layers."""
    rng = np.random.default_rng(1)
    worst = 0.0
    cases = []
    for it in range(220):
        layer = wl.random_layer(rng, max_c=32, max_hw=16, rs=(1, 2, 3, 5), groups=(1, 2, 4))
        N = int(rng.integers(1, 4))
        w, x = wl.random_tensors(rng, layer, N)
        cases.append((layer, w, x))
    if kernel == skc.SKC_KERNEL_AUTO:
        prewarm_jit([(layer, w) for layer, w, _ in cases], kernel)
    for it, (layer, w, x) in enumerate(cases):
        out, _ = run_gpu(w, x, layer, kernel)
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        worst = max(worst, check(out, ref, bound, f"it{it} {layer}"))
    print("max err/bound", worst)


def test_regtile_random_shapes():
    """The register-tiled kernel forced on random 3x3 / 5x5 stride-1 layers whose padded
    planes keep the TMA copies aligned: ragged K (not a multiple of M), C/g not a multiple
    of the chunk, batches that are not a multiple of the images per CTA, tiles that
    overhang the output, several lane groups, empty channels."""
    rng = np.random.default_rng(11)
    n_rt = 0
    for it in range(120):
        R = int(rng.choice([3, 5]))
        g = int(rng.choice([1, 2]))
        C = g * 4 * int(rng.integers(1, 9))
        K = g * int(rng.integers(1, 40))
        H = int(rng.integers(R - 2 if R > 2 else 1, 40))
        W = int(rng.integers(R - 2 if R > 2 else 1, 40))
        pad = (R - 1) // 2
        x_keep = float(rng.choice([1.0, 0.5, 0.1, 0.02]))
        layer = wl.Layer("rt", K, C, H, W, R, R, 1, pad, g, 1.0 - x_keep, 1.0)
        if layer.Ho < 1 or layer.Wo < 1:
            continue
        N = int(rng.integers(1, 12))
        w, x = wl.random_tensors(rng, layer, N)
        if it % 5 == 0:
            w[rng.integers(0, K)] = 0.0
        try:
            out, conv = run_gpu(w, x, layer, skc.SKC_KERNEL_REGTILE)
        except skc.SkcError as e:
            assert e.status == -5, e  # unsupported tiling only
            continue
        assert conv.geom["kernel"] == skc.SKC_KERNEL_REGTILE
        n_rt += 1
        ref, bound = oracle.conv2d_fp64(x, w, 1, pad, g)
        check(out, ref, bound, f"regtile it{it} {layer} {conv.geom}")
    assert n_rt >= 80, n_rt


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_tiles_and_ragged_tails(kernel):
    """Shapes spanning several channel blocks, stages, bands and lane tails."""
    rng = np.random.default_rng(2)
    cases = [
        wl.Layer("a", 40, 36, 13, 13, 3, 3, 1, 1, 1, 0.9, 1.0),     # K not multiple of 32
        wl.Layer("b", 70, 50, 27, 27, 5, 5, 1, 2, 2, 0.85, 1.0),    # odd C/g, 2 bands
        wl.Layer("c", 33, 17, 31, 29, 3, 3, 2, 1, 1, 0.5, 1.0),     # stride 2
        wl.Layer("d", 64, 64, 56, 56, 3, 3, 1, 1, 1, 0.7, 1.0),     # many bands
        wl.Layer("e", 24, 96, 7, 7, 3, 3, 1, 1, 1, 0.7, 1.0),       # 49 pixels, tiny T
        wl.Layer("f", 16, 8, 40, 3, 3, 3, 1, 1, 1, 0.5, 1.0),       # tall and narrow
        wl.Layer("g", 8, 4, 5, 70, 1, 7, 1, 3, 1, 0.3, 1.0),        # wide rows, 1x7 kernel
    ]
    for layer in cases:
        w, x = wl.random_tensors(rng, layer, 3)
        out, conv = run_gpu(w, x, layer, kernel)
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        check(out, ref, bound, f"{layer} {conv.geom}")


def test_edge_cases():
    rng = np.random.default_rng(3)
    layer = wl.Layer("z", 20, 12, 9, 9, 3, 3, 1, 1, 2, 0.0, 1.0)
    _, x = wl.random_tensors(rng, layer, 2)
    # all-zero weights -> exactly zero output
    out, _ = run_gpu(np.zeros((20, 6, 3, 3), np.float32), x, layer)
    assert not out.any()
    # single nonzero weight
    w = np.zeros((20, 6, 3, 3), np.float32)
    w[13, 4, 0, 2] = 1.5
    out, _ = run_gpu(w, x, layer)
    ref, bound = oracle.conv2d_fp64(x, w, 1, 1, 2)
    check(out, ref, bound, "single nnz")
    # some channels with nnz = 0 among dense ones, x = 1
    w = rng.standard_normal((20, 6, 3, 3)).astype(np.float32)
    w[[0, 5, 19]] = 0
    out, _ = run_gpu(w, x, layer)
    ref, bound = oracle.conv2d_fp64(x, w, 1, 1, 2)
    check(out, ref, bound, "empty rows")
    # N = 0 is a no-op
    conv = skc.SparseConv2d.from_dense(w, 9, 9, 1, 1, 2)
    skc.skc_sparse_conv_forward(conv.plan, 0, 0, 0)


def test_dense_equals_torch_conv2d_fp32():
    """P-O7: at 0% sparsity the sparse path equals torch conv2d in FP32 (TF32 off)."""
    rng = np.random.default_rng(4)
    layer = wl.Layer("d", 48, 32, 13, 13, 3, 3, 1, 1, 2, 0.0, 1.0)
    w, x = wl.random_tensors(rng, layer, 4)
    out, _ = run_gpu(w, x, layer)
    ref, bound = oracle.conv2d_fp64(x, w, 1, 1, 2)
    check(out, ref, bound, "dense")
    t = torch.nn.functional.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                                   padding=1, groups=2).cpu().numpy()
    check(t, ref, bound, "torch fp32")  # the library routine passes the same bar
    assert np.max(np.abs(out - t) / np.maximum(bound, 1e-30)) <= 2 * TOL


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_determinism_and_host_path(kernel):
    rng = np.random.default_rng(5)
    layer = wl.CONFIGS[2].layers[1]
    w = wl.gen_weights(2, 1, layer)
    x = wl.gen_input(2, 1, layer, 0, 8)
    conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                       kernel)
    xd = torch.from_numpy(x).cuda()
    a = conv.forward(xd).cpu().numpy()
    b = conv.forward(xd).cpu().numpy()
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
    # end-to-end host-buffer entry point (chunk-pipelined over 2 copy streams, ragged last
    # chunk) gives the same bits as the device path
    n = 37
    x2 = wl.gen_input(2, 1, layer, 0, n)
    ref = conv.forward(torch.from_numpy(x2).cuda()).cpu().numpy()
    h_in = torch.from_numpy(x2).pin_memory()
    h_out = torch.full(conv.out_shape(n), float("nan")).pin_memory()
    d_in = torch.empty(x2.shape, device="cuda")
    d_pad = torch.empty(conv.padded_shape(n), device="cuda")
    d_out = torch.empty(conv.out_shape(n), device="cuda")
    skc.skc_forward_host(conv.plan, h_in, h_out, n, d_in, d_pad, d_out)
    torch.cuda.current_stream().synchronize()
    np.testing.assert_array_equal(h_out.numpy().view(np.uint32), ref.view(np.uint32))
    np.testing.assert_array_equal(ref[:8].view(np.uint32), a.view(np.uint32))
    del rng


def sample_images(N, rng, k):
    idx = {0, N - 1}
    while len(idx) < min(k, N):
        idx.add(int(rng.integers(0, N)))
    return sorted(idx)


@pytest.mark.parametrize("cfg_id", [1, 2, 3, 4])
def test_config_parity_full_batch(cfg_id):
    """Every BASELINE config layer (configs 1-4, all 8 config-3 sparsity points) at its FULL
    batch, EVERY image checked against the fp64 oracle (full-batch
    oracle where host time allows -- about a minute of the box's cores), for the AUTO plan
    in the launch configuration bench.py times (tuned for the batch) and for the direct
    kernel; the oracle runs once per layer and serves both."""
    cfg = wl.CONFIGS[cfg_id]
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, layer)
        x = wl.gen_input(cfg_id, li, layer, 0, cfg.batch)
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        for kernel in (skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT):
            conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                               layer.groups, kernel)
            skc.skc_plan_verify(conv.plan)
            if kernel == skc.SKC_KERNEL_AUTO:
                conv.tune(cfg.batch)
            out = conv.forward(torch.from_numpy(x).cuda()).cpu().numpy()
            check(out, ref, bound, f"cfg{cfg_id} {layer.name} kernel {conv.geom['kernel']}")
            del out, conv
        del ref, bound


def test_small_batch_plans_vs_oracle():
    """Plans packed for small batches (skc_pack_csr_batch): AUTO's direct launch-time
    configurations below 16 images and the compiled-weights kernel from 16 up,
    every image checked against the fp64 oracle -- at the batch the plan was packed for, odd
    batches included, and at other batches (a configuration is a performance choice only)."""
    cases = [(1, 0), (2, 0), (2, 1), (4, 0)]
    for cfg_id, li in cases:
        cfg = wl.CONFIGS[cfg_id]
        layer = cfg.layers[li]
        w = wl.gen_weights(cfg_id, li, layer)
        x = wl.gen_input(cfg_id, li, layer, 0, 13)
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        for hint, Ns in ((1, (1, 6)), (2, (2,)), (3, (3, 1)), (5, (5, 13)), (8, (8, 3)), (13, (13,)),
                         (16, (13, 2))):
            conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                               layer.groups, batch_hint=hint)
            assert conv.geom["kernel"] == (skc.SKC_KERNEL_DIRECT if hint < 16 else skc.SKC_KERNEL_JIT)
            for N in Ns:
                out = conv.forward(torch.from_numpy(x[:N]).cuda()).cpu().numpy()
                check(out, ref[:N], bound[:N], f"cfg{cfg_id} {layer.name} hint {hint} N {N}")
            del conv


def test_small_batch_random_geometries():
    """Direct small-batch configurations (AUTO below 16 images) on 120 random layers (strides,
    groups, 1x1 to 5x5, ragged sizes, empty channels) at the batch they were packed for and at
    another one, every output against the fp64 oracle."""
    rng = np.random.default_rng(31)
    worst = 0.0
    for it in range(120):
        layer = wl.random_layer(rng, max_c=32, max_hw=20, rs=(1, 2, 3, 5), groups=(1, 2, 4))
        hint = int(rng.integers(1, 16))
        w, x = wl.random_tensors(rng, layer, hint + 2)
        if it % 7 == 0:
            w[rng.integers(0, layer.K)] = 0.0
        conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                           layer.groups, batch_hint=hint)
        assert conv.geom["kernel"] == skc.SKC_KERNEL_DIRECT
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        for N in (hint, hint + 2):
            out = conv.forward(torch.from_numpy(x[:N]).cuda()).cpu().numpy()
            worst = max(worst, check(out, ref[:N], bound[:N], f"it{it} {layer} hint {hint} N {N}"))
        del conv
    print("max err/bound", worst)


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_large_and_stem_geometries(kernel):
    """Network layers outside the BASELINE configs, at full size: the ResNet stem (3 -> 64,
    224x224, 7x7, stride 2, pad 3), AlexNet conv1 (3 -> 96, 227x227, 11x11, stride 4), a
    112x112 3x3 layer (many row bands), and a 1x1 projection with stride 2 -- odd channel
    counts and planes (no 16-byte TMA runs: AUTO falls back to the data-driven kernels), large
    strides and kernels, every output of 2 images against the fp64 oracle."""
    rng = np.random.default_rng(41)
    layers = [wl.Layer("resnet_stem", 64, 3, 224, 224, 7, 7, 2, 3, 1, 0.5, 1.0),
              wl.Layer("alexnet_conv1", 96, 3, 227, 227, 11, 11, 4, 0, 1, 0.5, 1.0),
              wl.Layer("c64_112", 64, 64, 112, 112, 3, 3, 1, 1, 1, 0.7, 1.0),
              wl.Layer("proj_s2", 128, 64, 56, 56, 1, 1, 2, 0, 1, 0.7, 1.0)]
    for layer in layers:
        w, x = wl.random_tensors(rng, layer, 2)
        try:
            out, conv = run_gpu(w, x, layer, kernel)
        except skc.SkcError as e:  # a forced kernel may not tile a shape; AUTO must
            assert kernel != skc.SKC_KERNEL_AUTO and e.status == -5, (layer.name, e)
            continue
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        check(out, ref, bound, f"{layer.name} kernel {conv.geom['kernel']}")
        del conv


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_beyond_2gib_offsets(kernel):
    """Maximum sizes: config 2's conv3 at 10240 images -- a 2.36 GB padded input and a 2.66 GB
    output, so image offsets pass 2^31 bytes in both -- pad + conv through the C-ABI, then
    sampled images (first, last, both sides of the 2 GiB boundaries, random) against the
    oracle."""
    layer = wl.CONFIGS[2].layers[1]
    N = 10240
    w = wl.gen_weights(2, 1, layer)
    conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                       kernel)
    x = torch.empty((N, layer.C, layer.H, layer.W), device="cuda")
    for n0 in range(0, N, 256):  # the seeded generator, in slices
        x[n0:n0 + 256] = torch.from_numpy(wl.gen_input(2, 1, layer, n0, n0 + 256))
    out = conv.forward(x)
    torch.cuda.synchronize()
    edges = [(1 << 31) // (layer.K * layer.Ho * layer.Wo * 4),                 # output
             (1 << 31) // (layer.C * (layer.H + 2 * layer.pad) * (layer.W + 2 * layer.pad) * 4)]
    assert all(e + 1 < N for e in edges)
    rng = np.random.default_rng(5)
    idx = sorted({0, N - 1, *[e + d for e in edges for d in (-1, 0, 1)],
                  *map(int, rng.integers(0, N, 3))})
    xs = x[idx].cpu().numpy()
    ref, bound = oracle.conv2d_fp64(xs, w, layer.stride, layer.pad, layer.groups)
    check(out[idx].cpu().numpy(), ref, bound, f"N={N} images {idx} kernel {conv.geom['kernel']}")
    del x, out, conv
    torch.cuda.empty_cache()


def test_concurrent_streams_separate_workspaces():
    """skc.h thread-safety contract: launches that use different workspaces may overlap.  The
    four AlexNet layers, plus a second upload of conv3's plan (its own workspace: the work-item
    counter and the first-item claim table), run at the same time on five streams, repeated;
    every output is bitwise equal to the same launch run alone."""
    cfg = wl.CONFIGS[2]
    N = 64
    convs, xs = [], []
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(2, li, layer)
        convs.append(skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                                 layer.groups))
        xs.append(torch.from_numpy(wl.gen_input(2, li, layer, 0, N)).cuda())
        if li == 1:
            convs.append(skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                                     layer.groups))
            xs.append(torch.from_numpy(wl.gen_input(2, li, layer, N, 2 * N)).cuda())
    alone = [c.forward(x) for c, x in zip(convs, xs)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in convs]
    for rep in range(5):
        outs = [None] * len(convs)
        for i, (c, x, st) in enumerate(zip(convs, xs, streams)):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                outs[i] = c.forward(x, stream=st)
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(zip(alone, outs)):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32)), (rep, i)


def test_config5_sharded_parity():
    """BASELINE.json configs[4]: config 2's layers at batch 4096, sharded over 8 GPUs.  On
    one GPU: the whole batch, and each of the 8 shards run separately (as the 8 ranks would,
    dist.shard_range) and concatenated -- the concatenation must equal the whole-batch run
    BIT FOR BIT, and 8 images of every shard (its first and last included: 64 per layer) must
    pass the oracle.  Uses bench.py's verify_gathered, the same check bench.py runs on the
    NCCL-gathered outputs of a multi-GPU run (and tests/test_dist_gloo.py on gloo)."""
    import bench
    from paper_1608_01409_b200 import dist as skd
    cfg = wl.CONFIGS[5]
    world = 8
    for li, layer in enumerate(cfg.layers):
        w = wl.gen_weights(5, li, layer)
        x = torch.from_numpy(wl.gen_input(5, li, layer, 0, cfg.batch)).cuda()
        conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups)
        shard = skd.shard_range(cfg.batch, world, 0)[1]
        conv.tune(shard)
        full = conv.forward(x).cpu().numpy()
        parts = [conv.forward(x[lo:hi]).cpu().numpy()
                 for lo, hi in (skd.shard_range(cfg.batch, world, r) for r in range(world))]
        res = bench.verify_gathered(np.concatenate(parts), full, 5, li, layer, w, cfg.batch, world)
        assert res["bitwise_vs_1gpu"], f"{layer.name}: sharded run differs from the whole batch"
        assert res["images"] >= 8 * world
        assert res["max_err_over_bound"] <= TOL, res
        del x, full, parts


def check_epi(out, ref, bound, bias, relu, what=""):
    """Reading R16: with a fused bias the per-element scale is sum|w*x| + |b|;
    ReLU is 1-Lipschitz, so the oracle's act(ref + b) carries the same bound."""
    b = bias.reshape(1, -1, 1, 1).astype(np.float64)
    exp = ref + b
    if relu:
        exp = np.maximum(exp, 0.0)
    scale = bound + np.abs(b)
    err = np.abs(out.astype(np.float64) - exp)
    zero = scale == 0
    assert np.all(out[zero] == 0), what
    worst = float(np.max(np.where(zero, 0.0, err / np.where(zero, 1.0, scale))))
    assert worst <= TOL, f"{what}: max err/scale {worst:.3e}"


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_DIRECT, skc.SKC_KERNEL_REGTILE,
                                    skc.SKC_KERNEL_JIT])
def test_fused_epilogue(kernel):
    """f1: conv + bias + ReLU written into the interior of an out_pad-wide halo; the halo is
    never touched (pre-filled sentinel survives)."""
    rng = np.random.default_rng(31)
    cases = [wl.Layer("e1", 20, 16, 13, 13, 3, 3, 1, 1, 2, 0.9, 1.0),
             wl.Layer("e2", 24, 8, 27, 27, 5, 5, 1, 2, 2, 0.85, 1.0),
             wl.Layer("e3", 9, 4, 9, 11, 3, 3, 1, 1, 1, 0.5, 1.0)]
    for layer in cases:
        w, x = wl.random_tensors(rng, layer, 3)
        bias = rng.standard_normal(layer.K).astype(np.float32)
        try:
            conv = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                               layer.groups, kernel)
        except skc.SkcError as e:
            assert e.status == -5
            continue
        skc.skc_plan_verify(conv.plan)
        xp = torch.empty(conv.padded_shape(3), device="cuda")
        skc.skc_pad_input(conv.plan, torch.from_numpy(x).cuda(), xp, 3)
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        db = torch.from_numpy(bias).cuda()
        zero = np.zeros_like(bias)
        # with and without a bias: the JIT kernel has separate epilogue code for each
        for relu, use_bias in ((False, True), (True, True), (False, False), (True, False)):
            for op in (0, 1, 2):
                out = torch.full((3, layer.K, layer.Ho + 2 * op, layer.Wo + 2 * op), 7.0,
                                 device="cuda")
                skc.skc_sparse_conv_forward_ex(conv.plan, xp, out, 3, db if use_bias else None,
                                               relu, op)
                torch.cuda.synchronize()
                o = out.cpu().numpy()
                inner = o[:, :, op:op + layer.Ho, op:op + layer.Wo]
                check_epi(inner, ref, bound, bias if use_bias else zero, relu,
                          f"{layer.name} relu={relu} bias={use_bias} pad={op}")
                halo = o.copy()
                halo[:, :, op:op + layer.Ho, op:op + layer.Wo] = 7.0
                assert np.all(halo == 7.0), "halo written"


def test_chain_conv3_to_conv5_no_pad_pass():
    """f1 in use: AlexNet conv3 -> conv4 -> conv5 (13x13, pad 1, ReLU between) where each
    layer writes bias + ReLU straight into the next layer's zero-padded input, in THAT plan's
    layout (skc_sparse_conv_forward_into: image-pair interleaved for JIT plans); every layer
    is checked against the oracle fed with exactly the GPU's input to that layer.  Run with
    AUTO plans (JIT, pair layout) and with direct plans (NCHW layout), and across the two."""
    cfg = wl.CONFIGS[2]
    rng = np.random.default_rng(33)
    layers = [cfg.layers[1], cfg.layers[2], cfg.layers[3]]
    biases = [(0.1 * rng.standard_normal(L.K)).astype(np.float32) for L in layers]
    for N, kernels in [(16, ("auto", "auto", "auto")), (13, ("direct", "direct", "direct")),
                       (7, ("auto", "direct", "auto"))]:
        km = {"auto": skc.SKC_KERNEL_AUTO, "direct": skc.SKC_KERNEL_DIRECT}
        convs = [skc.SparseConv2d.from_dense(wl.gen_weights(2, i + 1, L), L.H, L.W, L.stride,
                                             L.pad, L.groups, km[k])
                 for i, (L, k) in enumerate(zip(layers, kernels))]
        x = wl.gen_input(2, 1, layers[0], 0, N)
        xp = torch.empty(convs[0].padded_shape(N), device="cuda")
        skc.skc_pad_input(convs[0].plan, torch.from_numpy(x).cuda(), xp, N)
        for i, (L, conv, b) in enumerate(zip(layers, convs, biases)):
            last = i == len(layers) - 1
            if last:
                nxt = torch.zeros((N, L.K, L.Ho, L.Wo), device="cuda")
                skc.skc_sparse_conv_forward_ex(conv.plan, xp, nxt, N, torch.from_numpy(b).cuda(),
                                               True, 0)
            else:
                nxt = torch.zeros(convs[i + 1].padded_shape(N), device="cuda")
                skc.skc_sparse_conv_forward_into(conv.plan, xp, convs[i + 1].plan, nxt, N,
                                                 torch.from_numpy(b).cuda(), True)
            torch.cuda.synchronize()
            xin = skc.unpad_view(conv.geom, xp, N).cpu().numpy()[:, :, L.pad:L.pad + L.H,
                                                                 L.pad:L.pad + L.W]
            ref, bound = oracle.conv2d_fp64(np.ascontiguousarray(xin), wl.gen_weights(2, i + 1, L),
                                            L.stride, L.pad, L.groups)
            if last:
                o = nxt.cpu().numpy()
            else:
                op = layers[i + 1].pad
                full = skc.unpad_view(convs[i + 1].geom, nxt, N).cpu().numpy()
                o = full[:, :, op:op + L.Ho, op:op + L.Wo]
                halo = full.copy()
                halo[:, :, op:op + L.Ho, op:op + L.Wo] = 0
                assert not halo.any(), "halo written"
            check_epi(o, ref, bound, b, True, f"chain {kernels} {L.name}")
            xp = nxt


def test_im2col_equals_unfold():
    """f3: the lowering kernel equals the library routine torch.nn.functional.unfold
    (same (c, r, s) row order), bitwise."""
    rng = np.random.default_rng(41)
    for (N, C, H, W, R, st, p) in [(2, 3, 7, 9, 3, 1, 1), (1, 8, 13, 13, 3, 1, 1),
                                   (2, 4, 27, 27, 5, 1, 2), (3, 2, 11, 10, 3, 2, 0)]:
        x = rng.standard_normal((N, C, H, W), dtype=np.float32)
        plan = skc.skc_pack_csr(np.ones((1, C, R, R), np.float32), H, W, st, p, 1)
        g = plan.info()
        low = torch.empty((N, C * R * R, g["Ho"], g["Wo"]), device="cuda")
        skc.skc_im2col(plan, torch.from_numpy(x).cuda(), low, N)
        torch.cuda.synchronize()
        ref = torch.nn.functional.unfold(torch.from_numpy(x), R, padding=p, stride=st)
        np.testing.assert_array_equal(low.cpu().numpy().reshape(ref.shape).view(np.uint32),
                                      ref.numpy().view(np.uint32))


def test_im2col_pairs_equals_unfold():
    """f3: the image-pair lowering equals torch.nn.functional.unfold interleaved by image
    pairs, bitwise, with a zero second image for an odd batch."""
    rng = np.random.default_rng(43)
    for (N, C, H, W, R, st, p) in [(3, 3, 7, 9, 3, 1, 1), (2, 4, 27, 27, 5, 1, 2),
                                   (5, 2, 11, 10, 3, 2, 0)]:
        x = rng.standard_normal((N, C, H, W), dtype=np.float32)
        plan = skc.skc_pack_csr(np.ones((1, C, R, R), np.float32), H, W, st, p, 1)
        g = plan.info()
        P = (N + 1) // 2
        low = torch.full((P, C * R * R, g["Ho"], g["Wo"], 2), 7.0, device="cuda")
        skc.skc_im2col_ex(plan, torch.from_numpy(x).cuda(), low, N, skc.SKC_LAYOUT_PAIRS)
        torch.cuda.synchronize()
        ref = torch.nn.functional.unfold(torch.from_numpy(x), R, padding=p, stride=st).numpy()
        ref = ref.reshape(N, C * R * R, g["Ho"], g["Wo"])
        if N % 2:
            ref = np.concatenate([ref, np.zeros_like(ref[:1])])
        ref = ref.reshape(P, 2, C * R * R, g["Ho"], g["Wo"]).transpose(0, 2, 3, 4, 1)
        np.testing.assert_array_equal(low.cpu().numpy().view(np.uint32),
                                      np.ascontiguousarray(ref).view(np.uint32))
    with pytest.raises(skc.SkcError):
        skc.skc_im2col_ex(plan, torch.from_numpy(x).cuda(), low, N, skc.SKC_LAYOUT_RAW)


@pytest.mark.parametrize("N", [4, 5])
def test_lowered_auto_equals_direct_auto(N):
    """f3 with the compiled-weights kernel on both sides: im2col in the JIT plan's image-pair
    layout + the 1x1 JIT SpMDM equals the direct JIT convolution bit for bit."""
    rng = np.random.default_rng(44 + N)
    K, C, H, W, R = 24, 12, 13, 13, 3
    w = rng.standard_normal((K, C, R, R)).astype(np.float32)
    w[rng.random(w.shape) < 0.8] = 0.0
    x = rng.standard_normal((N, C, H, W), dtype=np.float32)
    direct = skc.SparseConv2d.from_dense(w, H, W, 1, 1, 1, skc.SKC_KERNEL_AUTO)
    low = skc.LoweredSparseConv2d(w, H, W, 1, 1, 1, kernel=skc.SKC_KERNEL_AUTO)
    assert low.conv.geom["kernel"] == skc.SKC_KERNEL_JIT
    xd = torch.from_numpy(x).cuda()
    a = direct.forward(xd)
    b = low.forward(xd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(b.cpu().numpy().view(np.uint32), a.cpu().numpy().view(np.uint32))
    ref, bound = oracle.conv2d_fp64(x, w, 1, 1, 1)
    check(b.cpu().numpy(), ref, bound, "lowered auto")


@pytest.mark.parametrize("li", [0, 1, 2, 3])
def test_lowered_equals_direct(li):
    """f3: sparse conv WITH lowering (im2col + SpMDM) gives bit-for-bit the direct sparse
    convolution's result (same nonzero order), and passes the oracle bar."""
    L = wl.CONFIGS[2].layers[li]
    w = wl.gen_weights(2, li, L)
    x = wl.gen_input(2, li, L, 0, 4)
    direct, _ = run_gpu(w, x, L, skc.SKC_KERNEL_DIRECT)
    low = skc.LoweredSparseConv2d(w, L.H, L.W, L.stride, L.pad, L.groups)
    skc.skc_plan_verify(low.conv.plan)
    out = low.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    np.testing.assert_array_equal(o.view(np.uint32), direct.view(np.uint32))
    ref, bound = oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups)
    check(o, ref, bound, f"lowered {L.name}")


def test_sparse_fc_alexnet():
    """f2: AlexNet fc6-fc8 (90% sparse) at batch 256 as SpMDM through skc_pack_fc against
    the library routine numpy float64 matmul; scale = |W| |X| per output element."""
    for i, L in enumerate(wl.ALEXNET_FC):
        w = wl.gen_fc_weights(i, L)
        x = wl.gen_fc_input(i, L, wl.FC_BATCH)
        fc = skc.SparseLinear(w, wl.FC_BATCH)
        assert fc.plan.info()["kernel"] == skc.SKC_KERNEL_SPMDM
        skc.skc_plan_verify(fc.plan)
        y = fc.forward(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        yo = y.cpu().numpy()
        yd, _ = _fc_run(w, x, skc.SKC_KERNEL_DIRECT)
        np.testing.assert_array_equal(yo.view(np.uint32), yd.view(np.uint32))
        ref = w.astype(np.float64) @ x.astype(np.float64)
        bound = np.abs(w).astype(np.float64) @ np.abs(x).astype(np.float64)
        check(yo, ref, bound, f"fc {L.name}")


def test_sparse_fc_small_vs_oracle():
    """f2 on small ragged shapes through the C oracle (the FC is its 1x1 special case)."""
    rng = np.random.default_rng(51)
    for (M, K, B) in [(1, 1, 1), (7, 13, 5), (40, 33, 64), (65, 100, 31)]:
        w = np.where(rng.random((M, K)) < 0.3, rng.standard_normal((M, K)), 0).astype(np.float32)
        x = np.maximum(rng.standard_normal((K, B)), 0).astype(np.float32)
        fc = skc.SparseLinear(w, B)
        y = fc.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        ref, bound = oracle.conv2d_fp64(x.reshape(1, K, 1, B), w.reshape(M, K, 1, 1))
        check(y.reshape(1, M, 1, B), ref, bound, f"fc {M}x{K}x{B}")


def _fc_run(w, x, kernel, bias=None, relu=False, out_pad=0):
    M, K = w.shape
    B = x.shape[1]
    p = skc.skc_pack_fc(w, B, kernel)
    p.upload("cuda")
    skc.skc_plan_verify(p)
    shape = (M, B) if out_pad == 0 else (M, 1 + 2 * out_pad, B + 2 * out_pad)
    y = torch.full(shape, -7.0, device="cuda")
    b = torch.from_numpy(bias).cuda() if bias is not None else None
    skc.skc_sparse_conv_forward_ex(p, torch.from_numpy(x).cuda(), y, 1, b, relu, out_pad)
    torch.cuda.synchronize()
    return y.cpu().numpy(), p.info()


@pytest.mark.parametrize("shape", [(1, 1, 4), (7, 13, 8), (65, 100, 132), (300, 257, 256),
                                   (1000, 4096, 256), (33, 700, 12), (129, 2000, 260)])
def test_spmdm_equals_direct_bitwise(shape):
    """f2: the SpMDM kernel (several row tiles, column blocks with a ragged last one, K over
    several chunks) gives bit for bit the direct kernel's result on the same FC plan, and
    passes the oracle bar (numpy float64 matmul)."""
    M, K, B = shape
    rng = np.random.default_rng(M + K + B)
    w = np.where(rng.random((M, K)) < 0.1, rng.standard_normal((M, K)), 0).astype(np.float32)
    w[M // 2] = 0  # an empty row
    x = rng.standard_normal((K, B)).astype(np.float32)
    ys, gi = _fc_run(w, x, skc.SKC_KERNEL_SPMDM)
    yd, gd = _fc_run(w, x, skc.SKC_KERNEL_DIRECT)
    assert gi["kernel"] == skc.SKC_KERNEL_SPMDM and gd["kernel"] == skc.SKC_KERNEL_DIRECT
    np.testing.assert_array_equal(ys.view(np.uint32), yd.view(np.uint32))
    ref = w.astype(np.float64) @ x.astype(np.float64)
    bound = np.abs(w).astype(np.float64) @ np.abs(x).astype(np.float64)
    check(ys, ref, bound, f"spmdm {shape}")


@pytest.mark.parametrize("out_pad", [0, 2])
def test_spmdm_epilogue_equals_direct(out_pad):
    """f2 + a6: bias, ReLU and a padded output (the general store path) bitwise as the
    direct kernel's epilogue; the halo is left untouched."""
    rng = np.random.default_rng(61 + out_pad)
    M, K, B = 90, 300, 136
    w = np.where(rng.random((M, K)) < 0.15, rng.standard_normal((M, K)), 0).astype(np.float32)
    x = rng.standard_normal((K, B)).astype(np.float32)
    bias = rng.standard_normal(M).astype(np.float32)
    ys, _ = _fc_run(w, x, skc.SKC_KERNEL_SPMDM, bias, True, out_pad)
    yd, _ = _fc_run(w, x, skc.SKC_KERNEL_DIRECT, bias, True, out_pad)
    np.testing.assert_array_equal(ys.view(np.uint32), yd.view(np.uint32))
    inner = ys if out_pad == 0 else ys[:, out_pad, out_pad:out_pad + B]
    ref = np.maximum(w.astype(np.float64) @ x.astype(np.float64) + bias[:, None], 0)
    assert np.allclose(inner, ref, rtol=1e-4, atol=1e-4)
    if out_pad:
        halo = ys.copy()
        halo[:, out_pad, out_pad:out_pad + B] = -7.0
        assert np.all(halo == -7.0)


def test_spmdm_1x1_conv_images():
    """The SpMDM kernel on a 1x1 conv plan with several images (grid z) = the direct kernel."""
    rng = np.random.default_rng(62)
    w = np.where(rng.random((48, 40, 1, 1)) < 0.25, rng.standard_normal((48, 40, 1, 1)), 0).astype(np.float32)
    x = rng.standard_normal((3, 40, 14, 14)).astype(np.float32)
    L = type("L", (), dict(H=14, W=14, stride=1, pad=0, groups=1))
    a, ca = run_gpu(w, x, L, skc.SKC_KERNEL_SPMDM)
    b, _ = run_gpu(w, x, L, skc.SKC_KERNEL_DIRECT)
    assert ca.geom["kernel"] == skc.SKC_KERNEL_SPMDM
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
    ref, bound = oracle.conv2d_fp64(x, w)
    check(a, ref, bound, "spmdm 1x1 conv")


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_batch_split_invariance(kernel):
    """a batch-sharded multi-GPU run must be bitwise identical to the
    1-GPU run.  CTAs stage NI images together, so this holds iff each image's result does
    not depend on which images share its CTA: run the full batch, then shards of it at odd
    offsets (as dist.shard_range produces), and compare bit for bit."""
    from paper_1608_01409_b200 import dist as skd
    for li in range(4):
        L = wl.CONFIGS[2].layers[li]
        w = wl.gen_weights(2, li, L)
        n = 37
        x = wl.gen_input(2, li, L, 0, n)
        full, conv = run_gpu(w, x, L, kernel)
        for world in (2, 3, 8):
            parts = []
            for r in range(world):
                lo, hi = skd.shard_range(n, world, r)
                xs = torch.from_numpy(x[lo:hi]).cuda()
                parts.append(conv.forward(xs).cpu().numpy())
            np.testing.assert_array_equal(np.concatenate(parts).view(np.uint32),
                                          full.view(np.uint32))


def run_jit_and_direct(w, x, layer):
    """Both kernels on the same padded input; returns (jit_out, direct_out, jit_conv)."""
    jit = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                      skc.SKC_KERNEL_JIT)
    skc.skc_plan_verify(jit.plan)
    direct = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                         layer.groups, skc.SKC_KERNEL_DIRECT)
    N = x.shape[0]
    xd = torch.from_numpy(x).cuda()
    xpj = torch.empty(jit.padded_shape(N), device="cuda")
    skc.skc_pad_input(jit.plan, xd, xpj, N)
    xpd = torch.empty(direct.padded_shape(N), device="cuda")
    skc.skc_pad_input(direct.plan, xd, xpd, N)
    yj = torch.full(jit.out_shape(N), float("nan"), device="cuda")
    jit.forward_padded(xpj, yj)
    yd = direct.forward_padded(xpd)
    torch.cuda.synchronize()
    return yj.cpu().numpy(), yd.cpu().numpy(), jit


def prewarm_jit(cases, kernel=skc.SKC_KERNEL_JIT):
    """Compile the JIT code of (layer, w) cases in parallel host threads into the on-disk
    cache, so the sequential test loop only loads it (a speed-up, results unaffected)."""
    import concurrent.futures as cf

    def one(case):
        layer, w = case
        try:
            skc.skc_plan_compile(skc.skc_pack_csr(w, layer.H, layer.W, layer.stride, layer.pad,
                                                  layer.groups, kernel))
        except skc.SkcError:
            pass
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(one, cases))


def test_jit_random_geometries():
    """The compiled-weights kernel forced on random layers (1x1..5x5, stride 1/2, groups,
    ragged K and C/g, batches not a multiple of the images per CTA, empty channels, tiles
    overhanging the output): within tolerance of the fp64 oracle and BITWISE equal to the
    direct kernel (same fp32 FMA sequence per output element, CSR order)."""
    rng = np.random.default_rng(21)
    n_jit = 0
    cases = []
    for it in range(150):
        if it % 2:
            layer = wl.random_layer(rng, max_c=32, max_hw=20, rs=(1, 2, 3, 5), groups=(1, 2, 4))
        else:
            R = int(rng.choice([1, 3, 5]))
            g = int(rng.choice([1, 2]))
            C = g * 4 * int(rng.integers(1, 9))
            K = g * int(rng.integers(1, 48))
            H, W = int(rng.integers(R, 32)), int(rng.integers(R, 32))
            layer = wl.Layer("j", K, C, H, W, R, R, int(rng.choice([1, 2])), (R - 1) // 2, g,
                             float(rng.choice([0.0, 0.5, 0.9, 0.98])), 1.0)
        N = int(rng.integers(1, 24))
        w, x = wl.random_tensors(rng, layer, N)
        if it % 5 == 0:
            w[rng.integers(0, layer.K)] = 0.0
        cases.append((layer, w, x))
    prewarm_jit([(layer, w) for layer, w, _ in cases])
    for it, (layer, w, x) in enumerate(cases):
        try:
            yj, yd, conv = run_jit_and_direct(w, x, layer)
        except skc.SkcError as e:
            assert e.status == -5, e  # unsupported staging alignment only
            continue
        n_jit += 1
        np.testing.assert_array_equal(yj.view(np.uint32), yd.view(np.uint32),
                                      err_msg=f"it{it} {layer} {conv.geom}")
        ref, bound = oracle.conv2d_fp64(x, w, layer.stride, layer.pad, layer.groups)
        check(yj, ref, bound, f"jit it{it} {layer}")
    assert n_jit >= 100, n_jit


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_jit_bitwise_equals_direct_full_batch(cfg_id):
    """Full batch (256) of every config-2 / config-4 layer: JIT output == direct output bit
    for bit (the direct kernel is checked against the oracle in test_config_parity)."""
    cfg = wl.CONFIGS[cfg_id]
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, L)
        x = wl.gen_input(cfg_id, li, L, 0, cfg.batch)
        yj, yd, conv = run_jit_and_direct(w, x, L)
        assert conv.geom["kernel"] == skc.SKC_KERNEL_JIT
        np.testing.assert_array_equal(yj.view(np.uint32), yd.view(np.uint32), err_msg=L.name)


@pytest.mark.parametrize("knobs", [
    {"SKC_JIT_ORDER": "0"}, {"SKC_JIT_ORDER": "1"}, {"SKC_JIT_DRY": "0"},
    {"SKC_JIT_L2HINT": "0"}, {"SKC_JIT_CLUSTER": "1"}, {"SKC_JIT_CLUSTER": "4"},
    {"SKC_JIT_PAIR": "0"}, {"SKC_JIT_PAIR": "1", "SKC_JIT_BANDS": "3"},
    {"SKC_JIT_NS": "4", "SKC_JIT_STAGE_KB": "24"}, {"SKC_JIT_NW": "8"}, {"SKC_JIT_NW": "24"},
    {"SKC_JIT_GRID": "7"}, {"SKC_JIT_DYN": "0"}, {"SKC_JIT_DYN": "1", "SKC_JIT_SPLIT": "2"},
    {"SKC_JIT_DYN": "2", "SKC_JIT_SPLIT": "1"}, {"SKC_JIT_DYN": "2", "SKC_JIT_GRID": "5"},
    {"SKC_JIT_DYN": "1", "SKC_JIT_SPLIT": "9", "SKC_JIT_GRID": "3"},
    {"SKC_JIT_XPF": "0"}, {"SKC_JIT_XPF": "1", "SKC_JIT_NS": "3", "SKC_JIT_STAGE_KB": "20", "SKC_JIT_GRID": "4"},
    {"SKC_JIT_XPF": "1", "SKC_JIT_NS": "2", "SKC_JIT_STAGE_KB": "12", "SKC_JIT_GRID": "1"},
    {"SKC_JIT_PMAJOR": "0"}, {"SKC_JIT_VID": "0"}, {"SKC_JIT_RAW": "1"},
    {"SKC_JIT_RAW": "1", "SKC_JIT_NS": "3", "SKC_JIT_STAGE_KB": "20"}, {"SKC_JIT_DEAL": "0"},
    {"SKC_JIT_DEAL": "1", "SKC_JIT_DYN": "1", "SKC_JIT_SPLIT": "2"}, {"SKC_JIT_LANES": "1"},
    {"SKC_JIT_LANES": "1", "SKC_JIT_DYN": "2"}, {"SKC_JIT_NP": "1"},
    {"SKC_JIT_NP": "1", "SKC_JIT_SCHED": "546"}, {"SKC_JIT_NP": "1", "SKC_JIT_SCHED": "17"},
    {"SKC_JIT_NP": "1", "SKC_JIT_GRID": "5", "SKC_JIT_CLUSTER": "1"}, {"SKC_JIT_LOOKAHEAD": "2"},
    {"SKC_JIT_DEAL": "1", "SKC_JIT_NP": "1"}, {"SKC_JIT_OPT": "-O1"},
])
def test_jit_tuning_knobs_bitwise(knobs, monkeypatch):
    """Every JIT tuning knob (work order, dry-run prefetch, L2 policy, cluster size, layout,
    row bands, staging depth, warps, grid size, dynamic scheduling, tail split, cross-item staging with rotated stages,
    position-major code) changes
    scheduling only: the output must stay
    bit-for-bit equal to the direct kernel's on ragged shapes (odd batch, 27x27 with bands,
    grouped 13x13)."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(44)
    for layer, N in [(wl.Layer("k1", 48, 32, 27, 27, 5, 5, 1, 2, 2, 0.85, 0.01), 7),
                     (wl.Layer("k2", 40, 64, 13, 13, 3, 3, 1, 1, 2, 0.9, 0.01), 9)]:
        w, x = wl.random_tensors(rng, layer, N)
        try:
            yj, yd, conv = run_jit_and_direct(w, x, layer)
        except skc.SkcError as e:
            assert e.status == -5, e
            continue
        np.testing.assert_array_equal(yj.view(np.uint32), yd.view(np.uint32),
                                      err_msg=f"{knobs} {layer.name} {conv.geom}")


@pytest.mark.gpu
@pytest.mark.parametrize("dyn", ["1", "2"])
def test_jit_dynamic_counter_resets_across_launches(dyn, monkeypatch):
    """Dynamic scheduling keeps a work-item counter in the plan workspace that the last CTA of
    every launch resets: back-to-back launches of ONE plan with different batch sizes (and
    grid sizes), and replays of a captured CUDA graph, must each compute every item exactly
    once -- bitwise equal to the direct kernel every time."""
    monkeypatch.setenv("SKC_JIT_DYN", dyn)
    monkeypatch.setenv("SKC_JIT_SPLIT", "2")
    rng = np.random.default_rng(46)
    layer = wl.Layer("d1", 48, 32, 13, 13, 3, 3, 1, 1, 2, 0.85, 0.01)
    w, x = wl.random_tensors(rng, layer, 40)
    jit = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                      skc.SKC_KERNEL_JIT)
    direct = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                         layer.groups, skc.SKC_KERNEL_DIRECT)
    assert jit.plan.info()["jit_split"] > 0
    xd = torch.from_numpy(x).cuda()
    xpj = torch.empty(jit.padded_shape(40), device="cuda")
    skc.skc_pad_input(jit.plan, xd, xpj, 40)
    xpd = torch.empty(direct.padded_shape(40), device="cuda")
    skc.skc_pad_input(direct.plan, xd, xpd, 40)
    yd = direct.forward_padded(xpd).cpu().numpy()
    for N in (40, 7, 1, 33, 40, 2, 40):
        yj = torch.full(jit.out_shape(N), float("nan"), device="cuda")
        jit.forward_padded(xpj, yj)  # the first N images (pairs are image-major)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(yj.cpu().numpy().view(np.uint32), yd[:N].view(np.uint32),
                                      err_msg=f"N={N}")
    # graph replays of the same launch
    yj = torch.full(jit.out_shape(40), float("nan"), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            jit.forward_padded(xpj, yj, stream=s)
    torch.cuda.synchronize()
    for _ in range(4):
        yj.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(yj.cpu().numpy().view(np.uint32), yd.view(np.uint32))


@pytest.mark.gpu
def test_plan_tune_keeps_outputs_bitwise():
    """skc_plan_tune times the launch-schedule variants on scratch buffers and keeps the
    fastest; the plan's outputs before and after tuning are bit-identical, and tuning a
    non-JIT plan is a no-op."""
    rng = np.random.default_rng(47)
    layer = wl.Layer("t1", 64, 48, 13, 13, 3, 3, 1, 1, 2, 0.9, 0.01)
    w, x = wl.random_tensors(rng, layer, 37)
    jit = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad, layer.groups,
                                      skc.SKC_KERNEL_JIT)
    xd = torch.from_numpy(x).cuda()
    xp = torch.empty(jit.padded_shape(37), device="cuda")
    skc.skc_pad_input(jit.plan, xd, xp, 37)
    y0 = jit.forward_padded(xp).cpu().numpy()
    ms = jit.tune(37)
    assert ms > 0
    y1 = jit.forward_padded(xp).cpu().numpy()
    np.testing.assert_array_equal(y0.view(np.uint32), y1.view(np.uint32))
    direct = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                         layer.groups, skc.SKC_KERNEL_DIRECT)
    assert direct.tune(37) == 0.0
    with pytest.raises(skc.SkcError):
        skc.skc_plan_tune(jit.plan, 0, xp, xp)


@pytest.mark.gpu
def test_sm_topology_is_a_gpc_major_permutation():
    """The topology probe (clusters never span a GPC; run by the first JIT upload on the
    device, in the plan workspace) yields a permutation of the SM ids in which every
    cluster-mate group is contiguous: the two SMs of a 2-CTA cluster (one TPC) always get
    neighbouring positions."""
    layer = wl.Layer("t0", 16, 16, 13, 13, 3, 3, 1, 1, 1, 0.5, 0.01)
    w, _ = wl.random_tensors(np.random.default_rng(49), layer, 1)
    skc.SparseConv2d.from_dense(w, 13, 13, 1, 1, 1, skc.SKC_KERNEL_JIT)  # uploads: probes
    vid = skc.skc_sm_topology()
    n = torch.cuda.get_device_properties(0).multi_processor_count
    assert len(vid) == n
    assert sorted(vid) == list(range(n))
    tpc_adjacent = sum(vid[2 * k + 1] == vid[2 * k] + 1 for k in range(n // 2))
    assert tpc_adjacent >= 0.9 * (n // 2), tpc_adjacent


@pytest.mark.gpu
@pytest.mark.parametrize("li", [0, 3])
def test_tuned_plan_full_batch_bitwise(li):
    """The launch configuration bench.py times: a config-2 layer's plan tuned for the full
    batch (skc_plan_tune picks the schedule), then the full batch of 256 -- bitwise equal to
    the direct kernel, whose output the oracle checks in test_config_parity."""
    cfg = wl.CONFIGS[2]
    L = cfg.layers[li]
    w = wl.gen_weights(2, li, L)
    x = wl.gen_input(2, li, L, 0, cfg.batch)
    jit = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_AUTO)
    assert jit.geom["kernel"] == skc.SKC_KERNEL_JIT
    assert jit.tune(cfg.batch) > 0
    assert jit.plan.info()["jit_sched"] >= 0
    direct = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups,
                                         skc.SKC_KERNEL_DIRECT)
    xd = torch.from_numpy(x).cuda()
    yj = jit.forward(xd).cpu().numpy()
    yd = direct.forward(xd).cpu().numpy()
    np.testing.assert_array_equal(yj.view(np.uint32), yd.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1, 3, 64])
def test_tune_small_layers_and_batches(N):
    """Tuning on tiny layers (several CTAs per SM, grid != #SMs: the GPC-major numbering must
    switch itself off) and small / odd batches: outputs stay bitwise equal to the direct
    kernel before and after tuning."""
    rng = np.random.default_rng(48 + N)
    for layer in (wl.Layer("s1", 8, 8, 6, 6, 3, 3, 1, 1, 1, 0.5, 0.01),
                  wl.Layer("s2", 24, 16, 9, 7, 1, 1, 1, 0, 2, 0.7, 0.01)):
        w, x = wl.random_tensors(rng, layer, N)
        try:
            jit = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                              layer.groups, skc.SKC_KERNEL_JIT)
        except skc.SkcError as e:
            assert e.status == -5
            continue
        direct = skc.SparseConv2d.from_dense(w, layer.H, layer.W, layer.stride, layer.pad,
                                             layer.groups, skc.SKC_KERNEL_DIRECT)
        xd = torch.from_numpy(x).cuda()
        yd = direct.forward(xd).cpu().numpy()
        y0 = jit.forward(xd).cpu().numpy()
        jit.tune(N)
        y1 = jit.forward(xd).cpu().numpy()
        np.testing.assert_array_equal(y0.view(np.uint32), yd.view(np.uint32), err_msg=layer.name)
        np.testing.assert_array_equal(y1.view(np.uint32), yd.view(np.uint32), err_msg=layer.name)


# every launch schedule skc_plan_tune can choose: bit 0 first round block-major, bit 1
# GPC-major (claimed) first items, bit 2 no dry-run prefetch, bit 3 contiguous lane table,
# bits 4-7 cluster size (1 or 2), bit 9 dry run by every CTA
SCHEDULES = [o3 | (v << 1) | (nd << 2) | (ln << 3) | (cs << 4) | (da << 9)
             for o3 in (0, 1) for v in (0, 1) for nd in (0, 1) for ln in (0, 1) for cs in (1, 2)
             for da in (0, 1)]


@pytest.mark.parametrize("np_mode", ["0", "1"])
def test_jit_every_schedule_bitwise(np_mode, monkeypatch):
    """The schedules the bench actually runs: every launch-schedule word the tuner can pick
    (forced with SKC_JIT_SCHED) on all four config-2 layers at the full batch of 256, in the
    plans AUTO builds (persistent whole-program kernel, and the non-persistent per-block-module
    kernel, SKC_JIT_NP=1) -- each BIT FOR BIT equal to the direct kernel (whose output the
    oracle checks in test_config_parity_full_batch)."""
    monkeypatch.setenv("SKC_JIT_NP", np_mode)
    cfg = wl.CONFIGS[2]
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(2, li, L)
        x = torch.from_numpy(wl.gen_input(2, li, L, 0, cfg.batch)).cuda()
        direct = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_DIRECT)
        yd = direct.forward(x)
        jit = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_AUTO)
        assert jit.geom["kernel"] == skc.SKC_KERNEL_JIT
        xp = torch.empty(jit.padded_shape(cfg.batch), device="cuda")
        skc.skc_pad_input(jit.plan, x, xp, cfg.batch)
        yj = torch.empty_like(yd)
        for sched in SCHEDULES:
            monkeypatch.setenv("SKC_JIT_SCHED", str(sched))
            yj.fill_(float("nan"))
            jit.forward_padded(xp, yj)
            torch.cuda.synchronize()
            assert torch.equal(yj.view(torch.int32), yd.view(torch.int32)), f"{L.name} sched {sched}"
        monkeypatch.delenv("SKC_JIT_SCHED")
        del x, yd, yj, xp


def test_gpc_major_items_claimed_when_sms_are_shared(monkeypatch):
    """GPC-major first items are CLAIMED (atomic compare-and-swap on a table in the
    workspace), not assumed from %smid: the launch is not cooperative, so when other kernels
    hold some SMs, CTAs of the persistent grid start late on SMs that earlier CTAs of the same
    grid already used.  Hold ~24 SMs with spinning kernels on side streams, launch the JIT
    kernel (GPC-major items forced, no clusters) meanwhile, repeatedly: every output must stay
    bitwise equal to the direct kernel (a duplicated first item would leave outputs unwritten)."""
    monkeypatch.setenv("SKC_JIT_SCHED", str((1 << 1) | (1 << 4)))
    L = wl.CONFIGS[2].layers[3]
    N = 256  # >= one item per SM: the grid is all SMs, the condition for GPC-major items
    w = wl.gen_weights(2, 3, L)
    x = torch.from_numpy(wl.gen_input(2, 3, L, 0, N)).cuda()
    direct = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_DIRECT)
    yd = direct.forward(x)
    jit = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_JIT)
    xp = torch.empty(jit.padded_shape(N), device="cuda")
    skc.skc_pad_input(jit.plan, x, xp, N)
    torch.cuda.synchronize()
    side = [torch.cuda.Stream() for _ in range(24)]
    main = torch.cuda.Stream()
    for rep in range(6):
        for s_ in side:
            with torch.cuda.stream(s_):
                torch.cuda._sleep(2_000_000 * (1 + rep % 3))  # ~1-3 ms per held SM
        yj = torch.full_like(yd, float("nan"))
        with torch.cuda.stream(main):
            jit.forward_padded(xp, yj, stream=main)
        torch.cuda.synchronize()
        assert torch.equal(yj.view(torch.int32), yd.view(torch.int32)), f"rep {rep}"


@pytest.mark.parametrize("kernel", [skc.SKC_KERNEL_AUTO, skc.SKC_KERNEL_DIRECT])
def test_first_forward_captured_in_graph(kernel):
    """skc_plan_upload prepares everything a launch needs (JIT code loaded, attributes,
    occupancy, SM order), so the VERY FIRST pad + forward of a fresh plan can be captured
    into a CUDA graph; replays match an ordinary launch of a second plan bit for bit."""
    L = wl.CONFIGS[2].layers[2]
    N = 12
    w = wl.gen_weights(2, 2, L)
    x = torch.from_numpy(wl.gen_input(2, 2, L, 0, N)).cuda()
    ref_conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kernel)
    ref = ref_conv.forward(x)
    conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kernel)
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    out = torch.full_like(ref, float("nan"))
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            skc.skc_pad_input(conv.plan, x, xp, N, s)
            skc.skc_sparse_conv_forward(conv.plan, xp, out, N, s)
    torch.cuda.synchronize()
    assert torch.isnan(out).all(), "capture must not execute"
    for _ in range(3):
        out.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32))


def test_bench_multirank_config5_gloo():
    """bench.py's multi-rank path run for real: 2 ranks (torchrun, gloo collectives) sharing
    this GPU on config 5 (BASELINE.json configs[4]) at a global batch of 96 -- strong scaling
    over shard_range, timed steps, then every layer's outputs gathered from both ranks,
    compared BIT FOR BIT with rank 0's one-device run of the whole batch, and 8 images per
    shard (first and last included) through the oracle.  The ranks' kernels never wait on
    each other (no collective on the data path), so sharing one GPU is only slower."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
           "--config", "5", "--batch", "96", "--steps", "3", "--warmup", "3", "--backend", "gloo",
           "--no-e2e", "--no-dense", "--no-cpu", "--no-peaks"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 96 and line["config"]["per_gpu_batch"] == 48
    par = line["parity"]
    assert par["bitwise_vs_1gpu"] is True and par["pass"] is True, par
    assert all(p["images"] >= 16 for p in par["per_layer"]), par
