"""JIT kernel probe: bitwise comparison against the direct kernel (same CSR accumulation
order => identical fp32 results) and CUDA-event timing, per AlexNet layer (config 2) and
per forced tile shape (SKC_JIT_TILE="TY,TX[,M]").  Writes one JSON line per case.

    python tools/jit_probe.py [--tiles "auto;1,13;3,4"] [--layers conv2,conv3] [--N 256]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_01409_b200 import skc  # noqa: E402
import workloads as wl  # noqa: E402


FLUSH = None


def time_ms(fn, reps=10):
    """Mean device time; with --flush the L2 is flushed (256 MiB write) before every rep,
    outside the events, as bench.py does (code and data start cold)."""
    fn()
    torch.cuda.synchronize()
    if FLUSH is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    tot = 0.0
    for _ in range(reps):
        FLUSH.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", default="auto")
    ap.add_argument("--layers", default="conv2,conv3,conv4,conv5")
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--out", default="")
    ap.add_argument("--warm", action="store_true", help="no L2 flush between reps")
    a = ap.parse_args()
    global FLUSH
    if not a.warm:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cfg = wl.CONFIGS[a.cfg]
    N = a.N
    lines = []
    for li, L in enumerate(cfg.layers):
        if L.name not in a.layers.split(","):
            continue
        w = wl.gen_weights(a.cfg, li, L)
        x = torch.from_numpy(wl.gen_input(a.cfg, li, L, 0, N)).cuda()
        ref = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_DIRECT)
        xp = torch.empty(ref.padded_shape(N), device="cuda")
        skc.skc_pad_input(ref.plan, x, xp, N)
        y_ref = ref.forward_padded(xp)
        nnz = ref.geom["nnz"]
        flops = 2.0 * nnz * ref.geom["Ho"] * ref.geom["Wo"] * N
        ms_ref = time_ms(lambda: ref.forward_padded(xp, y_ref))
        print(f"{L.name} direct {ms_ref:.3f} ms {flops / ms_ref / 1e9:.2f} TF", flush=True)
        for tile in a.tiles.split(";"):
            if tile == "auto":
                os.environ.pop("SKC_JIT_TILE", None)
            else:
                os.environ["SKC_JIT_TILE"] = tile
            t0 = time.time()
            try:
                j = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, skc.SKC_KERNEL_JIT)
            except Exception as e:  # noqa: BLE001
                print(L.name, tile, "FAILED", e, flush=True)
                continue
            t_build = time.time() - t0
            xpj = torch.empty(j.padded_shape(N), device="cuda")  # the JIT plan's layout
            skc.skc_pad_input(j.plan, x, xpj, N)
            y = torch.full_like(y_ref, float("nan"))
            j.forward_padded(xpj, y)
            torch.cuda.synchronize()
            same = bool(torch.equal(y, y_ref))
            ndiff = int((y != y_ref).sum().item())
            ms = time_ms(lambda: j.forward_padded(xpj, y))
            ms_pad = time_ms(lambda: skc.skc_pad_input(j.plan, x, xpj, N))
            inf = j.plan.info()
            rec = dict(layer=L.name, tile=tile, ms=ms, pad_ms=ms_pad, tflops=flops / ms / 1e9, direct_ms=ms_ref,
                       speedup_vs_direct=ms_ref / ms, bitwise_equal_direct=same, ndiff=ndiff,
                       build_s=t_build, cfg={k: inf[k] for k in (
                           "tile_h", "tile_w", "channels_per_warp", "warps", "images_per_cta",
                           "chunk_channels", "stages", "smem_bytes", "jit_blocks", "jit_split", "code_bytes",
                           "jit_compile_s", "jit_cache_hit", "model_instr_per_image", "layout")})
            lines.append(rec)
            print(json.dumps(rec), flush=True)
            del j
    if a.out:
        with open(a.out, "a") as f:
            for r in lines:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
