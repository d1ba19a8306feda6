#!/usr/bin/env python
"""Time the conv kernel of each layer for the direct kernel and every register-tile shape
(SKC_RT_SHAPE override) -- the measurements behind plan.cpp's shape choice.

    python tools/sweep_regtile.py --config 2 [--layers 0,1,2,3] [--nt 0]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402

SHAPES = {3: ["3,3,2,7,8", "3,3,2,7,4", "3,3,1,7,8", "3,3,1,7,4", "3,3,2,4,8", "3,3,1,7,16"],
          5: ["5,5,2,7,6", "5,5,2,7,3", "5,5,1,7,6", "5,5,1,7,12"]}


def time_conv(conv, xp, out, N, reps=5):
    for _ in range(2):
        skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layers", default="")
    ap.add_argument("--nt", default="0")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    layers = [int(v) for v in a.layers.split(",")] if a.layers else range(len(cfg.layers))
    N = cfg.batch
    res = []
    for li in layers:
        L = cfg.layers[li]
        w = wl.gen_weights(a.config, li, L)
        x = torch.from_numpy(wl.gen_input(a.config, li, L, 0, N)).cuda()
        base = None
        cands = [("direct", None, "0")] + [("regtile", s, nt) for s in SHAPES.get(L.R, [])
                                           for nt in a.nt.split(",")]
        for kind, shape, nt in cands:
            os.environ.pop("SKC_RT_SHAPE", None)
            os.environ["SKC_RT_NT"] = nt
            if shape:
                os.environ["SKC_RT_SHAPE"] = shape
            kern = skc.SKC_KERNEL_DIRECT if kind == "direct" else skc.SKC_KERNEL_REGTILE
            try:
                conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern)
            except skc.SkcError as e:
                print(f"{L.name} {kind} {shape}: {e}", flush=True)
                continue
            xp = torch.empty(conv.padded_shape(N), device="cuda")
            skc.skc_pad_input(conv.plan, x, xp, N)
            out = torch.empty(conv.out_shape(N), device="cuda")
            ms = time_conv(conv, xp, out, N)
            if base is None:
                base = out.clone()
            err = float((out - base).abs().max())
            tf = 2 * conv.geom["nnz"] * L.Ho * L.Wo * N / ms / 1e9
            g = conv.geom
            rec = dict(layer=L.name, kind=kind, shape=shape, nt=nt, ms=ms, nnz_gflops=tf,
                       warps=g["warps"], chunk=g["chunk_channels"], stages=g["stages"],
                       smem=g["smem_bytes"], ni=g["images_per_cta"], maxdiff_vs_direct=err)
            res.append(rec)
            print(json.dumps(rec), flush=True)
    os.environ.pop("SKC_RT_SHAPE", None)
    os.environ.pop("SKC_RT_NT", None)


if __name__ == "__main__":
    main()
