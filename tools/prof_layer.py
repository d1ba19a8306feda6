#!/usr/bin/env python
"""One config layer's conv launch, in the launch configuration bench.py times, as an ncu
target: plan built + tuned for the batch (as bench.py does), a warm-up launch, then ONE
launch inside the NVTX range "prof" (select it with ncu --nvtx --nvtx-include "prof/").

    python tools/prof_layer.py --config 2 --layer 1 [--batch 256] [--no-tune]
    ncu --set full --nvtx --nvtx-include "prof/" -c 1 -o gpurun_out/conv3 \
        python tools/prof_layer.py --config 2 --layer 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layer", type=int, default=1)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--kernel", default="auto", choices=["auto", "direct", "jit"])
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    L = cfg.layers[a.layer]
    N = a.batch or cfg.batch
    kern = {"auto": 0, "direct": 1, "jit": 3}[a.kernel]
    w = wl.gen_weights(a.config, a.layer, L)
    conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups, kern)
    if not a.no_tune:
        conv.tune(N)
    x = torch.from_numpy(wl.gen_input(a.config, a.layer, L, 0, N)).cuda()
    xp = torch.empty(conv.padded_shape(N), device="cuda")
    out = torch.empty(conv.out_shape(N), device="cuda")
    skc.skc_pad_input(conv.plan, x, xp, N)
    skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.fill_(1)  # cold L2, as between bench.py's timed steps
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    skc.skc_sparse_conv_forward(conv.plan, xp, out, N)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    info = conv.plan.info()
    print(f"{L.name} N={N} nnz={info['nnz']} kernel={info['kernel']} sched={info['jit_sched']} "
          f"Ho={L.Ho} Wo={L.Wo}")


if __name__ == "__main__":
    main()
