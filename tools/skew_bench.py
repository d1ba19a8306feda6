#!/usr/bin/env python
"""Row f4 stress test: AlexNet conv2-5 at batch 256 with per-output-channel densities skewed
log-normally around the layer's density (workloads.gen_weights_skewed), with and without the
nnz-sorted channel order the plan uses for load balance (SKC_NO_NNZ_SORT=1), against the
uniform masks of config 2.  AUTO plans (the JIT kernel), tuned for the batch as bench.py
does; L2 flushed before every timed launch.

    python tools/skew_bench.py > profiles/r02_skewed_masks_loadbalance.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from chain_bench import timed  # noqa: E402


def main():
    cfg = wl.CONFIGS[2]
    N = cfg.batch
    for li, L in enumerate(cfg.layers):
        x = torch.from_numpy(wl.gen_input(2, li, L, 0, N)).cuda()
        for mask in ("uniform", "skewed"):
            w = wl.gen_weights(2, li, L) if mask == "uniform" else wl.gen_weights_skewed(2, li, L, 1.0)
            nnz_k = np.count_nonzero(w.reshape(L.K, -1), axis=1)
            for sort in (True, False):
                if sort:
                    os.environ.pop("SKC_NO_NNZ_SORT", None)
                else:
                    os.environ["SKC_NO_NNZ_SORT"] = "1"
                conv = skc.SparseConv2d.from_dense(w, L.H, L.W, L.stride, L.pad, L.groups)
                conv.tune(N)
                xp = torch.empty(conv.padded_shape(N), device="cuda")
                skc.skc_pad_input(conv.plan, x, xp, N)
                out = torch.empty(conv.out_shape(N), device="cuda")
                ms = timed(lambda: skc.skc_sparse_conv_forward(conv.plan, xp, out, N))
                nnz = conv.geom["nnz"]
                print(json.dumps({"layer": L.name, "mask": mask, "nnz_sorted": sort,
                                  "kernel": conv.geom["kernel"], "nnz": nnz,
                                  "jit_blocks": conv.geom["jit_blocks"], "jit_split": conv.geom["jit_split"],
                                  "max_channel_nnz_over_mean": float(nnz_k.max() / nnz_k.mean()),
                                  "nnz_per_channel_cv": float(nnz_k.std() / nnz_k.mean()),
                                  "ms": ms,
                                  "nnz_tflops": 2 * nnz * L.Ho * L.Wo * N / (ms * 1e-3) / 1e12}),
                      flush=True)
    os.environ.pop("SKC_NO_NNZ_SORT", None)


if __name__ == "__main__":
    main()
