#!/usr/bin/env python
"""Row f2 measurement: AlexNet fc6-fc8 (90% element-wise sparse) at batch 256 as SpMDM with
the SpMDM kernel (AUTO) and the direct kernel, against dense FP32 cuBLAS SGEMM of the same
shape.  Roofline: shared-memory wavefronts."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from chain_bench import timed  # noqa: E402


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    B = wl.FC_BATCH
    for i, L in enumerate(wl.ALEXNET_FC):
        w = wl.gen_fc_weights(i, L)
        x = torch.from_numpy(wl.gen_fc_input(i, L, B)).cuda()
        fc = skc.SparseLinear(w, B)
        y = torch.empty((L.M, B), device="cuda")
        t_sp = timed(lambda: fc.forward(x, out=y))
        fd = skc.SparseLinear(w, B, skc.SKC_KERNEL_DIRECT)
        y2 = torch.empty((L.M, B), device="cuda")
        t_dir = timed(lambda: fd.forward(x, out=y2))
        wd = torch.from_numpy(w).cuda()
        t_dense = timed(lambda: torch.matmul(wd, x))
        g = fc.plan.info()
        nnz = g["nnz"]
        print(json.dumps({"layer": L.name, "M": L.M, "K": L.K, "batch": B, "nnz": nnz,
                          "kernel": g["kernel"], "LC": g["pixels_per_lane"],
                          "RWM": g["channels_per_warp"], "KC": g["chunk_channels"],
                          "stages": g["stages"], "smem": g["smem_bytes"],
                          "sparse_ms": t_sp, "direct_ms": t_dir, "sgemm_ms": t_dense,
                          "speedup": t_dense / t_sp, "vs_direct": t_dir / t_sp,
                          "bitwise_vs_direct": bool(torch.equal(y, y2)),
                          "nnz_tflops": 2.0 * nnz * B / (t_sp * 1e-3) / 1e12,
                          "sgemm_tflops": 2.0 * L.M * L.K * B / (t_dense * 1e-3) / 1e12}),
              flush=True)


if __name__ == "__main__":
    main()
