#!/usr/bin/env python
"""f2 tuning sweep: fold the FC batch axis into rows and split it into bands (more CTAs for
the single 'image'), per AlexNet FC layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402
from chain_bench import timed  # noqa: E402

B = wl.FC_BATCH
for i, L in enumerate(wl.ALEXNET_FC):
    w = wl.gen_fc_weights(i, L)
    x = torch.from_numpy(wl.gen_fc_input(i, L, B)).cuda()
    base = None
    for rows, bands, m in [(1, 1, 0), (8, 2, 0), (8, 4, 0), (8, 8, 0), (4, 4, 0), (8, 4, 2), (8, 8, 2), (8, 2, 2)]:
        os.environ["SKC_FC_ROWS"] = str(rows)
        os.environ["SKC_DIRECT_BANDS"] = str(bands)
        if m: os.environ["SKC_DIRECT_M"] = str(m)
        else: os.environ.pop("SKC_DIRECT_M", None)
        fc = skc.SparseLinear(w, B)
        y = torch.empty((L.M, B), device="cuda")
        ms = timed(lambda: fc.forward(x, out=y))
        if base is None:
            base = y.clone()
        g = fc.plan.info()
        print(L.name, "rows", rows, "bands", bands, "M", g["channels_per_warp"], "T", g["pixels_per_lane"],
              round(ms, 4), "ms", round(2 * g["nnz"] * B / ms / 1e9, 2), "TF", "eq", bool(torch.equal(y, base)), flush=True)
for k in ("SKC_FC_ROWS", "SKC_DIRECT_BANDS", "SKC_DIRECT_M"):
    os.environ.pop(k, None)
