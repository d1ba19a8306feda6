#!/usr/bin/env python
"""SURVEY.md Sec. 8(d) work check: the FP32 FMAs the conv kernel executed (ncu thread-level
counts, FFMA + 2 x FFMA2 -- an FFMA2 is two FMAs) against the algorithmic MACs
nnz x Ho x Wo x N, with the excess explained by the kernel's known waste:
  * idle lanes: a CTA's NW x 32 lanes hold NSL image pairs x the band's tiles; the rest
    mirror a neighbour and compute without storing;
  * the last image group: ceil(N / NI) x NI images are computed (missing ones on zeros);
  * the dry-run code prefetch: min(G, blocks x chunks) chunk segments (G with jit_sched
    bit 9) each execute one chunk of a block's code once more.

    python tools/ffma_check.py --sched conv2=553,conv3=32,... conv2=raw.csv ... \
        > profiles/r02_ffma_instruction_check.json
"""
import argparse
import csv
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl  # noqa: E402
from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--grid", type=int, default=148)
    ap.add_argument("--sched", default="", help="layer=jit_sched,... (the profiled launch's)")
    ap.add_argument("layers", nargs="+", help="name=ncu raw csv (ncu --page raw --csv)")
    a = ap.parse_args()
    sched = dict(kv.split("=") for kv in a.sched.split(",") if kv)
    cfg = wl.CONFIGS[a.config]
    out = []
    for item in a.layers:
        name, path = item.split("=", 1)
        li = [L.name for L in cfg.layers].index(name)
        L = cfg.layers[li]
        rows = list(csv.reader(open(path)))
        g = dict(zip(rows[0], rows[2]))
        num = lambda k: float(g[k].replace(",", ""))  # noqa: E731
        ffma = num("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum")
        ffma2 = num("smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum")
        w = wl.gen_weights(a.config, li, L)
        plan = skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups)
        i = plan.info()
        nnz, N = i["nnz"], a.batch
        macs = nnz * L.Ho * L.Wo * N
        executed = ffma + 2 * ffma2
        # waste model
        NI, NW, bands = i["images_per_cta"], i["warps"], max(1, i["bands"])
        pairs = NI // 2
        tiles_y = math.ceil(L.Ho / i["tile_h"]) if i["tile_h"] else L.Ho
        tiles_x = math.ceil(L.Wo / i["tile_w"]) if i["tile_w"] else L.Wo
        band_tiles = math.ceil(tiles_y / bands) * tiles_x  # the largest band
        lane_eff = pairs * band_tiles / (NW * 32)
        groups = math.ceil(N / NI)
        tail = groups * NI / N
        nchunks = math.ceil((L.C // L.groups) / i["chunk_channels"])
        items = groups * bands * i["jit_blocks"]
        s = int(sched.get(name, i["jit_sched"]))
        segs = a.grid if (s >= 0 and s & 512) else min(a.grid, i["jit_blocks"] * nchunks)
        dry = segs / (nchunks * items)
        predicted = (1.0 / lane_eff) * tail * (1.0 + dry)
        out.append({"layer": name, "nnz": nnz, "macs": macs, "ffma_thread_inst": ffma,
                    "ffma2_thread_inst": ffma2, "executed_fmas": executed,
                    "executed_over_macs": executed / macs,
                    "waste_model": {"lane_efficiency": lane_eff, "image_tail": tail,
                                    "dry_run_segments": segs, "dry_run_fraction": dry,
                                    "predicted_executed_over_macs": predicted},
                    "source": os.path.relpath(path)})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
