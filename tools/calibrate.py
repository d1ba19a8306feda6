#!/usr/bin/env python
"""Measure the B200 FP32 FFMA rate and the shared-memory word rate with libskc's
micro-benchmarks (the paper's SGEMM/STREAM calibration analogue).
Prints one JSON line; bench.py's roofline uses the guide-derived FP32 peak, these are
recorded beside it."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1608_01409_b200 import skc  # noqa: E402


def main():
    scratch = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for blocks in (148 * 4, 148 * 8):
        ms, fl = skc.skc_bench_ffma(scratch, blocks, 4096)
        res[f"ffma_tflops_b{blocks}"] = fl / ms / 1e9
        ms, by = skc.skc_bench_lds(scratch, blocks, 4096)
        res[f"lds_tbs_b{blocks}"] = by / ms / 1e9
    props = torch.cuda.get_device_properties(0)
    res["sm_count"] = props.multi_processor_count
    res["name"] = props.name
    print(json.dumps(res))


if __name__ == "__main__":
    main()
