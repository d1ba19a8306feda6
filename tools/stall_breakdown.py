#!/usr/bin/env python
"""Summarise an ncu --page source --csv --print-source sass export (gzip or plain): warp-stall
samples by opcode and by stall reason, and the share of samples in the inner code (FFMA2 +
LDS) versus everything else (staging waits, item set-up, epilogue, dry run).

    python tools/stall_breakdown.py gpurun_out/r02_conv_l1_source.csv.gz
"""
import csv
import gzip
import io
import json
import re
import sys
from collections import Counter


def main(path):
    raw = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    lines = raw.read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    i_src, i_samp = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    by_op, total = Counter(), 0
    reason = Counter()
    op_reason = {}
    reason_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    for r in rows[1:]:
        if len(r) <= i_samp:
            continue
        try:
            n = int(r[i_samp])
        except ValueError:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src])
        op = m.group(2) if m else "?"
        by_op[op] += n
        total += n
        for j in reason_cols:
            try:
                v = int(r[j])
            except (ValueError, IndexError):
                continue
            reason[hdr[j][6:]] += v
            op_reason.setdefault(op, Counter())[hdr[j][6:]] += v
    inner = by_op["FFMA2"] + by_op["LDS"]
    out = {"samples": total, "inner_code_share": inner / max(total, 1),
           "opcode_share": {k: round(v / total, 4) for k, v in by_op.most_common(14)},
           "reason_share": {k: round(v / max(sum(reason.values()), 1), 4) for k, v in reason.most_common(14)},
           "top_reasons_by_opcode": {op: {k: round(v / total, 4) for k, v in op_reason[op].most_common(4)}
                                     for op, _ in by_op.most_common(6) if op in op_reason}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
