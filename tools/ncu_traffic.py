#!/usr/bin/env python
"""Build profiles/ncu_traffic.json (read by bench.py for roofline.traffic) from per-layer
ncu --set full summaries (tools/ncu_summary.py output): DRAM bytes read + written per launch
of each layer's conv kernel, next to the layer's algorithmic bytes 4*N*(C*Hp*Wp + K*Ho*Wo)
(the padded input read once, the output written once).

    python tools/ncu_traffic.py --config 2 --batch 256 \
        conv2=profiles/r02_ncu_conv2_full.json conv3=... > profiles/ncu_traffic.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as wl  # noqa: E402


def scale(key: str) -> float:
    unit = key[key.index("[") + 1:key.index("]")] if "[" in key else "byte"
    return {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("layers", nargs="+", help="name=summary.json")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    by_name = {L.name: L for L in cfg.layers}
    out = {"kernel": a.kernel, "configs": [a.config] + ([5] if a.config == 2 else []),
           "batch": a.batch, "dram_bytes_per_launch": {}, "dram_read_bytes": {},
           "dram_write_bytes": {}, "algorithmic_bytes_per_launch": {}, "traffic_over_algorithmic": {},
           "kernel_us": {}, "sources": {}}
    for item in a.layers:
        name, path = item.split("=", 1)
        L = by_name[name]
        d = json.load(open(path))[0]
        rd = wr = t = None
        for k, v in d.items():
            if k.startswith("dram__bytes_read.sum"):
                rd = float(v) * scale(k)
            elif k.startswith("dram__bytes_write.sum"):
                wr = float(v) * scale(k)
            elif k.startswith("gpu__time_duration.sum"):
                t = float(v)
        alg = 4.0 * a.batch * (L.C * (L.H + 2 * L.pad) * (L.W + 2 * L.pad) + L.K * L.Ho * L.Wo)
        out["dram_read_bytes"][name] = rd
        out["dram_write_bytes"][name] = wr
        out["dram_bytes_per_launch"][name] = rd + wr
        out["algorithmic_bytes_per_launch"][name] = alg
        out["traffic_over_algorithmic"][name] = (rd + wr) / alg
        out["kernel_us"][name] = t
        out["sources"][name] = os.path.relpath(path, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
