#!/usr/bin/env python
"""Per-layer binding roof of the conv kernel from committed `ncu --set full` raw captures
(profiles/r02_ncu_conv{2,3,4,5}_raw.csv) -> profiles/r02_layer_roofs.json.

Two on-chip resources can bind the compiled-weights kernel:
  * the FP32 pipe: an SM retires 128 FMA lanes per clock, i.e. 2 warp-wide FFMA2 (64 FMAs) per
    clock -> floor_fma = FFMA2 warp-instructions per SM / 2 cycles;
  * the shared-memory crossbar: 128 B per clock per SM (B300_MICROARCH.md LDS/STS table;
    measured LDS.64 126.8 B/clk/SM in bench.py's peaks), i.e. one wavefront per clock, shared by
    the window loads (LDS wavefronts) and the TMA bulk copies that write the stages
    -> floor_smem = (LDS wavefronts + TMA bytes / 128) per SM cycles.
The layer's roof (in nnz-FLOP/s) = its algorithmic FLOPs (2*nnz*Ho*Wo*N) / max(floor_fma,
floor_smem) at the capture's SM clock; `frac` = that floor / the elapsed cycles, i.e. how close
the kernel runs to the resource that binds it.  FFMA2 thread-instruction counts come from
profiles/r02_ffma_instruction_check.json (same captures).  HBM is far from binding (DRAM
traffic per launch / duration is reported beside it).

    python tools/layer_roofs.py > profiles/r02_layer_roofs.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMS = 148
FFMA2_PER_CLK = 2.0        # warp-wide FFMA2 per clock per SM (128 FP32 lanes / 64)
SMEM_B_PER_CLK = 128.0     # shared-memory crossbar bytes per clock per SM


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    head, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for n, u, v in zip(head, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(u, 1.0)
        out[n] = x * mult
    return out


def main():
    checks = {d["layer"]: d for d in json.load(open(os.path.join(ROOT, "profiles/r02_ffma_instruction_check.json")))}
    res = {"method": __doc__.strip().splitlines()[0], "sms": SMS, "ffma2_per_clk_per_sm": FFMA2_PER_CLK,
           "smem_bytes_per_clk_per_sm": SMEM_B_PER_CLK, "layers": []}
    for layer in ("conv2", "conv3", "conv4", "conv5"):
        src = f"profiles/r02_ncu_{layer}_raw.csv"
        m = raw_metrics(os.path.join(ROOT, src))
        ck = checks[layer]
        dur = m["gpu__time_duration.sum"]
        cyc = m["sm__cycles_elapsed.avg"]
        clk = cyc / dur
        ffma2 = ck["ffma2_thread_inst"] / 32.0
        lds_wf = m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
        tma_b = m.get("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", 0.0)
        floor_fma = ffma2 / SMS / FFMA2_PER_CLK
        floor_lds = lds_wf / SMS
        floor_smem = floor_lds + tma_b / SMEM_B_PER_CLK / SMS
        floor = max(floor_fma, floor_smem)
        flops = 2.0 * ck["macs"]
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        res["layers"].append({
            "layer": layer, "source": src, "kernel_us": dur * 1e6, "sm_clock_ghz": clk / 1e9,
            "elapsed_cycles": cyc, "ffma2_warp_inst": ffma2, "lds_wavefronts": lds_wf,
            "tma_bytes": tma_b,
            "floor_cycles": {"fma_pipe": floor_fma, "smem_lds_only": floor_lds, "smem_with_tma": floor_smem},
            "binding": "fma_pipe" if floor_fma >= floor_smem else "smem",
            "roof_tflops": flops / (floor / clk) / 1e12,
            "achieved_tflops": flops / dur / 1e12,
            "frac_of_binding_roof": floor / cyc,
            "fma_pipe_share_of_elapsed": floor_fma / cyc,
            "smem_share_of_elapsed": floor_smem / cyc,
            "dram_tbs": dram / dur / 1e12,
        })
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
