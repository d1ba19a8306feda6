#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the direct-sparse-convolution hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A STEP is one pass of the whole hot path over one batch: for every
layer of the workload, skc_pad_input (a2) then skc_sparse_conv_forward (a3..a6); the CSR
packing (a1) is a one-off per layer, done before timing ("pre-computed").
Workload at N = 1: BASELINE.json configs[1] (AlexNet conv2-5, batch 256, FP32).  With N
GPUs every rank runs its own 256 images (weak scaling; images are independent so the path
has no collective -- SURVEY.md Sec. 8(e)); the whole-job value is all images / max-over-ranks time.

Printed by rank 0: ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

METRIC = "effective GFLOP/s (2·nnz MACs/s) and speedup vs dense, AlexNet conv2–5 batch 256"
N_SM, FP32_LANES, SMEM_WORDS_PER_CLK = 148, 128, 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: the config's)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "direct", "regtile", "jit"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time plain launches, no CUDA graph")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def nnz_flops(layer, nnz, n_images):
    return 2.0 * nnz * layer.Ho * layer.Wo * n_images


def dense_flops(layer, n_images):
    return 2.0 * layer.K * (layer.C // layer.groups) * layer.R * layer.S * layer.Ho * layer.Wo * n_images


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def start(self):
        """Launch nvidia-smi and wait (<= 5 s) for its first sample, before timing starts."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.01)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def mark(self):
        """Start of the timed region: only samples after this count."""
        self.lines.clear()

    def __enter__(self):
        if self.proc is None:
            self.start()
        self.mark()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic():
    """dram bytes per launch from a committed ncu --set full capture (profiles/), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except (OSError, ValueError):
            return None
    return None


# ----------------------------------------------------------------------------- oracle legs
def oracle_sample(cfg, budget_s):
    """Time the oracle (as it stands) on a bounded sample: whole images of every layer,
    doubling until the budget is used.  Returns (nnz_flops, dense_flops, seconds, images)."""
    import oracle
    ws = [wl.gen_weights(cfg.cfg_id, li, L) for li, L in enumerate(cfg.layers)]
    xs = [wl.gen_input(cfg.cfg_id, li, L, 0, 1) for li, L in enumerate(cfg.layers)]
    total_nnz = total_dense = total_t = 0.0
    n_img = 0
    reps = 1
    while True:
        t0 = time.perf_counter()
        for _ in range(reps):
            for L, w, x in zip(cfg.layers, ws, xs):
                oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups, want_bound=False)
        dt = time.perf_counter() - t0
        total_t += dt
        n_img += reps
        for L, w in zip(cfg.layers, ws):
            total_nnz += nnz_flops(L, np.count_nonzero(w), reps)
            total_dense += dense_flops(L, reps)
        if total_t >= budget_s / 3 or reps >= 64:
            break
        reps *= 2
    return total_nnz, total_dense, total_t, n_img


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle timed on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    ws = [wl.gen_weights(cfg.cfg_id, li, L) for li, L in enumerate(cfg.layers)]
    xs = [wl.gen_input(cfg.cfg_id, li, L, 0, 1) for li, L in enumerate(cfg.layers)]
    nnzs = [np.count_nonzero(w) for w in ws]

    def step():
        for L, w, x in zip(cfg.layers, ws, xs):
            oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups, want_bound=False)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    flops = sum(nnz_flops(L, z, 1) for L, z in zip(cfg.layers, nnzs))
    value = flops / t / 1e9
    sample = f"1 image of each of {len(cfg.layers)} layers per step (of {cfg.batch})"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name + " (BASELINE.json configs[%d])" % (cfg.cfg_id - 1),
                   "per_step_sample": sample, "oracle": "oracle/oracle_conv.c seven-loop, fp64, OpenMP"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": oracle.num_threads(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our leg
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1608_01409_b200 import skc

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: CUDA device required (there is no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    skc.lib()

    from paper_1608_01409_b200 import dist as skd
    per_gpu = args.batch or cfg.batch
    n0, n1 = skd.shard_range(per_gpu * world, world, rank)  # weak scaling: per_gpu images each
    kernel = {"auto": skc.SKC_KERNEL_AUTO, "direct": skc.SKC_KERNEL_DIRECT,
              "regtile": skc.SKC_KERNEL_REGTILE, "jit": skc.SKC_KERNEL_JIT}[args.kernel]
    stream = torch.cuda.current_stream(dev)

    layers = []
    t_build = time.time()
    # plan build (pack + JIT compile + upload): one-off, untimed; the JIT
    # compiles of the layers run concurrently (host threads; ctypes releases the GIL)
    plans = [skc.skc_pack_csr(wl.gen_weights(cfg.cfg_id, li, L), L.H, L.W, L.stride, L.pad,
                              L.groups, kernel) for li, L in enumerate(cfg.layers)]
    import concurrent.futures as cf
    # N ranks of one node: local rank 0 compiles first and fills the on-disk JIT cache, the
    # others then load the same code from it instead of N concurrent compiles
    if world > 1 and local_rank != 0:
        dist.barrier()
    with cf.ThreadPoolExecutor(max_workers=len(plans)) as ex:
        list(ex.map(skc.skc_plan_compile, plans))
    if world > 1 and local_rank == 0:
        dist.barrier()
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(cfg.cfg_id, li, L)
        conv = skc.SparseConv2d.from_plan(plans[li], dev)
        # launch-schedule tuning for this batch on this device (setup, untimed; outputs are
        # bitwise unaffected -- DESIGN.md Sec. 7.4)
        if os.environ.get("SKC_TUNE", "1") != "0":
            conv.tune(per_gpu)
        x_host = torch.from_numpy(wl.gen_input(cfg.cfg_id, li, L, n0, n1))
        x = x_host.to(dev)
        # (the raw layout is the NCHW input itself: the kernel pads while staging, and
        # skc_pad_input on the same buffer is a no-op)
        xp = x if conv.geom["layout"] == skc.SKC_LAYOUT_RAW else torch.empty(conv.padded_shape(per_gpu), device=dev)
        out = torch.empty(conv.out_shape(per_gpu), device=dev)
        layers.append(dict(L=L, w=w, conv=conv, x=x, xp=xp, out=out, x_host=x_host,
                           nnz=int(conv.geom["nnz"])))
        if world > 1 and not skd.check_same_plan(conv.plan, dev):
            raise SystemExit(f"bench.py: rank {rank} packed a different plan for {L.name}")

    t_build = time.time() - t_build
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step_on(st, evs=None):
        for i, d in enumerate(layers):
            skc.skc_pad_input(d["conv"].plan, d["x"], d["xp"], per_gpu, st)
            if evs is not None:
                evs[2 * i + 1].record(st)
            skc.skc_sparse_conv_forward(d["conv"].plan, d["xp"], d["out"], per_gpu, st)
            if evs is not None:
                evs[2 * i + 2].record(st)

    def step(evs=None):
        step_on(stream, evs)

    clk = ClockSampler(local_rank).start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # the step's 8 launches captured once in a CUDA graph (replayed per timed step: no
    # host launch gaps between the kernels); per-layer times come from an uncaptured pass
    graph = None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step_on(cap)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            graph = g
        except Exception as e:  # noqa: BLE001 -- report and time the plain launches
            print(f"bench.py: CUDA graph capture failed ({e}); timing plain launches",
                  file=sys.stderr)
            graph = None

    nev = 2 * len(layers) + 1
    per_kernel = np.zeros(nev - 1)
    step_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with clk:
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between timed steps (outside the events)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
            evs[0].record(stream)
            step(evs)
            torch.cuda.synchronize()
            ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(nev - 1)]
            per_kernel += ts
            step_ms.append(evs[0].elapsed_time(evs[-1]))
        if graph is not None:
            step_ms = []
            for _ in range(args.steps):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                graph.replay()
                b.record(stream)
                torch.cuda.synchronize()
                step_ms.append(a.elapsed_time(b))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_kernel /= args.steps
    t_step = float(np.mean(step_ms))
    if world > 1:
        t_step = skd.max_over_ranks(t_step, dev)

    step_nnz_flops = sum(nnz_flops(d["L"], d["nnz"], per_gpu) for d in layers)
    step_dense_flops = sum(dense_flops(d["L"], per_gpu) for d in layers)
    value = step_nnz_flops * world / (t_step * 1e-3) / 1e9

    # ---- dense FP32 baseline (cuDNN, TF32 off), same protocol
    dense = None
    if not args.no_dense:
        wd = [torch.from_numpy(d["w"]).to(dev) for d in layers]
        def dstep():
            for d, w in zip(layers, wd):
                torch.nn.functional.conv2d(d["x"], w, stride=d["L"].stride, padding=d["L"].pad,
                                           groups=d["L"].groups)
        for _ in range(3):
            dstep()
        torch.cuda.synchronize()
        dms = []
        for _ in range(max(3, args.steps // 2)):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); dstep(); b.record(stream)
            torch.cuda.synchronize()
            dms.append(a.elapsed_time(b))
        t_dense = float(np.mean(dms))
        del wd
        # the paper's proxy for dense convolution: FP32 SGEMM at the lowered shape
        # [K/g x C/g*R*S] x [C/g*R*S x Ho*Wo*N] per group
        sg_ms = 0.0
        for d in layers:
            L = d["L"]
            kk, cc, pp = L.K // L.groups, (L.C // L.groups) * L.R * L.S, L.Ho * L.Wo * per_gpu
            A = torch.randn(kk, cc, device=dev)
            B = torch.randn(cc, pp, device=dev)
            for _ in range(2):
                torch.matmul(A, B)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            a.record(stream)
            for _ in range(reps):
                torch.matmul(A, B)
            b.record(stream)
            torch.cuda.synchronize()
            sg_ms += a.elapsed_time(b) / reps * L.groups
            del A, B
        dense = {"cudnn_fp32_ms": t_dense, "speedup_vs_cudnn_fp32": t_dense / t_step,
                 "cudnn_dense_equiv_gflops": step_dense_flops / (t_dense * 1e-3) / 1e9,
                 "sgemm_proxy_ms": sg_ms, "speedup_vs_sgemm_proxy": sg_ms / t_step,
                 "sgemm_gflops": step_dense_flops / (sg_ms * 1e-3) / 1e9,
                 "note": "cuDNN FP32 (allow_tf32=False) may use Winograd/FFT, so its dense-"
                         "equivalent rate can exceed the FP32 FMA peak; the paper's own dense "
                         "baseline is the SGEMM proxy (PAPER.md:728-732)"}

    # ---- end to end through the C-ABI host entry point (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        hin = [d["x_host"].pin_memory() for d in layers]
        hout = [torch.empty(d["conv"].out_shape(per_gpu)).pin_memory() for d in layers]
        # the four layers are independent: each runs its H2D / pad + conv / D2H pipeline on
        # its own stream (forked from and joined back into the timed stream), so one layer's
        # output copy overlaps the next layer's input copy on the two copy engines
        side = [torch.cuda.Stream(dev) for _ in layers]

        def estep():
            fork = torch.cuda.Event()
            fork.record(stream)
            for s_, d, hi, ho in zip(side, layers, hin, hout):
                s_.wait_event(fork)
                skc.skc_forward_host(d["conv"].plan, hi, ho, per_gpu, d["x"], d["xp"], d["out"],
                                     s_)
            for s_ in side:
                j = torch.cuda.Event()
                j.record(s_)
                stream.wait_event(j)
        estep(); torch.cuda.synchronize()
        ems = []
        for _ in range(max(3, args.steps // 4)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream); estep(); b.record(stream)
            torch.cuda.synchronize()
            ems.append(a.elapsed_time(b))
        t_e2e = float(np.mean(ems))
        if world > 1:
            t_e2e = skd.max_over_ranks(t_e2e, dev)
        e2e = {"value": step_nnz_flops * world / (t_e2e * 1e-3) / 1e9, "unit": "GFLOP/s",
               "ms_per_step": t_e2e,
               "h2d_bytes_per_step": int(sum(h.numel() * 4 for h in hin)),
               "d2h_bytes_per_step": int(sum(h.numel() * 4 for h in hout))}

    if rank != 0:
        return
    clocks = clk.summary()
    # ---- roofline of the dominant kernel (the conv kernel of the layer with most time)
    conv_ms = per_kernel[1::2]
    pad_ms = per_kernel[0::2]
    dom = int(np.argmax(conv_ms))
    dl = layers[dom]
    achieved = nnz_flops(dl["L"], dl["nnz"], per_gpu) / (conv_ms[dom] * 1e-3) / 1e12
    f_max = (clocks["sm_max_mhz"] or 1965.0) * 1e6
    peak_fp32 = N_SM * FP32_LANES * 2 * f_max / 1e12
    peak_smem = N_SM * SMEM_WORDS_PER_CLK * 2 * f_max / 1e12
    traffic = load_traffic()
    tr = None
    if traffic and traffic.get("kernel_layer") == dl["L"].name and traffic.get("kernel") == args.kernel:
        tr = traffic.get("dram_bytes_per_launch")
    per_layer = []
    for d, cm, pm in zip(layers, conv_ms, pad_ms):
        L = d["L"]
        per_layer.append({
            "layer": L.name, "nnz": d["nnz"], "density": d["nnz"] / (L.K * (L.C // L.groups) * L.R * L.S),
            "conv_ms": float(cm), "pad_ms": float(pm),
            "conv_nnz_tflops": nnz_flops(L, d["nnz"], per_gpu) / (cm * 1e-3) / 1e12,
            "pad_gbs": per_gpu * 4 * (L.C * L.H * L.W + L.C * (L.H + 2 * L.pad) * (L.W + 2 * L.pad)) / (pm * 1e-3) / 1e9,
            "kernel_cfg": {k: d["conv"].plan.info()[k] for k in (
                "kernel", "band_rows", "chunk_channels", "stages", "warps", "channels_per_warp",
                "pixels_per_lane", "smem_bytes", "tile_h", "tile_w", "images_per_cta",
                "jit_blocks", "jit_split", "jit_sched", "code_bytes", "jit_compile_s", "jit_cache_hit")},
        })
    cpu = None
    if not args.no_cpu and world >= 1:
        import oracle
        oracle.build()
        nf, df, secs, nimg = oracle_sample(cfg, args.cpu_seconds)
        cpu = {"value": nf / secs / 1e9, "unit": "GFLOP/s", "cores": oracle.num_threads(),
               "kind": "oracle",
               "sample": f"{nimg} image(s) of each of the {len(cfg.layers)} layers ({secs:.1f} s)",
               "dense_equiv_gflops": df / secs / 1e9}
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name} (BASELINE.json configs[{cfg.cfg_id - 1}])",
                   "global_batch": per_gpu * world, "per_gpu_batch": per_gpu,
                   "layers": [l.name for l in cfg.layers], "parallelism": f"dp{world} (batch-sharded, no collective)",
                   "l2": "flushed between timed steps (256 MiB write)", "kernel": args.kernel,
                   "step": "per layer: skc_pad_input + skc_sparse_conv_forward"
                           + (", the step's 8 launches replayed as one CUDA graph" if graph is not None else "")},
        "dense_equiv_gflops": step_dense_flops * world / (t_step * 1e-3) / 1e9,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                     "frac": achieved / peak_fp32, "traffic": tr,
                     "kernel": f"skc_sparse_conv_forward ({dl['L'].name})",
                     "peak_basis": f"148 SM x 128 FP32 lanes x 2 x {f_max/1e6:.0f} MHz (CUDA-core FFMA)",
                     "smem_roof": peak_smem, "frac_smem_roof": achieved / peak_smem},
        "per_layer": per_layer,
        "dense": dense,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": 2 * len(layers) * args.steps,
        "plan_build_s": t_build,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    cfg = wl.CONFIGS[args.config]
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference(args, cfg, rank, world)
        else:
            run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1 and args.impl == "ours":
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
