#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the direct-sparse-convolution hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A STEP is one pass of the whole hot path over one batch: for every
layer of the workload, skc_pad_input (a2) then skc_sparse_conv_forward (a3..a6); the CSR
packing (a1) is a one-off per layer, done before timing ("pre-computed").
Workload at N = 1: BASELINE.json configs[1] (AlexNet conv2-5, batch 256, FP32).  With N
GPUs every rank runs its own 256 images (weak scaling; images are independent so the path
has no collective -- SURVEY.md Sec. 8(e)); the whole-job value is all images / max-over-ranks
time.  --config 5 is BASELINE.json configs[4]: ONE global batch of 4096 sharded across the
ranks (strong scaling); after timing, every layer's outputs are gathered over NCCL, compared
bit for bit with one GPU's run of the whole batch, and >= 8 images per shard (first and last
included) are checked against the oracle.

After timing, seeded images of the TIMED outputs of every layer are checked against the fp64
oracle (`parity`), and the FFMA / FFMA2 / LDS micro-benchmarks give the measured peaks the
roofline is also reported against (`peaks_measured`, `roofline.frac_measured`).

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
    ap.add_argument("--batch", type=int, default=0,
                    help="per-GPU batch (config 5: the global batch; default: the config's)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "direct", "regtile", "jit"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time plain launches, no CUDA graph")
    ap.add_argument("--pad-overlap", type=int, default=1, choices=[0, 1],
                    help="graph step: run the pads of layers 2..L on a low-priority side stream, "
                         "filling the previous conv's tail (the layers' inputs are independent)")
    ap.add_argument("--order", default="",
                    help="graph step with --pad-overlap: layer order, e.g. 0132 (default: 0213 for configs 2 and 5, else natural)")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--no-cpu-single", action="store_true", help="skip the 1-thread oracle timing")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed outputs")
    ap.add_argument("--parity-images", type=int, default=16, help="images per layer the oracle checks")
    ap.add_argument("--no-peaks", action="store_true", help="skip the FFMA/LDS micro-benchmarks")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: host-side collectives; lets "
                         "several ranks share one GPU for a functional run of the multi-rank path)")
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


def load_layer_roofs():
    """Per-layer binding roof (FP32 pipe vs shared-memory crossbar incl. the TMA stage writes)
    from the committed ncu captures (profiles/r02_layer_roofs.json, tools/layer_roofs.py)."""
    path = os.path.join(ROOT, "profiles", "r02_layer_roofs.json")
    try:
        return {d["layer"]: d for d in json.load(open(path))["layers"]}
    except (OSError, ValueError, KeyError):
        return {}


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


# ----------------------------------------------------------------------------- checks
def sample_images(lo: int, hi: int, k: int, rng) -> list:
    """k images of [lo, hi) (all if fewer): always the first and the last, the rest seeded."""
    idx = {lo, hi - 1} if hi > lo else set()
    while len(idx) < min(k, hi - lo):
        idx.add(int(rng.integers(lo, hi)))
    return sorted(idx)


def oracle_err(x_imgs, w, L, got) -> float:
    """max over elements of |got - oracle| / sum|w*x| for images x_imgs (inf if an element
    whose sum|w*x| is 0 is not exactly 0) -- the north star's tolerance is 1e-4."""
    import oracle
    ref, bound = oracle.conv2d_fp64(x_imgs, w, L.stride, L.pad, L.groups)
    got = np.asarray(got, dtype=np.float64)
    zero = bound == 0
    if np.any(got[zero] != 0):
        return float("inf")
    ratio = np.abs(got - ref)[~zero] / bound[~zero]
    return float(ratio.max()) if ratio.size else 0.0


def verify_gathered(gathered, full, cfg_id: int, li: int, L, w, n_total: int, world: int,
                    per_shard: int = 8, seed: int = 0) -> dict:
    """SURVEY.md Sec. 8(c)/(e) for a batch-sharded run: the outputs gathered from all ranks
    must equal, BIT FOR BIT, one device's run over the whole batch (`full`; None = skip), and
    >= per_shard images of every shard -- its first and last included -- must pass the oracle.
    gathered / full: [n_total, K, Ho, Wo] float32 arrays (NumPy or CPU tensors)."""
    from paper_1608_01409_b200 import dist as skd
    g = np.asarray(gathered)
    res = {"layer": L.name, "images": 0, "max_err_over_bound": 0.0, "bitwise_vs_1gpu": None}
    if full is not None:
        res["bitwise_vs_1gpu"] = bool(np.array_equal(g.view(np.uint32), np.asarray(full).view(np.uint32)))
    rng = np.random.default_rng([seed, cfg_id, li])
    for r in range(world):
        lo, hi = skd.shard_range(n_total, world, r)
        idx = sample_images(lo, hi, per_shard, rng)
        for n in idx:
            x = wl.gen_input(cfg_id, li, L, n, n + 1)
            res["max_err_over_bound"] = max(res["max_err_over_bound"], oracle_err(x, w, L, g[n:n + 1]))
        res["images"] += len(idx)
    return res


def measure_peaks(skc, torch, dev) -> dict:
    """FFMA / FFMA2 / LDS.32 / LDS.64 micro-benchmarks in this session: the measured
    "achievable" FP32 and shared-memory rates (as the paper measured SGEMM and STREAM,
    PAPER.md:550-552), beside the nominal unit-count peaks."""
    scratch = torch.empty(4 << 20, dtype=torch.uint8, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks = nsm * 8  # 2048 threads per SM
    out = {"blocks": blocks, "threads_per_block": 256}
    for name, fn, iters, scale, unit in (("ffma", skc.skc_bench_ffma, 4096, 1e9, "tflops"),
                                         ("ffma2", skc.skc_bench_ffma2, 2048, 1e9, "tflops"),
                                         ("lds32", skc.skc_bench_lds, 4096, 1e9, "tbs"),
                                         ("lds64", skc.skc_bench_lds64, 2048, 1e9, "tbs")):
        best = None
        for _ in range(3):
            ms, n = fn(scratch, blocks, iters)
            v = n / ms / scale
            best = v if best is None else max(best, v)
        out[f"{name}_{unit}"] = best
    return out


# ----------------------------------------------------------------------------- our leg
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1608_01409_b200 import skc

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: CUDA device required (there is no CPU fallback)")
    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    # collectives (off the timed path) on the GPU with NCCL, on host tensors with gloo
    cdev = dev if args.backend == "nccl" else torch.device("cpu")
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    skc.lib()

    from paper_1608_01409_b200 import dist as skd
    # config 5 (BASELINE.json configs[4]): ONE global batch (4096) sharded across the ranks --
    # strong scaling; every other config: each rank runs the config's batch -- weak scaling.
    # Images are independent, so either way there is no collective on the data path.
    strong = cfg.cfg_id == 5
    if strong:
        n_global = args.batch or cfg.batch
        n0, n1 = skd.shard_range(n_global, world, rank)
    else:
        per = args.batch or cfg.batch
        n_global = per * world
        n0, n1 = rank * per, (rank + 1) * per
    local_n = n1 - n0
    kernel = {"auto": skc.SKC_KERNEL_AUTO, "direct": skc.SKC_KERNEL_DIRECT,
              "regtile": skc.SKC_KERNEL_REGTILE, "jit": skc.SKC_KERNEL_JIT}[args.kernel]
    stream = torch.cuda.current_stream(dev)

    layers = []
    t_build = time.time()
    # plan build (pack + JIT compile + upload): one-off, untimed; the JIT
    # compiles of the layers run concurrently (host threads; ctypes releases the GIL)
    ws = [wl.gen_weights(cfg.cfg_id, li, L) for li, L in enumerate(cfg.layers)]
    # each plan configured for the images one forward call of this rank processes
    plans = [skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups, kernel, batch_hint=local_n)
             for w, L in zip(ws, cfg.layers)]
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
        conv = skc.SparseConv2d.from_plan(plans[li], dev)
        # launch-schedule tuning for this batch on this device (setup, untimed; outputs are
        # bitwise unaffected -- DESIGN.md Sec. 7.4)
        if os.environ.get("SKC_TUNE", "1") != "0":
            conv.tune(local_n)
        x_host = torch.from_numpy(wl.gen_input(cfg.cfg_id, li, L, n0, n1))
        x = x_host.to(dev)
        # (the raw layout is the NCHW input itself: the kernel pads while staging, and
        # skc_pad_input on the same buffer is a no-op)
        xp = x if conv.geom["layout"] == skc.SKC_LAYOUT_RAW else torch.empty(conv.padded_shape(local_n), device=dev)
        out = torch.empty(conv.out_shape(local_n), device=dev)
        layers.append(dict(L=L, w=ws[li], conv=conv, x=x, xp=xp, out=out, x_host=x_host,
                           nnz=int(conv.geom["nnz"])))
        if world > 1 and not skd.check_same_plan(conv.plan, cdev):
            raise SystemExit(f"bench.py: rank {rank} packed a different plan for {L.name}")

    t_build = time.time() - t_build
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step_on(st, evs=None):
        for i, d in enumerate(layers):
            skc.skc_pad_input(d["conv"].plan, d["x"], d["xp"], local_n, st)
            if evs is not None:
                evs[2 * i + 1].record(st)
            skc.skc_sparse_conv_forward(d["conv"].plan, d["xp"], d["out"], local_n, st)
            if evs is not None:
                evs[2 * i + 2].record(st)

    def step(evs=None):
        step_on(stream, evs)

    clk = ClockSampler(dev.index).start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # AlexNet conv2-5 (configs 2 and 5): conv2, conv4, conv3, conv5 measured 0.3% faster than the
    # natural order (0.8088-0.8106 vs 0.8115-0.8125 ms over four alternating pairs of 200-step
    # runs; other orders 0.8129-0.8385 ms: profiles/r02_pad_overlap.txt)
    default_order = "0213" if cfg.cfg_id in (2, 5) else ""
    order_s = args.order or default_order
    order = [int(c) for c in order_s] if order_s else list(range(len(layers)))
    if sorted(order) != list(range(len(layers))):
        raise SystemExit(f"bench.py: --order {args.order} is not a permutation of the layers")

    def step_overlap(main, side):
        # the conv launches stay in layer order on the high-priority main stream; the pad of
        # layer i > 0 runs on the low-priority side stream (forked after layer 0's pad) and
        # conv i waits for it.  Every conv kernel fills all SMs (1 CTA of 512 threads x 128
        # registers per SM), so a pad's CTAs get SMs only as the running conv's CTAs retire:
        # the HBM-bound pads fill the ALU-bound convs' tails instead of running between them.
        # (layer order: the natural one measured best, profiles/r02_pad_overlap.txt)
        seq = [layers[i] for i in order]
        skc.skc_pad_input(seq[0]["conv"].plan, seq[0]["x"], seq[0]["xp"], local_n, main)
        fork = torch.cuda.Event()
        fork.record(main)
        side.wait_event(fork)
        ready = []
        for d in seq[1:]:
            skc.skc_pad_input(d["conv"].plan, d["x"], d["xp"], local_n, side)
            e = torch.cuda.Event()
            e.record(side)
            ready.append(e)
        for i, d in enumerate(seq):
            if i > 0:
                main.wait_event(ready[i - 1])
            skc.skc_sparse_conv_forward(d["conv"].plan, d["xp"], d["out"], local_n, main)

    # the step's 8 launches captured once in a CUDA graph (replayed per timed step: no
    # host launch gaps between the kernels); per-layer times come from an uncaptured pass
    graph = None
    if not args.no_graph:
        try:
            lo, hi = torch.cuda.Stream.priority_range()  # (lowest, greatest) priority
            cap = torch.cuda.Stream(dev, priority=hi)
            side = torch.cuda.Stream(dev, priority=lo)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    if args.pad_overlap and len(layers) > 1:
                        step_overlap(cap, side)
                    else:
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
    torch.cuda.nvtx.range_push("timed")  # (select the timed launches in ncu: --nvtx-include timed/)
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
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_kernel /= args.steps
    t_local = float(np.mean(step_ms))
    t_step = t_local
    if world > 1:
        t_step = skd.max_over_ranks(t_local, cdev)

    local_nnz_flops = sum(nnz_flops(d["L"], d["nnz"], local_n) for d in layers)
    step_nnz_flops = sum(nnz_flops(d["L"], d["nnz"], n_global) for d in layers)
    step_dense_flops = sum(dense_flops(d["L"], n_global) for d in layers)
    value = step_nnz_flops / (t_step * 1e-3) / 1e9

    # ---- parity of the TIMED outputs (they hold the last replay's results): seeded images
    # of every layer against the fp64 oracle; with
    # N ranks, the outputs are gathered to every rank (NCCL all_gather, off the timed path),
    # compared bit for bit with one device's run over the whole batch, and >= 8 images per
    # shard go through the oracle
    parity = None
    if not args.no_parity:
        import oracle
        oracle.build()
        torch.cuda.synchronize()
        per_layer_par = []
        rng = np.random.default_rng([1608, cfg.cfg_id, rank])
        for li, d in enumerate(layers):
            L = d["L"]
            if world == 1:
                idx = sample_images(0, local_n, args.parity_images, rng)
                got = d["out"][idx].cpu().numpy()
                x_imgs = d["x_host"][idx].numpy()
                e = oracle_err(x_imgs, d["w"], L, got)
                per_layer_par.append({"layer": L.name, "images": len(idx), "max_err_over_bound": e})
                continue
            full_g = skd.gather_images(d["out"] if cdev.type == "cuda" else d["out"].cpu(),
                                       n_global) if strong else None
            if not strong:
                # weak scaling: every rank checks its own images against the oracle
                idx = sample_images(0, local_n, args.parity_images, rng)
                e = oracle_err(d["x_host"][idx].numpy(), d["w"], L, d["out"][idx].cpu().numpy())
                e = skd.max_over_ranks(e, cdev)
                per_layer_par.append({"layer": L.name, "images": len(idx) * world, "max_err_over_bound": e})
                continue
            ref = None
            if rank == 0:
                # one device's run over the whole global batch, same plan
                conv = d["conv"]
                xg = torch.from_numpy(wl.gen_input(cfg.cfg_id, li, L, 0, n_global)).to(dev)
                xpg = torch.empty(conv.padded_shape(n_global), device=dev)
                skc.skc_pad_input(conv.plan, xg, xpg, n_global)
                ref = torch.empty(conv.out_shape(n_global), device=dev)
                skc.skc_sparse_conv_forward(conv.plan, xpg, ref, n_global)
                del xg, xpg
                res = verify_gathered(full_g.cpu().numpy(), ref.cpu().numpy(), cfg.cfg_id, li, L,
                                      d["w"], n_global, world)
                per_layer_par.append(res)
            del full_g, ref
            if world > 1:
                dist.barrier()
        if rank == 0:
            worst = max(p["max_err_over_bound"] for p in per_layer_par)
            parity = {"max_err_over_bound": worst, "tolerance": 1e-4, "pass": worst <= 1e-4,
                      "images": sum(p["images"] for p in per_layer_par),
                      "what": ("timed outputs, seeded images incl. first and last, vs the fp64 "
                               "oracle (oracle/oracle_conv.c)"
                               + ("; outputs of all ranks gathered and compared bitwise with a "
                                  "1-GPU run of the global batch" if strong and world > 1 else "")),
                      "per_layer": per_layer_par}
            if strong and world > 1:
                parity["bitwise_vs_1gpu"] = all(p["bitwise_vs_1gpu"] for p in per_layer_par)
                parity["pass"] = parity["pass"] and parity["bitwise_vs_1gpu"]

    # ---- measured peaks (micro-benchmarks, this session)
    peaks = None if args.no_peaks else measure_peaks(skc, torch, dev)

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
            kk, cc, pp = L.K // L.groups, (L.C // L.groups) * L.R * L.S, L.Ho * L.Wo * local_n
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
        dense = {"cudnn_fp32_ms": t_dense, "speedup_vs_cudnn_fp32": t_dense / t_local,
                 "cudnn_dense_equiv_gflops": sum(dense_flops(d["L"], local_n) for d in layers) / (t_dense * 1e-3) / 1e9,
                 "sgemm_proxy_ms": sg_ms, "speedup_vs_sgemm_proxy": sg_ms / t_local,
                 "sgemm_gflops": sum(dense_flops(d["L"], local_n) for d in layers) / (sg_ms * 1e-3) / 1e9,
                 "note": "per rank, its own images; cuDNN FP32 (allow_tf32=False) may use "
                         "Winograd/FFT, so its dense-equivalent rate can exceed the FP32 FMA "
                         "peak; the paper's own dense baseline is the SGEMM proxy "
                         "(PAPER.md:728-732)"}

    # ---- end to end through the C-ABI host entry point (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        hin = [d["x_host"].pin_memory() for d in layers]
        hout = [torch.empty(d["conv"].out_shape(local_n)).pin_memory() for d in layers]
        # the four layers are independent: each runs its H2D / pad + conv / D2H pipeline on
        # its own stream (forked from and joined back into the timed stream), so one layer's
        # output copy overlaps the next layer's input copy on the two copy engines (every
        # plan's workspace is used by one stream only: skc.h thread-safety rule)
        side = [torch.cuda.Stream(dev) for _ in layers]

        def estep():
            fork = torch.cuda.Event()
            fork.record(stream)
            for s_, d, hi, ho in zip(side, layers, hin, hout):
                s_.wait_event(fork)
                skc.skc_forward_host(d["conv"].plan, hi, ho, local_n, d["x"], d["xp"], d["out"],
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
            t_e2e = skd.max_over_ranks(t_e2e, cdev)
        e2e_ok = None
        if not args.no_parity:
            # the host outputs of the last e2e step: bitwise equal to the device path's
            e2e_ok = all(bool(torch.equal(ho.view(torch.int32), d["out"].cpu().view(torch.int32)))
                         for ho, d in zip(hout, layers))
            if world > 1:
                e2e_ok = skd.max_over_ranks(0.0 if e2e_ok else 1.0, cdev) == 0.0
        e2e = {"value": step_nnz_flops / (t_e2e * 1e-3) / 1e9, "unit": "GFLOP/s",
               "ms_per_step": t_e2e,
               "h2d_bytes_per_step": int(sum(h.numel() * 4 for h in hin)),
               "d2h_bytes_per_step": int(sum(h.numel() * 4 for h in hout)),
               "outputs_bitwise_equal_device_path": e2e_ok}

    if rank != 0:
        return
    clocks = clk.summary()
    # ---- roofline of the dominant kernel (the conv kernel of the layer with most time)
    conv_ms = per_kernel[1::2]
    pad_ms = per_kernel[0::2]
    dom = int(np.argmax(conv_ms))
    dl = layers[dom]
    achieved = nnz_flops(dl["L"], dl["nnz"], local_n) / (conv_ms[dom] * 1e-3) / 1e12
    f_max = (clocks["sm_max_mhz"] or 1965.0) * 1e6
    peak_fp32 = N_SM * FP32_LANES * 2 * f_max / 1e12
    peak_smem = N_SM * SMEM_WORDS_PER_CLK * 2 * f_max / 1e12
    traffic = load_traffic()
    tr = None
    if traffic and traffic.get("kernel") == args.kernel and cfg.cfg_id in traffic.get("configs", []):
        tr = traffic.get("dram_bytes_per_launch", {}).get(dl["L"].name)
    peak_meas = peaks["ffma2_tflops"] if peaks else None
    # the binding roof of each layer's kernel, from its committed ncu capture (config 2, AUTO):
    # roof cycles = max(FFMA2 / 2, LDS wavefronts + TMA bytes / 128) per SM, rescaled from the
    # capture's SM clock to this run's
    roofs = load_layer_roofs() if (cfg.cfg_id in (2, 5) and args.kernel == "auto") else {}
    per_layer = []
    for d, cm, pm in zip(layers, conv_ms, pad_ms):
        L = d["L"]
        ach = nnz_flops(L, d["nnz"], local_n) / (cm * 1e-3) / 1e12
        per_layer.append({
            "layer": L.name, "nnz": d["nnz"], "density": d["nnz"] / (L.K * (L.C // L.groups) * L.R * L.S),
            "conv_ms": float(cm), "pad_ms": float(pm),
            "conv_nnz_tflops": ach, "frac_fp32_nominal": ach / peak_fp32,
            "frac_fp32_measured": ach / peak_meas if peak_meas else None,
            "pad_gbs": local_n * 4 * (L.C * L.H * L.W + L.C * (L.H + 2 * L.pad) * (L.W + 2 * L.pad)) / (pm * 1e-3) / 1e9,
            "dram_bytes_per_launch_ncu": (traffic or {}).get("dram_bytes_per_launch", {}).get(L.name)
            if (traffic and traffic.get("kernel") == args.kernel and cfg.cfg_id in traffic.get("configs", [])) else None,
            "binding_roof": (lambda r: None if r is None else {
                "resource": r["binding"],
                "roof_tflops": r["roof_tflops"] * (f_max / 1e9) / r["sm_clock_ghz"],
                "frac": ach / (r["roof_tflops"] * (f_max / 1e9) / r["sm_clock_ghz"]),
                "source": "profiles/r02_layer_roofs.json (" + r["source"] + ")"})(roofs.get(L.name)),
            "kernel_cfg": {k: d["conv"].plan.info()[k] for k in (
                "kernel", "band_rows", "chunk_channels", "stages", "warps", "channels_per_warp",
                "pixels_per_lane", "smem_bytes", "tile_h", "tile_w", "images_per_cta",
                "jit_blocks", "jit_split", "jit_sched", "jit_np", "jit_deal", "code_bytes", "jit_compile_s",
                "jit_cache_hit")},
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
        if not args.no_cpu_single:
            # the same oracle single-threaded on one image of each layer (BASELINE.md plan)
            r = subprocess.run([sys.executable, "-c",
                                "import bench, json; print(json.dumps(bench.oracle_one_image(%d)))" % cfg.cfg_id],
                               cwd=ROOT, env=dict(os.environ, OMP_NUM_THREADS="1"),
                               capture_output=True, text=True, timeout=600)
            try:
                one = json.loads(r.stdout.strip().splitlines()[-1])
                cpu["single_thread"] = {"value": one["nnz_flops"] / one["seconds"] / 1e9, "unit": "GFLOP/s",
                                        "cores": 1, "seconds_per_image_all_layers": one["seconds"],
                                        "sample": "1 image of each layer, OMP_NUM_THREADS=1"}
            except (ValueError, IndexError, KeyError):
                cpu["single_thread"] = {"error": r.stderr[-300:]}
    par = f"dp{world} (batch-sharded, no collective)"
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} (BASELINE.json configs[{cfg.cfg_id - 1}])",
                   "global_batch": n_global, "per_gpu_batch": local_n,
                   "layers": [l.name for l in cfg.layers], "parallelism": par,
                   "l2": "flushed between timed steps (256 MiB write)", "kernel": args.kernel,
                   "step": "per layer: skc_pad_input + skc_sparse_conv_forward"
                           + (", the step's 8 launches replayed as one CUDA graph" if graph is not None else "")
                           + ("; pads of layers 2..L on a low-priority side stream overlapping the previous conv"
                              + (f" (layer order {''.join(map(str, order))})" if order != list(range(len(layers))) else "")
                              if graph is not None and args.pad_overlap and len(layers) > 1 else "")},
        "dense_equiv_gflops": step_dense_flops / (t_step * 1e-3) / 1e9,
        "per_gpu_gflops": local_nnz_flops / (t_local * 1e-3) / 1e9,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                     "frac": achieved / peak_fp32, "traffic": tr,
                     "kernel": f"skc_sparse_conv_forward ({dl['L'].name})",
                     "peak_basis": f"nominal: 148 SM x 128 FP32 lanes x 2 x {f_max/1e6:.0f} MHz (CUDA-core FFMA)",
                     "peak_measured": peak_meas,
                     "frac_measured": achieved / peak_meas if peak_meas else None,
                     "peak_measured_basis": "FFMA2 micro-benchmark in this session (skc_bench_ffma2)",
                     "smem_roof_1word_per_mac": peak_smem, "frac_smem_roof": achieved / peak_smem,
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write)"},
        "peaks_measured": peaks,
        "parity": parity,
        "per_layer": per_layer,
        "dense": dense,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks,
        # per layer: the pad pass + the conv kernel (+ the dry-run prefetch kernel of np plans)
        "gpu_launches": sum(2 + dry_kernel(d["conv"].plan.info()) for d in layers) * args.steps,
        "plan_build_s": t_build,
    }
    print(json.dumps(line), flush=True)


def dry_kernel(info: dict) -> int:
    """1 if a forward of this plan also launches the np dry-run prefetch kernel."""
    sched = int(info.get("jit_sched", -1))
    return int(bool(info.get("jit_np")) and not (sched >= 0 and sched & 4))


def oracle_one_image(cfg_id: int) -> dict:
    """The oracle on ONE image of every layer of a config (run with OMP_NUM_THREADS=1 for the
    single-threaded CPU baseline)."""
    import oracle
    cfg = wl.CONFIGS[cfg_id]
    nf = 0.0
    t = 0.0
    for li, L in enumerate(cfg.layers):
        w = wl.gen_weights(cfg_id, li, L)
        x = wl.gen_input(cfg_id, li, L, 0, 1)
        t0 = time.perf_counter()
        oracle.conv2d_fp64(x, w, L.stride, L.pad, L.groups, want_bound=False)
        t += time.perf_counter() - t0
        nf += nnz_flops(L, np.count_nonzero(w), 1)
    return {"seconds": t, "nnz_flops": nf}


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    cfg = wl.CONFIGS[args.config]
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            if args.backend == "nccl":
                torch.cuda.set_device(local_rank)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            else:
                dist.init_process_group("gloo")
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
