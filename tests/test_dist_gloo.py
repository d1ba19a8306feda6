"""Multi-process (world_size 2, gloo, CPU) tests of the batch-sharded multi-GPU host logic:
shards partition the batch, per-64-image-block seeding makes a shard's images identical to
the same images of the whole batch, plans agree across ranks, timing takes the max over
ranks, and gathering shards reproduces the whole batch bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as wl
from paper_1608_01409_b200 import dist as skd


def test_shard_range_partitions():
    for n in (0, 1, 7, 256, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            ranges = [skd.shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        skd.shard_range(4, 2, 2)


def test_shard_inputs_match_whole_batch():
    L = wl.CONFIGS[5].layers[1]
    whole = wl.gen_input(5, 1, L, 0, 150)
    for world in (2, 4):
        for r in range(world):
            lo, hi = skd.shard_range(150, world, r)
            np.testing.assert_array_equal(wl.gen_input(5, 1, L, lo, hi), whole[lo:hi])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1608_01409_b200 import skc
        L = wl.CONFIGS[2].layers[3]
        w = wl.gen_weights(2, 3, L)
        plan = skc.skc_pack_csr(w, L.H, L.W, L.stride, L.pad, L.groups)
        same = skd.check_same_plan(plan)
        # a rank whose weights differ must be detected
        w2 = w.copy()
        if rank == 1:
            w2[0, 0, 0, 0] = 1.0
        plan2 = skc.skc_pack_csr(w2, L.H, L.W, L.stride, L.pad, L.groups)
        differ = not skd.check_same_plan(plan2)
        t = skd.max_over_ranks(1.5 + rank)
        lo, hi = skd.shard_range(9, world, rank)
        local = torch.arange(lo * 4, hi * 4, dtype=torch.float32).reshape(hi - lo, 2, 2)
        full = skd.gather_images(local, 9)
        # bench.py's check of a sharded run, on real conv outputs: each rank's shard of a
        # 10-image batch (computed here by the oracle, cast to fp32, as a stand-in for the
        # GPU's), gathered over the process group, must equal one "device's" whole batch bit
        # for bit and pass the oracle on >= 3 images per shard; a corrupted element must fail
        import bench
        import oracle
        n_total = 10
        lo2, hi2 = skd.shard_range(n_total, world, rank)
        mine = oracle.conv2d_fp64(wl.gen_input(2, 3, L, lo2, hi2), w, L.stride, L.pad, L.groups,
                                  want_bound=False)[0].astype(np.float32)
        bad = mine.copy()
        if rank == 1:
            bad[0, 5, 3, 3] = np.nextafter(bad[0, 5, 3, 3], np.float32(np.inf))
        g_ok = skd.gather_images(torch.from_numpy(mine), n_total).numpy()
        g_bad = skd.gather_images(torch.from_numpy(bad), n_total).numpy()
        ver = None
        if rank == 0:
            whole = oracle.conv2d_fp64(wl.gen_input(2, 3, L, 0, n_total), w, L.stride, L.pad,
                                       L.groups, want_bound=False)[0].astype(np.float32)
            ok = bench.verify_gathered(g_ok, whole, 2, 3, L, w, n_total, world, per_shard=3)
            nok = bench.verify_gathered(g_bad, whole, 2, 3, L, w, n_total, world, per_shard=3)
            ver = (ok["bitwise_vs_1gpu"], ok["images"], ok["max_err_over_bound"], nok["bitwise_vs_1gpu"])
        q.put((rank, same, differ, t, full.numpy().tolist(), ver))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, differ, t, full, ver in res:
        assert same and differ
        assert t == 2.5
        np.testing.assert_array_equal(np.array(full), np.arange(36, dtype=np.float32).reshape(9, 2, 2))
        if rank == 0:
            bitwise_ok, images, err, bitwise_bad = ver
            assert bitwise_ok and images >= 6 and err <= 1e-4, ver
            assert bitwise_bad is False
