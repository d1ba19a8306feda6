"""Batch sharding across GPUs.

Images are independent units of direct sparse convolution (each output image depends on one
input image and the shared weights), so the path shards by contiguous image ranges with the
weights replicated and NO collective on the data path -- the paper's own parallelisation over
hardware threads by image ("batch sizes ... multiples of the number of
hardware threads").  torch.distributed is used only off the timed path: to check that every
rank packed the identical plan, to take the max over ranks of the timed region, and to gather
outputs for checking.  Works with the "nccl" backend (one process per GPU) and "gloo" (CPU
tests).
"""
from __future__ import annotations

import hashlib

import numpy as np


def shard_range(n_images: int, world: int, rank: int):
    """Contiguous images [lo, hi) of `rank`: sizes differ by at most one, ranks in order."""
    if world < 1 or not (0 <= rank < world) or n_images < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_images, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def plan_digest(plan) -> bytes:
    """SHA-256 of the canonical CSR (rowptr, colidx, value bits) and the channel order."""
    rowptr, colidx, values = plan.csr()
    h = hashlib.sha256()
    for a in (rowptr, colidx, values.view(np.uint32), plan.perm()):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.digest()


def _as_tensor(b: bytes, device):
    import torch
    return torch.tensor(list(b), dtype=torch.uint8, device=device)


def check_same_plan(plan, device=None) -> bool:
    """all_gather the plan digests; True iff every rank packed the same weights."""
    import torch
    import torch.distributed as dist
    mine = _as_tensor(plan_digest(plan), device or "cpu")
    allv = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(allv, mine)
    return all(bool(torch.equal(v, allv[0])) for v in allv)


def max_over_ranks(value: float, device=None) -> float:
    """The whole-job time of a timed region: the slowest rank's."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_images(local, n_total: int, device=None):
    """Concatenate every rank's [n_r, ...] output shard in rank order (off the timed path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)
