"""Multi-rank plumbing around libadapt.so: one process per GPU.

Host logic only; every collective of the training path runs inside the
library (NCCL over NVLink, or the caller's host-staged hooks):

* ``shard_bounds``      — rank r's contiguous row shard [r*N/P, (r+1)*N/P)
                          (§8(b) "multi-rank rules": adapt_record_table takes
                          the rank's contiguous shard).
* ``init_nccl``         — rank 0 draws the ncclUniqueId, torch.distributed
                          broadcasts its 128 bytes, every rank calls adapt_init.
* ``gloo_hooks``        — torch.distributed (gloo) implementations of the two
                          host-staged collectives of adapt_init_host_comm;
                          several ranks can then share ONE GPU (NCCL refuses
                          duplicate devices), which is how the tree's
                          P-invariance is tested on a 1-GPU box.
* ``max_over_ranks``    — device timings are reported as the max over ranks.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous shard of n rows; shards tile [0, n)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad n/rank/world")
    return rank * n // world, (rank + 1) * n // world


def gloo_hooks(group=None):
    """(all_gather, all_reduce_u64) over a torch.distributed process group.

    all_gather(send uint8[b]) -> uint8[world*b], rank order.
    all_reduce_u64(buf uint64[k]) -> uint64[k], the sum mod 2^64 (computed on
    the int64 view: two's-complement addition gives the same bits)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def all_gather(send: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(send, dtype=np.uint8))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        return torch.cat(parts).numpy()

    def all_reduce_u64(buf: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.uint64).view(np.int64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.numpy().view(np.uint64)

    return all_gather, all_reduce_u64


def share_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 draws a 128-byte ncclUniqueId; every rank returns the same bytes."""
    import torch.distributed as dist

    from . import _binding as b

    uid = [b.adapt_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    if not isinstance(uid[0], bytes) or len(uid[0]) != 128:
        raise RuntimeError("ncclUniqueId broadcast failed")
    return uid[0]


def init_nccl(device: int, rank: int, world: int, group=None) -> None:
    """adapt_init for world ranks; the ncclUniqueId travels by torch.distributed."""
    from . import _binding as b

    if world == 1:
        b.adapt_init(device, 0, 1)
        return
    b.adapt_init(device, rank, world, share_unique_id(rank, group))


def init_host_comm(device: int, rank: int, world: int, group=None) -> None:
    """adapt_init_host_comm with the gloo hooks of `group`."""
    from . import _binding as b

    ag, ar = gloo_hooks(group)
    b.adapt_init_host_comm(device, rank, world, ag, ar)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
