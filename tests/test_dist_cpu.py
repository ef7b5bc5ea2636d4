"""Multi-rank host logic on CPU: world_size 2 (and 3) over gloo.

The training collectives themselves run inside libadapt.so; what is checked
here is the Python plumbing around them — contiguous shards, the ncclUniqueId
broadcast, the gloo implementations of the host-staged collective hooks
(adapt_init_host_comm) and max-over-ranks timing — plus the C entry point's
argument checks.  The same hooks drive the 2-rank training parity test in
tests/test_gpu_multirank.py on a GPU box."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2303_08873_b200 as ad
from paper_2303_08873_b200 import dist as adist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        ag, ar = adist.gloo_hooks()
        # all_gather: rank order, ragged content irrelevant (same byte count)
        send = np.arange(5, dtype=np.uint8) + 10 * rank
        out["ag"] = ag(send)
        # all_reduce_u64: sums incl. values past 2^63 and wrap-around mod 2^64
        buf = np.array([1, 2**40 + rank, 2**63 + rank, 2**64 - 1], dtype=np.uint64)
        out["ar"] = ar(buf)
        out["max"] = adist.max_over_ranks(float(rank) + 0.5)
        out["uid"] = adist.share_unique_id(rank)
        out["shard"] = adist.shard_bounds(1001, rank, world)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_collectives_and_shards(world):
    res = _run(world)
    ag_expect = np.concatenate([np.arange(5, dtype=np.uint8) + 10 * r for r in range(world)])
    M = 2**64
    ar_expect = np.array([world, (world * 2**40 + sum(range(world))) % M,
                          (world * 2**63 + sum(range(world))) % M, (world * (M - 1)) % M],
                         dtype=np.uint64)
    for r in range(world):
        o = res[r]
        assert np.array_equal(o["ag"], ag_expect)
        assert o["ar"].dtype == np.uint64 and np.array_equal(o["ar"], ar_expect)
        assert o["max"] == world - 0.5
        assert len(o["uid"]) == 128 and o["uid"] == res[0]["uid"]
    shards = [res[r]["shard"] for r in range(world)]
    assert shards[0][0] == 0 and shards[-1][1] == 1001
    assert all(shards[i][1] == shards[i + 1][0] for i in range(world - 1))


def test_shard_bounds_tile():
    for n in (0, 1, 7, 100, 10**8 + 3):
        for world in (1, 2, 3, 8):
            b = [adist.shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
    with pytest.raises(ValueError):
        adist.shard_bounds(10, 2, 2)


def test_host_comm_entry_checks():
    lib = ad.lib()
    # null hooks -> INVALID_ARG before any device query
    assert lib.adapt_init_host_comm(0, 0, 2, None) == ad.ADAPT_E_INVALID_ARG
    assert lib.adapt_init_host_comm(0, 2, 2, None) == ad.ADAPT_E_INVALID_ARG
    # valid hooks without a GPU fail loudly (no CPU fallback)
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_init_host_comm(0, 0, 2, lambda s: s, lambda b: b)
    assert e.value.code == ad.ADAPT_E_CUDA
