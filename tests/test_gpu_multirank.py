"""Multi-rank training parity on ONE GPU (test T3 "P-invariant
tree").  World ranks run as separate processes sharing cuda:0, each recording
its contiguous shard; the library's collectives (value-table all-gather,
per-level histogram and error-flag sums) go through the host-staged hooks of
adapt_init_host_comm over gloo — NCCL refuses two ranks on one device, and the
collective arithmetic is the same integer sum either way.  Every rank must
return the oracle's tree for the WHOLE table, labels / bins of its own shard,
and the oracle's selections for its shard; errors raised by one rank's data
must fail every rank with the same code."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, job, q):
    import torch
    import torch.distributed as dist

    import paper_2303_08873_b200 as ad
    from paper_2303_08873_b200 import dist as adist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if job.get("comm"):  # per-level histogram exchange (engine.cpp hist_comm_rs)
        os.environ["ADAPT_HIST_COMM"] = job["comm"]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        adist.init_host_comm(0, rank, world)
        if "regions" in job:  # adapt_train_many over rank shards of several regions (fused path)
            s = torch.cuda.current_stream()
            hs, keep = [], []
            for r, (X, T) in enumerate(job["regions"]):
                lo, hi = adist.shard_bounds(len(X), rank, world)
                h = ad.adapt_region_create(f"mr_region{r}", X.shape[1], T.shape[1], f"dtree,depth={job['D']}", 0)
                dX = torch.from_numpy(np.ascontiguousarray(X[lo:hi])).cuda()
                dT = torch.from_numpy(np.ascontiguousarray(T[lo:hi])).cuda()
                keep.append((dX, dT))
                ad.adapt_record_table(h, dX, dT, hi - lo, True, s)
                hs.append(h)
            ad.adapt_train_many(hs, s)
            q.put((rank, {"trees": [ad.adapt_get_tree(h) for h in hs]}))
            return
        X, T, D = job["X"], job["T"], job["D"]
        lo, hi = adist.shard_bounds(len(X), rank, world)
        Xs, Ts = np.ascontiguousarray(X[lo:hi]), np.ascontiguousarray(T[lo:hi])
        n, F = Xs.shape
        h = ad.adapt_region_create("mr", F, T.shape[1], job.get("model", f"dtree,depth={D}"), 0)
        s = torch.cuda.current_stream()
        dX = torch.from_numpy(Xs).cuda()
        if job.get("host"):
            ad.adapt_record_table(h, Xs, Ts, n, False, s)
        else:
            ad.adapt_record_table(h, dX, torch.from_numpy(Ts).cuda(), n, True, s)
        out = {"lo": lo, "hi": hi}
        try:
            ad.adapt_train(h, s)
        except ad.AdaptError as e:
            out["error"] = e.code
            q.put((rank, out))
            return
        out["tree"] = ad.adapt_get_tree(h)
        out["forest"] = [ad.adapt_get_forest_tree(h, t) for t in range(ad.adapt_forest_size(h))]
        out["labels"] = ad.adapt_get_labels(h, n)
        out["bins"] = ad.adapt_get_bins(h, n, F)
        sel = torch.empty(n, dtype=torch.int32, device="cuda")
        ad.adapt_select_batch(h, dX, n, sel, s)
        torch.cuda.synchronize()
        out["select"] = sel.cpu().numpy()
        if "kfold" in job:  # the K-fold harness is collective too (R22: global row ids)
            K, m, S, seed = job["kfold"]
            ad.adapt_record_table(h, dX, torch.from_numpy(Ts).cuda(), n, True, s)
            out["kfold"] = ad.adapt_kfold(h, K, m, S, seed, s)
            out["kfold_trees"] = [ad.adapt_get_kfold_tree(h, i) for i in range(S * K)]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _check(res, X, T, D):
    y = oracle.labels(T)
    ref = oracle.train(X, y, T.shape[1], D)
    bins = oracle.bins(X)
    for r, o in sorted(res.items()):
        lo, hi = o["lo"], o["hi"]
        assert "error" not in o, f"rank {r} failed: {o.get('error')}"
        got = o["tree"]
        assert len(got) == len(ref), f"rank {r}: {len(got)} nodes vs oracle {len(ref)}"
        for k in ("feature", "left", "right", "label", "depth", "n"):
            assert np.array_equal(got[k], ref[k]), f"rank {r}: {k} differs"
        assert got["threshold"].tobytes() == ref["threshold"].tobytes()
        np.testing.assert_allclose(got["gini"], ref["gini"], rtol=1e-12, atol=0)
        assert np.array_equal(o["labels"], y[lo:hi]), f"rank {r}: labels"
        assert np.array_equal(o["bins"], bins[lo:hi]), f"rank {r}: bins (global value table)"
        assert np.array_equal(o["select"], oracle.select(ref, X[lo:hi])), f"rank {r}: select"


@pytest.mark.parametrize("world", [2, 3])
def test_p_invariant_tree_c3(world):
    X, T = synth.generate("C3", 0, 200_003)
    _check(_run(world, {"X": X, "T": T, "D": 12, "comm": "allreduce"}), X, T, 12)


def test_p_invariant_tree_c4_slice_host_records():
    X, T = synth.generate("C4", 0, 60_001)
    _check(_run(2, {"X": X, "T": T, "D": 12, "host": True}), X, T, 12)


def test_p_invariant_forest():
    # bootstrap draws run over the GLOBAL row index (R19): every rank counts
    # the draws landing in its shard, so the forest is the single-GPU one
    X, T = synth.generate("C3", 0, 30_001)
    res = _run(2, {"X": X, "T": T, "D": 6, "model": "rfc,3,6,seed=4"})
    y = oracle.labels(T)
    ref = oracle.train_forest(X, y, T.shape[1], 6, 3, 4)
    expect = oracle.select_forest(ref, X)
    for r, o in sorted(res.items()):
        assert "error" not in o
        assert len(o["forest"]) == 3
        for t in range(3):
            assert o["forest"][t].tobytes() == ref[t].tobytes(), f"rank {r} tree {t}"
        assert np.array_equal(o["select"], expect[o["lo"]:o["hi"]])


def test_empty_shard_rank():
    # 1 row over 2 ranks: rank 0 records an empty shard, the tree is one leaf
    X, T = synth.generate("C1", 0, 1)
    _check(_run(2, {"X": X, "T": T, "D": 4}), X, T, 4)


def test_errors_fail_every_rank():
    X, T = synth.generate("C3", 0, 4000)
    X = X.copy()
    X[3500, 2] = np.nan  # in rank 1's shard only
    res = _run(2, {"X": X, "T": T, "D": 4})
    assert [res[r].get("error") for r in range(2)] == [-6, -6]
    # each shard has <= 256 distinct values of feature 0, the union has 300
    X, T = synth.generate("C3", 0, 600)
    X = X.copy()
    X[:300, 0] = np.arange(300, dtype=np.float32) % 200          # rank 0: 0..199
    X[300:, 0] = 100 + np.arange(300, dtype=np.float32) % 200    # rank 1: 100..299
    res = _run(2, {"X": X, "T": T, "D": 4})
    assert [res[r].get("error") for r in range(2)] == [-7, -7]


def test_p_invariant_kfold():
    # every rank returns the single-GPU K-fold results: the models' trees are the
    # oracle's CART on the fold's rows of the WHOLE table, counts summed over ranks
    X, T = synth.generate("C3", 0, 30_001)
    K, m, S, seed, D = 4, 2, 2, 9, 6
    res = _run(2, {"X": X, "T": T, "D": D, "kfold": (K, m, S, seed)})
    ref, trees = oracle.kfold(X, T, D, K, m, S, seed)
    for r, o in sorted(res.items()):
        assert "error" not in o
        for i, (got, want) in enumerate(zip(o["kfold"], ref)):
            for k in ("n_train", "n_test", "n_correct", "n_nodes"):
                assert got[k] == want[k], (r, i, k)
            np.testing.assert_allclose(got["t_selected"], want["t_selected"], rtol=len(X) * 2.0**-52)
            np.testing.assert_allclose(got["t_best"], want["t_best"], rtol=len(X) * 2.0**-52)
            assert o["kfold_trees"][i].tobytes() == trees[i].tobytes(), (r, i)


def test_p_invariant_quantile_bins():
    # R23 with 2 ranks: each rank's sorted distinct keys are all-gathered and
    # merged, so the quantiser (and the tree) is the single-table one
    rng = np.random.default_rng(3)
    n = 40001
    X = np.stack([rng.normal(size=n), rng.integers(0, 7, n), rng.uniform(0, 1e4, n)], 1).astype(np.float32)
    X[: n // 2, 2] += 1e4  # rank 0 and rank 1 see disjoint value ranges
    T = rng.random((n, 4)).astype(np.float32)
    T[:, 1] -= (X[:, 0] > 0.3) * 0.4
    T[:, 2] -= (X[:, 2] < 5e3) * 0.6
    res = _run(2, {"X": X, "T": T, "D": 7, "model": "dtree,depth=7,bins=quantile"})
    y = oracle.labels(T)
    ref = oracle.train_quantile(X, y, 4, 7)
    for r, o in sorted(res.items()):
        assert "error" not in o
        assert o["tree"].tobytes() == ref.tobytes(), f"rank {r}"
        assert np.array_equal(o["select"], oracle.select(ref, X[o["lo"]:o["hi"]]))


def test_p_invariant_train_many_fused():
    # three regions' trees in one multi-root frontier over the union of the
    # ranks' shards: every rank gets every region's single-table tree
    cfg = synth.CONFIGS["C2"]
    X, T = synth.generate(cfg, 0, 30_000)
    regions = []
    for r in range(3):
        rows = np.arange(r, len(X), 3)
        regions.append((np.ascontiguousarray(X[rows]), np.ascontiguousarray(T[rows])))
    res = _run(2, {"regions": regions, "D": 6})
    for r, o in sorted(res.items()):
        for (Xr, Tr), got in zip(regions, o["trees"]):
            ref = oracle.train(Xr, oracle.labels(Tr), Tr.shape[1], 6)
            assert got.tobytes() == ref.tobytes(), f"rank {r}"


# ---- reduce-scatter of the level's histograms by node
# ownership, owner split search, all-gather of the winner records
# (ADAPT_HIST_COMM=rs, the default with more than one rank; the tests above
# without "comm" run it too, the ones below force each mode): every rank must
# still get the single-table tree ----
@pytest.mark.parametrize("world", [2, 3])
def test_p_invariant_tree_reduce_scatter(world):
    X, T = synth.generate("C3", 0, 200_003)
    _check(_run(world, {"X": X, "T": T, "D": 12, "comm": "rs"}), X, T, 12)


def test_reduce_scatter_c4_deep_and_empty_shard():
    X, T = synth.generate("C4", 0, 60_001)
    _check(_run(3, {"X": X, "T": T, "D": 16, "comm": "rs"}), X, T, 16)
    X, T = synth.generate("C1", 0, 1)
    _check(_run(2, {"X": X, "T": T, "D": 4, "comm": "rs"}), X, T, 4)


def test_allreduce_forest_kfold_many():
    # the same workloads through the all-reduce mode (the default above is rs)
    X, T = synth.generate("C3", 0, 30_001)
    res = _run(2, {"X": X, "T": T, "D": 6, "model": "rfc,3,6,seed=4", "comm": "allreduce"})
    ref = oracle.train_forest(X, oracle.labels(T), T.shape[1], 6, 3, 4)
    for r, o in sorted(res.items()):
        assert "error" not in o
        for t in range(3):
            assert o["forest"][t].tobytes() == ref[t].tobytes(), f"rank {r} tree {t}"
    K, m, S, seed, D = 4, 2, 2, 9, 6
    res = _run(2, {"X": X, "T": T, "D": D, "kfold": (K, m, S, seed), "comm": "allreduce"})
    _, trees = oracle.kfold(X, T, D, K, m, S, seed)
    for r, o in sorted(res.items()):
        assert "error" not in o
        for i, want in enumerate(trees):
            assert o["kfold_trees"][i].tobytes() == want.tobytes(), (r, i)
    cfg = synth.CONFIGS["C2"]
    X, T = synth.generate(cfg, 0, 30_000)
    regions = [(np.ascontiguousarray(X[r::3]), np.ascontiguousarray(T[r::3])) for r in range(3)]
    res = _run(2, {"regions": regions, "D": 6, "comm": "allreduce"})
    for r, o in sorted(res.items()):
        for (Xr, Tr), got in zip(regions, o["trees"]):
            assert got.tobytes() == oracle.train(Xr, oracle.labels(Tr), Tr.shape[1], 6).tobytes()
