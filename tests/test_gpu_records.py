"""GPU record path (§8(c) step 0): long-format records are
aggregated on the device into wide rows, bit-identical to the oracle's
aggregation (oracle_aggregate: sort-based grouping, R1, R3, R4,
S:58), then trained on exactly like a wide table."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2303_08873_b200 as ad  # noqa: E402

DEV = torch.device("cuda:0")
_uid = [0]


@pytest.fixture(scope="module", autouse=True)
def _init():
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    yield


def _region(F, V, D=6):
    _uid[0] += 1
    return ad.adapt_region_create(f"rec{_uid[0]}", F, V, f"dtree,depth={D}", 0)


def _records(seed, m, F, V, grid=5, neg_zero=True):
    rng = np.random.default_rng(seed)
    vals = np.array([0.0, 1.5, -2.25, 1e-3, 3e6, 7.0, 11.0, 0.5][:grid], np.float32)
    X = vals[rng.integers(0, len(vals), size=(m, F))].astype(np.float32)
    if neg_zero:  # -0.0 and +0.0 are the same value (R4)
        z = (X == 0) & (rng.random((m, F)) < 0.5)
        X[z] = np.float32(-0.0)
    var = rng.integers(0, V, size=m).astype(np.int32)
    ns = rng.integers(1, 10**12, size=m, dtype=np.uint64)
    return X, var, ns


def _check_tree(h, wf, wt, V, D):
    y = oracle.labels(wt)
    ref = oracle.train(wf, y, V, D)
    got = ad.adapt_get_tree(h)
    assert len(got) == len(ref)
    for k in ("feature", "left", "right", "label", "depth", "n"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["threshold"].tobytes() == ref["threshold"].tobytes()


@pytest.mark.parametrize("seed,m,F,V", [(1, 1, 1, 1), (2, 5000, 3, 5), (3, 20000, 2, 9),
                                        (4, 3000, 7, 48), (5, 777, 1, 2)])
def test_batch_records_match_oracle(seed, m, F, V):
    X, var, ns = _records(seed, m, F, V)
    h = _region(F, V)
    half = m // 2  # two batches: host pointers then device tensors
    ad.adapt_record_batch(h, X[:half], var[:half], ns[:half], half, False)
    ad.adapt_record_batch(h, torch.from_numpy(X[half:]).to(DEV), torch.from_numpy(var[half:]).to(DEV),
                          torch.from_numpy(ns[half:].view(np.int64)).to(DEV), m - half, True)
    assert ad.adapt_distinct_pairs(h) == oracle.distinct_pairs(X, var)
    ad.adapt_train(h)
    wf, wt = ad.adapt_get_wide_table(h)
    of, ot = oracle.aggregate(X, var, ns, V)
    assert wf.tobytes() == of.tobytes(), "wide features differ"
    assert wt.tobytes() == ot.tobytes(), "wide times differ"
    _check_tree(h, of, ot, V, 6)


def test_batch_then_single_records_order():
    # the device store first, then the adapt_record() ones in call order
    X, var, ns = _records(7, 3000, 3, 4)
    Y, vy, ny = _records(8, 500, 3, 4)
    h = _region(3, 4)
    ad.adapt_record_batch(h, X, var, ns)
    for i in range(len(Y)):
        ad.adapt_record(h, Y[i], int(vy[i]), int(ny[i]))
    ad.adapt_train(h)
    wf, wt = ad.adapt_get_wide_table(h)
    of, ot = oracle.aggregate(np.concatenate([X, Y]), np.concatenate([var, vy]),
                              np.concatenate([ns, ny]), 4)
    assert wf.tobytes() == of.tobytes() and wt.tobytes() == ot.tobytes()
    # training again re-aggregates the same records: same table, same tree
    ad.adapt_train(h)
    wf2, wt2 = ad.adapt_get_wide_table(h)
    assert wf2.tobytes() == of.tobytes() and wt2.tobytes() == ot.tobytes()


def test_single_records_go_through_the_gpu_aggregation():
    X, var, ns = _records(9, 400, 2, 3)
    h = _region(2, 3)
    for i in range(len(X)):
        ad.adapt_record(h, X[i], int(var[i]), int(ns[i]))
    ad.adapt_train(h)
    wf, wt = ad.adapt_get_wide_table(h)
    of, ot = oracle.aggregate(X, var, ns, 3)
    assert wf.tobytes() == of.tobytes() and wt.tobytes() == ot.tobytes()


def test_large_batch_properties():
    # 2e6 records over ~4e4 distinct vectors: the oracle's O(R*G) grouping is
    # too slow, so check what defines the result: distinct rows in order of
    # first appearance, and sampled rows against the oracle on their records
    rng = np.random.default_rng(11)
    m, F, V = 2_000_000, 4, 6
    X = rng.integers(0, 14, size=(m, F)).astype(np.float32)
    var = rng.integers(0, V, size=m).astype(np.int32)
    ns = rng.integers(1, 10**9, size=m, dtype=np.uint64)
    h = _region(F, V, 8)
    ad.adapt_record_batch(h, torch.from_numpy(X).to(DEV), torch.from_numpy(var).to(DEV),
                          torch.from_numpy(ns.view(np.int64)).to(DEV), m, True)
    ad.adapt_train(h)
    wf, wt = ad.adapt_get_wide_table(h)
    _, first, inv = np.unique(X, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first)
    assert np.array_equal(wf, X[first[order]])
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    row_of = rank[inv.reshape(-1)]
    for g in rng.choice(len(wf), size=12, replace=False):
        sel = row_of == g
        of, ot = oracle.aggregate(X[sel], var[sel], ns[sel], V)
        assert of.shape[0] == 1 and wt[g].tobytes() == ot[0].tobytes()


def test_bad_variant_and_errors():
    h = _region(2, 3)
    X = np.zeros((4, 2), np.float32)
    ad.adapt_record_batch(h, X, np.array([0, 1, 3, 2], np.int32), np.ones(4, np.uint64))
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h)
    assert e.value.code == ad.ADAPT_E_BAD_VALUE
    h2 = _region(2, 3)
    Xn = np.array([[1.0, np.nan]], np.float32)
    ad.adapt_record_batch(h2, Xn, np.array([0], np.int32), np.ones(1, np.uint64))
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h2)
    assert e.value.code == ad.ADAPT_E_BAD_VALUE
    h3 = _region(2, 3)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_get_wide_table(h3)
    assert e.value.code == ad.ADAPT_E_NOT_TRAINED
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h3)
    assert e.value.code == ad.ADAPT_E_INSUFFICIENT_DATA
