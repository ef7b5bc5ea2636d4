"""GPU parity of the lossy quantile bins (model "dtree,...,bins=quantile";
SURVEY §8(f) f4; DESIGN R23) against oracle.train_quantile: value tables (the
256 bin lower bounds), bins, tree (byte-identical, raw thresholds at the
quantiser's cut points) and selections on raw vectors; exact mode still
rejects > 256 values; 2 ranks merge the distinct sets (P-invariance)."""
import numpy as np
import pytest

import oracle
import synth

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


def _parity(X, T, D, on_device=True):
    n, F = X.shape
    V = T.shape[1]
    _uid[0] += 1
    h = ad.adapt_region_create(f"q{_uid[0]}", F, V, f"dtree,depth={D},bins=quantile", 0)
    s = torch.cuda.current_stream()
    if on_device:
        ad.adapt_record_table(h, torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV), n, True, s)
    else:
        ad.adapt_record_table(h, X, T, n, False, s)
    ad.adapt_train(h, s)
    y = oracle.labels(T)
    q = oracle.quantizer(X)
    Xq = oracle.quantize(X, q)
    for f in range(F):
        assert np.array_equal(ad.adapt_get_value_table(h, f), oracle.value_table(Xq, f)), f
    assert np.array_equal(ad.adapt_get_bins(h, n, F), oracle.bins(Xq))
    ref = oracle.train_quantile(X, y, V, D)
    got = ad.adapt_get_tree(h)
    assert got.tobytes() == ref.tobytes()
    out = torch.empty(n, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), n, out, s)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(ref, X))
    ad.adapt_region_destroy(h)
    return q


def test_continuous_features():
    rng = np.random.default_rng(1)
    n = 50000
    X = np.stack([rng.normal(size=n), rng.integers(0, 50, n), rng.exponential(size=n),
                  -rng.uniform(0, 1e6, n)], 1).astype(np.float32)
    X[::7, 0] = -0.0
    T = np.stack([X[:, 0] * 3 + X[:, 2], X[:, 1] * 0.1 + 1, 2 - X[:, 0], X[:, 3] * 1e-6 + 2], 1)
    T = (T + rng.random(T.shape)).astype(np.float32)
    q = _parity(X, T, 10)
    assert set(q) == {0, 2, 3}


@pytest.mark.parametrize("n", [257, 3001, 1_500_000])
def test_sizes_incl_sampled_discovery(n):
    # 1.5e6 rows > the sampled-discovery threshold: the sample may not see > 256
    # values, the bin pass then flags unseen values and the full discovery overflows
    rng = np.random.default_rng(n)
    X = np.stack([rng.integers(0, 1000, n), rng.integers(0, 9, n)], 1).astype(np.float32)
    T = rng.random((n, 5)).astype(np.float32)
    T[:, 0] -= (X[:, 0] > 500) * 0.3
    _parity(X, T, 6, on_device=n != 3001)


def test_exact_mode_still_rejects():
    rng = np.random.default_rng(2)
    X = rng.normal(size=(1000, 1)).astype(np.float32)
    T = rng.random((1000, 2)).astype(np.float32)
    h = ad.adapt_region_create("q_exact", 1, 2, "dtree,depth=3", 0)
    ad.adapt_record_table(h, X, T, 1000, False, None)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, None)
    assert e.value.code == ad.ADAPT_E_TOO_MANY_DISTINCT
    ad.adapt_region_destroy(h)


def _continuous_table(n, seed):
    rng = np.random.default_rng(seed)
    X = np.stack([rng.normal(size=n), rng.integers(0, 5, n), rng.uniform(0, 1e3, n)], 1).astype(np.float32)
    T = rng.random((n, 4)).astype(np.float32)
    T[:, 1] -= (X[:, 0] > 0.2) * 0.5
    T[:, 3] -= (X[:, 2] < 300) * 0.4
    return X, T


def test_kfold_with_quantile_bins():
    # the table is quantised once (its own quantiser); every fold's model is the
    # exact CART of its quantised rows with raw thresholds from that quantiser
    X, T = _continuous_table(6000, 4)
    h = ad.adapt_region_create("q_kfold", 3, 4, "dtree,depth=5,bins=quantile", 0)
    s = torch.cuda.current_stream()
    ad.adapt_record_table(h, torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV), len(X), True, s)
    got = ad.adapt_kfold(h, 4, 2, 2, 5, s)
    q = oracle.quantizer(X)
    y = oracle.labels(T)
    for i, r in enumerate(got):
        g = oracle.kfold_groups(5, int(r["shuffle"]), len(X), 4)
        tr = np.isin(g, [(int(r["fold"]) + j) % 4 for j in range(2)])
        ref = oracle.train_quantile(X[tr], y[tr], 4, 5, q=q)
        assert ad.adapt_get_kfold_tree(h, i).tobytes() == ref.tobytes(), i
        te = ~tr
        sel = oracle.select(ref, X[te])
        assert r["n_test"] == te.sum() and r["n_correct"] == int((sel == y[te]).sum())
    ad.adapt_region_destroy(h)


def test_forest_with_quantile_bins():
    X, T = _continuous_table(5000, 6)
    h = ad.adapt_region_create("q_rfc", 3, 4, "rfc,3,4,seed=2,bins=quantile", 0)
    s = torch.cuda.current_stream()
    ad.adapt_record_table(h, torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV), len(X), True, s)
    ad.adapt_train(h, s)
    q = oracle.quantizer(X)
    y = oracle.labels(T)
    for t in range(3):
        w = oracle.bootstrap(2, t, len(X)).astype(np.int64)
        ref = oracle.train_quantile(np.repeat(X, w, axis=0), np.repeat(y, w), 4, 4, q=q)
        assert ad.adapt_get_forest_tree(h, t).tobytes() == ref.tobytes(), t
    ad.adapt_region_destroy(h)
