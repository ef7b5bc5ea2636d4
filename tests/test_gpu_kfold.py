"""GPU parity of the K-fold harness (DESIGN R22)
against oracle.kfold: per model (shuffle, fold) the tree is byte-identical to
the oracle's CART on the fold's training rows, n_train / n_test / n_correct are
exact, and the time sums agree within the summation-order bound of R22
(|err| <= n u sum, u = 2^-53, all terms positive)."""
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


def _region(F, V, spec):
    _uid[0] += 1
    return ad.adapt_region_create(f"kf{_uid[0]}", F, V, spec, 0)


def _kfold_parity(X, T, D, K, m, S, seed, on_device=True):
    n, F = X.shape
    V = T.shape[1]
    h = _region(F, V, f"dtree,depth={D}")
    s = torch.cuda.current_stream()
    if on_device:
        ad.adapt_record_table(h, torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV), n, True, s)
    else:
        ad.adapt_record_table(h, X, T, n, False, s)
    got = ad.adapt_kfold(h, K, m, S, seed, s)
    ref, trees = oracle.kfold(X, T, D, K, m, S, seed)
    assert len(got) == len(ref) == S * K
    rtol = max(n, 1) * 2.0**-53
    for i, (g, r) in enumerate(zip(got, ref)):
        assert (g["shuffle"], g["fold"]) == (r["shuffle"], r["fold"])
        for k in ("n_train", "n_test", "n_correct", "n_nodes"):
            assert g[k] == r[k], (i, k, g[k], r[k])
        np.testing.assert_allclose(g["t_selected"], r["t_selected"], rtol=rtol)
        np.testing.assert_allclose(g["t_best"], r["t_best"], rtol=rtol)
        assert ad.adapt_get_kfold_tree(h, i).tobytes() == trees[i].tobytes(), f"model {i} tree"
    ad.adapt_region_destroy(h)
    return got


@pytest.mark.parametrize("m", [1, 2, 3])
def test_c1_adaptive_25_50_75(m):
    # the paper's protocol at C1's shape: K = 4, m = 1/2/3 groups, 10 shuffles
    cfg = synth.CONFIGS["C1"]
    X, T = synth.generate(cfg, 0, cfg.N)
    _kfold_parity(X, T, cfg.D, 4, m, 10, seed=1)


@pytest.mark.parametrize("m", [1, 3])
def test_c2_region(m):
    cfg = synth.CONFIGS["C2"]
    X, T = synth.generate(cfg, 0, cfg.N)
    r0 = synth.region_rows(cfg, 0)[:20_000]
    _kfold_parity(np.ascontiguousarray(X[r0]), np.ascontiguousarray(T[r0]), cfg.D, 4, m, 2, seed=3)


def test_random_tables_and_host_path():
    rng = np.random.default_rng(7)
    for t in range(6):
        n = int(rng.integers(3, 3000))
        F = int(rng.choice([1, 3, 8, 16]))
        V = int(rng.integers(2, 9))
        K = int(rng.integers(2, min(n, 9) + 1))
        m = int(rng.integers(1, K))
        X = rng.choice(np.arange(30, dtype=np.float32), size=(n, F)).astype(np.float32)
        T = rng.integers(1, 5, size=(n, V)).astype(np.float32)
        if t % 2:
            T[rng.random(T.shape) < 0.2] = np.inf  # unmeasured: never the label, may be selected
            T[np.all(np.isinf(T), axis=1), 0] = 1.0
        _kfold_parity(X, T, int(rng.integers(0, 7)), K, m, 2, seed=t, on_device=bool(t % 3))


def test_model_kept_and_errors():
    cfg = synth.CONFIGS["C1"]
    X, T = synth.generate(cfg, 0, cfg.N)
    dX, dT = torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV)
    s = torch.cuda.current_stream()
    h = _region(cfg.F, cfg.V, f"dtree,depth={cfg.D}")
    ad.adapt_record_table(h, dX, dT, cfg.N, True, s)
    ad.adapt_train(h, s)
    before = ad.adapt_get_tree(h)
    ad.adapt_record_table(h, dX, dT, cfg.N, True, s)
    ad.adapt_kfold(h, 4, 1, 2, 0, s)
    assert ad.adapt_get_tree(h).tobytes() == before.tobytes()
    out = torch.empty(cfg.N, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, dX, cfg.N, out, s)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(before, X))
    for K, m, S in ((1, 1, 1), (4, 0, 1), (4, 4, 1), (4, 1, 0), (65, 1, 1)):
        ad.adapt_record_table(h, dX, dT, cfg.N, True, s)
        with pytest.raises(ad.AdaptError) as e:
            ad.adapt_kfold(h, K, m, S, 0, s)
        assert e.value.code == ad.ADAPT_E_INVALID_ARG
    ad.adapt_record_table(h, dX[:3], dT[:3], 3, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_kfold(h, 4, 1, 1, 0, s)
    assert e.value.code == ad.ADAPT_E_INSUFFICIENT_DATA
    f = _region(cfg.F, cfg.V, "rfc,2,2")
    ad.adapt_record_table(f, dX, dT, cfg.N, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_kfold(f, 4, 1, 1, 0, s)
    assert e.value.code == ad.ADAPT_E_USAGE
    ad.adapt_region_destroy(h)
    ad.adapt_region_destroy(f)


def test_kfold_on_recorded_samples():
    # the Apollo flow: long-format records -> the GPU aggregation to wide
    # rows (first appearance order, mean times) -> the K-fold harness over them
    rng = np.random.default_rng(12)
    R, F, V = 20000, 2, 4
    grid = rng.choice(np.arange(60, dtype=np.float32), size=(700, F)).astype(np.float32)
    feat = grid[rng.integers(0, len(grid), R)]
    var = rng.integers(0, V, R).astype(np.int32)
    ns = (1000 + 37 * feat[:, 0] * (var + 1) + rng.integers(0, 500, R)).astype(np.uint64)
    h = _region(F, V, "dtree,depth=5")
    ad.adapt_record_batch(h, torch.from_numpy(feat).to(DEV), torch.from_numpy(var).to(DEV),
                          torch.from_numpy(ns.astype(np.int64)).to(DEV), R, True)
    got = ad.adapt_kfold(h, 4, 3, 2, 8)
    Xw, Tw = oracle.aggregate(feat, var, ns, V)
    ref, trees = oracle.kfold(Xw, Tw, 5, 4, 3, 2, 8)
    for i, (g, r) in enumerate(zip(got, ref)):
        for k in ("n_train", "n_test", "n_correct", "n_nodes"):
            assert g[k] == r[k], (i, k)
        assert ad.adapt_get_kfold_tree(h, i).tobytes() == trees[i].tobytes()
    ad.adapt_region_destroy(h)
