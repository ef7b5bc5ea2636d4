"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element, on seeded inputs.  Bit-exact for labels, value tables,
bins, tree topology / features / thresholds / labels / counts and selections;
Gini within 1e-12 relative (north_star), which the engine in fact meets exactly."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2303_08873_b200 as ad  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module", autouse=True)
def _init():
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    yield


_uid = [0]


def _region(F, V, D):
    _uid[0] += 1
    return ad.adapt_region_create(f"t{_uid[0]}", F, V, f"dtree,depth={D}", 0)


def _train(X, T, D, on_device=True):
    n, F = X.shape
    V = T.shape[1]
    h = _region(F, V, D)
    s = torch.cuda.current_stream()
    if on_device:
        dX, dT = torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV)
        ad.adapt_record_table(h, dX, dT, n, True, s)
    else:
        ad.adapt_record_table(h, X, T, n, False, s)
    ad.adapt_train(h, s)
    return h


def assert_tree_equal(got, ref):
    assert len(got) == len(ref), f"{len(got)} nodes vs oracle {len(ref)}"
    for k in ("feature", "left", "right", "label", "depth", "n"):
        bad = np.nonzero(got[k] != ref[k])[0]
        assert bad.size == 0, f"{k} differs at nodes {bad[:10]}"
    assert got["threshold"].tobytes() == ref["threshold"].tobytes(), "thresholds differ"
    np.testing.assert_allclose(got["gini"], ref["gini"], rtol=1e-12, atol=0)


def full_parity(X, T, D, select_X=None, on_device=True):
    n, F = X.shape
    V = T.shape[1]
    h = _train(X, T, D, on_device)
    y = oracle.labels(T)
    assert np.array_equal(ad.adapt_get_labels(h, n), y), "labels differ"
    for f in range(F):
        assert np.array_equal(ad.adapt_get_value_table(h, f), oracle.value_table(X, f))
    assert np.array_equal(ad.adapt_get_bins(h, n, F), oracle.bins(X)), "bins differ"
    ref = oracle.train(X, y, V, D)
    got = ad.adapt_get_tree(h)
    assert_tree_equal(got, ref)
    Xs = X if select_X is None else select_X
    m = len(Xs)
    out = torch.empty(m, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(np.ascontiguousarray(Xs)).to(DEV), m, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(ref, Xs)), "selections differ"
    # host walk (Table-1 get_policy) agrees with the batch kernel
    for i in range(0, m, max(1, m // 50)):
        assert ad.adapt_select(h, Xs[i]) == int(out[i])
    ad.adapt_region_destroy(h)
    return got


# ------------------------------------------------------------ generator --
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_synth_device_matches_host(name):
    cfg = synth.CONFIGS[name]
    n = min(cfg.N, 20000)
    row0 = 12345 if cfg.N > 100000 else 0
    X, T = synth.generate(cfg, row0, n)
    flat, off = cfg.grid_table
    g = torch.from_numpy(flat).to(DEV)
    o = torch.from_numpy(off).to(DEV)
    dX = torch.empty((n, cfg.F), dtype=torch.float32, device=DEV)
    dT = torch.empty((n, cfg.V), dtype=torch.float32, device=DEV)
    synth.generate_device(cfg, row0, n, dX.data_ptr(), dT.data_ptr(), g.data_ptr(), o.data_ptr())
    torch.cuda.synchronize()
    assert dX.cpu().numpy().tobytes() == X.tobytes()
    assert dT.cpu().numpy().tobytes() == T.tobytes()


# ------------------------------------------------------------ configs --
def test_c1_full():
    cfg = synth.CONFIGS["C1"]
    X, T = synth.generate(cfg, 0, cfg.N)
    full_parity(X, T, cfg.D)


def test_c2_three_regions():
    cfg = synth.CONFIGS["C2"]
    X, T = synth.generate(cfg, 0, cfg.N)
    hs, refs = [], []
    s = torch.cuda.current_stream()
    keep = []
    for r in range(cfg.regions):
        rows = synth.region_rows(cfg, r)
        Xr, Tr = np.ascontiguousarray(X[rows]), np.ascontiguousarray(T[rows])
        h = _region(cfg.F, cfg.V, cfg.D)
        dX, dT = torch.from_numpy(Xr).to(DEV), torch.from_numpy(Tr).to(DEV)
        keep.append((dX, dT))
        ad.adapt_record_table(h, dX, dT, len(rows), True, s)
        hs.append(h)
        refs.append(oracle.train(Xr, oracle.labels(Tr), cfg.V, cfg.D))
    ad.adapt_train_many(hs, s)
    for h, ref in zip(hs, refs):
        assert_tree_equal(ad.adapt_get_tree(h), ref)


def test_train_many_fused_and_fallbacks():
    # fused (one multi-root frontier over the union table): trees and labels per
    # region; bins are ranks in the union's value tables.  Fallbacks: a union
    # with > 256 values of a feature (each region <= 256), different specs, an
    # empty region (its error, as adapt_train would raise it).
    rng = np.random.default_rng(21)
    s = torch.cuda.current_stream()
    keep = []

    def region(X, T, D):
        h = _region(X.shape[1], T.shape[1], D)
        dX, dT = torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV)
        keep.append((dX, dT))
        ad.adapt_record_table(h, dX, dT, len(X), True, s)
        return h

    tabs = []
    for r in range(4):
        n = int(rng.integers(50, 4000))
        X = rng.choice(np.arange(40, dtype=np.float32) + 100 * r, size=(n, 3)).astype(np.float32)
        T = rng.random((n, 5)).astype(np.float32)
        tabs.append((X, T))
    hs = [region(X, T, 6) for X, T in tabs]
    ad.adapt_train_many(hs, s)
    Xu = np.concatenate([X for X, _ in tabs])
    for h, (X, T) in zip(hs, tabs):
        y = oracle.labels(T)
        assert_tree_equal(ad.adapt_get_tree(h), oracle.train(X, y, 5, 6))
        assert np.array_equal(ad.adapt_get_labels(h, len(X)), y)
        assert np.array_equal(ad.adapt_get_value_table(h, 1), oracle.value_table(Xu, 1))
        assert np.array_equal(ad.adapt_get_bins(h, len(X), 3),
                              np.stack([np.searchsorted(oracle.value_table(Xu, f), X[:, f]) for f in range(3)],
                                       1).astype(np.uint8))
        out = torch.empty(len(X), dtype=torch.int32, device=DEV)
        ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), len(X), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), oracle.select(oracle.train(X, y, 5, 6), X))
    # union of 3 x 200 distinct values > 256: one by one
    tabs2 = [(rng.choice(np.arange(200, dtype=np.float32) + 1000 * r, size=(3000, 2)).astype(np.float32),
              rng.random((3000, 4)).astype(np.float32)) for r in range(3)]
    hs2 = [region(X, T, 5) for X, T in tabs2]
    ad.adapt_train_many(hs2, s)
    for h, (X, T) in zip(hs2, tabs2):
        assert_tree_equal(ad.adapt_get_tree(h), oracle.train(X, oracle.labels(T), 4, 5))
        assert np.array_equal(ad.adapt_get_value_table(h, 0), oracle.value_table(X, 0))
    # different depths: one by one
    hs3 = [region(*tabs[0], 3), region(*tabs[1], 4)]
    ad.adapt_train_many(hs3, s)
    assert_tree_equal(ad.adapt_get_tree(hs3[1]), oracle.train(tabs[1][0], oracle.labels(tabs[1][1]), 5, 4))
    # an empty region: the error adapt_train raises for it
    hs4 = [region(*tabs[0], 3), region(tabs[1][0][:0], tabs[1][1][:0], 3)]
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train_many(hs4, s)
    assert e.value.code == ad.ADAPT_E_INSUFFICIENT_DATA
    for h in hs + hs2 + hs3 + hs4:
        ad.adapt_region_destroy(h)


def test_c3_full():
    cfg = synth.CONFIGS["C3"]
    X, T = synth.generate(cfg, 0, cfg.N)
    got = full_parity(X, T, cfg.D, select_X=X[:200000])
    assert got["depth"].max() == cfg.D


def test_c4_slice_depth12():
    # C4's 16 features x 48 classes (feature groups, class chunks) on 2e5 rows
    cfg = synth.CONFIGS["C4"]
    X, T = synth.generate(cfg, 777, 200000)
    full_parity(X, T, cfg.D)


def test_host_table_path():
    cfg = synth.CONFIGS["C3"]
    X, T = synth.generate(cfg, 5, 30000)
    full_parity(X, T, 6, on_device=False)


# ------------------------------------------------------------ edge cases --
@pytest.mark.parametrize("seed", range(8))
def test_random_small_tables(seed):
    rng = np.random.default_rng(seed)
    for _ in range(6):
        n = int(rng.integers(1, 3000))
        F = int(rng.choice([1, 2, 3, 5, 8, 13, 16, 24]))
        V = int(rng.integers(1, 12))
        D = int(rng.integers(0, 9))
        G = int(rng.integers(1, 40))
        grid = np.unique(rng.normal(size=G).astype(np.float32) * 10)
        X = rng.choice(grid, size=(n, F)).astype(np.float32)
        T = rng.integers(1, 6, size=(n, V)).astype(np.float32)  # many label ties
        if rng.random() < 0.3:
            T[rng.random(size=T.shape) < 0.3] = np.inf
            T[np.all(np.isinf(T), axis=1), 0] = 1.0
        full_parity(X, T, D)


def test_degenerate_cases():
    # single row; all rows identical; one class; -0 vs +0; XOR (zero-gain splits)
    full_parity(np.array([[1.5, 2.0]], np.float32), np.array([[3.0, 1.0]], np.float32), 4)
    X = np.ones((100, 3), np.float32)
    T = np.random.default_rng(0).random((100, 4)).astype(np.float32)
    full_parity(X, T, 5)
    X = np.random.default_rng(1).integers(0, 9, (500, 2)).astype(np.float32)
    full_parity(X, np.tile(np.array([[1, 2, 3]], np.float32), (500, 1)), 3)
    X = np.array([[-0.0], [0.0], [1.0], [2.0]] * 10, np.float32)
    full_parity(X, np.array([[1, 2], [2, 1], [1, 2], [2, 1]] * 10, np.float32), 3)
    X = np.array([[0, 0], [0, 1], [1, 0], [1, 1]] * 7, np.float32)
    T = np.array([[1, 2], [2, 1], [2, 1], [1, 2]] * 7, np.float32)
    got = full_parity(X, T, 8)
    assert len(got) == 7


def _degenerate_tables():
    rng = np.random.default_rng(0)
    yield "single row", np.array([[1.5, 2.0]], np.float32), np.array([[3.0, 1.0]], np.float32), 4
    yield "identical rows", np.ones((100, 3), np.float32), rng.random((100, 4)).astype(np.float32), 5
    yield ("one class", np.random.default_rng(1).integers(0, 9, (500, 2)).astype(np.float32),
           np.tile(np.array([[1, 2, 3]], np.float32), (500, 1)), 3)
    yield ("-0/+0", np.array([[-0.0], [0.0], [1.0], [2.0]] * 10, np.float32),
           np.array([[1, 2], [2, 1], [1, 2], [2, 1]] * 10, np.float32), 3)
    yield ("XOR", np.array([[0, 0], [0, 1], [1, 0], [1, 1]] * 7, np.float32),
           np.array([[1, 2], [2, 1], [2, 1], [1, 2]] * 7, np.float32), 8)


@pytest.mark.parametrize("how", ["wide_classes", "many_rows", "many_features"])
def test_degenerate_cases_general_path(how):
    """The degenerate cases of test_degenerate_cases past the one-block
    small-table limits (n <= 512, F <= 8, V <= 16), so R10 (zero-gain XOR
    splits, no-candidate leaves), one class, -0/+0 and the single row run
    through the general level loop (hist / split / winner kernels and the host
    leaf logic that C4 uses):
      wide_classes  : times padded with unmeasured (+inf) variants to V = 20;
      many_rows     : every row repeated to >= 600 rows (multiplicity counts, R5);
      many_features : 8 constant features appended (F > 8; never a candidate)."""
    for name, X, T, D in _degenerate_tables():
        if how == "wide_classes":
            T = np.concatenate([T, np.full((len(T), 20 - T.shape[1]), np.inf, np.float32)], 1)
        elif how == "many_rows":
            k = -(-600 // len(X))  # > 512 rows
            X, T = np.repeat(X, k, axis=0), np.repeat(T, k, axis=0)
        else:
            X = np.concatenate([X, np.full((len(X), 8), 4.25, np.float32)], 1)
        n, F = X.shape
        h = _train(X, T, D)
        assert len(ad.adapt_train_stats(h)) >= 1, f"{name}: did not run the level loop"
        ad.adapt_region_destroy(h)
        got = full_parity(X, T, D)
        if name == "XOR":
            assert len(got) == 7  # zero-gain splits taken (R10)
        if name in ("single row", "identical rows", "one class"):
            assert len(got) == 1  # no candidate cut / pure (R10)


def test_max_distinct_and_classes():
    rng = np.random.default_rng(3)
    n = 60000
    X = np.stack([rng.permutation(np.arange(n) % 256), rng.integers(0, 256, n)], 1).astype(np.float32)
    T = rng.random((n, 200)).astype(np.float32)
    full_parity(X, T, 3)


@pytest.mark.parametrize("V", [127, 128])
def test_two_level_class_limit(V, monkeypatch):
    """Two-level row moves mark rows with label bit 7, so they run only below 128
    classes: V = 127 takes the TAG / MOVE4 schedule with class slabs (4 x 256
    values x 127 classes exceed one CTA), V = 128 the per-level partition; both
    against the oracle, several levels deep."""
    rng = np.random.default_rng(11 + V)
    n = 90000
    X = rng.integers(0, 256, size=(n, 8)).astype(np.float32)
    T = rng.random((n, V)).astype(np.float32)
    T[:, : V // 4] *= 0.9  # fewer classes win often: deeper nodes hold few classes
    monkeypatch.setenv("ADAPT_TWO_LEVEL", "1")  # (the engine reads it per train)
    full_parity(X, T, 6)


@pytest.mark.parametrize("depth", [1, 12, 16])
def test_select_synthetic_complete_tree(depth):
    # a complete depth-16 tree (131071 nodes: deeper than the
    # shared-memory top) on C4-shaped vectors, vs the oracle's walk
    cfg = synth.CONFIGS["C4"]
    cols = synth.random_tree(cfg, depth, seed=6)
    tree = np.zeros(len(cols["feature"]), oracle.NODE_DTYPE)
    for k, v in cols.items():
        tree[k] = v
    X, _ = synth.generate(cfg, 0, 300001, seed=7)
    X[::97, 3] = np.nan  # NaN goes right (R8)
    h = _region(cfg.F, cfg.V, depth)
    ad.adapt_set_tree(h, tree)
    out = torch.empty(len(X), dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), len(X), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(tree, X))
    hout = np.empty(len(X), np.int32)
    ad.adapt_select_batch_host(h, X, len(X), hout)
    assert np.array_equal(hout, oracle.select(tree, X))
    ad.adapt_region_destroy(h)


@pytest.mark.parametrize("F", [16, 5])
def test_select_deep_irregular_trees(F):
    # trained trees deeper than the shared-memory top (> 8191 nodes, leaves at
    # every depth): the walk continues in the 3-level bottom blocks, whose
    # pass-through nodes stand in for leaves above the block bottom; F=5 runs
    # the generic-F kernel
    rng = np.random.default_rng(11 + F)
    n = 60000
    X = rng.choice(np.arange(256, dtype=np.float32) * 0.5, size=(n, F)).astype(np.float32)
    T = rng.random((n, 9)).astype(np.float32)
    T[X[:, 0] < 20, 0] = 0  # a pure region: leaves high up the tree
    h = _train(X, T, 22)
    y = oracle.labels(T)
    ref = oracle.train(X, y, 9, 22)
    got = ad.adapt_get_tree(h)
    assert_tree_equal(got, ref)
    assert len(got) > 8191 and got["depth"].max() > 16
    Xs = np.concatenate([X, rng.choice(np.arange(260, dtype=np.float32) * 0.5 - 1, size=(20001, F))
                         .astype(np.float32)])
    Xs[::31, F - 1] = np.nan  # NaN goes right (R8)
    out = torch.empty(len(Xs), dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(Xs).to(DEV), len(Xs), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(ref, Xs))
    ad.adapt_region_destroy(h)


def test_select_set_tree_chain():
    # a depth-24 caterpillar given through adapt_set_tree (BFS-valid, one child a
    # leaf at every level) and a tree with two parents for a node (rejected)
    F, V, D = 4, 7, 24
    nodes = np.zeros(2 * D + 1, oracle.NODE_DTYPE)
    for d in range(D):
        k = 2 * d  # internal node of level d; its leaf sibling is 2d - 1
        nodes[k] = (d % F, k + 1, k + 2, 0, d, 0, 70.0 + d, 0, 0.0)
        nodes[k + 1] = (-1, -1, -1, d % V, d + 1, 0, 0.0, 0, 0.0)
    nodes[2 * D] = (-1, -1, -1, 3, D, 0, 0.0, 0, 0.0)
    h = _region(F, V, D)
    ad.adapt_set_tree(h, nodes)
    rng = np.random.default_rng(2)
    X = rng.uniform(70, 105, size=(50000, F)).astype(np.float32)
    out = torch.empty(len(X), dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), len(X), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.select(nodes, X))
    bad = np.zeros(5, oracle.NODE_DTYPE)  # nodes 1 and 2 both have children 3, 4
    bad[0] = (0, 1, 2, 0, 0, 0, 1.0, 0, 0.0)
    bad[1] = (0, 3, 4, 0, 1, 0, 0.5, 0, 0.0)
    bad[2] = (0, 3, 4, 0, 1, 0, 1.5, 0, 0.0)
    bad[3] = (-1, -1, -1, 1, 2, 0, 0.0, 0, 0.0)
    bad[4] = (-1, -1, -1, 2, 2, 0, 0.0, 0, 0.0)
    with pytest.raises(ad.AdaptError):
        ad.adapt_set_tree(h, bad)
    ad.adapt_region_destroy(h)


def test_select_table_of_host_recorded_table():
    """adapt_select_table: the selections of the recorded (host) table's own
    vectors from the library's device copy, to host and to device memory."""
    cfg = synth.CONFIGS["C3"]
    X, T = synth.generate(cfg, 0, 50_001)
    h = _train(X, T, 9, on_device=False)
    ref = oracle.train(X, oracle.labels(T), cfg.V, 9)
    want = oracle.select(ref, X)
    hout = np.empty(len(X), np.int32)
    ad.adapt_select_table(h, hout)
    assert np.array_equal(hout, want)
    dout = torch.empty(len(X), dtype=torch.int32, device=DEV)
    ad.adapt_select_table(h, dout, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(dout.cpu().numpy(), want)
    ad.adapt_region_destroy(h)
    h = _train(X, T, 9, on_device=True)  # borrowed device table: released by train
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_select_table(h, hout)
    assert e.value.code == ad.ADAPT_E_USAGE
    ad.adapt_region_destroy(h)


def test_errors():
    s = torch.cuda.current_stream()
    h = _region(1, 2, 2)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, s)
    assert e.value.code == ad.ADAPT_E_INSUFFICIENT_DATA
    X = torch.tensor([[1.0], [float("nan")]], device=DEV)
    T = torch.ones((2, 2), device=DEV)
    ad.adapt_record_table(h, X, T, 2, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, s)
    assert e.value.code == ad.ADAPT_E_BAD_VALUE
    X = torch.tensor([[1.0], [2.0]], device=DEV)
    T = torch.tensor([[1.0, float("nan")], [1.0, 2.0]], device=DEV)
    ad.adapt_record_table(h, X, T, 2, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, s)
    assert e.value.code == ad.ADAPT_E_BAD_VALUE
    T = torch.tensor([[float("inf"), float("inf")], [1.0, 2.0]], device=DEV)
    ad.adapt_record_table(h, X, T, 2, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, s)
    assert e.value.code == ad.ADAPT_E_BAD_VALUE
    X = torch.arange(300, dtype=torch.float32, device=DEV).reshape(-1, 1)
    T = torch.ones((300, 2), device=DEV)
    ad.adapt_record_table(h, X, T, 300, True, s)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_train(h, s)
    assert e.value.code == ad.ADAPT_E_TOO_MANY_DISTINCT
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_select(h, np.zeros(1, np.float32))
    assert e.value.code == ad.ADAPT_E_NOT_TRAINED


def test_record_path_and_shim():
    # long-format records -> aggregated wide rows -> tree; and the
    # Table-1 shim: round-robin exploration then auto-train at end
    rng = np.random.default_rng(7)
    R = 4000
    feat = rng.choice(np.arange(1, 40, dtype=np.float32), size=(R, 2))
    var = rng.integers(0, 3, R).astype(np.int32)
    ns = (feat[:, 0] * (var + 1) * 100 + rng.integers(0, 50, R)).astype(np.uint64)
    h = _region(2, 3, 4)
    for i in range(R):
        ad.adapt_record(h, feat[i], int(var[i]), int(ns[i]))
    assert ad.adapt_distinct_pairs(h) == oracle.distinct_pairs(feat, var)
    ad.adapt_train(h)
    wf, wt = oracle.aggregate(feat, var, ns, 3)
    assert_tree_equal(ad.adapt_get_tree(h), oracle.train(wf, oracle.labels(wt), 3, 4))

    r = ad.__adapt_region_create("shim_vecadd", 1, 2, "DecisionTree,explore=RoundRobin", 4)
    assert r
    pol = []
    for N in [10.0, 20.0, 30.0, 40.0]:
        ad.__adapt_region_begin(r)
        ad.__adapt_region_set_feature(r, N)
        pol.append(ad.__adapt_region_get_policy(r))
        ad.__adapt_region_end(r)
    assert pol == [0, 1, 0, 1]  # round robin before training
    info = ad.adapt_region_info(r)
    assert info["trained"]  # 4 distinct (feature, variant) pairs = min_train_data


@pytest.mark.parametrize("rare", [False, True])
def test_sampled_discovery_is_exact(rare):
    # tables above 4.2M rows discover their values on a 1M-row sample first;
    # the bin pass checks every value and falls back to the full discovery
    # when the sample missed one (a value that only occurs outside the sample)
    rng = np.random.default_rng(21)
    n, F, V = 4_500_000, 3, 3
    grid = np.array([1.0, 2.5, 4.0, 8.0, 16.0, 0.0, -3.0], np.float32)
    X = grid[rng.integers(0, len(grid), size=(n, F))]
    T = rng.random((n, V), dtype=np.float32) + 1.0
    T[np.arange(n), (X[:, 0] > 3).astype(int) + (X[:, 1] > 5).astype(int)] = 0.5
    if rare:  # rows 40000 and 4.4e6 lie between the sample chunks
        X[40_000, 1] = 123.25
        X[4_400_000, 2] = -7.5
    h = _train(X, T, 3)
    for f in range(F):
        assert np.array_equal(ad.adapt_get_value_table(h, f), oracle.value_table(X, f)), f
    bins = ad.adapt_get_bins(h, n, F)
    ref_bins = np.stack([np.searchsorted(oracle.value_table(X, f), X[:, f]) for f in range(F)], 1)
    assert np.array_equal(bins, ref_bins.astype(np.uint8))
    y = oracle.labels(T)
    assert_tree_equal(ad.adapt_get_tree(h), oracle.train(X, y, V, 3))
