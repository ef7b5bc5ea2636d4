"""Pins for the CPU oracle (no GPU).  Each test cites what fixes the expected
value: a SPEC/paper worked example (tests/golden/), exact rational brute force
(tests/exact_checker.py), a closed form or an invariant."""
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import exact_checker as ex


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


def _frac(s):
    return Fraction(s)


# ---------------------------------------------------------------- labelling --
def test_golden_labelling(golden_dir):
    g = _load(golden_dir, "spec_labelling.json")
    for case in g["cases"]:
        feat = np.array([r[0] for r in case["records"]], np.float32)
        var = np.array([r[1] for r in case["records"]], np.int32)
        ns = np.array([r[2] for r in case["records"]], np.uint64)
        wf, wt = oracle.aggregate(feat, var, ns, case["V"])
        assert wf.tolist() == case["expect_features"], case["name"]
        assert oracle.labels(wt).tolist() == case["expect_labels"], case["name"]


def test_golden_distinct_pairs(golden_dir):
    g = _load(golden_dir, "spec_distinct.json")
    for case in g["cases"]:
        if not case["records"]:
            feat = np.zeros((0, case["F"]), np.float32)
            var = np.zeros(0, np.int32)
        else:
            feat = np.array([r[0] for r in case["records"]], np.float32)
            var = np.array([r[1] for r in case["records"]], np.int32)
        assert oracle.distinct_pairs(feat, var) == case["expect"], case["name"]


def test_labels_match_exact_checker_random():
    rng = random.Random(11)
    for _ in range(300):
        n, V = rng.randint(1, 6), rng.randint(1, 6)
        t = np.array([[rng.choice([1.0, 2.0, 3.0, 0.5, float("inf"), -0.0, 0.0])
                       for _ in range(V)] for _ in range(n)], np.float32)
        for i in range(n):  # keep at least one measured variant per row
            if np.all(np.isinf(t[i])):
                t[i, rng.randrange(V)] = 1.0
        assert oracle.labels(t).tolist() == ex.labels_exact(t.tolist())


def test_labels_crossover_closed_form():
    # device-select cost model t_v(N) = a_v N + b_v: label = [N > N*],
    # N* = (b1-b0)/(a0-a1), exact tie at N* -> 0 (R2).
    a0, b0, a1, b1 = 2.0, 10.0, 0.5, 40.0
    nstar = (b1 - b0) / (a0 - a1)  # = 20
    Ns = np.arange(1, 64, dtype=np.float32)
    t = np.stack([a0 * Ns + b0, a1 * Ns + b1], 1).astype(np.float32)
    assert oracle.labels(t).tolist() == [int(N > nstar) for N in Ns]


def test_labels_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.labels(np.array([[np.inf, np.inf]], np.float32))
    assert e.value.code == oracle.E_BAD_VALUE
    with pytest.raises(oracle.OracleError) as e:
        oracle.labels(np.array([[1.0, np.nan]], np.float32))
    assert e.value.code == oracle.E_BAD_VALUE


def test_labelling_stable_under_slower_duplicate():
    # adding a strictly slower measurement of a non-winning variant never
    # changes a label.
    rng = random.Random(3)
    for _ in range(100):
        R, V = rng.randint(1, 8), 3
        feat = np.array([[float(rng.randint(0, 2))] for _ in range(R)], np.float32)
        var = np.array([rng.randrange(V) for _ in range(R)], np.int32)
        ns = np.array([rng.randint(1, 100) for _ in range(R)], np.uint64)
        wf, wt = oracle.aggregate(feat, var, ns, V)
        lab = oracle.labels(wt)
        for g in range(len(wf)):
            losers = [v for v in range(V) if v != lab[g] and np.isfinite(wt[g, v])]
            if not losers:
                continue
            v = losers[0]
            slow = np.uint64(int(wt[g, v]) * 10 + 1000)
            wf2, wt2 = oracle.aggregate(np.vstack([feat, wf[g:g + 1]]), np.append(var, v),
                                        np.append(ns, slow), V)
            assert oracle.labels(wt2).tolist() == lab.tolist()


def test_aggregate_mean_and_first_appearance():
    feat = np.array([[2.0], [1.0], [2.0], [-0.0], [0.0]], np.float32)
    var = np.array([0, 1, 0, 1, 1], np.int32)
    ns = np.array([3, 7, 4, 9, 10], np.uint64)
    wf, wt = oracle.aggregate(feat, var, ns, 2)
    # order of first appearance; -0 and +0 are one vector (R4)
    assert wf[:, 0].tolist() == [2.0, 1.0, 0.0]
    assert math.copysign(1.0, float(wf[2, 0])) == 1.0
    assert wt[0].tolist() == [3.5, float("inf")]
    assert wt[1].tolist() == [float("inf"), 7.0]
    assert wt[2].tolist() == [float("inf"), 9.5]


# ------------------------------------------------------------- value tables --
def test_value_table_and_bins():
    rng = np.random.default_rng(0)
    X = rng.choice(np.array([3.5, -1.0, 0.0, -0.0, 7.25, 1e-30], np.float32), size=(200, 3))
    for f in range(3):
        vt = oracle.value_table(X, f)
        ref = sorted(set(float(v) + 0.0 for v in X[:, f]))
        assert vt.tolist() == ref
    b = oracle.bins(X)
    for f in range(3):
        vt = oracle.value_table(X, f)
        assert np.all(vt[b[:, f]] == X[:, f])


def test_value_table_too_many_distinct():
    X = np.arange(300, dtype=np.float32).reshape(-1, 1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.value_table(X, 0)
    assert e.value.code == oracle.E_TOO_MANY_DISTINCT
    assert len(oracle.value_table(X[:256], 0)) == 256


def test_nonfinite_features_rejected():
    for bad in (np.nan, np.inf, -np.inf):
        X = np.array([[1.0], [bad]], np.float32)
        with pytest.raises(oracle.OracleError) as e:
            oracle.train(X, np.array([0, 1], np.uint8), 2, 2)
        assert e.value.code == oracle.E_BAD_VALUE


# --------------------------------------------------------------------- Gini --
def test_gini_closed_forms():
    assert oracle.gini_counts([5, 0, 0]) == 0.0  # pure
    for k in range(1, 9):
        assert oracle.gini_counts([7] * k) == pytest.approx(1 - 1 / k, abs=1e-15)
    for a, b in [(1, 3), (2, 2), (5, 11), (1000, 1)]:
        p = a / (a + b)
        assert oracle.gini_counts([a, b]) == pytest.approx(2 * p * (1 - p), rel=1e-14)


# ------------------------------------------------------------------- trees --
def _check_tree(got, expect):
    assert len(got) == len(expect)
    for g, e in zip(got, expect):
        assert int(g["feature"]) == e["feature"]
        assert int(g["label"]) == e["label"]
        assert int(g["depth"]) == e["depth"]
        assert int(g["n"]) == e["n"]
        # gini is the double formula 1 - S/(n*n): within a few ulps of the exact value
        assert float(g["gini"]) == pytest.approx(float(_frac(e["gini"])), rel=1e-15, abs=1e-16)
        if e["feature"] >= 0:
            assert float(g["threshold"]) == float(_frac(e["threshold"]))
            assert int(g["left"]) == e["left"] and int(g["right"]) == e["right"]


def test_golden_spec_train_predict(golden_dir):
    g = _load(golden_dir, "spec_train_predict.json")
    for case in g["train"]:
        t = oracle.train(np.array(case["X"], np.float32), np.array(case["y"], np.uint8),
                         case["C"], case["D"])
        _check_tree(t, case["expect"])
    tree = np.zeros(len(g["predict_tree"]), oracle.NODE_DTYPE)
    for i, nd in enumerate(g["predict_tree"]):
        for k, v in nd.items():
            tree[i][k] = v
    for case in g["predict"]:
        assert oracle.select(tree, np.array([case["x"]], np.float32))[0] == case["expect"]


def test_golden_appendix_a(golden_dir):
    g = _load(golden_dir, "survey_appendix_a.json")
    for key in ("A1", "A3b"):
        c = g[key]
        X = np.array(c["X"], np.float32)
        y = np.array(c["y"], np.uint8)
        t = oracle.train(X, y, c["C"], c["D"])
        _check_tree(t, c["expect"])
        assert float(t[0]["gini"]) == pytest.approx(float(_frac(c["root_gini"])), rel=1e-15)
    a1 = g["A1"]
    X = np.array(a1["X"], np.float32)
    y = np.array(a1["y"], np.uint8)
    acc = Fraction(int(np.sum(oracle.select(oracle.train(X, y, 2, 2), X) == y)), len(y))
    assert acc == _frac(a1["train_accuracy"])
    # greedy < exhaustive here (SPEC's acceptance criterion 4 is false)
    best = ex.exhaustive_best_accuracy([Fraction(v) for v in X[:, 0].tolist()], y.tolist(), 2, 2)
    assert Fraction(best, len(y)) == _frac(a1["exhaustive_depth2_accuracy"])
    # hand values of the three cuts at the root
    for thr, wg in a1["cut_weighted_gini"].items():
        L = [int(v) for v, x in zip(y, X[:, 0]) if x <= float(thr)]
        R = [int(v) for v, x in zip(y, X[:, 0]) if x > float(thr)]
        w = (len(L) * ex.gini(ex._counts(L, 2)) + len(R) * ex.gini(ex._counts(R, 2))) / 4
        assert w == _frac(wg)


def _random_table(rng, n, F, C, grid):
    X = np.array([[rng.choice(grid) for _ in range(F)] for _ in range(n)], np.float32)
    y = np.array([rng.randrange(C) for _ in range(n)], np.uint8)
    return X, y


def _compare_with_exact(X, y, C, D):
    t = oracle.train(X, y, C, D)
    e = ex.cart_exact(X.tolist(), y.tolist(), C, D)
    assert len(t) == len(e)
    for g, h in zip(t, e):
        assert int(g["feature"]) == h["feature"]
        assert int(g["left"]) == h["left"] and int(g["right"]) == h["right"]
        assert int(g["label"]) == h["label"]
        assert int(g["n"]) == h["n"]
        assert int(g["depth"]) == h["depth"]
        assert float(g["gini"]) == pytest.approx(float(h["gini"]), rel=1e-15, abs=1e-16)
        if h["feature"] >= 0:
            # oracle thr = RN((double)u_j + (double)u_{j+1}) / 2 = RN(exact midpoint)
            assert float(g["threshold"]) == float(h["threshold"])
    return t, e


@pytest.mark.parametrize("seed", range(6))
def test_tree_matches_exact_bruteforce(seed):
    rng = random.Random(seed)
    grids = [[1.0, 2.0, 3.0], [0.5, -1.0, 4.0, 4.5, 9.0], [0.0, 1.0], [1.5, 2.5, 3.5, 4.5, 5.5, 6.5]]
    for _ in range(40):
        n = rng.randint(1, 12)
        F = rng.randint(1, 3)
        C = rng.randint(1, 4)
        D = rng.randint(0, 4)
        X, y = _random_table(rng, n, F, C, rng.choice(grids))
        _compare_with_exact(X, y, C, D)


def test_tree_invariants_random():
    rng = random.Random(99)
    for _ in range(60):
        n, F, C = rng.randint(2, 30), rng.randint(1, 3), rng.randint(2, 4)
        X, y = _random_table(rng, n, F, C, [float(v) for v in range(8)])
        prev_acc = -1
        for D in range(0, 7):
            t = oracle.train(X, y, C, D)
            pred = oracle.select(t, X)
            acc = int(np.sum(pred == y))
            assert acc >= prev_acc  # training accuracy non-decreasing in D
            prev_acc = acc
            for k, nd in enumerate(t):
                if nd["feature"] < 0:
                    continue
                # S:288 threshold soundness: strictly between left max and right min of the node
                rows = _rows_of_node(t, X, k)
                xs = X[rows, nd["feature"]].astype(np.float64)
                L, R = xs[xs <= nd["threshold"]], xs[xs > nd["threshold"]]
                assert L.size and R.size and L.max() < nd["threshold"] < R.min()
                # S:289 Gini monotonicity, as R10 reads it: the weighted child Gini
                # never exceeds the parent's, and is strictly below it whenever
                # some candidate at that node lowers it.
                l, r = t[nd["left"]], t[nd["right"]]
                w = (l["n"] * Fraction(l["gini"]) + r["n"] * Fraction(r["gini"])) / nd["n"]
                w_exact = _weighted_exact(X, y, rows, nd["feature"], nd["threshold"], C)
                parent = ex.gini(ex._counts(y[rows].tolist(), C))
                assert w_exact <= parent
                if ex.best_split(X.tolist(), y.tolist(), rows.tolist(), C)[0][0] < parent:
                    assert w_exact < parent
                assert abs(w - w_exact) < 1e-12
        # depth-unlimited on distinct vectors -> 100% training accuracy
        _, keep = np.unique(X, axis=0, return_index=True)
        Xd, yd = X[np.sort(keep)], y[np.sort(keep)]
        t = oracle.train(Xd, yd, C, 40, cap=4 * len(yd) + 1)
        assert np.all(oracle.select(t, Xd) == yd)


def _weighted_exact(X, y, rows, f, thr, C):
    L = [int(y[i]) for i in rows if X[i, f] <= thr]
    R = [int(y[i]) for i in rows if X[i, f] > thr]
    return (len(L) * ex.gini(ex._counts(L, C)) + len(R) * ex.gini(ex._counts(R, C))) / len(rows)


def test_xor_node_splits_with_zero_gain():
    # R10: a node whose every cut has zero gain (XOR) is still split, so the
    # depth-unlimited tree reproduces the labels (north_star invariant).
    X = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], np.float32)
    y = np.array([0, 1, 1, 0], np.uint8)
    t = oracle.train(X, y, 2, 8)
    assert t[0]["feature"] == 0 and t[0]["threshold"] == 0.5  # all tie: lowest f, thr
    assert np.all(oracle.select(t, X) == y)
    assert len(t) == 7


def _rows_of_node(t, X, k):
    rows = []
    for i in range(len(X)):
        j = 0
        path = [0]
        while t[j]["feature"] >= 0 and j != k:
            j = t[j]["left"] if X[i, t[j]["feature"]] <= t[j]["threshold"] else t[j]["right"]
            path.append(j)
        if k in path:
            rows.append(i)
    return np.array(rows, np.int64)


def test_greedy_not_better_than_exhaustive():
    # greedy depth-<=2 accuracy <= exhaustive optimum (never >)
    rng = random.Random(5)
    for _ in range(150):
        n = rng.randint(1, 7)
        xs = sorted(rng.sample(range(1, 20), n))
        y = [rng.randrange(3) for _ in range(n)]
        X = np.array(xs, np.float32).reshape(-1, 1)
        t = oracle.train(X, np.array(y, np.uint8), 3, 2)
        g = int(np.sum(oracle.select(t, X) == np.array(y)))
        assert g <= ex.exhaustive_best_accuracy([Fraction(v) for v in xs], y, 3, 2)


def test_row_permutation_invariance():
    rng = np.random.default_rng(4)
    X = rng.integers(0, 6, size=(300, 3)).astype(np.float32)
    y = rng.integers(0, 3, size=300).astype(np.uint8)
    t = oracle.train(X, y, 3, 5)
    for _ in range(3):
        p = rng.permutation(300)
        t2 = oracle.train(X[p], y[p], 3, 5)
        assert t.tobytes() == t2.tobytes()


def test_step_function_special_case():
    # one feature, labels = [x > t]: a depth-1 tree splitting at the midpoint of
    # the two grid values straddling t (SURVEY §8(c) "special case").
    grid = np.array([1, 2, 4, 8, 16, 32, 64], np.float32)
    for tcut in (1.5, 3.0, 10.0, 50.0):
        X = np.repeat(grid, 3).reshape(-1, 1)
        y = (X[:, 0] > tcut).astype(np.uint8)
        t = oracle.train(X, y, 2, 3)
        lo, hi = grid[grid <= tcut].max(), grid[grid > tcut].min()
        assert len(t) == 3 and t[0]["feature"] == 0
        assert t[0]["threshold"] == (float(lo) + float(hi)) / 2


def test_select_special_cases():
    leaf = np.zeros(1, oracle.NODE_DTYPE)
    leaf[0]["feature"] = -1
    leaf[0]["label"] = 3
    X = np.array([[1.0], [np.nan], [-5.0]], np.float32)
    assert oracle.select(leaf, X).tolist() == [3, 3, 3]
    stump = np.zeros(3, oracle.NODE_DTYPE)
    stump[0] = (0, 1, 2, 0, 0, 0, 0.5, 0, 0.0)
    stump[1] = (-1, -1, -1, 7, 1, 0, 0.0, 0, 0.0)
    stump[2] = (-1, -1, -1, 9, 1, 0, 0.0, 0, 0.0)
    X = np.array([[0.5], [np.nextafter(np.float32(0.5), np.float32(1))], [np.nan], [-np.inf]],
                 np.float32)
    assert oracle.select(stump, X).tolist() == [7, 9, 9, 7]  # == -> left, NaN -> right (R8)


def test_negative_zero_canonical():
    X = np.array([[-0.0], [0.0], [1.0], [1.0]], np.float32)
    y = np.array([0, 0, 1, 1], np.uint8)
    t = oracle.train(X, y, 2, 2)
    assert t[0]["threshold"] == 0.5 and len(t) == 3
    vt = oracle.value_table(X, 0)
    assert vt.tolist() == [0.0, 1.0] and math.copysign(1, float(vt[0])) == 1


def test_openmp_build_is_identical():
    """The all-cores build (liboracle_omp.so: the same oracle.c with -fopenmp,
    features of a node scanned in parallel and reduced in feature order) gives
    byte-identical trees and selections — it only serves timing and the
    full-size expected outputs (scripts/oracle_fullsize.py)."""
    import synth

    X, T = synth.generate("C4", 0, 20_000)
    y = oracle.labels(T)
    a = oracle.train(X, y, 48, 8)
    b = oracle.train(X, y, 48, 8, omp=True)
    assert len(a) > 100 and a.tobytes() == b.tobytes()
    assert np.array_equal(oracle.select(a, X), oracle.select(a, X, omp=True))
