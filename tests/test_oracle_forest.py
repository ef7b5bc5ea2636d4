"""Pins of the oracle's random forest ("rfc"; SPEC train_rfc /
predict; readings R19-R21 in DESIGN.md §3)."""
import math

import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module", autouse=True)
def _build():
    oracle.build()


M64 = (1 << 64) - 1


def _splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_splitmix64_reference_value():
    # Vigna's SplitMix64 seeded with 0 returns 0xe220a8397b1dcdaf first; the
    # generator R19 uses is that mixer (state + golden gamma, then mix)
    assert _splitmix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("seed,tree,n", [(0, 0, 1), (0, 0, 10), (7, 3, 1000), (2**63 + 5, 9, 4097)])
def test_bootstrap_is_n_draws_with_replacement(seed, tree, n):
    w = oracle.bootstrap(seed, tree, n)
    assert w.dtype == np.uint32 and len(w) == n and int(w.sum()) == n
    # exact re-derivation of R19 with Python integers
    key = _splitmix64(seed ^ _splitmix64(tree + 0x5851F42D4C957F2D))
    ref = np.zeros(n, np.int64)
    for j in range(n):
        ref[(_splitmix64(key ^ _splitmix64(j)) * n) >> 64] += 1
    assert np.array_equal(w, ref)


def test_bootstrap_multiplicities_are_binomial():
    # a size-n resample with replacement: w_i ~ Binomial(n, 1/n) -> Poisson(1)
    n = 200_000
    w = oracle.bootstrap(3, 1, n)
    freq = np.bincount(w, minlength=6)[:5] / n
    pois = np.array([math.exp(-1) / math.factorial(k) for k in range(5)])
    assert np.all(np.abs(freq - pois) < 5 * np.sqrt(pois / n) + 1e-4)
    # different trees / seeds give different resamples; the same ones repeat exactly
    assert not np.array_equal(w, oracle.bootstrap(3, 2, n))
    assert not np.array_equal(w, oracle.bootstrap(4, 1, n))
    assert np.array_equal(w, oracle.bootstrap(3, 1, n))


def _leaf(label):
    t = np.zeros(1, oracle.NODE_DTYPE)
    t["feature"] = -1
    t["left"] = t["right"] = -1
    t["label"] = label
    return t


@pytest.mark.parametrize("labels,expect", [([0, 1, 1], 1), ([0, 1], 0), ([2, 1, 1, 2], 1),
                                           ([3], 3), ([4, 4, 0, 1, 1, 4], 4)])
def test_majority_vote_ties_lowest(labels, expect):
    # SPEC predict: "forest of 3 trees voting {0,1,1} -> 1"; ties -> lowest (R20)
    X = np.zeros((3, 2), np.float32)
    assert np.all(oracle.select_forest([_leaf(l) for l in labels], X) == expect)


def test_single_row_forest_is_the_tree():
    # n = 1: every bootstrap is the table itself, so each tree is train_dtree's
    X = np.array([[1.0, 2.0]], np.float32)
    y = np.array([1], np.uint8)
    for t in oracle.train_forest(X, y, 3, 4, 5, seed=11):
        assert oracle.select(t, X)[0] == 1 and len(t) == 1


def test_single_label_data_predicts_that_label():
    rng = np.random.default_rng(0)
    X = rng.integers(0, 9, size=(300, 3)).astype(np.float32)
    y = np.full(300, 2, np.uint8)
    trees = oracle.train_forest(X, y, 4, 3, 6, seed=1)
    assert np.all(oracle.select_forest(trees, X) == 2)


def test_forest_trees_are_trees_of_the_resamples_and_deterministic():
    rng = np.random.default_rng(5)
    X = rng.integers(0, 6, size=(400, 2)).astype(np.float32)
    y = ((X[:, 0] + X[:, 1]) > 5).astype(np.uint8) + (X[:, 0] > 4).astype(np.uint8)
    a = oracle.train_forest(X, y, 3, 3, 4, seed=9)
    b = oracle.train_forest(X, y, 3, 3, 4, seed=9)
    for t, (ta, tb) in enumerate(zip(a, b)):
        assert ta.tobytes() == tb.tobytes()
        w = oracle.bootstrap(9, t, len(X))
        assert ta["n"][0] == int(w.sum())  # root holds the whole resample
        counts = np.bincount(y, weights=w, minlength=3)
        assert ta["label"][0] == int(np.argmax(counts))  # majority of the resample
