"""Pins of the oracle's K-fold harness (DESIGN R22) against what the
paper and the mathematics fix: the shuffle is a permutation (brute force), the
K groups are equal-sized (closed form), every input is in the training set of
exactly m folds and in the test set of K-m (the paper's "each input appears at
least once in the training set and in the testing set"), and the accuracy of
a depth-1 model on a separable crossover table equals a rule derived by hand
from the uniqueness of the perfect cut (independent of the CART code)."""
import math

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("N", [1, 2, 3, 5, 16, 17, 100, 1000, 4097])
@pytest.mark.parametrize("seed,shuffle", [(0, 0), (7, 3), (2**63 + 5, 9)])
def test_pos_is_a_permutation(N, seed, shuffle):
    pos = [oracle.kfold_pos(seed, shuffle, N, r) for r in range(N)]
    assert sorted(pos) == list(range(N))


def test_pos_bad_args():
    assert oracle.kfold_pos(0, 0, 10, 10) == -1
    assert oracle.kfold_pos(0, 0, 0, 0) == -1
    assert oracle.kfold_pos(0, -1, 10, 0) == -1


def test_shuffles_differ_and_spread():
    N = 1000
    p0 = [oracle.kfold_pos(1, 0, N, r) for r in range(N)]
    p1 = [oracle.kfold_pos(1, 1, N, r) for r in range(N)]
    assert p0 != p1 and p0 != list(range(N))
    # row 0's group over 4000 shuffles: roughly uniform over K = 4 (chi-square, 3 dof, p ~ 1e-6)
    g = [oracle.kfold_groups(5, s, 37, 4)[0] for s in range(4000)]
    cnt = np.bincount(g, minlength=4)
    exp = 4000 * np.array([10, 9, 9, 9]) / 37  # group sizes of N=37, K=4
    assert ((cnt - exp) ** 2 / exp).sum() < 30


@pytest.mark.parametrize("N,K", [(1, 2), (7, 4), (100, 4), (1001, 4), (10, 3), (4097, 7)])
def test_groups_equal_sized(N, K):
    g = oracle.kfold_groups(3, 2, N, K)
    sizes = np.bincount(g, minlength=K)
    # |{pos : floor(pos K / N) = j}| = ceil((j+1) N / K) - ceil(j N / K)
    want = [-((-(j + 1) * N) // K) + ((-j * N) // K) for j in range(K)]
    assert list(sizes) == want and sizes.sum() == N
    assert sizes.max() - sizes.min() <= 1


@pytest.mark.parametrize("m", [1, 2, 3])
def test_fold_coverage(m):
    rng = np.random.default_rng(m)
    N, K = 40, 4
    X = rng.integers(0, 5, size=(N, 2)).astype(np.float32)
    T = rng.random((N, 3)).astype(np.float32)
    res, trees = oracle.kfold(X, T, 2, K, m, 3, seed=11)
    assert len(res) == len(trees) == 3 * K
    for s in range(3):
        g = oracle.kfold_groups(11, s, N, K)
        in_train = np.zeros(N, int)
        for k in range(K):
            in_train += np.isin(g, [(k + j) % K for j in range(m)])
        assert (in_train == m).all()  # trained on m folds, tested on K - m >= 1
    for r in res:
        assert r["n_train"] + r["n_test"] == N


def test_single_label_table():
    X = np.arange(20, dtype=np.float32)[:, None]
    T = np.stack([np.ones(20), np.full(20, 2.0)], 1).astype(np.float32)
    res, _ = oracle.kfold(X, T, 3, 4, 2, 2, seed=1)
    for r in res:
        assert r["n_correct"] == r["n_test"] == 10
        assert r["t_selected"] == r["t_best"] == 10.0


@pytest.mark.parametrize("m", [1, 2, 3])
def test_crossover_accuracy_by_hand(m):
    # SURVEY A3's crossover: t_cpu = 2x + 10, t_gpu = 0.5x + 40 -> label 0 iff
    # x <= 20 (tie at 20 -> 0).  A depth-1 tree on a training set with both
    # classes has exactly one perfect cut candidate, (max0 + min1) / 2 between
    # the largest class-0 and the smallest class-1 training input; a training
    # set with one class is a leaf of that class.
    x = np.arange(10, 210, 10, dtype=np.float32)
    T = np.stack([2 * x + 10, 0.5 * x + 40], 1).astype(np.float32)
    y = (x > 20).astype(int)
    res, _ = oracle.kfold(x[:, None], T, 1, 4, m, 5, seed=4)
    for r in res:
        g = oracle.kfold_groups(4, r["shuffle"], len(x), 4)
        tr = np.isin(g, [(r["fold"] + j) % 4 for j in range(m)])
        te = ~tr
        if len(set(y[tr])) == 2:
            thr = (float(x[tr][y[tr] == 0].max()) + float(x[tr][y[tr] == 1].min())) / 2
            pred = (x[te] > thr).astype(int)
        else:
            pred = np.full(te.sum(), y[tr][0])
        assert r["n_correct"] == int((pred == y[te]).sum())
        assert r["t_best"] == math.fsum(float(T[i, y[i]]) for i in np.nonzero(te)[0])
        assert r["t_selected"] == math.fsum(float(T[i, p]) for i, p in zip(np.nonzero(te)[0], pred))
