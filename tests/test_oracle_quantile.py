"""Pins of the oracle's lossy quantile binning (DESIGN R23)
against what the definition and the mathematics fix: <= 256 distinct values
leave the table and the tree exactly as the pinned exact path; bins hold
floor/ceil(D/256) distinct values each (closed form) and are monotone; a
1-feature root split equals a brute-force exact-Fraction search over the 255
fixed cut points c_b = (u[e_b - 1] + u[e_b]) / 2; every reported threshold
routes the raw training rows exactly as the quantised split."""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def test_few_values_unchanged():
    rng = np.random.default_rng(0)
    X = rng.choice(np.arange(200, dtype=np.float32), size=(3000, 3))
    T = rng.random((3000, 4)).astype(np.float32)
    assert oracle.quantizer(X) == {}
    y = oracle.labels(T)
    assert oracle.train_quantile(X, y, 4, 5).tobytes() == oracle.train(X, y, 4, 5).tobytes()


@pytest.mark.parametrize("D", [257, 300, 1000, 4097])
def test_equal_count_bins(D):
    rng = np.random.default_rng(D)
    vals = np.unique(rng.normal(size=3 * D).astype(np.float32))[:D]
    X = rng.permutation(np.concatenate([vals, rng.choice(vals, 500)]))[:, None].astype(np.float32)
    q = oracle.quantizer(X)
    lb, prev = q[0]
    assert len(lb) == 256 and np.all(np.diff(lb) > 0) and np.all(prev[1:] < lb[1:])
    Xq = oracle.quantize(X, q)
    b = np.searchsorted(lb, vals, side="right") - 1  # bin of each distinct value
    sizes = np.bincount(b, minlength=256)
    want = [((j + 1) * D) // 256 - (j * D) // 256 for j in range(256)]
    assert list(sizes) == want and set(sizes) <= {D // 256, -(-D // 256)}
    assert np.all(np.diff(b) >= 0)  # monotone
    assert len(np.unique(Xq[:, 0])) == 256
    for j in range(1, 256):  # prev_b is the largest value of bin b-1
        assert prev[j] == vals[b == j - 1].max() and lb[j] == vals[b == j].min()


def _brute_root(x, y, C, cuts):
    best = None
    n = len(x)
    tot = np.bincount(y, minlength=C)
    for c in cuts:
        left = x.astype(np.float64) <= c
        nl = int(left.sum())
        if nl in (0, n):
            continue
        cl = np.bincount(y[left], minlength=C)
        cr = tot - cl
        # R10: every cut with two non-empty sides competes,
        # zero-gain ones included; they score exactly S/n, below any improving cut
        s = Fraction(int((cl.astype(object) ** 2).sum()), nl) + \
            Fraction(int((cr.astype(object) ** 2).sum()), n - nl)
        if best is None or s > best[0]:  # strict: ties keep the lowest cut
            best = (s, c)
    return best[1]


@pytest.mark.parametrize("seed", range(4))
def test_root_split_brute_force(seed):
    rng = np.random.default_rng(seed)
    vals = np.unique(rng.uniform(0, 100, size=900).astype(np.float32))[:700]
    x = rng.choice(vals, size=2000).astype(np.float32)
    y = ((x > 37) ^ (rng.random(2000) < 0.15)).astype(np.uint8) + (x > 80).astype(np.uint8)
    tree = oracle.train_quantile(x[:, None], y, 3, 1)
    u = np.unique(x)
    e = (np.arange(256) * len(u)) // 256
    cuts = [(float(u[e[b] - 1]) + float(u[e[b]])) / 2 for b in range(1, 256)]
    assert tree["feature"][0] == 0 and tree["threshold"][0] == _brute_root(x, y, 3, cuts)


def test_thresholds_route_like_the_quantised_split():
    rng = np.random.default_rng(9)
    n = 20000
    X = np.stack([rng.normal(size=n), rng.integers(0, 50, n), rng.exponential(size=n)], 1).astype(np.float32)
    T = np.stack([X[:, 0] * 3 + X[:, 2], X[:, 1] * 0.1 + 1, 2 - X[:, 0]], 1).astype(np.float32)
    T += rng.random(T.shape).astype(np.float32)
    y = oracle.labels(T)
    q = oracle.quantizer(X)
    assert set(q) == {0, 2}
    Xq = oracle.quantize(X, q)
    raw = oracle.train_quantile(X, y, 3, 8)
    ref = oracle.train(Xq, y, 3, 8)
    for k in ("feature", "left", "right", "label", "depth", "n"):
        assert np.array_equal(raw[k], ref[k])
    assert np.array_equal(raw["threshold"][ref["feature"] == 1], ref["threshold"][ref["feature"] == 1])
    # the raw tree walks the raw rows exactly as the quantised tree walks Xq
    assert np.array_equal(oracle.select(raw, X), oracle.select(ref, Xq))
