"""CPU oracle for the adaptive-OpenMP model-building path.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2303_08873_b200``) never imports it and has
no CPU fallback.

This is a ctypes wrapper (argument marshalling only) over ``oracle.c``, a plain
single-threaded C implementation written from PAPER.md and the readings in
DESIGN.md §3.  See ``oracle.h`` for the per-function citations.  Every function
is pinned by ``tests/test_oracle_*.py`` (exact rational brute force, closed
forms and the worked examples under ``tests/golden/``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SO_OMP = os.path.join(_HERE, "liboracle_omp.so")  # same source, -fopenmp (bench timing only)
_SRC = os.path.join(_HERE, "oracle.c")

OK = 0
E_INVALID_ARG = -1
E_INSUFFICIENT_DATA = -4
E_BAD_VALUE = -6
E_TOO_MANY_DISTINCT = -7
E_CAPACITY = -12

NODE_DTYPE = np.dtype(
    [
        ("feature", np.int32),
        ("left", np.int32),
        ("right", np.int32),
        ("label", np.int32),
        ("depth", np.int32),
        ("pad_", np.int32),
        ("threshold", np.float64),
        ("n", np.int64),
        ("gini", np.float64),
    ]
)
assert NODE_DTYPE.itemsize == 48


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no FMA contraction) and the
    all-cores build liboracle_omp.so of the same source (-fopenmp: features of
    a node scanned in parallel, vectors walked in parallel; same results)."""
    srcs_mtime = max(os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h")))
    for so, extra in ((_SO, []), (_SO_OMP, ["-fopenmp"])):
        if force or not os.path.exists(so) or os.path.getmtime(so) < srcs_mtime:
            subprocess.check_call(
                ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", *extra,
                 "-shared", "-o", so, _SRC, "-lm"]
            )
    return _SO


_libs = {}


def lib(omp: bool = False):
    if omp not in _libs:
        build()
        L = ctypes.CDLL(_SO_OMP if omp else _SO)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.oracle_canon_features.argtypes = [P, i64, ctypes.c_int, P]
        L.oracle_labels.argtypes = [P, i64, ctypes.c_int, P]
        L.oracle_aggregate.argtypes = [P, P, P, i64, ctypes.c_int, ctypes.c_int, P, P, i64, P]
        L.oracle_distinct_pairs.argtypes = [P, P, i64, ctypes.c_int]
        L.oracle_distinct_pairs.restype = i64
        L.oracle_value_table.argtypes = [P, i64, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P]
        L.oracle_train.argtypes = [P, P, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, i32, P]
        L.oracle_select.argtypes = [P, i32, P, i64, ctypes.c_int, P]
        L.oracle_bootstrap.argtypes = [ctypes.c_uint64, ctypes.c_int, i64, P]
        L.oracle_kfold_pos.argtypes = [ctypes.c_uint64, ctypes.c_int, i64, i64]
        L.oracle_kfold_pos.restype = i64
        L.oracle_kfold_groups.argtypes = [ctypes.c_uint64, ctypes.c_int, i64, ctypes.c_int, P]
        L.oracle_gini_counts.argtypes = [P, ctypes.c_int]
        L.oracle_gini_counts.restype = ctypes.c_double
        _libs[omp] = L
    return _libs[omp]


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(X, F=None):
    X = np.ascontiguousarray(X, dtype=np.float32)
    if F is not None:
        X = X.reshape(-1, F)
    return X


def canon_features(X: np.ndarray) -> np.ndarray:
    X = _f32(X)
    n, F = X.shape
    out = np.empty_like(X)
    rc = lib().oracle_canon_features(_p(X), n, F, _p(out))
    if rc:
        raise OracleError(rc, "canon_features")
    return out


def labels(times: np.ndarray) -> np.ndarray:
    """Fastest-variant label per row."""
    t = _f32(times)
    n, V = t.shape
    out = np.empty(n, np.uint8)
    rc = lib().oracle_labels(_p(t), n, V, _p(out))
    if rc:
        raise OracleError(rc, "labels")
    return out


def aggregate(feat: np.ndarray, var: np.ndarray, ns: np.ndarray, V: int):
    """Long-format records -> (wide features [n][F], wide times [n][V])."""
    feat = _f32(feat)
    R, F = feat.shape
    var = np.ascontiguousarray(var, dtype=np.int32)
    ns = np.ascontiguousarray(ns, dtype=np.uint64)
    of = np.empty((max(R, 1), F), np.float32)
    ot = np.empty((max(R, 1), V), np.float32)
    n_out = np.zeros(1, np.int64)
    rc = lib().oracle_aggregate(_p(feat), _p(var), _p(ns), R, F, V, _p(of), _p(ot), max(R, 1),
                                _p(n_out))
    if rc:
        raise OracleError(rc, "aggregate")
    n = int(n_out[0])
    return of[:n].copy(), ot[:n].copy()


def distinct_pairs(feat: np.ndarray, var: np.ndarray) -> int:
    feat = _f32(feat)
    R, F = feat.shape
    var = np.ascontiguousarray(var, dtype=np.int32)
    return int(lib().oracle_distinct_pairs(_p(feat), _p(var), R, F))


def value_table(X: np.ndarray, f: int) -> np.ndarray:
    """Sorted distinct values of feature f (a2)."""
    X = _f32(X)
    n, F = X.shape
    vals = np.empty(max(n, 1), np.float32)
    cnt = np.zeros(1, np.int32)
    rc = lib().oracle_value_table(_p(X), n, F, f, _p(vals), vals.size, _p(cnt))
    if rc:
        raise OracleError(rc, "value_table")
    return vals[: int(cnt[0])].copy()


def bins(X: np.ndarray) -> np.ndarray:
    """Rank of each value in its feature's value table (a3), u8 [n][F]."""
    X = canon_features(X)
    n, F = X.shape
    out = np.empty((n, F), np.uint8)
    for f in range(F):
        out[:, f] = np.searchsorted(value_table(X, f), X[:, f]).astype(np.uint8)
    return out


def train(X: np.ndarray, y: np.ndarray, C: int, D: int, cap: int | None = None,
          omp: bool = False) -> np.ndarray:
    """Exact greedy CART, canonical BFS node array (structured NODE_DTYPE).
    omp=True: the all-cores build (same tree; bench timing only)."""
    X = _f32(X)
    n, F = X.shape
    y = np.ascontiguousarray(y, dtype=np.uint8)
    if cap is None:
        cap = int(min(2 * n + 1, (1 << (D + 1)) - 1 if D < 30 else 2 * n + 1))
    out = np.zeros(max(cap, 1), NODE_DTYPE)
    nn = np.zeros(1, np.int32)
    rc = lib(omp).oracle_train(_p(X), _p(y), n, F, C, D, _p(out), max(cap, 1), _p(nn))
    if rc:
        raise OracleError(rc, "train")
    return out[: int(nn[0])].copy()


def select(tree: np.ndarray, X: np.ndarray, omp: bool = False) -> np.ndarray:
    X = _f32(X)
    m, F = X.shape
    tree = np.ascontiguousarray(tree, dtype=NODE_DTYPE)
    out = np.empty(m, np.int32)
    rc = lib(omp).oracle_select(_p(tree), len(tree), _p(X), m, F, _p(out))
    if rc:
        raise OracleError(rc, "select")
    return out


def gini_counts(counts) -> float:
    c = np.ascontiguousarray(counts, dtype=np.int64)
    return float(lib().oracle_gini_counts(_p(c), c.size))


# ---- random forest ("rfc"; SPEC train_rfc / predict; R19-R21) ----
def bootstrap(seed: int, tree: int, n: int) -> np.ndarray:
    """Multiplicities of the size-n bootstrap resample of tree `tree` (R19)."""
    w = np.zeros(max(n, 1), np.uint32)
    rc = lib().oracle_bootstrap(ctypes.c_uint64(seed), int(tree), int(n), _p(w))
    if rc:
        raise OracleError(rc, "bootstrap")
    return w[:n]


def train_forest(X: np.ndarray, y: np.ndarray, V: int, D: int, T: int, seed: int) -> list:
    """Tree t = the plain CART (train) on the bootstrap resample of tree t:
    every row repeated w[i] times (SPEC train_rfc; no feature subsampling)."""
    trees = []
    for t in range(T):
        w = bootstrap(seed, t, len(X)).astype(np.int64)
        trees.append(train(np.repeat(X, w, axis=0), np.repeat(y, w), V, D))
    return trees


def select_forest(trees: list, X: np.ndarray) -> np.ndarray:
    """Majority vote of the trees' selections, ties -> lowest variant (R20)."""
    votes = np.stack([select(t, X) for t in trees])  # [T][m]
    out = np.empty(votes.shape[1], np.int32)
    for i in range(votes.shape[1]):
        labels, counts = np.unique(votes[:, i], return_counts=True)  # ascending labels
        out[i] = labels[np.argmax(counts)]  # first maximum = lowest label
    return out


# ---- K-fold harness (Adaptive-25/50/75; R22) ----
def kfold_pos(seed: int, shuffle: int, N: int, r: int) -> int:
    """Position of row r in shuffle `shuffle` (a permutation of range(N))."""
    return int(lib().oracle_kfold_pos(ctypes.c_uint64(seed), int(shuffle), ctypes.c_int64(N),
                                      ctypes.c_int64(r)))


def kfold_groups(seed: int, shuffle: int, N: int, K: int) -> np.ndarray:
    g = np.zeros(max(N, 1), np.int32)
    rc = lib().oracle_kfold_groups(ctypes.c_uint64(seed), int(shuffle), ctypes.c_int64(N), int(K), _p(g))
    if rc:
        raise OracleError(rc, "kfold_groups")
    return g[:N]


def kfold(X: np.ndarray, T: np.ndarray, D: int, K: int, m: int, shuffles: int, seed: int):
    """The paper's K-fold methodology on one wide table: per shuffle
    s and fold k, train the plain CART on the rows whose group is in
    {(k + j) mod K : j < m} (in row order) and test it on the other rows:
    n_correct = test rows whose selection is their label (the fastest
    variant), t_selected / t_best = the exactly rounded sums (math.fsum) of the
    test rows' times of the selected / the fastest variant.
    Returns (results: list of dicts in (s, k) order, trees: list)."""
    import math

    y = labels(T)
    N = len(X)
    res, trees = [], []
    for s in range(shuffles):
        g = kfold_groups(seed, s, N, K)
        for k in range(K):
            train_mask = np.isin(g, [(k + j) % K for j in range(m)])
            tree = train(X[train_mask], y[train_mask], T.shape[1], D)
            test = np.nonzero(~train_mask)[0]
            sel = select(tree, X[test])
            res.append({"shuffle": s, "fold": k, "n_nodes": len(tree), "n_train": int(train_mask.sum()),
                        "n_test": int(len(test)), "n_correct": int((sel == y[test]).sum()),
                        "t_selected": math.fsum(float(T[i, v]) for i, v in zip(test, sel)),
                        "t_best": math.fsum(float(T[i, y[i]]) for i in test)})
            trees.append(tree)
    return res, trees


# ---- lossy quantile bins for > 256 distinct values (R23) ----
def quantizer(X: np.ndarray, bins: int = 256):
    """Per feature with more than `bins` distinct values (global, -0 -> +0): the
    sorted distinct values u (np.unique as the sort primitive), bin b = distinct
    indices [floor(b D / bins), floor((b+1) D / bins)), lower bounds lb_b =
    u[e_b] and prev_b = u[e_b - 1] (the largest value of bin b-1, b >= 1).
    Returns {f: (lb, prev)}; features with <= bins values are absent (exact)."""
    Xc = canon_features(X)
    out = {}
    for f in range(Xc.shape[1]):
        u = np.unique(Xc[:, f])
        D = len(u)
        if D <= bins:
            continue
        e = (np.arange(bins, dtype=np.int64) * D) // bins
        prev = np.concatenate([[u[0]], u[e[1:] - 1]]).astype(np.float32)
        out[f] = (u[e].astype(np.float32), prev)
    return out


def quantize(X: np.ndarray, q: dict) -> np.ndarray:
    """x -> lb_{q(x)}, q(x) = #{b : lb_b <= x} - 1, on the quantised features."""
    Xq = canon_features(X).copy()
    for f, (lb, _) in q.items():
        Xq[:, f] = lb[np.searchsorted(lb, Xq[:, f], side="right") - 1]
    return Xq


def train_quantile(X: np.ndarray, y: np.ndarray, C: int, D: int, q: dict | None = None) -> np.ndarray:
    """R23: the exact CART (train) of the quantised table; a split of a quantised
    feature f between the node's bins a < b' then reports the raw threshold
    ((double)prev_{a+1} + (double)lb_{a+1}) / 2, a = the largest quantised value
    of the node's rows that goes left (rows routed through the tree by Xq).
    q: the quantiser (default: the one of X itself; the K-fold harness and
    forests train on subsets / resamples with the WHOLE table's quantiser)."""
    q = quantizer(X) if q is None else q
    Xq = quantize(X, q)
    tree = train(Xq, y, C, D)
    node_rows = {0: np.arange(len(X))}
    for k in range(len(tree)):
        rows = node_rows.pop(k, np.arange(0))
        f = int(tree["feature"][k])
        if f < 0:
            continue
        v = Xq[rows, f].astype(np.float64)
        go_left = v <= tree["threshold"][k]
        node_rows[int(tree["left"][k])] = rows[go_left]
        node_rows[int(tree["right"][k])] = rows[~go_left]
        if f in q:
            lb, prev = q[f]
            a = int(np.searchsorted(lb, v[go_left].max(), side="left"))  # lb[a] == that value
            tree["threshold"][k] = (float(prev[a + 1]) + float(lb[a + 1])) / 2
    return tree
