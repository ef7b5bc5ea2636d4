"""Independent exact checker for the oracle (pins, not a second oracle).

Pure Python, exact rational arithmetic (``fractions.Fraction``), brute force.
It shares no code with ``oracle/`` and uses a different formulation on
purpose: the oracle maximises the score SL/nL + SR/nR (sum of squared class
counts over child size) by sort-and-scan, comparing rationals by quotient and
remainder; this checker re-partitions the rows for every midpoint and
minimises the weighted child Gini as Fractions.  The two agree by the identity
weighted_gini = 1 - score/n, so a transposed operand, a dropped term or a
wrong index in either shows up as a disagreement.

Only for tiny inputs (it is O(n^2 F) per node).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction


def labels_exact(times):
    """Fastest variant per row; +inf = unmeasured; ties -> lowest (R2, R3)."""
    out = []
    for row in times:
        vals = [float(t) for t in row]
        if any(math.isnan(v) for v in vals):
            raise ValueError("NaN time")
        finite = [(v, i) for i, v in enumerate(vals) if not (math.isinf(v) and v > 0)]
        if not finite:
            raise ValueError("all unmeasured")
        out.append(min(finite)[1])  # tuple order: smallest value, then smallest index
    return out


def gini(counts) -> Fraction:
    n = sum(counts)
    if n == 0:
        return Fraction(0)
    return 1 - sum(Fraction(c * c, n * n) for c in counts)


def _counts(ys, C):
    c = [0] * C
    for y in ys:
        c[y] += 1
    return c


def best_split(X, y, rows, C):
    """All (f, node-local midpoint) candidates; min weighted Gini; ties lowest f, thr.
    Zero-gain candidates compete too (R10); None only if no cut exists."""
    n = len(rows)
    best = None
    F = len(X[0])
    for f in range(F):
        vals = sorted({Fraction(float(X[i][f])) for i in rows})
        for a, b in zip(vals, vals[1:]):
            thr = (a + b) / 2
            L = [i for i in rows if Fraction(float(X[i][f])) <= thr]
            R = [i for i in rows if Fraction(float(X[i][f])) > thr]
            w = (len(L) * gini(_counts([y[i] for i in L], C))
                 + len(R) * gini(_counts([y[i] for i in R], C))) / n
            key = (w, f, thr)
            if best is None or key < best[0]:
                best = (key, f, thr, L, R)
    return best


def majority(ys, C):
    c = _counts(ys, C)
    m = max(c)
    return c.index(m)


def cart_exact(X, y, C, D):
    """Greedy CART in BFS order.  Returns list of dicts with exact Fraction thresholds."""
    nodes = [{"rows": list(range(len(y))), "depth": 0}]
    k = 0
    while k < len(nodes):
        nd = nodes[k]
        rows = nd.pop("rows")
        ys = [y[i] for i in rows]
        nd.update(n=len(rows), label=majority(ys, C), gini=gini(_counts(ys, C)),
                  feature=-1, left=-1, right=-1, threshold=None)
        if nd["depth"] < D and len(set(ys)) > 1:
            b = best_split(X, y, rows, C)
            if b is not None:
                _, f, thr, L, R = b
                nd.update(feature=f, threshold=thr, left=len(nodes), right=len(nodes) + 1)
                nodes.append({"rows": L, "depth": nd["depth"] + 1})
                nodes.append({"rows": R, "depth": nd["depth"] + 1})
        k += 1
    return nodes


def predict_exact(nodes, x):
    k = 0
    while nodes[k]["feature"] >= 0:
        v = float(x[nodes[k]["feature"]])
        if math.isnan(v):
            k = nodes[k]["right"]
            continue
        k = nodes[k]["left"] if Fraction(v) <= nodes[k]["threshold"] else nodes[k]["right"]
    return nodes[k]["label"]


def exhaustive_best_accuracy(x1d, y, C, D):
    """Best training accuracy (count of correct rows) over ALL threshold trees of
    depth <= D on one feature (leaves labelled by majority).  Tiny inputs only."""
    vals = sorted(set(x1d))
    cuts = [(a + b) / 2 for a, b in zip(vals, vals[1:])]

    def best(rows, d):
        ys = [y[i] for i in rows]
        if not rows:
            return 0
        leaf = max(_counts(ys, C))
        if d == 0:
            return leaf
        acc = leaf
        for t in cuts:
            L = [i for i in rows if x1d[i] <= t]
            R = [i for i in rows if x1d[i] > t]
            if L and R:
                acc = max(acc, best(L, d - 1) + best(R, d - 1))
        return acc

    return best(list(range(len(y))), D)


def all_label_tuples(n, C):
    return itertools.product(range(C), repeat=n)
