"""Expected outputs at BASELINE.json's full sizes, written by the ORACLE only.

Calls nothing but ``oracle/`` (the plain CPU oracle) and ``synth/`` (the seeded
input recipe); never the CUDA path.  Runs on the CPU container (tens of minutes
single-threaded per config) and commits small files under
``tests/golden/fullsize/`` that ``tests/test_gpu_fullsize.py`` compares the GPU
outputs against (whole trees byte for byte, SHA-256 of every 1e7-row chunk of
labels / bins / selections).

  c4  : C4 = 1e8 rows, F=16, V=48, seed 4, depth 12 (SURVEY §8(a) sizes table):
        labels, value tables, bins, the depth-12 tree, oracle.select of the
        1e8 training vectors with that tree.
  c5t : the C5 training table, 1e7 C4-shaped rows, seed 5, depth 16: the tree.
  c5s : C5 = 1e9 C4-shaped vectors, seed 7: oracle.select with the c5t tree and
        with the synthetic complete depth-16 tree (seed 6), hashed per 1e8.

Every file carries ``oracle_sha`` = SHA-256 of the oracle's C source and the
input generator (oracle.c, oracle.h, synth/__init__.py); the test refuses a stale file (re-run this script after any change
there, and name the justifying passage in the commit, tier rule ③)."""
from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize")
CHUNK = 10_000_000
OMP_NOTE = ("liboracle_omp.so: oracle.c built with -fopenmp (features of a node / vectors in "
            "parallel); byte-identical to the plain build (tests/test_oracle.py::"
            "test_openmp_build_is_identical)")


def source_sha() -> str:
    h = hashlib.sha256()
    for p in ("oracle/oracle.c", "oracle/oracle.h", "synth/__init__.py"):
        with open(os.path.join(ROOT, p), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def log(msg: str) -> None:
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def c4() -> None:
    cfg = synth.CONFIGS["C4"]
    N, F, V, D = cfg.N, cfg.F, cfg.V, cfg.D
    X = np.empty((N, F), np.float32)
    y = np.empty(N, np.uint8)
    t0 = time.time()
    for r0 in range(0, N, CHUNK):
        Xc, Tc = synth.generate(cfg, r0, min(CHUNK, N - r0))
        X[r0:r0 + len(Xc)] = Xc
        y[r0:r0 + len(Xc)] = oracle.labels(Tc)
        log(f"c4 rows {r0 + len(Xc)}")
    t_lab = time.time() - t0
    vals = [oracle.value_table(X, f) for f in range(F)]
    log("c4 value tables")
    bins_sha = []
    for r0 in range(0, N, CHUNK):
        Xc = oracle.canon_features(X[r0:r0 + CHUNK])
        b = np.empty(Xc.shape, np.uint8)
        for f in range(F):
            b[:, f] = np.searchsorted(vals[f], Xc[:, f])
        bins_sha.append(sha(b))
    log("c4 bins")
    t0 = time.time()
    tree = oracle.train(X, y, V, D, omp=True)
    t_train = time.time() - t0
    log(f"c4 tree {len(tree)} nodes in {t_train:.0f} s")
    t0 = time.time()
    sel_sha = [sha(oracle.select(tree, X[r0:r0 + CHUNK], omp=True)) for r0 in range(0, N, CHUNK)]
    t_sel = time.time() - t0
    np.savez_compressed(os.path.join(OUT, "c4_tree.npz"), tree=tree)
    meta = dict(config="C4", N=N, F=F, V=V, D=D, seed=cfg.seed, chunk=CHUNK,
                oracle_sha=source_sha(), tree_sha=sha(tree), n_nodes=len(tree),
                labels_sha=[sha(y[r0:r0 + CHUNK]) for r0 in range(0, N, CHUNK)],
                bins_sha=bins_sha, select_sha=sel_sha,
                value_tables_sha=[sha(v) for v in vals],
                label_counts=np.bincount(y, minlength=V).tolist(),
                oracle_seconds=dict(generate_and_label=round(t_lab, 1), train=round(t_train, 1),
                                    select=round(t_sel, 1), threads=os.cpu_count(), build=OMP_NOTE))
    with open(os.path.join(OUT, "c4.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    log("c4 done")


def c5_cfg():
    return dataclasses.replace(synth.CONFIGS["C4"], D=16)


def c5t() -> None:
    cfg = c5_cfg()
    Nt = 10_000_000
    X, T = synth.generate(cfg, 0, Nt, seed=5)
    y = oracle.labels(T)
    del T
    t0 = time.time()
    tree = oracle.train(X, y, cfg.V, 16, omp=True)
    t_train = time.time() - t0
    np.savez_compressed(os.path.join(OUT, "c5_trained_tree.npz"), tree=tree)
    meta = dict(config="C5 training table", N=Nt, F=cfg.F, V=cfg.V, D=16, seed=5,
                oracle_sha=source_sha(), tree_sha=sha(tree), n_nodes=len(tree),
                labels_sha=sha(y), oracle_seconds=dict(train=round(t_train, 1), threads=os.cpu_count(), build=OMP_NOTE))
    with open(os.path.join(OUT, "c5_trained.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    log(f"c5t tree {len(tree)} nodes in {t_train:.0f} s")


def complete_tree(cfg) -> np.ndarray:
    cols = synth.random_tree(cfg, 16, seed=6)
    t = np.zeros(len(cols["feature"]), oracle.NODE_DTYPE)
    for k, v in cols.items():
        t[k] = v
    return t


def c5s() -> None:
    cfg = c5_cfg()
    trained = np.load(os.path.join(OUT, "c5_trained_tree.npz"))["tree"]
    complete = complete_tree(cfg)
    M = 1_000_000_000
    ch = 100_000_000
    res = {"trained": [], "complete": []}
    t_sel = 0.0
    for r0 in range(0, M, ch):
        parts = []
        for s0 in range(r0, r0 + ch, CHUNK):
            parts.append(synth.generate(cfg, s0, CHUNK, seed=7, times=False)[0])
        X = np.concatenate(parts)
        del parts
        t0 = time.time()
        res["trained"].append(sha(oracle.select(trained, X, omp=True)))
        res["complete"].append(sha(oracle.select(complete, X, omp=True)))
        t_sel += time.time() - t0
        log(f"c5s vectors {r0 + ch}")
    meta = dict(config="C5", M=M, F=cfg.F, seed=7, chunk=ch, oracle_sha=source_sha(),
                trained_tree_sha=sha(trained), complete_tree_sha=sha(complete),
                select_sha=res, oracle_seconds=dict(select_both_trees=round(t_sel, 1), threads=os.cpu_count(), build=OMP_NOTE))
    with open(os.path.join(OUT, "c5_select.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    log("c5s done")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for what in sys.argv[1:]:
        {"c4": c4, "c5t": c5t, "c5s": c5s}[what]()
