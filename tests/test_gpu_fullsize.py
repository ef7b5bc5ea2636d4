"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (tier rules ③), against expected outputs the ORACLE wrote
(scripts/oracle_fullsize.py, committed under tests/golden/fullsize/, keyed by
the SHA-256 of the oracle's C source and the input generator):
  * C4 (1e8 rows, 16 features, 48 variants, depth 12, seed 4): the whole
    8191-node tree byte for byte; labels, bins and the selections of all 1e8
    training vectors by SHA-256 of every 1e7-row chunk; every value table;
  * C5: the depth-16 tree the engine trains on the 1e7-row C5 training table
    (seed 5) byte for byte, and the selections of all 1e9 vectors (seed 7) by
    that tree and by the synthetic complete depth-16 tree (seed 6), SHA-256 per
    1e8-vector chunk.
Independently of the oracle, the C4 root split is also checked against an
exact Fraction search over the full root histogram (built test-side)."""
import hashlib
import json
import os
from fractions import Fraction

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
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "fullsize")


def _source_sha() -> str:  # as scripts/oracle_fullsize.py computes it
    h = hashlib.sha256()
    for p in ("oracle/oracle.c", "oracle/oracle.h", "synth/__init__.py"):
        with open(os.path.join(ROOT, p), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _golden(name: str) -> dict:
    with open(os.path.join(GOLD, name)) as fh:
        meta = json.load(fh)
    assert meta["oracle_sha"] == _source_sha(), \
        f"{name} is stale: re-run scripts/oracle_fullsize.py after the oracle/generator change"
    return meta


def _tree(name: str) -> np.ndarray:
    return np.load(os.path.join(GOLD, name))["tree"]


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _exact_root_split(H, vals):
    """H[f] = int64 [D_f][C] counts. Best cut by R10/R13x/R9: max SL/nL + SR/nR
    over cuts between consecutive nonempty bins, ties -> lowest f, lowest thr."""
    best = None
    for f, Hf in enumerate(H):
        tot = Hf.sum(0)
        n = int(tot.sum())
        nonempty = np.nonzero(Hf.sum(1))[0]
        cl = np.zeros(Hf.shape[1], np.int64)
        prev = None
        cum = np.cumsum(Hf, 0)
        for b in nonempty:
            if prev is not None:
                left = cum[prev]
                nl = int(left.sum())
                right = tot - left
                nr = n - nl
                score = Fraction(int((left.astype(object) ** 2).sum()), nl) + \
                    Fraction(int((right.astype(object) ** 2).sum()), nr)
                thr = (float(vals[f][prev]) + float(vals[f][b])) / 2
                key = (score, -f, -thr)
                if best is None or key > best[0]:
                    best = (key, f, thr)
            prev = b
    return best[1], best[2]


def test_c4_full_size_parity():
    cfg = synth.CONFIGS["C4"]
    N, F, V = cfg.N, cfg.F, cfg.V
    meta = _golden("c4.json")
    ref = _tree("c4_tree.npz")
    assert meta["N"] == N and meta["D"] == cfg.D and _sha(ref) == meta["tree_sha"]
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(DEV), torch.from_numpy(off).to(DEV)
    X = torch.empty((N, F), dtype=torch.float32, device=DEV)
    T = torch.empty((N, V), dtype=torch.float32, device=DEV)
    s = torch.cuda.current_stream()
    synth.generate_device(cfg, 0, N, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(),
                          s.cuda_stream)
    h = ad.adapt_region_create("fullsize_c4", F, V, f"dtree,depth={cfg.D}", 0)
    ad.adapt_record_table(h, X, T, N, True, s)
    ad.adapt_train(h, s)
    tree = ad.adapt_get_tree(h)
    # the whole tree, byte for byte (topology, features, thresholds, labels, n, gini)
    assert tree.tobytes() == ref.tobytes(), "C4 tree differs from the oracle's"
    ch = meta["chunk"]
    labels = ad.adapt_get_labels(h, N)
    assert [_sha(labels[r:r + ch]) for r in range(0, N, ch)] == meta["labels_sha"], "labels differ"
    assert np.bincount(labels, minlength=V).tolist() == meta["label_counts"]
    vals = [ad.adapt_get_value_table(h, f) for f in range(F)]
    assert [_sha(v) for v in vals] == meta["value_tables_sha"], "value tables differ"
    bins = ad.adapt_get_bins(h, N, F)
    assert [_sha(bins[r:r + ch]) for r in range(0, N, ch)] == meta["bins_sha"], "bins differ"
    del bins
    out = torch.empty(N, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, X, N, out, s)
    torch.cuda.synchronize()
    sel = out.cpu().numpy()
    assert [_sha(sel[r:r + ch]) for r in range(0, N, ch)] == meta["select_sha"], "selections differ"
    # independent of the oracle: the root split by exact Fractions over the
    # full root histogram, built test-side (torch as library code)
    y = torch.argmin(T, dim=1)  # first minimum = lowest variant (R2)
    H = []
    for f in range(F):
        u = torch.from_numpy(vals[f]).to(DEV)
        r = torch.searchsorted(u, X[:, f].contiguous())
        H.append(torch.bincount(r * V + y, minlength=len(vals[f]) * V).view(len(vals[f]), V)
                 .cpu().numpy().astype(np.int64))
    f_star, thr_star = _exact_root_split(H, vals)
    assert tree["feature"][0] == f_star and tree["threshold"][0] == thr_star
    ad.adapt_region_destroy(h)
    del X, T, out
    torch.cuda.empty_cache()


def test_c5_full_size_parity():
    """C5 at full size, in bench.py's launch configuration: the engine trains the
    depth-16 tree on the 1e7-row C5 training table (seed 5) — byte-identical to
    the oracle's — and one adapt_select_batch per tree walks all 1e9 C4-shaped
    vectors (seed 7; 64 GB); every 1e8-vector chunk of selections hashes to the
    oracle's, for that tree and for the synthetic complete depth-16 tree."""
    import dataclasses

    meta_t = _golden("c5_trained.json")
    meta_s = _golden("c5_select.json")
    ref_trained = _tree("c5_trained_tree.npz")
    assert _sha(ref_trained) == meta_t["tree_sha"] == meta_s["trained_tree_sha"]
    cfg = dataclasses.replace(synth.CONFIGS["C4"], D=16)
    F, V = cfg.F, cfg.V
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    s = torch.cuda.current_stream()
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(DEV), torch.from_numpy(off).to(DEV)
    Nt = meta_t["N"]
    Xt = torch.empty((Nt, F), dtype=torch.float32, device=DEV)
    Tt = torch.empty((Nt, V), dtype=torch.float32, device=DEV)
    synth.generate_device(cfg, 0, Nt, Xt.data_ptr(), Tt.data_ptr(), g.data_ptr(), o.data_ptr(),
                          s.cuda_stream, seed=5)
    trained = ad.adapt_region_create("fullsize_c5_trained", F, V, "dtree,depth=16", 0)
    ad.adapt_record_table(trained, Xt, Tt, Nt, True, s)
    ad.adapt_train(trained, s)
    assert _sha(ad.adapt_get_labels(trained, Nt)) == meta_t["labels_sha"]
    got = ad.adapt_get_tree(trained)
    assert got.tobytes() == ref_trained.tobytes(), "C5 training tree differs from the oracle's"
    del Xt, Tt
    cols = synth.random_tree(cfg, 16, seed=6)
    ctree = np.zeros(len(cols["feature"]), oracle.NODE_DTYPE)
    for k, v in cols.items():
        ctree[k] = v
    assert _sha(ctree) == meta_s["complete_tree_sha"]
    complete = ad.adapt_region_create("fullsize_c5_complete", F, V, "dtree,depth=16", 0)
    ad.adapt_set_tree(complete, ctree)
    M = meta_s["M"]
    ch = meta_s["chunk"]
    X = torch.empty((M, F), dtype=torch.float32, device=DEV)
    synth.generate_device(cfg, 0, M, X.data_ptr(), 0, g.data_ptr(), o.data_ptr(), s.cuda_stream, seed=7)
    out = torch.empty(M, dtype=torch.int32, device=DEV)
    for name, h in (("trained", trained), ("complete", complete)):
        out.fill_(-1)
        ad.adapt_select_batch(h, X, M, out, s)
        torch.cuda.synchronize()
        sel = out.cpu().numpy()
        assert [_sha(sel[r:r + ch]) for r in range(0, M, ch)] == meta_s["select_sha"][name], \
            f"C5 selections ({name} tree) differ from the oracle's"
    assert len(got) > 8191  # deeper than the shared-memory top
    ad.adapt_region_destroy(trained)
    ad.adapt_region_destroy(complete)
    del X, out
    torch.cuda.empty_cache()
