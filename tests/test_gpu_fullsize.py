"""Parity at BASELINE.json's full size (C4: 1e8 rows, 16 features, 48 variants,
depth 12) in the launch configuration bench.py times, on what can be checked
one by one or exactly from a small summary (tier rules ③):
  * labels of 20k sampled rows against the oracle (row-local definition);
  * every value table = the sorted distinct values of the feature (computed
    test-side), bins of sampled rows = ranks in it;
  * the ROOT split against an exact Fraction search over the full root
    histogram (built test-side from test-side labels and ranks);
  * every node's n = its children's sum, thresholds strictly inside the value
    gaps, and selections of sampled vectors against the oracle's tree walk.
Test-side reductions use torch on the GPU as plain library code; nothing here
reads the engine's intermediate buffers to build its expectations."""
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


def test_c4_full_size_sampled_parity():
    cfg = synth.CONFIGS["C4"]
    N, F, V = cfg.N, cfg.F, cfg.V
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
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(N, size=20_000, replace=False))
    ti = torch.from_numpy(idx).to(DEV)
    Xs, Ts = X[ti].cpu().numpy(), T[ti].cpu().numpy()
    # labels (row-local definition)
    labels = ad.adapt_get_labels(h, N)
    assert np.array_equal(labels[idx], oracle.labels(Ts))
    # value tables and sampled bins
    vals = []
    for f in range(F):
        u = torch.unique(torch.where(X[:, f] == 0, torch.zeros_like(X[:, f]), X[:, f])).cpu().numpy()
        got = ad.adapt_get_value_table(h, f)
        assert np.array_equal(got, u), f"value table {f}"
        vals.append(u)
    # test-side labels and ranks of every row -> the root histogram
    y = torch.argmin(T, dim=1)  # first minimum = lowest variant (R2)
    assert np.array_equal(y[ti].cpu().numpy(), labels[idx])
    H = []
    for f in range(F):
        u = torch.from_numpy(vals[f]).to(DEV)
        r = torch.searchsorted(u, X[:, f].contiguous())
        H.append(torch.bincount(r * V + y, minlength=len(vals[f]) * V).view(len(vals[f]), V)
                 .cpu().numpy().astype(np.int64))
    # sampled bins = ranks in the value tables
    got_bins = ad.adapt_get_bins(h, N, F)[idx]
    for f in range(F):
        assert np.array_equal(got_bins[:, f], np.searchsorted(vals[f], Xs[:, f]).astype(np.uint8)), f
    f_star, thr_star = _exact_root_split(H, vals)
    assert tree["feature"][0] == f_star and tree["threshold"][0] == thr_star
    assert tree["n"][0] == N
    counts = H[0].sum(0)
    assert tree["label"][0] == int(np.argmax(counts))
    # structure: n conserved, thresholds strictly inside value gaps
    for k in np.nonzero(tree["feature"] >= 0)[0]:
        l, r = tree["left"][k], tree["right"][k]
        assert tree["n"][l] + tree["n"][r] == tree["n"][k]
        vf = vals[tree["feature"][k]]
        t = tree["threshold"][k]
        j = np.searchsorted(vf.astype(np.float64), t)
        assert 0 < j < len(vf) and vf[j - 1] < t < vf[j]
    # selections of the sampled vectors: the oracle's walk of this tree
    out = torch.empty(N, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, X, N, out, s)
    torch.cuda.synchronize()
    assert np.array_equal(out[ti].cpu().numpy(), oracle.select(tree, Xs))
    ad.adapt_region_destroy(h)


def test_c5_full_size_sampled_selection():
    """C5 at full size, in bench.py's launch configuration: one adapt_select_batch
    over 1e9 C4-shaped vectors (seed 7; 64 GB) with (i) a depth-16 tree the
    engine trains on a 1e7-row C4-shaped table (seed 5) and (ii) the synthetic
    complete depth-16 tree (seed 6).  Sampled vectors (random + the ragged tail)
    against the oracle's walk of the same tree (R8: x <= thr -> left)."""
    import dataclasses

    cfg = dataclasses.replace(synth.CONFIGS["C4"], D=16)
    F, V = cfg.F, cfg.V
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    s = torch.cuda.current_stream()
    flat, off = cfg.grid_table
    g, o = torch.from_numpy(flat).to(DEV), torch.from_numpy(off).to(DEV)
    Nt = 10_000_000
    Xt = torch.empty((Nt, F), dtype=torch.float32, device=DEV)
    Tt = torch.empty((Nt, V), dtype=torch.float32, device=DEV)
    synth.generate_device(cfg, 0, Nt, Xt.data_ptr(), Tt.data_ptr(), g.data_ptr(), o.data_ptr(),
                          s.cuda_stream, seed=5)
    trained = ad.adapt_region_create("fullsize_c5_trained", F, V, "dtree,depth=16", 0)
    ad.adapt_record_table(trained, Xt, Tt, Nt, True, s)
    ad.adapt_train(trained, s)
    del Xt, Tt
    cols = synth.random_tree(cfg, 16, seed=6)
    ctree = np.zeros(len(cols["feature"]), oracle.NODE_DTYPE)
    for k, v in cols.items():
        ctree[k] = v
    complete = ad.adapt_region_create("fullsize_c5_complete", F, V, "dtree,depth=16", 0)
    ad.adapt_set_tree(complete, ctree)
    M = 1_000_000_000
    X = torch.empty((M, F), dtype=torch.float32, device=DEV)
    synth.generate_device(cfg, 0, M, X.data_ptr(), 0, g.data_ptr(), o.data_ptr(), s.cuda_stream, seed=7)
    out = torch.empty(M, dtype=torch.int32, device=DEV)
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.choice(M, size=100_000, replace=False),
                                    np.arange(M - 1000, M)]))
    ti = torch.from_numpy(idx).to(DEV)
    Xs = X[ti].cpu().numpy()
    # the device generator is the host one (test_synth_device_matches_host); spot-check here too
    Xh, _ = synth.generate(cfg, int(idx[0]), 1, seed=7)
    assert np.array_equal(Xh[0], Xs[0])
    for h in (trained, complete):
        tree = ad.adapt_get_tree(h)
        assert tree["depth"].max() <= 16
        out.fill_(-1)
        ad.adapt_select_batch(h, X, M, out, s)
        torch.cuda.synchronize()
        assert np.array_equal(out[ti].cpu().numpy(), oracle.select(tree, Xs))
        assert int((out < 0).sum()) == 0 and int((out >= V).sum()) == 0
    assert len(ad.adapt_get_tree(trained)) > 8191  # deeper than the shared-memory top
    ad.adapt_region_destroy(trained)
    ad.adapt_region_destroy(complete)
    del X, out
    torch.cuda.empty_cache()
