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
