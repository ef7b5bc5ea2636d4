"""GPU random forests ("rfc"): every tree
bit-identical to the oracle's CART on the same bootstrap resample (R19), the
batched majority vote identical to the oracle's (R20), on seeded tables."""
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
_uid = [0]


@pytest.fixture(scope="module", autouse=True)
def _init():
    torch.cuda.set_device(DEV)
    ad.adapt_init(0, 0, 1)
    yield


def _forest(X, T, params, on_device=True):
    _uid[0] += 1
    n, F = X.shape
    h = ad.adapt_region_create(f"rf{_uid[0]}", F, T.shape[1], params, 0)
    if on_device:
        ad.adapt_record_table(h, torch.from_numpy(X).to(DEV), torch.from_numpy(T).to(DEV), n, True)
    else:
        ad.adapt_record_table(h, X, T, n, False)
    ad.adapt_train(h)
    return h


def _assert_tree(got, ref, t):
    assert len(got) == len(ref), f"tree {t}: {len(got)} nodes vs {len(ref)}"
    for k in ("feature", "left", "right", "label", "depth", "n"):
        assert np.array_equal(got[k], ref[k]), f"tree {t}: {k}"
    assert got["threshold"].tobytes() == ref["threshold"].tobytes(), f"tree {t}: thresholds"
    np.testing.assert_allclose(got["gini"], ref["gini"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("cfg,rows,T,D,seed", [("C3", 30_011, 5, 6, 7), ("C2", 20_000, 3, 8, 0),
                                               ("C1", 512, 8, 4, 123), ("C4", 8_000, 2, 5, 99)])
def test_forest_matches_oracle(cfg, rows, T, D, seed):
    X, Tm = synth.generate(cfg, 0, rows)
    h = _forest(X, Tm, f"rfc,trees={T},depth={D},seed={seed}")
    assert ad.adapt_forest_size(h) == T
    y = oracle.labels(Tm)
    ref = oracle.train_forest(X, y, Tm.shape[1], D, T, seed)
    for t in range(T):
        _assert_tree(ad.adapt_get_forest_tree(h, t), ref[t], t)
    out = torch.empty(rows, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), rows, out)
    torch.cuda.synchronize()
    expect = oracle.select_forest(ref, X)
    assert np.array_equal(out.cpu().numpy(), expect), "forest votes differ"
    for i in range(0, rows, max(1, rows // 40)):  # Table-1 get_policy: host vote
        assert ad.adapt_select(h, X[i]) == expect[i]


def test_forest_params_and_degenerate_cases():
    X, Tm = synth.generate("C1", 0, 1)
    h = _forest(X, Tm, "rfc(3,2)", on_device=False)  # n = 1: every resample is the row
    assert ad.adapt_forest_size(h) == 3
    for t in range(3):
        assert len(ad.adapt_get_forest_tree(h, t)) == 1
    X, Tm = synth.generate("C3", 0, 2000)
    Tm = Tm.copy()
    Tm[:, 2] = 0.0  # variant 2 always fastest: single-label data
    h = _forest(X, Tm, "RandomForest")  # defaults: 10 trees of depth 2
    assert ad.adapt_forest_size(h) == 10
    out = torch.empty(2000, dtype=torch.int32, device=DEV)
    ad.adapt_select_batch(h, torch.from_numpy(X).to(DEV), 2000, out)
    torch.cuda.synchronize()
    assert np.all(out.cpu().numpy() == 2)
    for bad in ("rfc,trees=0", "rfc,trees=65", "rfc,3,99", "gbt"):
        with pytest.raises(ad.AdaptError) as e:
            ad.adapt_region_create("rf_bad", 2, 2, bad, 0)
        assert e.value.code == ad.ADAPT_E_INVALID_ARG
    ad.adapt_region_create("rf_spec", 2, 2, "rfc,2,2,seed=1", 0)
    with pytest.raises(ad.AdaptError) as e:
        ad.adapt_region_create("rf_spec", 2, 2, "rfc,2,2,seed=2", 0)
    assert e.value.code == ad.ADAPT_E_SPEC_MISMATCH


def test_forest_is_deterministic():
    X, Tm = synth.generate("C3", 0, 5000)
    a = _forest(X, Tm, "rfc,4,5,seed=3")
    b = _forest(X, Tm, "rfc,4,5,seed=3")
    for t in range(4):
        assert ad.adapt_get_forest_tree(a, t).tobytes() == ad.adapt_get_forest_tree(b, t).tobytes()
