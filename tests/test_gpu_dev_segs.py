"""Histogram segments built on the device vs on the host; two-level row moves
vs the per-level partition.

On one rank without weights the level loop plans every direct node's size from
its parent's winner record and lets `build_hist_segs_kernel` turn the
partition's share reports into the histogram segments (no host round trip
between the partition and the histogram pass; levels of 2^22 rows and more, or
any level with ADAPT_DEV_SEGS=1 as here).  ADAPT_HOST_SEGS=1 forces the
host-built segments (the path multi-rank and forest runs take).  Both must give
byte-identical trees: a single tree (C3, depth 12), a deep tree on random data
(ragged small nodes, the flat pass), and the multi-root frontier of
adapt_train_many (C2's three regions).

Two-level row moves (the default on one rank for tables of 2^24
rows and more; ADAPT_TWO_LEVEL=1 forces it at the sizes here): the TAG pass
marks the rows, the next level's histogram counts the marked rows from the
parents' pieces and MOVE4 moves them one level later.  ADAPT_ONE_LEVEL=1 keeps
a partition at every level, ADAPT_TAG_LAST=1 tags into the last frontier level
too; all schedules must give byte-identical trees, including shallow depths
where the schedule degenerates (depth 2: no TAG pass; depth 3: MOVE4 straight
into the last level)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2303_08873_b200 as ad, synth
torch.cuda.set_device(0)
ad.adapt_init(0, 0, 1)
out = []
keep = []
def tree(name, X, T, model):
    h = ad.adapt_region_create(name, X.shape[1], T.shape[1], model, 0)
    dX, dT = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
    keep.append((dX, dT))
    ad.adapt_record_table(h, dX, dT, len(X), True)
    ad.adapt_train(h)
    out.append(ad.adapt_get_tree(h).tobytes())
X, T = synth.generate("C3", 0, 300_000)
tree("c3", X, T, "dtree,depth=12")
rng = np.random.default_rng(5)
Xr = rng.integers(0, 40, size=(60_000, 6)).astype(np.float32)
Tr = rng.random((60_000, 9)).astype(np.float32)
tree("rnd", Xr, Tr, "dtree,depth=18")
for d in (2, 3, 4, 5):
    tree("rnd%d" % d, Xr[: 20_000 * d], Tr[: 20_000 * d], "dtree,depth=%d" % d)
# 1-3 features: bins rows of 1, 2 and 4 bytes (the single-plane layouts)
for F in (1, 2, 3):
    tree("f%d" % F, np.ascontiguousarray(Xr[:, :F]), Tr, "dtree,depth=9")
cfg = synth.CONFIGS["C2"]
X2, T2 = synth.generate(cfg, 0, cfg.N)
hs = []
for r in range(cfg.regions):
    rows = synth.region_rows(cfg, r)
    Xq, Tq = np.ascontiguousarray(X2[rows]), np.ascontiguousarray(T2[rows])
    h = ad.adapt_region_create("c2_%d" % r, cfg.F, cfg.V, "dtree,depth=%d" % cfg.D, 0)
    dX, dT = torch.from_numpy(Xq).cuda(), torch.from_numpy(Tq).cuda()
    keep.append((dX, dT))
    ad.adapt_record_table(h, dX, dT, len(rows), True)
    hs.append(h)
ad.adapt_train_many(hs)
for h in hs:
    out.append(ad.adapt_get_tree(h).tobytes())
np.save(sys.argv[2], np.frombuffer(b"|".join(out), np.uint8))
print("bytes", [len(o) for o in out])
"""


_runs = [0]


def _run(tmp_path, env_extra):
    _runs[0] += 1
    f = tmp_path / f"o{_runs[0]}.npy"
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(f)], check=True, env=env,
                       timeout=600, capture_output=True, text=True)
    return np.load(f).tobytes(), p.stdout


def test_device_built_segments_match_host_built(tmp_path):
    dev, log_d = _run(tmp_path, {"ADAPT_DEV_SEGS": "1"})
    host, log_h = _run(tmp_path, {"ADAPT_HOST_SEGS": "1"})
    assert len(dev) > 1000, log_d
    assert dev == host, (log_d, log_h)


def test_two_level_moves_match_one_level(tmp_path):
    two, log_t = _run(tmp_path, {"ADAPT_TWO_LEVEL": "1"})
    one, log_o = _run(tmp_path, {"ADAPT_ONE_LEVEL": "1"})
    tag_last, log_l = _run(tmp_path, {"ADAPT_TWO_LEVEL": "1", "ADAPT_TAG_LAST": "1"})
    # the histogram segments after each MOVE4 built on the device
    two_dev, log_d = _run(tmp_path, {"ADAPT_TWO_LEVEL": "1", "ADAPT_DEV_SEGS": "1"})
    assert len(two) > 1000, log_t
    assert two == one, (log_t, log_o)
    assert two == tag_last, (log_t, log_l)
    assert two == two_dev, (log_t, log_d)
