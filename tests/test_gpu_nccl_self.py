"""The NCCL transport on one GPU: with ADAPT_NCCL_SELF=1 a world-1 run gets a
1-rank NCCL communicator, so every collective of the training path (value-table
all-gather, histogram / flag / row-count all-reduces, the forest's row-offset
all-gather; with ADAPT_HIST_COMM=rs the histogram reduce-scatter and the winner
all-gather) is a real NCCL call; results must equal the plain run's and the
oracle's.  (Multi-rank NCCL itself needs several GPUs; the multi-rank logic is
tested through the host-staged hooks in test_gpu_multirank.py.)"""
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
X, T = synth.generate("C3", 0, 100_000)
out = {}
for name, model in (("tree", "dtree,depth=10"), ("forest", "rfc,3,5,seed=1")):
    h = ad.adapt_region_create(name, 8, 6, model, 0)
    ad.adapt_record_table(h, torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda(), len(X), True)
    ad.adapt_train(h)
    out[name] = b"".join(ad.adapt_get_forest_tree(h, t).tobytes() for t in range(ad.adapt_forest_size(h)))
np.save(sys.argv[2], np.frombuffer(out["tree"] + b"|" + out["forest"], np.uint8))
"""


def _run(tmp_path, env_extra):
    f = tmp_path / f"o{len(env_extra)}.npy"
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(f)], check=True, env=env,
                       timeout=600, capture_output=True, text=True)
    return np.load(f).tobytes(), p.stdout + p.stderr


def test_nccl_self_communicator_matches_plain_run(tmp_path):
    plain, _ = _run(tmp_path, {})
    nccl, log = _run(tmp_path, {"ADAPT_NCCL_SELF": "1", "NCCL_DEBUG": "INFO"})
    assert "NCCL INFO" in log, "no NCCL communicator was created"
    assert plain == nccl
    # the reduce-scatter exchange (the default with more than one rank) forced
    # on the 1-rank communicator: ncclReduceScatter of the padded owner ranges
    # and ncclAllGather of the winner records are real NCCL calls
    rs, log = _run(tmp_path, {"ADAPT_NCCL_SELF": "1", "ADAPT_HIST_COMM": "rs", "NCCL_DEBUG": "INFO"})
    assert "NCCL INFO" in log
    assert plain == rs
