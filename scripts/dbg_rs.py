import os, sys, subprocess, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2303_08873_b200 as ad, synth
torch.cuda.set_device(0)
ad.adapt_init(0, 0, 1)
X, T = synth.generate("C3", 0, 100_000)
res = {}
for name, model in (("tree", "dtree,depth=10"), ("forest", "rfc,3,5,seed=1"), ("tree5", "dtree,depth=5")):
    h = ad.adapt_region_create(name, 8, 6, model, 0)
    ad.adapt_record_table(h, torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda(), len(X), True)
    ad.adapt_train(h)
    res[name] = [ad.adapt_get_forest_tree(h, t) for t in range(ad.adapt_forest_size(h))]
np.save(sys.argv[2], np.array([res], dtype=object), allow_pickle=True)
"""
outs = {}
for tag, env in (("plain", {}), ("rs", {"ADAPT_NCCL_SELF": "1", "ADAPT_HIST_COMM": "rs"}), ("ar", {"ADAPT_NCCL_SELF": "1"})):
    f = f"/tmp/dbg_{tag}.npy"
    subprocess.run([sys.executable, "-c", CHILD, ROOT, f], check=True, env=dict(os.environ, **env))
    outs[tag] = np.load(f, allow_pickle=True)[0]
for tag in ("rs", "ar"):
    for name in outs["plain"]:
        for t, (a, b) in enumerate(zip(outs["plain"][name], outs[tag][name])):
            if a.tobytes() != b.tobytes():
                n = min(len(a), len(b))
                bad = [i for i in range(n) if a[i].tobytes() != b[i].tobytes()]
                print(tag, name, "tree", t, "nodes", len(a), len(b), "first diff", bad[:3], a[bad[0]] if bad else None, b[bad[0]] if bad else None)
            else:
                print(tag, name, "tree", t, "ok", len(a))
