"""K-fold harness timing breakdown (profiling aid; not part of the product)."""
import sys, time
import torch
sys.path.insert(0, ".")
import synth
import paper_2303_08873_b200 as ad

ad.adapt_init(0, 0, 1)
dev = torch.device("cuda:0")
s = torch.cuda.current_stream()
for name, rows in (("C1", 512), ("C3", 1_000_000)):
    cfg = synth.CONFIGS[name]
    X, T = synth.generate(cfg, 0, rows)
    dX, dT = torch.from_numpy(X).to(dev), torch.from_numpy(T).to(dev)
    h = ad.adapt_region_create(f"kp{name}", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)
    for m in (1, 3):
        for it in range(2):
            ad.adapt_profile_reset(); ad.adapt_profile_enable(True)
            ad.adapt_record_table(h, dX, dT, rows, True, s)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            ad.adapt_kfold(h, 4, m, 10, 1, s)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            ad.adapt_profile_enable(False)
        prof = ad.adapt_profile_get()
        tot = sum(v["ms"] for v in prof.values())
        print(name, "m", m, "wall ms %.1f" % (dt * 1e3), "gpu phases ms %.1f" % tot,
              {k: round(v["ms"], 2) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])[:8]})
