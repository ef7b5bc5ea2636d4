"""C1 small-path timing (profiling aid): kernel time vs adapt_train wall time."""
import sys, time
import torch
sys.path.insert(0, ".")
import synth
import paper_2303_08873_b200 as ad

ad.adapt_init(0, 0, 1)
cfg = synth.CONFIGS["C1"]
X, T = synth.generate(cfg, 0, cfg.N)
dX, dT = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
s = torch.cuda.current_stream()
h = ad.adapt_region_create("sp", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)
for it in range(30):
    ad.adapt_record_table(h, dX, dT, cfg.N, True, s)
    if it == 20:
        ad.adapt_profile_reset(); ad.adapt_profile_enable(True)
    t0 = time.perf_counter(); ad.adapt_train(h, s); dt = time.perf_counter() - t0
ad.adapt_profile_enable(False)
print("wall us", dt * 1e6, {k: (v["launches"], round(v["ms"] * 1e3 / max(v["launches"], 1), 1)) for k, v in ad.adapt_profile_get().items()})
