mkdir -p gpurun_out
timeout 600 python scripts/kfold_prof.py > gpurun_out/kfold_prof.log 2>&1; echo rc=$?; cat gpurun_out/kfold_prof.log | tail -5
ADAPT_TRACE_HOST=3 timeout 600 python - > gpurun_out/kfold_trace.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, ".")
import synth, paper_2303_08873_b200 as ad
ad.adapt_init(0, 0, 1)
cfg = synth.CONFIGS["C3"]
X, T = synth.generate(cfg, 0, 1_000_000)
dX, dT = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
h = ad.adapt_region_create("kt", cfg.F, cfg.V, "dtree,depth=12", 0)
s = torch.cuda.current_stream()
for it in range(2):
    ad.adapt_record_table(h, dX, dT, len(X), True, s)
    ad.adapt_kfold(h, 4, 2, 10, 1, s)
PY
grep -n "host:\|cudaMalloc" gpurun_out/kfold_trace.log | tail -60
