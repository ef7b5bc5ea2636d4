"""C3 train time (adapt_record_table + adapt_train per step, CUDA events) for A/B of engine env knobs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_08873_b200 as ad
import synth

torch.cuda.set_device(0)
ad.adapt_init(0, 0, 1)
cfg = synth.CONFIGS["C3"]
flat, off = cfg.grid_table
dev = torch.device("cuda:0")
g, o = torch.from_numpy(flat).to(dev), torch.from_numpy(off).to(dev)
X = torch.empty((cfg.N, cfg.F), dtype=torch.float32, device=dev)
T = torch.empty((cfg.N, cfg.V), dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
synth.generate_device(cfg, 0, cfg.N, X.data_ptr(), T.data_ptr(), g.data_ptr(), o.data_ptr(), s.cuda_stream)
h = ad.adapt_region_create("c3", cfg.F, cfg.V, f"dtree,depth={cfg.D}", 0)
def step():
    ad.adapt_record_table(h, X, T, cfg.N, True, s)
    ad.adapt_train(h, s)
for _ in range(5):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(20):
    step()
e1.record(s)
torch.cuda.synchronize()
print(os.environ.get("TAG", ""), "C3 train ms", round(e0.elapsed_time(e1) / 20, 3))
