"""Summarise a round's ncu evidence into profiles/: per-kernel share of one
bench step from the launch list (gpu__time_duration.sum, --clock-control none)
and the key counters of each `ncu --set full` capture.

    python scripts/profile_summary.py ROUND gpurun_out/launches.csv gpurun_out/prof_*.ncu-rep
"""
import collections
import csv
import re
import subprocess
import sys

import json
import os

rnd, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
PHASE = {"partition_kernel": "partition", "partition4_kernel": "partition", "tag_kernel": "tag",
         "hist_kernel": "hist", "label_bin_kernel": "ingest",
         "discover_kernel": "discover", "select_kernel_c": "select", "select_kernel_h": "select",
         "split_kernel": "split"}
traffic = {}
out = [f"# Round {rnd} ncu summary", ""]

# ---- launch list: one bench step (steps=1, warmup=0), engine kernels only ----
rows = [r for r in csv.reader(l for l in open(launches) if l.startswith('"'))][1:]
per = collections.OrderedDict()
for r in rows:
    name = re.sub(r"^(<unnamed>|adapt)::", "", r[4]).split("(")[0]
    name = re.sub(r"<.*>", "", name.split("::")[-1])
    if name == "gen_kernel":  # synthetic-input generator (not timed by bench.py)
        continue
    ns = float(r[14])
    d = per.setdefault(name, [0, 0.0])
    d[0] += 1
    d[1] += ns / 1e6
# bench.py runs the timed step and then a separately profiled step (per-phase
# events): the list holds whole steps, one ingest launch each
nst = max(1, per.get("label_bin_kernel", [1, 0])[0])
for v in per.values():
    v[0] /= nst
    v[1] /= nst
tot = sum(v[1] for v in per.values())
out += ["## Launch list (per step, serialised, cold-cache)", "",
        f"Source: `{launches}` — `ncu --metrics gpu__time_duration.sum --clock-control none "
        "python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy` "
        f"({nst} steps in the list: the timed step and bench.py's profiled step; figures per step).", "",
        "| kernel | launches | ms | share of step |", "|---|---:|---:|---:|"]
for k, (n, ms) in sorted(per.items(), key=lambda x: -x[1][1]):
    out.append(f"| {k} | {n:g} | {ms:.3f} | {100 * ms / tot:.1f}% |")
out += [f"| **total** | {sum(v[0] for v in per.values()):g} | {tot:.3f} | 100% |", ""]

# ---- full captures ----
out += ["## Full captures (`ncu --set full --clock-control none --import-source on`)", "",
        "| report | kernel | ms | DRAM read GB | DRAM write GB | DRAM TB/s | DRAM active % | "
        "smem wavefronts % | occupancy % | IPC | regs | top stalls (cycles per issue) |",
        "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    if len(r) < 3:
        continue
    d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ms": 1, "s": 1e3}
    dur = float(d["gpu__time_duration.sum"]) * scale.get(u["gpu__time_duration.sum"], 1e-6)
    gb = lambda k: float(d[k]) * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1}.get(u[k], 1)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    st = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(v)
          for k, v in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v}
    top = ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4])
    kname = re.sub(r"\(.*", "", d.get("Kernel Name", "?"))
    base = re.sub(r"<.*", "", kname.split("::")[-1])
    if base in PHASE and "c5" not in os.path.basename(rep):  # the C4 step's kernels
        # several captures of one phase (e.g. a tagged and a plain histogram
        # level): their mean stands for the phase's average launch
        t = traffic.setdefault(PHASE[base], {"dram_bytes_per_launch": 0.0, "ms": 0.0, "n": 0,
                                             "source": f"profiles/round{rnd}/ncu_summary.md", "capture": ""})
        t["dram_bytes_per_launch"] = (t["dram_bytes_per_launch"] * t["n"] + (rd + wr) * 1e9) / (t["n"] + 1)
        t["ms"] = (t["ms"] * t["n"] + dur) / (t["n"] + 1)
        t["n"] += 1
        t["capture"] = (t["capture"] + " + " if t["capture"] else "") + os.path.basename(rep)
    out.append(f"| `{rep.split('/')[-1]}` | {kname} | {dur:.3f} | {rd:.3f} | {wr:.3f} | "
               f"{(rd + wr) / dur:.2f} | "
               f"{float(d.get('dram__cycles_active.avg.pct_of_peak_sustained_elapsed', 0)):.0f} | "
               f"{float(d.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 0)):.0f} | "
               f"{float(d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0)):.0f} | "
               f"{float(d.get('sm__inst_executed.avg.per_cycle_active', 0)):.2f} | "
               f"{d.get('launch__registers_per_thread', '?')} | {top} |")
print("\n".join(out))
with open(f"profiles/round{rnd}/ncu_traffic.json", "w") as fh:
    json.dump(traffic, fh, indent=1)
