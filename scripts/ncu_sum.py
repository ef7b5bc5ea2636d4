"""One-line summary per ncu report: duration, DRAM bytes/throughput, occupancy, top stalls."""
import csv
import subprocess
import sys

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    d = dict(zip(r[0], r[2]))
    u = dict(zip(r[0], r[1]))
    dur = float(d["gpu__time_duration.sum"]) * {"ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}.get(u["gpu__time_duration.sum"], 1)
    gb = lambda k: float(d[k]) * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1}.get(u[k], 1)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    st = {k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(v)
          for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v}
    top = sorted(st.items(), key=lambda x: -x[1])[:4]
    print(f"{rep}: {dur:.3f} ms  dram rd {rd:.2f} GB wr {wr:.2f} GB  -> {(rd+wr)/dur:.2f} TB/s  "
          f"occ {float(d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0)):.0f}%  "
          f"ipc {float(d.get('sm__inst_executed.avg.per_cycle_active', 0)):.2f}  "
          f"l1 {float(d.get('l1tex__throughput.avg.pct_of_peak_sustained_active', 0)):.0f}%  "
          f"stalls {[(k, round(v, 2)) for k, v in top]}")
