"""Summarise an ncu --set full report's source page: hottest SASS lines by stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = rows[1:]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
top = sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in top:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} {st}")
