"""Top source lines by warp-stall samples of one ncu report (all source files):
python tools/ncu_hot.py rep [n] [launch_index]"""
import csv
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    args += ["--launch-skip", sys.argv[3], "--launch-count", "1"]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
lines, fname, hdr = [], "?", None
for r in rows:
    if r and r[0] == "File Path":
        fname = os.path.basename(r[1])
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
        try:
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        top = sorted(((float(r[i]) if r[i] else 0.0, h) for i, h in enumerate(hdr)
                      if h.startswith("stall_") and "Not Issued" not in h), reverse=True)[:2]
        lines.append((s, f"{fname}:{r[0]}", r[1].strip()[:90], ",".join(f"{h[6:]}" for v, h in top if v)))
tot = sum(l[0] for l in lines) or 1
for s, loc, src, why in sorted(lines, reverse=True)[:n]:
    print(f"{s / tot:6.1%} {loc:22s} [{why}] {src}")
