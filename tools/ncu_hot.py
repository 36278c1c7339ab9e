"""Top source lines by warp-stall samples of one ncu report: python tools/ncu_hot.py rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
samp, inst = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
cuda = []
for r in rows[hi + 1:]:
    if len(r) == len(hdr) and r[2] == "-":
        try:
            cuda.append((float(r[samp]), int(r[0]), r[1][:110], int(r[inst])))
        except ValueError:
            pass
tot = sum(c[0] for c in cuda) or 1
for c in sorted(cuda, reverse=True)[:n]:
    print(f"{c[0] / tot:6.1%} L{c[1]:4d} inst={c[3]:>11} {c[2]}")
