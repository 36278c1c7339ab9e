"""Top SASS instructions by warp-stall samples from an ncu report (source page):
python tools/ncu_hot_sass.py report.ncu-rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
tot = sum(float(r[i_s] or 0) for r in data)
print(f"{len(data)} instructions, {tot:.0f} samples")
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][i_s] or 0))[:n]:
    print(f"{idx:6d} {float(r[i_s]) / tot:6.1%}  {r[i_src].strip()[:90]}")
