"""Aggregate one ncu report's SASS by opcode: executed warp instructions and stall samples.
python tools/ncu_sass_ops.py rep [launch_index] [n]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    args += ["--launch-skip", sys.argv[2], "--launch-count", "1"]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
ops = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    sass = d.get("Source", "").strip()
    if not sass:
        continue
    tok = sass.split()
    op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
    op = op.split(".")[0]
    try:
        ops[op][0] += int(d.get("Instructions Executed", "0") or 0)
        ops[op][1] += float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        pass
ti = sum(v[0] for v in ops.values()) or 1
ts = sum(v[1] for v in ops.values()) or 1
print(f"total warp instructions {ti}")
for op, (i, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{op:12s} {i:>12d} {i / ti:6.1%}   stall samples {s / ts:6.1%}")
