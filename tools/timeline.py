"""Stream timeline of one compression (NC_TIMELINE diagnostics): python tools/timeline.py [workload] [plan]
plan: optional NC_SLAB_PLAN (comma-separated slab lengths)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NC_TIMELINE"] = "1"
if len(sys.argv) > 2:
    os.environ["NC_SLAB_PLAN"] = sys.argv[2]
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import numpy as np  # noqa: E402
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
data = open(ensure_text(wl.name), "rb").read()
model = nc.Model(ensure_model(wl.shape), 0)
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits)
for i in range(3):
    blob = nc.nc_compress(model, data, prm)
    print(f"run {i}: {len(blob)} B, stats {nc.nc_last_stats()}", file=sys.stderr, flush=True)
