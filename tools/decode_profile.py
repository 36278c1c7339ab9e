"""Per-kernel-class device time of one decompression (config2 by default), per decode step.
python tools/decode_profile.py [workload] [bytes per chunk: decode only the first B bytes of
every chunk, as bench.py's decompress sample does]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
data = open(ensure_text(wl.name), "rb").read()
if len(sys.argv) > 2:
    cuts = nc.nc_host_split(data, wl.n_chunks)
    b = int(sys.argv[2])
    data = b"".join(data[cuts[c]:min(cuts[c + 1], cuts[c] + b)] for c in range(len(cuts) - 1))
model = nc.Model(ensure_model(wl.shape), 0)
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits)
blob = nc.nc_compress(model, data, prm)
steps = None
nc.nc_set_profiling(True)
t0 = time.perf_counter()
back = nc.nc_decompress(model, blob, prm)
dt = time.perf_counter() - t0
prof = nc.nc_profile()
nc.nc_set_profiling(False)
assert back == data
st = nc.nc_last_stats()
n_steps = max(1, max(1, len(data)) and st.get("steps", 0) or 1)
tot = sum(v["ms"] for v in prof.values())
print(f"decompress {len(data)} B in {dt:.2f} s ({len(data) / dt:.0f} B/s); stats {st}")
for k, v in sorted(prof.items(), key=lambda x: -x[1]["ms"]):
    if v["launches"]:
        print(f"  {k:12s} {v['ms']:9.1f} ms  {v['launches']:7d} launches  {1e3 * v['ms'] / v['launches']:8.1f} us/launch")
print(f"  kernel time {tot:.0f} ms of {1e3 * dt:.0f} ms wall")
