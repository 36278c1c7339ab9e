"""Wall time of one decompression (graph-replayed decode steps, no profiling).
python tools/decode_time.py [workload] [bytes per chunk] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
data = open(ensure_text(wl.name), "rb").read()
b = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cuts = nc.nc_host_split(data, wl.n_chunks)
data = b"".join(data[cuts[c]:min(cuts[c + 1], cuts[c] + b)] for c in range(len(cuts) - 1))
model = nc.Model(ensure_model(wl.shape), 0)
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits)
blob = nc.nc_compress(model, data, prm)
assert nc.nc_decompress(model, blob, prm) == data
best = 1e9
for _ in range(reps):
    t0 = time.perf_counter()
    nc.nc_decompress(model, blob, prm)
    best = min(best, time.perf_counter() - t0)
print(f"{wl.name} {len(data)} B: decompress {best:.3f} s, {len(data) / best:.0f} B/s "
      f"(NC_NO_WPREFETCH={'1' if os.environ.get('NC_NO_WPREFETCH') else '0'})")
