"""Diagnostics: device time of the config3 compress step through nc_compress_tokens, the same
call bench.py times (CUDA events on the stream, L2 flushed between steps).  With
NC_DIAG_NO_WALK=1 the walk is not launched (the call then fails at the host encoder; the
forward's time is what is measured).   python tools/step_time.py [workload] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
data = open(ensure_text(wl.name), "rb").read()
model = nc.Model(ensure_model(wl.shape), 0)
cuts = nc.nc_host_split(data, wl.n_chunks)
toks = [nc.nc_tokenize(model, data[cuts[c]:cuts[c + 1]], 1)[0] for c in range(len(cuts) - 1)]
ntok = np.array([len(t) for t in toks], np.uint32)
tok_dev = torch.from_numpy(np.concatenate(toks).view(np.int32).copy()).cuda()
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=len(toks), cdf_bits=wl.cdf_bits)
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(K + 2):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    try:
        nc.nc_compress_tokens(model, tok_dev.data_ptr(), ntok, prm, stream.cuda_stream)
    except nc.NcError:
        pass
    e1.record(stream)
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"{wl.name}: {np.median(ts):.1f} ms per step (min {min(ts):.1f}) NC_DIAG_NO_WALK={os.environ.get('NC_DIAG_NO_WALK', '0')}")
if os.environ.get("PROFILE"):   # one more step with per-kernel events (eager; no PDL overlap between kernels)
    nc.nc_set_profiling(True)
    try:
        nc.nc_compress_tokens(model, tok_dev.data_ptr(), ntok, prm, stream.cuda_stream)
    except nc.NcError:
        pass
    torch.cuda.synchronize()
    pr = nc.nc_profile()
    nc.nc_set_profiling(False)
    print({k: (v["launches"], round(v["ms"], 1), round(1e3 * v["ms"] / max(1, v["launches"]), 1)) for k, v in pr.items() if v["launches"]})
