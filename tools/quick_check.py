"""Quick GPU check of a kernel change: config-2/3 compress step time (device-resident tokens,
CUDA events) and the forward's logits error against the fp64 oracle (30 layers, L = 2048,
two slides).  usage: python tools/quick_check.py [workload] [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
path = ensure_model(wl.shape)
model = nc.Model(path, 0)
data = open(ensure_text(wl.name), "rb").read()
tokens, ntok = nc.nc_tokenize(model, data, wl.n_chunks)
tok = torch.from_numpy(tokens.view(np.int32).copy()).cuda()
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits,
                           flags=int(os.environ.get("QC_FLAGS", "3")))
s = torch.cuda.current_stream()
for _ in range(2):
    nc.nc_compress_tokens(model, tok.data_ptr(), ntok, prm, s.cuda_stream)
ts = []
for _ in range(steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    blob = nc.nc_compress_tokens(model, tok.data_ptr(), ntok, prm, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{wl.name}: {np.median(ts):.1f} ms/step ({len(data) / np.median(ts) / 1e3:.3f} MB/s), {len(blob)} B")
nc.nc_set_profiling(True)
nc.nc_compress_tokens(model, tok.data_ptr(), ntok, prm, s.cuda_stream)
torch.cuda.synchronize()
for k, v in nc.nc_profile().items():
    if v["launches"]:
        print(f"  {k:12s} {v['ms']:8.2f} ms  {v['work'] / (v['ms'] / 1e3) / 1e12 if v['ms'] else 0:7.1f} T/s")
nc.nc_set_profiling(False)
if os.environ.get("QC_ERR", "1") == "1":
    from oracle.lm import LM
    from oracle.ncw import Weights
    w = Weights(path)
    rng = np.random.default_rng(11)
    n = 2600
    x = [0] + list(rng.integers(3, w.V, n - 1))
    t0 = time.time()
    z = nc.nc_debug_forward(model, x, nc.nc_params_default(), 0)
    ref = LM(w).forward_blocked(x, 2048, 512)
    print(f"30-layer logits max err / max|z| = {np.abs(z - ref).max() / np.abs(ref).max():.3e} "
          f"(oracle {time.time() - t0:.0f} s)")
