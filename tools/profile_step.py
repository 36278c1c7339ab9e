"""One warm-up + one measured compress step of the bench workload (for ncu runs).
Usage: python tools/profile_step.py [workload] [n_steps] [flags]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
data = open(ensure_text(wl.name), "rb").read()
model = nc.Model(ensure_model(wl.shape), 0)
tokens, ntok = nc.nc_tokenize(model, data, wl.n_chunks)
tok = torch.from_numpy(tokens.view(np.int32).copy()).cuda()
kw = {"flags": int(sys.argv[3])} if len(sys.argv) > 3 else {}
prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits, **kw)
for i in range(steps):
    blob = nc.nc_compress_tokens(model, tok.data_ptr(), ntok, prm, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print(f"ok {len(data)} B -> {len(blob)} B, launches/step {nc.nc_last_stats()['kernel_launches']}")
