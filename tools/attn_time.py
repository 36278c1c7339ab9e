"""Time the tensor-core attention kernel alone (nc_debug_attention, profiling on).
usage: NC_ATTN_REPS=5 [NC_ATTN_DEBUG=k] python tools/attn_time.py [n]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2602_19626_b200 as nc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
q = rng.standard_normal((n, 576)).astype(np.float32)
k = rng.standard_normal((n, 192)).astype(np.float32)
v = rng.standard_normal((n, 192)).astype(np.float32)
nc.nc_set_profiling(True)
nc.nc_debug_attention(q, k, v, 9, 3, 2048, 512, 0)
pr = nc.nc_profile()["attention"]
ms = pr["ms"] / max(1, pr["launches"])
print(f"debug={os.environ.get('NC_ATTN_DEBUG', '0')} n={n} launches={pr['launches']} ms/launch={ms:.3f} "
      f"TFLOP/s={pr['work'] / pr['launches'] / ms / 1e9:.1f}")
