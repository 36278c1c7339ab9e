import sys, numpy as np
sys.path.insert(0, '/root/repo')
import __graft_entry__; __graft_entry__.build()
import paper_2602_19626_b200 as nc
rng = np.random.default_rng(1)
n, H, KV, L, C = 130, 9, 3, 256, 128
q = rng.standard_normal((n, H * 64)).astype(np.float32)
k = rng.standard_normal((n, KV * 64)).astype(np.float32)
v = rng.standard_normal((n, KV * 64)).astype(np.float32)
np.set_printoptions(precision=3, linewidth=220, suppress=True)
o = nc.nc_debug_attention(q, k, v, H, KV, L, C, 0)   # debug: o_hi + o_lo summed; o_hi has S, o_lo has l,m,Opart
S_ref = (q[:, :64].astype(np.float64) @ k[:32, :64].T.astype(np.float64))
print("S row0 ours", o[0, :6], "ref", S_ref[0, :6])
print("S row5 ours", o[5, :6], "ref", S_ref[5, :6])
print("l,m row0", o[0, 32:34], " row5", o[5, 32:34])
p5 = np.exp(S_ref[5, :6] / 8 - (S_ref[5, :6] / 8).max())
print("Opart row0", o[0, 34:40], "v0", v[0, :6])
print("Opart row5", o[5, 34:40], "ref", (p5 @ v[:6, :64])[:6])
import os
if os.environ.get("NC_ATTN_DEBUG") == "2":
    ref2 = (q[:, 0:32].astype(np.float64) @ v[:32, :64].astype(np.float64))
    print("debug2 Opart row0", o[0, 34:40], "ref QV", ref2[0, :6])
if os.environ.get("NC_ATTN_DEBUG") == "3":
    ref3 = (q[:, 0:32].astype(np.float64) @ k[:32, 0:32].T.astype(np.float64))
    print("debug3 Opart row0", o[0, 34:40], "ref QK(d0-31)", ref3[0, :6])
