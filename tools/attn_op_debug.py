import sys, numpy as np
sys.path.insert(0, '/root/repo')
import __graft_entry__; __graft_entry__.build()
import paper_2602_19626_b200 as nc
from oracle.lm import window_start
rng = np.random.default_rng(1)
n, H, KV, L, C = int(sys.argv[1]) if len(sys.argv) > 1 else 200, 9, 3, 256, 128
q = rng.standard_normal((n, H * 64)).astype(np.float32)
k = rng.standard_normal((n, KV * 64)).astype(np.float32)
v = rng.standard_normal((n, KV * 64)).astype(np.float32)
ref = np.zeros((n, H * 64))
for j in range(n):
    w0 = window_start(j, L, C)
    for h in range(H):
        g = h // 3
        s = k[w0:j + 1, g * 64:(g + 1) * 64].astype(np.float64) @ q[j, h * 64:(h + 1) * 64] / 8
        p = np.exp(s - s.max()); p /= p.sum()
        ref[j, h * 64:(h + 1) * 64] = p @ v[w0:j + 1, g * 64:(g + 1) * 64]
np.set_printoptions(precision=3, linewidth=220, suppress=True)
for mode in (1, 0):
    o = nc.nc_debug_attention(q, k, v, H, KV, L, C, mode)
    e = np.abs(o - ref).max(axis=1)
    print("mode", mode, "max err", e.max(), "rows bad", (e > 1e-4).sum(), "first", np.argmax(e > 1e-4))
    if mode == 0:
        print("row0 h0 ours", o[0, :8], "\n ref", ref[0, :8], "\n v0", v[0, :8])
        print("row1 h0 ours", o[1, :8], "\n ref", ref[1, :8])
