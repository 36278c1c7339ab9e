import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import __graft_entry__; __graft_entry__.build()
import paper_2602_19626_b200 as nc
from synth import ensure_model
from oracle.ncw import Weights
from oracle.lm import LM
path = ensure_model("smollm2-2l")
m = nc.Model(path, 0); w = Weights(path)
rng = np.random.default_rng(7)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
x = [0] + list(rng.integers(3, w.V, n - 1))
prm = nc.nc_params_default(window=256, slide=128, max_slab_rows=256)
z = nc.nc_debug_forward(m, x, prm, 0)
ref = LM(w).forward_blocked(x, 256, 128)
e = np.abs(z - ref).max(axis=1) / np.abs(ref).max()
np.set_printoptions(precision=2, linewidth=200)
print("rows 0..40:", e[:40])
print("rows around 32:", e[28:40], "64:", e[60:70], "128:", e[124:134])
print("max", e.max(), "argmax", e.argmax(), "n bad", (e > 1e-4).sum(), "first bad", np.argmax(e > 1e-4))
