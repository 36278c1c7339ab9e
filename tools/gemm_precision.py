import numpy as np, sys
sys.path.insert(0, '/root/repo')
import __graft_entry__; __graft_entry__.build()
import paper_2602_19626_b200 as nc
rng = np.random.default_rng(0)
for K in (64, 576, 1536):
    for kind in ("gauss", "pos"):
        M, N = 256, 256
        if kind == "gauss":
            A = rng.standard_normal((M, K)).astype(np.float32); B = (rng.standard_normal((N, K)) / 24).astype(np.float32)
        else:
            A = rng.random((M, K)).astype(np.float32); B = rng.random((N, K)).astype(np.float32)
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        for mode in (0,):
            out = nc.nc_debug_gemm(A, B, mode)
            err = out - ref
            scale = np.abs(ref).max()
            print(f"K={K:5d} {kind:5s} mode={mode} maxrel={np.abs(err).max()/scale:.2e} meanrel(bias)={err.mean()/scale:+.2e} rms={np.sqrt((err**2).mean())/scale:.2e}")
