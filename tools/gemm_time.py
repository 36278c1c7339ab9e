"""Time the tcgen05 GEMM alone at the forward's shapes (diagnostics; needs a GPU).
python tools/gemm_time.py   (env NC_GEMM_REPS / NC_GEMM_EPI / NC_GEMM_NOSTORE are set here per case)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("qkv", 8192, 960, 576), ("o", 8192, 576, 576), ("gateup", 8192, 3072, 576), ("down", 8192, 576, 1536),
         ("head", 8192, 49152, 576)]
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2602_19626_b200 as nc
    M, N, K = map(int, sys.argv[2:5])
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K), dtype=np.float32)
    B = rng.standard_normal((N, K), dtype=np.float32)
    nc.nc_debug_gemm(A, B, 0)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "cases":
    CASES = [tuple([c.split(":")[0]] + [int(v) for v in c.split(":")[1:]]) for c in sys.argv[2:]]
for name, M, N, K in CASES:
    for epi in (["head", "resid"] if name in ("o", "down") else ["head"]):
        for nostore in (0, 1):
            env = dict(os.environ, NC_GEMM_REPS="20", NC_GEMM_EPI=epi)
            if nostore:
                env["NC_GEMM_NOSTORE"] = "1"
            r = subprocess.run([sys.executable, __file__, "one", str(M), str(N), str(K)], env=env,
                               capture_output=True, text=True)
            print(name, (r.stderr.strip().splitlines() or ["?"])[-1], flush=True)
