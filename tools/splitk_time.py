"""Time the tcgen05 GEMM at decode shapes (M = rows per step) with split-K on and off
(diagnostics; needs a GPU).  python tools/splitk_time.py [M]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
CASES = [("qkv", 960, 576, "head"), ("o", 576, 576, "resid"), ("gateup", 3072, 576, "head"),
         ("down", 576, 1536, "resid"), ("head", 49152, 576, "head")]
for name, N, K, epi in CASES:
    for split in ("0", "1"):
        env = dict(os.environ, NC_GEMM_REPS="50", NC_GEMM_EPI=epi, NC_GEMM_SPLIT=split)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gemm_time.py"), "one", str(M), str(N), str(K)],
                           env=env, capture_output=True, text=True)
        lines = r.stderr.strip().splitlines() or ["?"]
        print(f"{name:7s} split={split}", *[l for l in lines if "gemm" in l][-3:], flush=True)
