"""Build libnc.so in-tree for sm_100a with nvcc (no JIT cache: the built .so
travels to the GPU box with the repo snapshot)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG.parent / "build" / "nc"
LIB = PKG / "libnc.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", f"-I{PKG.parent / 'include'}"]
# diagnostics builds only (e.g. NC_NVCC_EXTRA=-DNC_ATT_TIMING); a change of flags rebuilds everything
EXTRA = os.environ.get("NC_NVCC_EXTRA", "").split()
SOURCES = ["host_runtime.cpp", "host_nc06.cpp", "hf_loader.cpp", "api.cpp", "comm.cpp", "engine.cu", "k_embed_rms.cu", "k_walk.cu",
           "k_gemm_tc.cu", "k_attn_tc.cu"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists() or _flags_changed:
        return True
    deps = [src] + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.inc")) + \
        [PKG.parent / "include" / "nc.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def _compile(src: str):
    s = CSRC / src
    o = BUILD / (src + ".o")
    if not _stale(o, s):
        return None
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(s), "-o", str(o)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return src


_flags_changed = False


def build(verbose: bool = False) -> Path:
    global _flags_changed
    BUILD.mkdir(parents=True, exist_ok=True)
    stamp = BUILD / "flags.txt"
    _flags_changed = not stamp.exists() or stamp.read_text() != " ".join(EXTRA)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        done = [x for x in ex.map(_compile, SOURCES) if x]
    stamp.write_text(" ".join(EXTRA))
    objs = [str(BUILD / (s + ".o")) for s in SOURCES]
    if done or not LIB.exists() or any(Path(o).stat().st_mtime > LIB.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *objs, "-ldl", "-lpthread", "-lz"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(f"built {LIB} (recompiled: {done})", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
