"""Randomised round-trip soak on the GPU (diagnostics): random inputs (prose, MediaWiki-like,
mixed text/binary, random bytes, tiny and empty), random parameters (chunks, CDF-16/24, flags,
window variants, coder, window/slide, temperature, warmup), through nc_compress / nc_decompress
and nc_compress_file / nc_decompress_file on the 2-layer model.  Every case must round-trip.
    python tools/fuzz_roundtrip.py [seconds] [seed]"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import ensure_model, make_text  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 600
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 2602)
m = nc.Model(ensure_model("smollm2-2l"), 0)
t_end = time.time() + secs
n = fails = 0
while time.time() < t_end:
    kind = rng.choice(["alice", "enwik", "mixed", "bytes", "tiny"])
    size = rng.choice([0, 1, 7, 300, 3000, 20000, 60000])
    if kind == "bytes":
        data = bytes(rng.getrandbits(8) for _ in range(min(size, 5000)))
    elif kind == "tiny":
        data = bytes(rng.choice(b"ab\n \x00\xff") for _ in range(rng.randint(0, 40)))
    else:
        data = make_text(kind, size, rng.randint(0, 10 ** 6)) if size else b""
    window = rng.choice([256, 512, 1024])
    slide = rng.choice([s for s in (128, 256, 512) if s < window])
    prm = nc.nc_params_default(window=window, slide=slide, n_chunks=rng.choice([1, 2, 3, 7, 16]),
                               cdf_bits=rng.choice([16, 24]), flags=rng.choice([0, 1, 2, 3, 7]),
                               window_variant=rng.choice([0, 0, 1, 2, 3]), coder=rng.choice([0, 1]),
                               temperature=rng.choice([1.0, 0.8, 1.25]), warmup=rng.choice([100, 0, 7]),
                               max_slab_rows=rng.choice([1024, 4096, 32768]))
    use_file = kind in ("mixed", "bytes") or rng.random() < 0.2
    desc = (f"case {n}: kind={kind} n={len(data)} file={use_file} L={window} C={slide} chunks={prm.n_chunks} "
            f"bits={prm.cdf_bits} flags={prm.flags} wv={prm.window_variant} coder={prm.coder} "
            f"tau={prm.temperature} warmup={prm.warmup} slab={prm.max_slab_rows}")
    try:
        if use_file:
            back = nc.nc_decompress_file(m, nc.nc_compress_file(m, data, prm), prm)
        else:
            back = nc.nc_decompress(m, nc.nc_compress(m, data, prm), prm)
        ok = back == data
    except nc.NcError as e:
        ok = False
        desc += f" error {e}"
    if not ok:
        fails += 1
        print("FAIL", desc, flush=True)
    n += 1
print(f"fuzz: {n} cases, {fails} failures")
