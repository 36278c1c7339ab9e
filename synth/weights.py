"""Random-init weight file writer (NCW1) and the on-disk cache of generated inputs.

NCW1 layout (little-endian; our own flat format):

  off  0  magic  b"NCW1"
  off  4  u32    version = 1
  off  8  u32 x9 n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab, bos_id, n_special
  off 44  f64    rope_theta
  off 52  f64    rms_eps
  off 60  u32    reserved (0)
  off 64  fp32 tensors, row-major, in this order:
            embed [V, d]
            per layer: attn_norm [d], wq [H*dh, d], wk [KV*dh, d], wv [KV*dh, d],
                       wo [d, H*dh], mlp_norm [d], wg [d_ff, d], wu [d_ff, d], wd [d, d_ff]
            final_norm [d]
  then    u32 V, then V x (u16 len, bytes)          -- the vocabulary (token id order)

Weights: every matrix ~ N(0, (1/24)^2) from numpy PCG64(seed) drawn in file
order; norm gains 1, or U(lo, hi) from PCG64(seed + 1000) in file
order for shapes with ``gain_range`` (test variants).  The head is tied to ``embed`` (D16).
"""
import os
import struct
from pathlib import Path

import numpy as np

from .configs import SHAPES, WORKLOADS, ModelShape
from .text import make_text
from .vocab import make_vocab

MAGIC = b"NCW1"
HEADER_BYTES = 64


def cache_dir() -> Path:
    d = Path(os.environ.get("NC_CACHE", Path(__file__).resolve().parent.parent / ".nc_cache"))
    d.mkdir(parents=True, exist_ok=True)
    return d


def tensor_layout(s: ModelShape):
    """[(name, shape)] in file order."""
    d, H, KV, dh, f, V = s.d_model, s.n_heads, s.n_kv_heads, s.head_dim, s.d_ff, s.vocab
    out = [("embed", (V, d))]
    for i in range(s.n_layers):
        out += [(f"l{i}.attn_norm", (d,)), (f"l{i}.wq", (H * dh, d)), (f"l{i}.wk", (KV * dh, d)),
                (f"l{i}.wv", (KV * dh, d)), (f"l{i}.wo", (d, H * dh)), (f"l{i}.mlp_norm", (d,)),
                (f"l{i}.wg", (f, d)), (f"l{i}.wu", (f, d)), (f"l{i}.wd", (d, f))]
    out.append(("final_norm", (d,)))
    return out


def write_ncw(path, s: ModelShape, seed: int = None):
    seed = s.weight_seed if seed is None else seed
    rng = np.random.default_rng(seed)
    grng = np.random.default_rng(seed + 1000)
    vocab = make_vocab(s.vocab)
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as f:
        hdr = MAGIC + struct.pack("<10I", 1, s.n_layers, s.d_model, s.n_heads, s.n_kv_heads,
                                  s.head_dim, s.d_ff, s.vocab, 0, 3)
        hdr += struct.pack("<dd", s.rope_theta, s.rms_eps) + struct.pack("<I", 0)
        assert len(hdr) == HEADER_BYTES
        f.write(hdr)
        for name, shape in tensor_layout(s):
            if len(shape) == 1:
                a = np.ones(shape, dtype=np.float32) if s.gain_range is None else \
                    grng.uniform(s.gain_range[0], s.gain_range[1], shape).astype(np.float32)
            else:
                a = (rng.standard_normal(shape, dtype=np.float32) * np.float32(s.init_std))
            f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())
        f.write(struct.pack("<I", len(vocab)))
        for t in vocab:
            f.write(struct.pack("<H", len(t)) + t)
    os.replace(tmp, path)


def ensure_model(shape_name: str) -> Path:
    s = SHAPES[shape_name]
    p = cache_dir() / f"{s.name}.seed{s.weight_seed}.ncw"
    if not p.exists():
        write_ncw(p, s)
    return p


def ensure_text(workload_name: str) -> Path:
    w = WORKLOADS[workload_name]
    p = cache_dir() / f"{w.text_kind}.{w.n_bytes}.seed{w.text_seed}.txt"
    if not p.exists():
        data = make_text(w.text_kind, w.n_bytes, w.text_seed)
        tmp = str(p) + ".tmp"
        with open(tmp, "wb") as f:
            f.write(data)
        os.replace(tmp, p)
    return p
