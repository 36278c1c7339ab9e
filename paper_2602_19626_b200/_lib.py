"""Thin ctypes binding of libnc.so (include/nc.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
fallback: if libnc.so is missing or no GPU is present, calls raise."""
import ctypes as C
import os
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libnc.so"

NC_OK, NC_ERR_FORMAT, NC_ERR_BACKEND, NC_ERR_INVALID, NC_ERR_NOMEM, NC_ERR_TRUNCATED, NC_ERR_INTEGRITY = range(7)
STATUS_NAMES = {0: "NC_OK", 1: "NC_ERR_FORMAT", 2: "NC_ERR_BACKEND", 3: "NC_ERR_INVALID", 4: "NC_ERR_NOMEM",
                5: "NC_ERR_TRUNCATED", 6: "NC_ERR_INTEGRITY"}
FLAG_NGRAM, FLAG_HEAD, FLAG_SKIP = 1, 2, 4
WINDOW_REFRESH, WINDOW_LMAX_M1 = 1, 2          # nc_params.window_variant (NEXT-4)
CODER_WNC, CODER_ANS = 0, 1                    # nc_params.coder (NEXT-4, D39)

# every symbol declared in include/nc.h (checked by tests/test_abi.py)
EXPORTS = [
    "nc_params_default", "nc_set_allocator", "nc_model_load", "nc_model_load_hf", "nc_model_free",
    "nc_host_bpe_encode", "nc_model_info",
    "nc_compress", "nc_decompress", "nc_compress_file", "nc_decompress_file", "nc_tokenize",
    "nc_host_segment", "nc_host_blob_encode", "nc_host_blob_decode", "nc_compress_tokens", "nc_comm_unique_id",
    "nc_comm_init", "nc_comm_free", "nc_compress_shard", "nc_decompress_shard", "nc_free",
    "nc_last_error", "nc_last_stats", "nc_debug_quantize", "nc_debug_walk", "nc_debug_walk_dump", "nc_debug_forward",
    "nc_host_split", "nc_host_wnc_encode", "nc_host_ans_encode", "nc_host_tokenize_vocab", "nc_host_shard_range", "nc_host_walk_ctas",
    "nc_host_shard_part", "nc_set_profiling", "nc_profile", "nc_debug_set_splitk", "nc_debug_gemm", "nc_debug_attention",
]


class NcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class nc_params(C.Structure):
    _fields_ = [("cdf_bits", C.c_uint32), ("flags", C.c_uint32), ("temperature", C.c_float),
                ("window", C.c_uint32), ("slide", C.c_uint32), ("warmup", C.c_uint32),
                ("eta", C.c_double), ("alpha", C.c_double), ("ngram_orders", C.c_uint32),
                ("ngram_cap", C.c_uint32), ("n_chunks", C.c_uint32), ("chunks_per_gpu", C.c_uint32),
                ("max_slab_rows", C.c_uint32), ("debug_dump", C.c_uint32),
                ("window_variant", C.c_uint32), ("coder", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise NcError(NC_ERR_BACKEND, f"{_LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(str(_LIB_PATH))
        P, u8p, u32p, f32p, szp, u64p = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), \
            C.POINTER(C.c_float), C.POINTER(C.c_size_t), C.POINTER(C.c_uint64)
        pp = C.POINTER(C.c_void_p)
        sig = {
            "nc_params_default": (None, [C.POINTER(nc_params)]),
            "nc_model_load": (C.c_int, [C.c_char_p, C.c_int, pp]),
            "nc_model_free": (None, [P]),
            "nc_model_load_hf": (C.c_int, [C.c_char_p, C.c_int, pp]),
            "nc_host_bpe_encode": (C.c_int, [C.c_char_p, C.c_uint32, P, C.c_size_t, pp, szp]),
            "nc_model_info": (C.c_int, [P, u32p, u32p, u32p]),
            "nc_compress": (C.c_int, [P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp]),
            "nc_decompress": (C.c_int, [P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp]),
            "nc_compress_file": (C.c_int, [P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp]),
            "nc_decompress_file": (C.c_int, [P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp]),
            "nc_host_segment": (C.c_int, [P, C.c_size_t, pp, pp, szp]),
            "nc_host_blob_encode": (C.c_int, [P, C.c_size_t, u8p, pp, szp]),
            "nc_host_blob_decode": (C.c_int, [C.c_uint8, P, C.c_size_t, C.c_size_t, pp, szp]),
            "nc_tokenize": (C.c_int, [P, P, C.c_size_t, C.c_uint32, pp, szp, pp, u32p]),
            "nc_compress_tokens": (C.c_int, [P, P, u32p, C.c_uint32, C.POINTER(nc_params), P, pp, szp]),
            "nc_comm_unique_id": (C.c_int, [u8p]),
            "nc_comm_init": (C.c_int, [C.c_int, C.c_int, u8p, C.c_int, pp]),
            "nc_comm_free": (None, [P]),
            "nc_compress_shard": (C.c_int, [P, P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp, u64p, u64p]),
            "nc_decompress_shard": (C.c_int, [P, P, P, C.c_size_t, C.POINTER(nc_params), P, pp, szp, u64p, u64p]),
            "nc_free": (None, [P]),
            "nc_set_profiling": (C.c_int, [C.c_int]),
            "nc_debug_set_splitk": (C.c_int, [C.c_int]),
            "nc_profile": (C.c_int, [C.c_int, u64p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_char_p)]),
            "nc_last_error": (C.c_char_p, []),
            "nc_last_stats": (C.c_int, [u64p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
            "nc_debug_quantize": (C.c_int, [f32p, C.c_uint32, C.c_uint32, u32p]),
            "nc_debug_walk": (C.c_int, [C.c_int, f32p, u32p, C.c_uint32, C.c_uint32, C.POINTER(nc_params),
                                        u32p, u32p, f32p]),
            "nc_debug_walk_dump": (C.c_int, [C.c_int, f32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.POINTER(nc_params),
                                             u32p, u32p, f32p, f32p, u32p, C.c_uint32, f32p, f32p, u32p]),
            "nc_debug_forward": (C.c_int, [P, u32p, C.c_uint32, C.POINTER(nc_params), C.c_int, f32p]),
            "nc_debug_attention": (C.c_int, [C.c_int, f32p, f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_uint32, C.c_uint32, C.c_int, f32p]),
            "nc_debug_gemm": (C.c_int, [C.c_int, f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, f32p]),
            "nc_host_split": (C.c_int, [P, C.c_size_t, C.c_uint32, u64p, u32p]),
            "nc_host_wnc_encode": (C.c_int, [u32p, u32p, C.c_size_t, C.c_uint32, pp, szp, u64p]),
            "nc_host_ans_encode": (C.c_int, [u32p, u32p, C.c_size_t, C.c_uint32, pp, szp, u64p]),
            "nc_host_tokenize_vocab": (C.c_int, [P, u32p, C.c_uint32, C.c_uint32, P, C.c_size_t, pp, szp]),
            "nc_host_shard_range": (C.c_int, [C.c_uint32, C.c_int, C.c_int, u32p, u32p]),
            "nc_host_walk_ctas": (C.c_int, [C.c_uint32, C.c_uint32, u32p]),
            "nc_host_shard_part": (C.c_int, [u32p, C.c_uint32, C.c_uint8, C.c_uint16, C.c_int, C.c_int, P,
                                             C.c_size_t, pp, szp, u64p, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st != NC_OK:
        raise NcError(st, lib().nc_last_error().decode(errors="replace"))


def _take_bytes(ptr, n):
    try:
        return C.string_at(ptr, n) if n else b""
    finally:
        if ptr:
            lib().nc_free(ptr)


def _take_array(ptr, n, dtype):
    try:
        if not n:
            return np.zeros(0, dtype=dtype)
        buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
        return np.frombuffer(bytes(buf), dtype=dtype).copy()
    finally:
        if ptr:
            lib().nc_free(ptr)


def nc_params_default(**overrides) -> nc_params:
    p = nc_params()
    lib().nc_params_default(C.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint32))


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


class Model:
    """A loaded NCW1 model on one device (nc_model_load / nc_model_free)."""

    def __init__(self, path, device=0):
        """path: an NCW1 file, or an HF checkpoint directory (config.json, model.safetensors,
        tokenizer.json; nc_model_load_hf)."""
        h = C.c_void_p()
        if os.path.isdir(str(path)):
            _check(lib().nc_model_load_hf(str(path).encode(), int(device), C.byref(h)))
        else:
            _check(lib().nc_model_load(str(path).encode(), int(device), C.byref(h)))
        self.h = h
        V, L, d = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib().nc_model_info(h, C.byref(V), C.byref(L), C.byref(d)))
        self.vocab, self.n_layers, self.d_model = V.value, L.value, d.value

    def close(self):
        if self.h:
            lib().nc_model_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nc_compress(model: Model, data: bytes, params: nc_params, stream=None) -> bytes:
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_compress(model.h, data, len(data), C.byref(params), stream, C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_decompress(model: Model, blob: bytes, params: nc_params, stream=None) -> bytes:
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_decompress(model.h, blob, len(blob), C.byref(params), stream, C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_compress_file(model: Model, data: bytes, params: nc_params, stream=None) -> bytes:
    """any bytes -> NC06 (hybrid text / binary, NEXT-3)."""
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_compress_file(model.h, data, len(data), C.byref(params), stream, C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_decompress_file(model: Model, blob: bytes, params: nc_params, stream=None) -> bytes:
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_decompress_file(model.h, blob, len(blob), C.byref(params), stream, C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_host_segment(data: bytes):
    k, l_, n = C.c_void_p(), C.c_void_p(), C.c_size_t()
    _check(lib().nc_host_segment(data, len(data), C.byref(k), C.byref(l_), C.byref(n)))
    kinds = _take_array(k.value, n.value, np.uint8)
    lens = _take_array(l_.value, n.value, np.uint64)
    return [(int(a), int(b)) for a, b in zip(kinds, lens)]


def nc_host_blob_encode(data: bytes):
    m, out, n = C.c_uint8(), C.c_void_p(), C.c_size_t()
    _check(lib().nc_host_blob_encode(data, len(data), C.byref(m), C.byref(out), C.byref(n)))
    return m.value, _take_bytes(out.value, n.value)


def nc_host_blob_decode(method: int, payload: bytes, expect_n: int):
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_host_blob_decode(method, payload, len(payload), expect_n, C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_tokenize(model: Model, data: bytes, n_chunks: int):
    t, nt, ntok, nch = C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_uint32()
    _check(lib().nc_tokenize(model.h, data, len(data), n_chunks, C.byref(t), C.byref(nt), C.byref(ntok),
                             C.byref(nch)))
    return _take_array(t.value, nt.value, np.uint32), _take_array(ntok.value, nch.value, np.uint32)


def nc_compress_tokens(model: Model, tokens_dev_ptr: int, chunk_ntok, params: nc_params, stream=None) -> bytes:
    nt, ntp = _u32(chunk_ntok)
    out, n = C.c_void_p(), C.c_size_t()
    _check(lib().nc_compress_tokens(model.h, C.c_void_p(tokens_dev_ptr), ntp, len(nt), C.byref(params), stream,
                                    C.byref(out), C.byref(n)))
    return _take_bytes(out.value, n.value)


def nc_last_stats():
    k, w, f, h = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
    _check(lib().nc_last_stats(C.byref(k), C.byref(w), C.byref(f), C.byref(h)))
    return dict(kernel_launches=k.value, walk_ms=w.value, forward_ms=f.value, head_ms=h.value)


def nc_debug_set_splitk(mode: int):
    _check(lib().nc_debug_set_splitk(int(mode)))


def nc_set_profiling(on: bool):
    _check(lib().nc_set_profiling(1 if on else 0))


def nc_profile():
    """{class name: dict(launches, ms, work)} since the last nc_set_profiling."""
    out = {}
    for cls in range(10):
        n, ms, w, name = C.c_uint64(), C.c_double(), C.c_double(), C.c_char_p()
        _check(lib().nc_profile(cls, C.byref(n), C.byref(ms), C.byref(w), C.byref(name)))
        out[name.value.decode()] = dict(launches=n.value, ms=ms.value, work=w.value)
    return out


def nc_debug_quantize(p, cdf_bits: int):
    p, pp = _f32(p)
    out = np.zeros(len(p), dtype=np.uint32)
    _check(lib().nc_debug_quantize(pp, len(p), cdf_bits, out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out


def nc_debug_walk(logits, tok, params: nc_params, device=0):
    lg, lp = _f32(logits)
    n, V = lg.shape
    tk, tp = _u32(tok)
    cum = np.zeros(n, np.uint32)
    freq = np.zeros(n, np.uint32)
    pt = np.zeros(n, np.float32)
    _check(lib().nc_debug_walk(device, lp, tp, n, V, C.byref(params), cum.ctypes.data_as(C.POINTER(C.c_uint32)),
                               freq.ctypes.data_as(C.POINTER(C.c_uint32)), pt.ctypes.data_as(C.POINTER(C.c_float))))
    return cum, freq, pt


def nc_debug_walk_dump(logits, tok, params: nc_params, rows=(), device=0):
    """nc_debug_walk + p~(t) of every row + full (p~, p, counts) vectors of `rows`.
    len(logits) < len(tok): token j uses logits[j % len(logits)] (cyclic rows).

    Returns dict(cum, freq, p_true, pt_true, rows, pt_rows [k,V], p_rows [k,V], c_rows [k,V])."""
    lg, lp = _f32(logits)
    n_lr, V = lg.shape
    tk, tp = _u32(tok)
    n = len(tk)
    if n_lr < n and n_lr == 0:
        raise NcError(NC_ERR_INVALID, "no logits rows")
    rv, rp = _u32(sorted(set(int(r) for r in rows)))
    k = len(rv)
    cum, freq = np.zeros(n, np.uint32), np.zeros(n, np.uint32)
    p_true, pt_true = np.zeros(n, np.float32), np.zeros(n, np.float32)
    pt_rows, p_rows = np.zeros((k, V), np.float32), np.zeros((k, V), np.float32)
    c_rows = np.zeros((k, V), np.uint32)
    u32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32))
    f32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
    _check(lib().nc_debug_walk_dump(device, lp, min(n_lr, n), tp, n, V, C.byref(params), u32(cum), u32(freq), f32(p_true),
                                    f32(pt_true), rp, k, f32(pt_rows), f32(p_rows), u32(c_rows)))
    return dict(cum=cum, freq=freq, p_true=p_true, pt_true=pt_true, rows=rv.tolist(), pt_rows=pt_rows,
                p_rows=p_rows, c_rows=c_rows)


def nc_debug_forward(model: Model, x, params: nc_params, mode: int = 0):
    xv, xp = _u32(x)
    out = np.zeros((len(xv), model.vocab), np.float32)
    _check(lib().nc_debug_forward(model.h, xp, len(xv), C.byref(params), mode,
                                  out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def nc_debug_gemm(A, B, mode: int = 0, device: int = 0):
    """out = A @ B.T through the forward's GEMM (mode 0 tcgen05 3xTF32, 1 SIMT fp32)."""
    a, ap = _f32(A)
    b, bp = _f32(B)
    M, K = a.shape
    N = b.shape[0]
    out = np.zeros((M, N), np.float32)
    _check(lib().nc_debug_gemm(device, ap, bp, M, N, K, mode, out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def nc_debug_attention(q, k, v, H, KV, window, slide, mode=0, device=0):
    """one attention layer of one chunk (q rotated): mode 0 tensor cores, 1 SIMT."""
    qa, qp = _f32(q)
    ka, kp = _f32(k)
    va, vp = _f32(v)
    n = qa.shape[0]
    out = np.zeros((n, H * 64), np.float32)
    _check(lib().nc_debug_attention(device, qp, kp, vp, n, H, KV, window, slide, mode,
                                    out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def nc_host_split(data: bytes, n_chunks: int):
    cuts = np.zeros(max(1, n_chunks) + 1, np.uint64)
    n = C.c_uint32()
    _check(lib().nc_host_split(data, len(data), n_chunks, cuts.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(n)))
    return cuts[: n.value].tolist()


def nc_host_wnc_encode(cum, freq, cdf_bits: int):
    c, cp = _u32(cum)
    f, fp = _u32(freq)
    s, sn, bits = C.c_void_p(), C.c_size_t(), C.c_uint64()
    _check(lib().nc_host_wnc_encode(cp, fp, len(c), cdf_bits, C.byref(s), C.byref(sn), C.byref(bits)))
    return _take_bytes(s.value, sn.value), bits.value


def nc_host_ans_encode(cum, freq, cdf_bits: int):
    """rANS stream of (cum, freq) pairs in coding order (NC_CODER_ANS, D39)."""
    c, cp = _u32(cum)
    f, fp = _u32(freq)
    s, sn, bits = C.c_void_p(), C.c_size_t(), C.c_uint64()
    _check(lib().nc_host_ans_encode(cp, fp, len(c), cdf_bits, C.byref(s), C.byref(sn), C.byref(bits)))
    return _take_bytes(s.value, sn.value), bits.value


def nc_host_tokenize_vocab(vocab, data: bytes, n_special: int = 3):
    blob = b"".join(vocab)
    lens, lp = _u32([len(v) for v in vocab])
    t, nt = C.c_void_p(), C.c_size_t()
    _check(lib().nc_host_tokenize_vocab(blob, lp, len(vocab), n_special, data, len(data), C.byref(t), C.byref(nt)))
    return _take_array(t.value, nt.value, np.uint32).tolist()


def nc_host_bpe_encode(tokenizer_json, vocab: int, data: bytes):
    t, nt = C.c_void_p(), C.c_size_t()
    _check(lib().nc_host_bpe_encode(str(tokenizer_json).encode(), vocab, data, len(data), C.byref(t), C.byref(nt)))
    return _take_array(t.value, nt.value, np.uint32).tolist()


def nc_host_walk_ctas(V: int, n_chunks: int) -> int:
    n = C.c_uint32()
    _check(lib().nc_host_walk_ctas(V, n_chunks, C.byref(n)))
    return n.value


def nc_host_shard_range(n_chunks: int, world: int, rank: int):
    a, b = C.c_uint32(), C.c_uint32()
    _check(lib().nc_host_shard_range(n_chunks, world, rank, C.byref(a), C.byref(b)))
    return a.value, b.value


def nc_host_shard_part(table, flags, tau_milli, world, rank, my_streams: bytes):
    t, tp = _u32(np.asarray(table).reshape(-1))
    part, pn, off, tot = C.c_void_p(), C.c_size_t(), C.c_uint64(), C.c_uint64()
    _check(lib().nc_host_shard_part(tp, len(t) // 3, flags, tau_milli, world, rank, my_streams, len(my_streams),
                                    C.byref(part), C.byref(pn), C.byref(off), C.byref(tot)))
    return _take_bytes(part.value, pn.value), off.value, tot.value


class Comm:
    """NCCL communicator (nc_comm_init); the unique id travels over torch.distributed."""

    def __init__(self, rank, world, uid: bytes, device=0):
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().nc_comm_init(rank, world, buf, device, C.byref(h)))
        self.h, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().nc_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.h:
            lib().nc_comm_free(self.h)
            self.h = None


def nc_compress_shard(model: Model, comm: Comm, data: bytes, params: nc_params, stream=None):
    part, pn, off, tot = C.c_void_p(), C.c_size_t(), C.c_uint64(), C.c_uint64()
    _check(lib().nc_compress_shard(model.h, comm.h, data, len(data), C.byref(params), stream, C.byref(part),
                                   C.byref(pn), C.byref(off), C.byref(tot)))
    return _take_bytes(part.value, pn.value), off.value, tot.value


def nc_decompress_shard(model: Model, comm: Comm, blob: bytes, params: nc_params, stream=None):
    part, pn, off, tot = C.c_void_p(), C.c_size_t(), C.c_uint64(), C.c_uint64()
    _check(lib().nc_decompress_shard(model.h, comm.h, blob, len(blob), C.byref(params), stream, C.byref(part),
                                     C.byref(pn), C.byref(off), C.byref(tot)))
    return _take_bytes(part.value, pn.value), off.value, tot.value


__all__ = [n for n in dir() if n.startswith("nc_")] + ["Model", "Comm", "NcError", "lib", "EXPORTS"]
