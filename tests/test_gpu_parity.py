"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): integer CDFs bit-exact given identical float
inputs; per-token probabilities within 1e-4 relative of the oracle; compressed
size within 0.5 %; GPU decompress(GPU compress(x)) == x; prefill and decode
logits bit-identical (D15).  Logits: 1e-5 of max |z| (fp32-accurate forward,
SURVEY T-K)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P_TOL = 1e-4
Z_TOL = 1e-5


@pytest.fixture(scope="module")
def nc():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2602_19626_b200 as m
    assert torch.cuda.is_available()
    return m


@pytest.fixture(scope="module")
def m2(nc):
    from synth import ensure_model
    return nc.Model(ensure_model("smollm2-2l"), 0)


@pytest.fixture(scope="module")
def w2():
    from synth import ensure_model
    from oracle.ncw import Weights
    return Weights(ensure_model("smollm2-2l"))


def _softmax32(z):
    e = np.exp(z - z.max())
    return (e / e.sum()).astype(np.float32)


# ------------------------------------------------------------ quantizer ----
@pytest.mark.parametrize("bits", [16, 24])
def test_quantize_bitexact(nc, bits):
    from oracle.cdf import quantize
    rng = np.random.default_rng(bits)
    V = 49152
    for scale in (0.3, 1.0, 4.0, 12.0):
        p = _softmax32(rng.standard_normal(V) * scale)
        assert np.array_equal(nc.nc_debug_quantize(p, bits), quantize(p, 1 << bits))
    p = np.zeros(V, np.float32)
    p[77] = 1.0
    assert np.array_equal(nc.nc_debug_quantize(p, bits), quantize(p, 1 << bits))
    p = np.full(V, 1.0 / V, np.float32)          # ties -> lowest index
    assert np.array_equal(nc.nc_debug_quantize(p, bits), quantize(p, 1 << bits))


def test_quantize_negative_residual(nc):
    from oracle.cdf import quantize
    p = np.zeros(256, np.float32)
    p[3] = 1.05                                   # sum p > 1, floors saturated (D6)
    assert np.array_equal(nc.nc_debug_quantize(p, 16), quantize(p, 1 << 16))


# ---------------------------------------------------------------- walker ---
def _markov_tokens(V, n, seed, k=8):
    rng = np.random.default_rng(seed)
    succ = rng.integers(0, V, (V, k))
    t = [int(rng.integers(V))]
    for _ in range(n - 1):
        t.append(int(succ[t[-1], rng.integers(k)]) if rng.random() < 0.7 else int(rng.integers(V)))
    return t


@pytest.mark.parametrize("V,n,flags,bits", [(49152, 400, 3, 24), (49152, 300, 1, 16), (256, 1500, 3, 24),
                                            (256, 800, 2, 24), (16, 600, 3, 24), (4, 300, 3, 16),
                                            (8192, 600, 3, 24),      # 4-CTA clusters (4096 <= V < 32768)
                                            (16, 800, 7, 24)])       # skip flag (tiny V: confident N-gram)
def test_walk_parity_synthetic(nc, V, n, flags, bits):
    from oracle.ensemble import Params, encode_tokens
    rng = np.random.default_rng(V + n)
    Z = (rng.standard_normal((n, V)) * (1.0 + rng.random((n, 1)) * 2)).astype(np.float32)
    toks = _markov_tokens(V, n, V)
    warm = 50
    prm = nc.nc_params_default(flags=flags, cdf_bits=bits, warmup=warm)
    cum, freq, p_gpu = nc.nc_debug_walk(Z, toks, prm)
    ref = encode_tokens(Z.astype(np.float64), toks, V, Params(flags=flags, cdf_bits=bits, warmup=warm))
    p_ref = np.array(ref["p_true"])
    rel = np.abs(p_gpu - p_ref) / p_ref
    assert rel.max() < P_TOL, rel.max()
    T = 1 << bits
    assert (freq >= 1).all() and (cum.astype(np.int64) + freq <= T).all()
    # the integer counts themselves are checked bit for bit against the oracle quantizer on
    # the walk's own p in tests/test_gpu_walk_dump.py (every sampled row); here: code length
    ideal_gpu = -np.log2(freq / T).sum()
    ideal_ref = -np.log2(np.array(ref["freq"]) / T).sum()
    assert abs(ideal_gpu - ideal_ref) <= 0.005 * ideal_ref + 1


def test_walk_gpu_stream_decodes_with_oracle_decoder_when_counts_match(nc):
    """host encoder on GPU (cum, freq) == oracle encoder on the same pairs."""
    from oracle.coder import Encoder
    V, n = 49152, 200
    rng = np.random.default_rng(5)
    Z = rng.standard_normal((n, V)).astype(np.float32)
    toks = list(rng.integers(0, V, n))
    cum, freq, _ = nc.nc_debug_walk(Z, toks, nc.nc_params_default())
    enc = Encoder()
    for c, f in zip(cum, freq):
        enc.encode(int(c), int(f), 1 << 24)
    assert nc.nc_host_wnc_encode(cum, freq, 24) == enc.finish()


# --------------------------------------------------------------- forward ---
def test_forward_parity_and_window(nc, m2, w2):
    from oracle.lm import LM
    rng = np.random.default_rng(7)
    n = 700
    x = [0] + list(rng.integers(3, w2.V, n - 1))
    prm = nc.nc_params_default(window=256, slide=128, max_slab_rows=256)
    z_gpu = nc.nc_debug_forward(m2, x, prm, 0)
    z_ref = LM(w2).forward_blocked(x, 256, 128)
    err = np.abs(z_gpu - z_ref).max() / np.abs(z_ref).max()
    assert err < Z_TOL, err


def test_forward_parity_nonunit_gains(nc):
    """RMSNorm gains ~ U(0.5, 1.5) (smollm2-2l-g; the GPU folds them into W_qkv, W_gate/up
    and E_head on load): logits within 1e-5 of max|z| of the fp64 oracle, with slides, and
    prefill == decode; the same weights pass the HF pin on CPU (tests/test_oracle_lm.py)."""
    from oracle.lm import LM
    from oracle.ncw import Weights
    from synth import ensure_model
    path = ensure_model("smollm2-2l-g")
    w = Weights(path)
    assert np.abs(w.final_norm - 1).max() > 0.1
    m = nc.Model(path, 0)
    rng = np.random.default_rng(17)
    n = 600
    x = [0] + list(rng.integers(3, w.V, n - 1))
    prm = nc.nc_params_default(window=256, slide=128, max_slab_rows=256)
    z = nc.nc_debug_forward(m, x, prm, 0)
    ref = LM(w).forward_blocked(x, 256, 128)
    err = np.abs(z - ref).max() / np.abs(ref).max()
    assert err < Z_TOL, err
    assert np.array_equal(z[:200], nc.nc_debug_forward(m, x[:200], prm, 1))
    m.close()


def test_prefill_decode_bit_identity(nc, m2, w2):
    rng = np.random.default_rng(8)
    n = 420
    x = [0] + list(rng.integers(3, w2.V, n - 1))
    prm = nc.nc_params_default(window=256, slide=128, max_slab_rows=256)
    a = nc.nc_debug_forward(m2, x, prm, 0)
    b = nc.nc_debug_forward(m2, x, prm, 1)
    assert np.array_equal(a, b)
    prm2 = nc.nc_params_default(window=256, slide=128, max_slab_rows=128)
    assert np.array_equal(a, nc.nc_debug_forward(m2, x, prm2, 0))     # slab size invariance


def test_splitk_bit_identity(nc, m2, w2):
    """Split-K GEMMs (decode steps: a few rows, the k loop spread over CTAs) sum the
    same per-span TMEM partials in the same order as the unsplit kernel (D15), so the
    logits are bit-identical whichever way every GEMM of the forward runs."""
    rng = np.random.default_rng(9)
    n = 300
    x = [0] + list(rng.integers(3, w2.V, n - 1))
    prm = nc.nc_params_default(window=256, slide=128, max_slab_rows=256)
    try:
        nc.nc_debug_set_splitk(0)
        a = nc.nc_debug_forward(m2, x, prm, 0)          # prefill, no split
        b0 = nc.nc_debug_forward(m2, x[:40], prm, 1)    # decode, no split
        nc.nc_debug_set_splitk(1)
        b = nc.nc_debug_forward(m2, x, prm, 1)          # decode, split-K
        c = nc.nc_debug_forward(m2, x, prm, 0)          # prefill, split where the grid is small
    finally:
        nc.nc_debug_set_splitk(1)
    assert np.array_equal(a[:40], b0)
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)


# ------------------------------------------------------------ end to end ---
def _oracle_size_and_p(w, data, prm_o):
    from oracle.chunking import split_chunks
    from oracle.ensemble import encode_tokens
    from oracle.lm import LM
    from oracle.tokenizer import Tokenizer
    tk, lm = getattr(w, "tokenizer", None) or Tokenizer(w.vocab), LM(w)
    size, ps, xs, ts = 9, [], [], []
    for ch in split_chunks(data, prm_o.n_chunks):
        t = tk.encode(ch)
        x = [w.bos] + t[:-1] if t else []
        Z = lm.forward_blocked(x, prm_o.window, prm_o.slide)
        r = encode_tokens(Z, t, w.V, prm_o)
        size += 12 + (r["bits"] + 7) // 8
        ps.append(np.array(r["p_true"]))
        xs.append(x)
        ts.append(t)
    return size, ps, xs, ts


@pytest.mark.parametrize("n_chunks,flags,bits", [(1, 3, 24), (3, 3, 24), (2, 1, 16), (1, 0, 24)])
def test_config1_roundtrip_size_and_p(nc, m2, w2, n_chunks, flags, bits):
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("alice", 4096, 1001)
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=n_chunks, flags=flags, cdf_bits=bits)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    size, ps, xs, ts = _oracle_size_and_p(w2, data, Params(window=512, slide=128, n_chunks=n_chunks,
                                                            flags=flags, cdf_bits=bits))
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    for x, t, p_ref in zip(xs, ts, ps):
        z = nc.nc_debug_forward(m2, x, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(z, t, prm)
        assert (np.abs(p_gpu - p_ref) / p_ref).max() < P_TOL


@pytest.mark.parametrize("n_chunks", [1, 2])
def test_skip_roundtrip_size_and_p(nc, m2, w2, n_chunks):
    """confidence-based LLM skip (NEXT-1, flags bit 2): round trip on repetitive text (the
    N-gram becomes confident), size within 0.5 % of the oracle, p(t) within P_TOL of the
    oracle on every token whose oracle H(p_ng) is not within 1e-3 of 1.5 bits (there fp32
    and fp64 may decide the skip differently: compare what is unique)."""
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("alice", 300, 4242) * 14       # oracle: 562 (1 chunk) / 256 (2 chunks) skips
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=n_chunks, flags=7, cdf_bits=24)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    prm_o = Params(window=512, slide=128, n_chunks=n_chunks, flags=7, cdf_bits=24)
    from oracle.chunking import split_chunks
    from oracle.lm import LM
    from oracle.ensemble import encode_tokens
    from oracle.tokenizer import Tokenizer
    tk, lm = Tokenizer(w2.vocab), LM(w2)
    size, n_cmp, n_all, n_skip = 0, 0, 0, 0
    for ch in split_chunks(data, n_chunks):
        t = tk.encode(ch)
        x = [w2.bos] + t[:-1] if t else []
        Z = lm.forward_blocked(x, 512, 128)
        r = encode_tokens(Z, t, w2.V, prm_o)
        size += 12 + (r["bits"] + 7) // 8
        n_skip += sum(r["skipped"])
        z = nc.nc_debug_forward(m2, x, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(z, t, prm)
        p_ref = np.array(r["p_true"])
        ok = np.array([h is None or abs(h - 1.5) > 1e-3 for h in r["h_ng"]])
        n_cmp += int(ok.sum())
        n_all += len(t)
        assert (np.abs(p_gpu[ok] - p_ref[ok]) / p_ref[ok]).max() < P_TOL
    assert n_skip > 100, n_skip                       # the skip path is exercised
    assert n_cmp >= 0.98 * n_all
    assert abs(len(blob) - (9 + size)) <= 0.005 * size, (len(blob), size)


def _chunk_stream_alone(nc, m, data, n_chunks, prm_fw):
    """(token_count, bit_count, stream) of one chunk computed ALONE: its own debug forward
    (one chunk, its own slab plan / decode-free prefill) and walk -- with the walk's cluster
    size of an n_chunks container (the rule's input) -- then the host WNC encoder."""
    t, _ = nc.nc_tokenize(m, data, 1)
    t = [int(v) for v in t]
    z = nc.nc_debug_forward(m, [0] + t[:-1], prm_fw, 0)
    cum, freq, _ = nc.nc_debug_walk(z, t, nc.nc_params_default(window=prm_fw.window, slide=prm_fw.slide,
                                                              n_chunks=n_chunks))
    stream, bits = nc.nc_host_wnc_encode(cum, freq, 24)
    return len(t), bits, stream


def test_chunk_streams_independent_of_batch(nc, m2):
    """Chunks are independent: a chunk's bitstream inside a 16-chunk container
    (slabs of 16 x len rows, 16 decode rows per step) equals the stream of that chunk's
    forward and walk run alone (batch and slab independence of every kernel, D15), and the
    16-chunk container round-trips.  (The walk's cluster size is a function of the
    container's chunk count, so the lone walk takes the 16-chunk container's.)"""
    import struct
    from synth import make_text
    data = make_text("alice", 24000, 77)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=16)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    n = struct.unpack_from("<BHH", blob, 4)[2]   # NC05 header: magic, flags u8, tau u16, chunks u16
    assert n == len(nc.nc_host_split(data, 16)) - 1
    table = [struct.unpack_from("<III", blob, 9 + 12 * c) for c in range(n)]
    offs = [9 + 12 * n]
    for t in table:
        offs.append(offs[-1] + t[2])
    cuts = nc.nc_host_split(data, 16)
    prm1 = nc.nc_params_default(window=256, slide=128, n_chunks=1)
    for c in (0, 7, n - 1):
        ntk, bits, stream = _chunk_stream_alone(nc, m2, data[cuts[c]:cuts[c + 1]], n, prm1)
        assert (ntk, bits) == table[c][:2], (c, ntk, bits, table[c])
        assert stream == blob[offs[c]:offs[c + 1]], c


def test_edge_inputs_roundtrip(nc, m2):
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=4)
    for data in (b"", b"a", b"\x00\x00\xff\n", b"\n" * 9, bytes(range(256)) * 3):
        assert nc.nc_decompress(m2, nc.nc_compress(m2, data, prm), prm) == data


def test_decompress_detects_wrong_params_and_corruption(nc, m2):
    """tampering is an error or output != input.  Wrong params and single bit flips
    early / in the middle of a stream, in the coder's finish bits and in the padding end in
    NC_ERR_INTEGRITY: the decoder's bit count must equal bit_count and the stream's tail must
    be exactly the finish() of the decoder's final state (D8).  (D38: without a checksum in
    NC05, a flip among the last data bits can only alter the final symbols.)"""
    import struct
    from synth import make_text
    data = make_text("alice", 1500, 5)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=1)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    bad = nc.nc_params_default(window=256, slide=128, n_chunks=1, warmup=7)
    with pytest.raises(nc.NcError) as ei:
        nc.nc_decompress(m2, blob, bad)
    assert ei.value.status == nc._lib.NC_ERR_INTEGRITY
    bits = struct.unpack_from("<I", blob, 13)[0]
    s0 = 21                                   # stream start: 9-byte header + one 12-byte entry
    # Flips that derail the decoder (early / middle), hit the coder's finish bits or the
    # padding are integrity errors.  NC05 has no checksum field (reading D38): a
    # flip in the last few DATA bits can change only the final symbol(s) into ones with the
    # same counts and renormalisation -- it may decode silently, but only the last bytes differ.
    for bit in [3, 40, bits // 3, bits // 2, bits - 2, bits - 1] + ([bits + 1] if bits % 8 else []):
        corrupt = bytearray(blob)
        corrupt[s0 + bit // 8] ^= 0x80 >> (bit % 8)
        with pytest.raises(nc.NcError) as ei:
            nc.nc_decompress(m2, bytes(corrupt), prm)
        assert ei.value.status == nc._lib.NC_ERR_INTEGRITY, bit
    corrupt = bytearray(blob)
    corrupt[s0 + (bits - 9) // 8] ^= 0x80 >> ((bits - 9) % 8)
    try:
        out = nc.nc_decompress(m2, bytes(corrupt), prm)
        assert len(out) >= len(data) - 16 and out[:len(data) - 16] == data[:len(data) - 16]
    except nc.NcError as e:
        assert e.status == nc._lib.NC_ERR_INTEGRITY
    with pytest.raises(nc.NcError):
        nc.nc_decompress(m2, b"NC99" + blob[4:], prm)
    with pytest.raises(nc.NcError):
        nc.nc_decompress(m2, blob[:-3], prm)
    # a crafted header asking for 10^8 tokens coded in 0 bits is refused before any allocation
    crafted = b"NC05" + bytes([3]) + struct.pack("<HH", 1000, 1) + struct.pack("<III", 10 ** 8, 0, 0)
    with pytest.raises(nc.NcError) as ei:
        nc.nc_decompress(m2, crafted, prm)
    assert ei.value.status == nc._lib.NC_ERR_INTEGRITY


def test_compress_tokens_rejects_out_of_vocab_ids(nc, m2):
    """nc_compress_tokens takes caller device ids: an id >= V is NC_ERR_INVALID, not an
    out-of-bounds read of E / b / cu."""
    ids = torch.tensor([5, 7, m2.vocab + 3, 9], dtype=torch.int32, device="cuda")
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=1)
    with pytest.raises(nc.NcError) as ei:
        nc.nc_compress_tokens(m2, ids.data_ptr(), np.array([4], np.uint32), prm,
                              torch.cuda.current_stream().cuda_stream)
    assert ei.value.status == nc._lib.NC_ERR_INVALID


# --------------------------------------------------- full-size sampled rows ---
@pytest.mark.slow
def test_full_model_sampled_rows(nc):
    """30-layer model, L=2048/C=512 as bench.py runs it: the first 2,600 rows of
    one chunk (two slides) against the oracle, plus decode bit-identity on a
    sample of rows."""
    from oracle.lm import LM
    from oracle.ncw import Weights
    from synth import ensure_model
    path = ensure_model("smollm2-135m")
    m = nc.Model(path, 0)
    w = Weights(path)
    rng = np.random.default_rng(11)
    n = 2600
    x = [0] + list(rng.integers(3, w.V, n - 1))
    prm = nc.nc_params_default()
    z = nc.nc_debug_forward(m, x, prm, 0)
    ref = LM(w).forward_blocked(x, 2048, 512)
    err = np.abs(z - ref).max() / np.abs(ref).max()
    assert err < Z_TOL, err
    m.close()


# ------------------------------------------------------- op-level kernels ---
def test_attention_op_vs_numpy(nc):
    """one attention layer (block-window causal GQA, D9-D10) of the tensor-core kernel
    against fp64 numpy, with slides (n > L)."""
    from oracle.lm import window_start
    rng = np.random.default_rng(21)
    n, H, KV, L, C = 390, 9, 3, 256, 128
    q = rng.standard_normal((n, H * 64)).astype(np.float32)
    k = rng.standard_normal((n, KV * 64)).astype(np.float32)
    v = rng.standard_normal((n, KV * 64)).astype(np.float32)
    ref = np.zeros((n, H * 64))
    for j in range(n):
        w0 = window_start(j, L, C)
        for h in range(H):
            g = h // (H // KV)
            s = k[w0:j + 1, g * 64:(g + 1) * 64].astype(np.float64) @ q[j, h * 64:(h + 1) * 64] / 8
            p = np.exp(s - s.max())
            ref[j, h * 64:(h + 1) * 64] = (p / p.sum()) @ v[w0:j + 1, g * 64:(g + 1) * 64]
    o = nc.nc_debug_attention(q, k, v, H, KV, L, C, 0)
    assert np.abs(o - ref).max() < 1e-5


@pytest.mark.parametrize("K", [576, 1536])
def test_tc_gemm_op_vs_numpy(nc, K):
    """tcgen05 3xTF32 GEMM with fp32-RN promotion: at least SIMT-fp32 accuracy."""
    rng = np.random.default_rng(K)
    A = rng.standard_normal((300, K)).astype(np.float32)
    B = (rng.standard_normal((448, K)) / 24).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    out = nc.nc_debug_gemm(A, B, 0)
    assert np.abs(out - ref).max() / np.abs(ref).max() < 2e-6
    P = rng.random((256, K)).astype(np.float32)              # positive data: no cancellation of bias
    Q = rng.random((128, K)).astype(np.float32)
    r2 = P.astype(np.float64) @ Q.astype(np.float64).T
    assert abs(((nc.nc_debug_gemm(P, Q, 0) - r2) / r2).mean()) < 1e-6


def test_shard_path_one_rank_nccl(nc, m2):
    """nc_compress_shard / nc_decompress_shard through a real 1-rank NCCL communicator
    (SURVEY 8(e)): the part equals nc_compress with the same n_chunks, covers [0, total),
    and decompresses back.  (Several ranks need several GPUs; the multi-rank host plan is
    covered by tests/test_multi_gloo.py.)"""
    from synth import make_text
    data = make_text("alice", 2500, 606)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=3)
    comm = nc.Comm(0, 1, nc.Comm.unique_id(), 0)
    try:
        part, off, tot = nc.nc_compress_shard(m2, comm, data, prm)
        ref = nc.nc_compress(m2, data, prm)
        assert off == 0 and tot == len(part) and part == ref
        out, o2, t2 = nc.nc_decompress_shard(m2, comm, part, prm)
        assert o2 == 0 and t2 == len(data) and out == data
    finally:
        comm.close()


@pytest.mark.slow
def test_config2_full_size_chunk0(nc):
    """config2 at full size in bench.py's launch configuration (152,089 B, 30 layers,
    L = 2048 / C = 512, 8 chunks, the two-slab plan, 8-CTA walk clusters): the container
    round-trips; chunk 0 (3,899 tokens, four window slides) is recomputed by the oracle
    (blocked fp64 LM + the step-by-step walk) -- p(t) within 1e-4 at every row, logits
    within 1e-5 of max|z| on sampled rows, bit count within 0.5 %; and the chunk's stream
    in the 8-chunk container equals the host WNC encoding of the (cum, freq) the debug
    forward + walk give for that chunk alone (batch / slab independence at full size), so
    the §8(c) coder bound can be checked on the container's own bit count."""
    import struct
    from oracle.chunking import split_chunks
    from oracle.ensemble import Params, encode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from oracle.tokenizer import Tokenizer
    from synth import WORKLOADS, ensure_model, ensure_text
    wl = WORKLOADS["config2"]
    path = ensure_model(wl.shape)
    data = open(ensure_text("config2"), "rb").read()
    m = nc.Model(path, 0)
    prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks)
    blob = nc.nc_compress(m, data, prm)
    assert nc.nc_decompress(m, blob, prm) == data
    n = struct.unpack_from("<BHH", blob, 4)[2]
    assert n == wl.n_chunks
    table = [struct.unpack_from("<III", blob, 9 + 12 * c) for c in range(n)]
    assert all(t[2] == (t[1] + 7) // 8 for t in table)
    assert len(blob) == 9 + 12 * n + sum(t[2] for t in table)
    s0 = blob[9 + 12 * n:9 + 12 * n + table[0][2]]

    w = Weights(path)
    ch0 = split_chunks(data, n)[0]
    toks = Tokenizer(w.vocab).encode(ch0)
    assert len(toks) == table[0][0] and len(toks) > wl.window + 3 * wl.slide   # four slides
    x = [w.bos] + toks[:-1]
    z = nc.nc_debug_forward(m, x, prm, 0)
    cum, freq, p_gpu = nc.nc_debug_walk(z, toks, prm)
    stream, bits = nc.nc_host_wnc_encode(cum, freq, 24)
    assert bits == table[0][1] and stream == s0
    T = 1 << 24
    f = freq.astype(np.float64)
    bound = (-np.log2(f / T) - np.log2(1.0 - 2.0 ** (24 - 30) / f)).sum() + 64
    assert bits <= bound, (bits, bound)

    Z = LM(w).forward_blocked(x, wl.window, wl.slide)
    rows = sorted(set([0, 1, 99, 100, 2047, 2048, 2559, 2560, len(x) - 1] + list(range(0, len(x), 97))))
    zerr = np.abs(z[rows] - Z[rows]).max() / np.abs(Z[rows]).max()
    assert zerr < Z_TOL, zerr
    ref = encode_tokens(Z, toks, w.V, Params(window=wl.window, slide=wl.slide, n_chunks=1))
    p_ref = np.array(ref["p_true"])
    rel = np.abs(p_gpu - p_ref) / p_ref
    assert rel.max() < P_TOL, rel.max()
    assert abs(bits - ref["bits"]) <= 0.005 * ref["bits"], (bits, ref["bits"])
    m.close()


@pytest.mark.slow
@pytest.mark.parametrize("L,bits", [(512, 24), (1024, 16)])
def test_config5_windows_full_model(nc, L, bits):
    """Config 5 variants on the 30-layer model: window L with C = L/4 (D11) over enough
    rows for several slides, CDF-16 and CDF-24 -- GPU logits within 1e-5 of max|z| of the
    blocked fp64 oracle, and the walk's p(t) within 1e-4 of the oracle walk on them."""
    from oracle.ensemble import Params, encode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from synth import ensure_model, make_text
    path = ensure_model("smollm2-135m")
    m = nc.Model(path, 0)
    w = Weights(path)
    C = L // 4
    toks, _ = nc.nc_tokenize(m, make_text("alice", 12000, 1005), 1)
    assert len(toks) >= L + 3 * C + 37
    toks = [int(t) for t in toks[:L + 3 * C + 37]]          # three slides and a ragged tail
    x = [w.bos] + toks[:-1]
    prm = nc.nc_params_default(window=L, slide=C, cdf_bits=bits)
    z = nc.nc_debug_forward(m, x, prm, 0)
    Z = LM(w).forward_blocked(x, L, C)
    err = np.abs(z - Z).max() / np.abs(Z).max()
    assert err < Z_TOL, err
    _, freq, p_gpu = nc.nc_debug_walk(z, toks, prm)
    ref = encode_tokens(z.astype(np.float64), toks, w.V, Params(window=L, slide=C, cdf_bits=bits))
    rel = np.abs(p_gpu - np.array(ref["p_true"])) / np.array(ref["p_true"])
    assert rel.max() < P_TOL, rel.max()
    assert (freq >= 1).all()
    m.close()


def test_enwik_shaped_roundtrip_size_and_p(nc, m2, w2):
    """Config 4's input kind (MediaWiki XML with ~1-2 % non-ASCII UTF-8, which exercises the
    byte-fallback tokens) on the 2-layer model, 3 chunks: GPU round trip, size within 0.5 %
    of the oracle, p(t) within 1e-4 at every row."""
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("enwik", 6000, 1004)
    assert any(b >= 0x80 for b in data)
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=3)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    size, ps, xs, ts = _oracle_size_and_p(w2, data, Params(window=512, slide=128, n_chunks=3))
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    for x, t, p_ref in zip(xs, ts, ps):
        z = nc.nc_debug_forward(m2, x, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(z, t, prm)
        assert (np.abs(p_gpu - p_ref) / p_ref).max() < P_TOL


@pytest.mark.parametrize("V,n,over", [(49152, 400, {"temperature": 0.7}), (49152, 400, {"temperature": 1.3}),
                                      (8192, 600, {"eta": 0.1}), (8192, 600, {"alpha": 5e-3}),
                                      (256, 1500, {"ngram_orders": 3}),      # SPEC's reading of D18
                                      (256, 1500, {"ngram_cap": 16}),        # capacity freeze, D22
                                      (16, 800, {"ngram_orders": 1, "eta": 0.5})])
def test_walk_parity_param_variants(nc, V, n, over):
    """The walk under the non-default parameters nc_params carries (temperature D29, mixer
    rate eta D24, head rate alpha, number of N-gram context tables D18, table capacity D22):
    p(t) within 1e-4 of the oracle walk on the same fp32 logits, counts valid."""
    from oracle.ensemble import Params, encode_tokens
    rng = np.random.default_rng(V + n + len(over))
    Z = (rng.standard_normal((n, V)) * (1.0 + rng.random((n, 1)) * 2)).astype(np.float32)
    toks = _markov_tokens(V, n, V + 1)
    prm = nc.nc_params_default(warmup=50, **over)
    cum, freq, p_gpu = nc.nc_debug_walk(Z, toks, prm)
    ref = encode_tokens(Z.astype(np.float64), toks, V, Params(warmup=50, **over))
    p_ref = np.array(ref["p_true"])
    rel = np.abs(p_gpu - p_ref) / p_ref
    assert rel.max() < P_TOL, rel.max()
    assert (freq >= 1).all() and (cum.astype(np.int64) + freq <= (1 << 24)).all()


def test_many_chunks_roundtrip(nc, m2):
    """300 chunks in one call (chunk_count > 255 in the u16 header field; walk clusters in
    several waves; ~30-token chunks, most shorter than the warmup): round trip, and chunks
    0 / 150 / 299 carry the same stream as their forward and walk run alone."""
    import struct
    from synth import make_text
    data = make_text("alice", 45000, 55)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=300)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    n = struct.unpack_from("<BHH", blob, 4)[2]
    cuts = nc.nc_host_split(data, 300)
    assert n == len(cuts) - 1 == 300
    table = [struct.unpack_from("<III", blob, 9 + 12 * c) for c in range(n)]
    offs = [9 + 12 * n]
    for t in table:
        offs.append(offs[-1] + t[2])
    assert offs[-1] == len(blob)
    prm1 = nc.nc_params_default(window=256, slide=128, n_chunks=1)
    for c in (0, 150, n - 1):
        ntk, bits, stream = _chunk_stream_alone(nc, m2, data[cuts[c]:cuts[c + 1]], n, prm1)
        assert (ntk, bits) == table[c][:2], (c, ntk, bits, table[c])
        assert stream == blob[offs[c]:offs[c + 1]], c


def test_compress_tokens_equals_compress(nc, m2):
    """The entry point bench.py times as `value` (nc_compress_tokens: token ids already in
    HBM) produces the same container as the public nc_compress on host bytes (`e2e`)."""
    from synth import make_text
    data = make_text("alice", 20000, 66)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=5)
    blob = nc.nc_compress(m2, data, prm)
    cuts = nc.nc_host_split(data, 5)
    toks, ntok = [], []
    for c in range(len(cuts) - 1):
        t, _ = nc.nc_tokenize(m2, data[cuts[c]:cuts[c + 1]], 1)
        toks.append(t)
        ntok.append(len(t))
    td = torch.from_numpy(np.concatenate(toks).view(np.int32).copy()).cuda()
    s = torch.cuda.current_stream()
    blob2 = nc.nc_compress_tokens(m2, td.data_ptr(), np.array(ntok, np.uint32), prm, s.cuda_stream)
    torch.cuda.synchronize()
    assert blob2 == blob


# ------------------------------------------------------ NEXT-4 window variants ---
VARIANTS = [(1, "refresh"), (2, "lmax-1"), (3, "refresh+lmax-1")]


@pytest.mark.parametrize("wv,name", VARIANTS)
def test_forward_window_variants(nc, m2, w2, wv, name):
    """NEXT-4 on the GPU forward: refresh semantics (every window block evaluated fresh,
    P:489-492) and/or L_max = L - 1 (D10): logits within 1e-5 of max|z| of the fp64 oracle
    (oracle/lm.py, pinned to HF on CPU), over several slides with a ragged tail; and the
    decode-step path (with the refresh re-prefill at every block start) bit-identical to the
    prefill path (D15)."""
    from oracle.lm import LM
    rng = np.random.default_rng(30 + wv)
    L, C, n = 256, 128, 777
    x = [0] + list(rng.integers(3, w2.V, n - 1))
    prm = nc.nc_params_default(window=L, slide=C, max_slab_rows=256, window_variant=wv)
    z = nc.nc_debug_forward(m2, x, prm, 0)
    lmax = L - 1 if wv & 2 else L
    ref = LM(w2).forward_refresh_blocked(x, L, C, lmax) if wv & 1 else LM(w2).forward_blocked(x, lmax, C)
    err = np.abs(z - ref).max() / np.abs(ref).max()
    assert err < Z_TOL, err
    z1 = nc.nc_debug_forward(m2, x, prm, 1)
    assert np.array_equal(z, z1)
    # the variant really changes the logits past the first slide
    base = nc.nc_debug_forward(m2, x, nc.nc_params_default(window=L, slide=C, max_slab_rows=256), 0)
    assert np.abs(base[L + C:] - z[L + C:]).max() > 1e-4


@pytest.mark.parametrize("wv,name", VARIANTS)
@pytest.mark.parametrize("n_chunks", [1, 3])
def test_window_variants_roundtrip_size_and_p(nc, m2, w2, wv, name, n_chunks):
    """NEXT-4 end to end: GPU round trip, size within 0.5 % of the oracle pipeline with the
    same variant, p(t) within 1e-4 at every row; decoding with the wrong variant fails the
    integrity checks (the variant is not stored in the container, like L and C)."""
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("alice", 4096, 1001)
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=n_chunks, window_variant=wv, max_slab_rows=1024)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    po = Params(window=512, slide=128, n_chunks=n_chunks, refresh=bool(wv & 1), lmax_minus_one=bool(wv & 2))
    from oracle.chunking import split_chunks
    from oracle.ensemble import encode_tokens
    from oracle.lm import LM
    from oracle.tokenizer import Tokenizer
    tk, lm = Tokenizer(w2.vocab), LM(w2)
    size = 9
    for ch in split_chunks(data, n_chunks):
        t = tk.encode(ch)
        x = [w2.bos] + t[:-1]
        Z = lm.forward_refresh_blocked(x, 512, 128, po.lmax) if po.refresh else lm.forward_blocked(x, po.lmax, 128)
        r = encode_tokens(Z, t, w2.V, po)
        size += 12 + (r["bits"] + 7) // 8
        z = nc.nc_debug_forward(m2, x, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(z, t, prm)
        p_ref = np.array(r["p_true"])
        assert (np.abs(p_gpu - p_ref) / p_ref).max() < P_TOL
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    if n_chunks == 1:
        # with the N-gram on, random-init weights leave the LLM a negligible mixer weight after
        # ~150 tokens, so a wrong variant can still decode; with the head alone (flags = 2)
        # p = p~ depends on the LLM everywhere, and decoding with the other variant must fail
        hp = nc.nc_params_default(window=512, slide=128, n_chunks=1, window_variant=wv, flags=2)
        hblob = nc.nc_compress(m2, data, hp)
        assert nc.nc_decompress(m2, hblob, hp) == data
        other = nc.nc_params_default(window=512, slide=128, n_chunks=1, window_variant=wv ^ 1, flags=2)
        with pytest.raises(nc.NcError) as ei:
            nc.nc_decompress(m2, hblob, other)
        assert ei.value.status == nc._lib.NC_ERR_INTEGRITY


# ------------------------------------------------------------- NEXT-3: NC06 ---
def test_nc06_roundtrip_and_oracle_sections(nc, m2, w2):
    """NC06 hybrid files through the C ABI: round trip of a mixed text / binary
    file; the container parses with the oracle's reader, its entry table equals the oracle
    segmentation (rules 1-4), its binary section decodes (Python lzma / zlib) to the
    oracle's binary blob with the oracle's method choice, and its text section is within
    0.5 % of the oracle's NC05 size for the same text document with p(t) within 1e-4."""
    from oracle import nc06
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("mixed", 30000, 77)
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=3)
    blob = nc.nc_compress_file(m2, data, prm)
    assert nc.nc_decompress_file(m2, blob, prm) == data
    flags, tau, regs, method, payload, chunks = nc06.read_nc06(blob)
    assert regs == nc06.segment(data) and len(regs) > 4
    text, binary = nc06.split(data, regs)
    assert method == nc06.blob_encode(binary)[0] and nc06.blob_decode(method, payload) == binary
    size, ps, xs, ts = _oracle_size_and_p(w2, text, Params(window=512, slide=128, n_chunks=3))
    text_section = 2 + sum(12 + len(s) for _, _, s in chunks)
    assert abs(text_section - (size - 7)) <= 0.005 * size, (text_section, size)
    assert [n for n, _, _ in chunks] == [len(t) for t in ts]
    for x, t, p_ref in zip(xs, ts, ps):
        z = nc.nc_debug_forward(m2, x, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(z, t, prm)
        assert (np.abs(p_gpu - p_ref) / p_ref).max() < P_TOL
    # a corrupted binary section is an integrity error, never silent output
    off = 10 + 5 * len(regs) + 5
    bad = bytearray(blob)
    bad[off + len(payload) // 2] ^= 0x10
    with pytest.raises(nc.NcError) as ei:
        nc.nc_decompress_file(m2, bytes(bad), prm)
    assert ei.value.status == nc._lib.NC_ERR_INTEGRITY


def test_nc06_edge_inputs(nc, m2):
    """pure binary (one binary entry, no text tokens), pure text, empty input; and a plain
    NC05 container is accepted by nc_decompress_file."""
    from oracle import nc06
    from synth import make_text
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=2)
    rnd = bytes(np.random.default_rng(3).integers(128, 256, 5000).astype(np.uint8))
    for data in (rnd, make_text("alice", 3000, 8), b"", b"\x00" * 10000, rnd[:40]):
        blob = nc.nc_compress_file(m2, data, prm)
        assert nc.nc_decompress_file(m2, blob, prm) == data
        regs = nc06.read_nc06(blob)[2]
        assert sum(ln for _, ln in regs) == len(data)
    blob5 = nc.nc_compress(m2, b"hello NC05\n" * 40, prm)
    assert nc.nc_decompress_file(m2, blob5, prm) == b"hello NC05\n" * 40


# ------------------------------------------------- NEXT-2: HF checkpoint + BPE ---
def test_hf_checkpoint_forward_tokenizer_roundtrip(nc):
    """An HF-format SmolLM2-shaped checkpoint (config.json + BF16 model.safetensors +
    tokenizer.json, synth/hf.py) loaded by nc_model_load_hf: the model's BPE tokenization
    equals the HF tokenizers library's; logits within 1e-5 of max|z| of the oracle's
    independent safetensors reader + fp64 LM; GPU round trip; size within 0.5 % of the
    oracle pipeline (tokenizing with the HF library) and p(t) within 1e-4."""
    from oracle.ensemble import Params
    from oracle.hf import HfWeights
    from oracle.lm import LM
    from synth import make_text
    from synth.hf import ensure_hf_model
    d = ensure_hf_model("hf-smollm2-2l")
    m = nc.Model(d, 0)
    w = HfWeights(d)
    data = make_text("enwik", 6000, 1004)
    toks, ntok = nc.nc_tokenize(m, data, 1)
    assert toks.tolist() == w.tokenizer.encode(data)
    x = [w.bos] + toks.tolist()[:-1]
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=2)
    z = nc.nc_debug_forward(m, x, prm, 0)
    ref = LM(w).forward_blocked(x, 512, 128)
    assert np.abs(z - ref).max() / np.abs(ref).max() < Z_TOL
    blob = nc.nc_compress(m, data, prm)
    assert nc.nc_decompress(m, blob, prm) == data
    size, ps, xs, ts = _oracle_size_and_p(w, data, Params(window=512, slide=128, n_chunks=2))
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    for x_, t, p_ref in zip(xs, ts, ps):
        zz = nc.nc_debug_forward(m, x_, prm, 0)
        _, _, p_gpu = nc.nc_debug_walk(zz, t, prm)
        assert (np.abs(p_gpu - p_ref) / p_ref).max() < P_TOL
    m.close()


@pytest.mark.slow
def test_config3_full_size_chunk_stream_and_p(nc):
    """config3 at full size in bench.py's launch configuration (10 MB, 64 chunks, 30 layers,
    L = 2048 / C = 512, 512-position slabs, 4-CTA walk clusters): the container's structure;
    chunk 17's stream (~39K tokens) equals the host WNC encoding of its forward + walk run
    alone (batch / slab independence at full size); the §8(c) coder bound on its bit count;
    and the fp64 oracle (blocked LM + walk) on the chunk's first 2,600 rows (one slide):
    logits within 1e-5 of max|z| on sampled rows, p(t) within 1e-4 at every one of them."""
    import struct
    from oracle.chunking import split_chunks
    from oracle.ensemble import Params, encode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from oracle.tokenizer import Tokenizer
    from synth import WORKLOADS, ensure_model, ensure_text
    wl = WORKLOADS["config3"]
    path = ensure_model(wl.shape)
    data = open(ensure_text("config3"), "rb").read()
    m = nc.Model(path, 0)
    prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks)
    toks, ntok = nc.nc_tokenize(m, data, wl.n_chunks)
    td = torch.from_numpy(toks.view(np.int32).copy()).cuda()
    blob = nc.nc_compress_tokens(m, td.data_ptr(), ntok, prm, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    n = struct.unpack_from("<BHH", blob, 4)[2]
    assert n == wl.n_chunks == len(ntok)
    table = [struct.unpack_from("<III", blob, 9 + 12 * c) for c in range(n)]
    assert [t[0] for t in table] == list(ntok)
    assert len(blob) == 9 + 12 * n + sum(t[2] for t in table)
    c = 17
    off = 9 + 12 * n + sum(t[2] for t in table[:c])
    t = [int(v) for v in toks[int(sum(ntok[:c])):int(sum(ntok[:c + 1]))]]
    assert len(t) > 30000
    x = [0] + t[:-1]
    z = nc.nc_debug_forward(m, x, nc.nc_params_default(window=wl.window, slide=wl.slide), 0)
    cum, freq, p_gpu = nc.nc_debug_walk(z, t, prm)            # prm.n_chunks = 64: the container's walk
    stream, bits = nc.nc_host_wnc_encode(cum, freq, 24)
    assert bits == table[c][1] and stream == blob[off:off + table[c][2]]
    T = 1 << 24
    f = freq.astype(np.float64)
    assert bits <= (-np.log2(f / T) - np.log2(1.0 - 2.0 ** (24 - 30) / f)).sum() + 64
    w = Weights(path)
    nr = 2600
    Z = LM(w).forward_blocked(x[:nr], wl.window, wl.slide)
    rows = sorted(set([0, 99, 100, 2047, 2048, nr - 1] + list(range(0, nr, 131))))
    assert np.abs(z[rows] - Z[rows]).max() / np.abs(Z[rows]).max() < Z_TOL
    ref = encode_tokens(Z, t[:nr], w.V, Params(window=wl.window, slide=wl.slide))
    p_ref = np.array(ref["p_true"])
    assert (np.abs(p_gpu[:nr] - p_ref) / p_ref).max() < P_TOL
    m.close()


@pytest.mark.slow
def test_full_model_head_only_end_to_end(nc):
    """The LLM visible end to end: with the N-gram off (flags = 2) the coded distribution is
    the head's p~ = softmax(z + b) on every row, so the 30-layer forward drives every code.
    GPU compress -> decompress round trip; size within 0.5 % of the oracle pipeline (fp64
    blocked LM + walk) and p(t) within 1e-4 at every row (3 window slides)."""
    from oracle.ensemble import Params
    from oracle.ncw import Weights
    from synth import ensure_model, make_text
    path = ensure_model("smollm2-135m")
    m = nc.Model(path, 0)
    w = Weights(path)
    data = make_text("alice", 16000, 2024)
    prm = nc.nc_params_default(window=1024, slide=256, n_chunks=1, flags=2)
    blob = nc.nc_compress(m, data, prm)
    assert nc.nc_decompress(m, blob, prm) == data
    size, ps, xs, ts = _oracle_size_and_p(w, data, Params(window=1024, slide=256, n_chunks=1, flags=2))
    assert len(ts[0]) > 1024 + 2 * 256
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    z = nc.nc_debug_forward(m, xs[0], prm, 0)
    _, _, p_gpu = nc.nc_debug_walk(z, ts[0], prm)
    assert (np.abs(p_gpu - ps[0]) / ps[0]).max() < P_TOL
    m.close()


# ------------------------------------------------------------------ rANS ---
@pytest.mark.parametrize("n_chunks,flags", [(1, 3), (3, 3), (2, 1)])
def test_ans_coder_roundtrip_size_and_streams(nc, m2, w2, n_chunks, flags):
    """NEXT-4 rANS (D39): NC_CODER_ANS containers round-trip through the device rANS decoder;
    the size is within 0.5 % of the oracle pipeline with coder="ans"; every chunk stream is
    the oracle rANS encoder's bytes of the walk's own (cum, freq) pairs (the coder is the
    same function on both sides, the pairs come from the GPU walk); and the coder costs at
    most 12 bytes per chunk over the WNC container of the same input (the 64-bit flush plus
    a partial word)."""
    import struct
    from oracle.ans import AnsEncoder
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("alice", 4096, 1001)
    prm = nc.nc_params_default(window=512, slide=128, n_chunks=n_chunks, flags=flags, coder=nc._lib.CODER_ANS)
    blob = nc.nc_compress(m2, data, prm)
    assert nc.nc_decompress(m2, blob, prm) == data
    size, _, xs, ts = _oracle_size_and_p(w2, data, Params(window=512, slide=128, n_chunks=n_chunks,
                                                           flags=flags, coder="ans"))
    assert abs(len(blob) - size) <= 0.005 * size, (len(blob), size)
    wnc = nc.nc_compress(m2, data, nc.nc_params_default(window=512, slide=128, n_chunks=n_chunks, flags=flags))
    assert len(wnc) - 2 * n_chunks <= len(blob) <= len(wnc) + 12 * n_chunks, (len(blob), len(wnc))
    n = struct.unpack_from("<BHH", blob, 4)[2]
    table = [struct.unpack_from("<III", blob, 9 + 12 * c) for c in range(n)]
    off = 9 + 12 * n
    for c in range(n):
        z = nc.nc_debug_forward(m2, xs[c], prm, 0)
        cum, freq, _ = nc.nc_debug_walk(z, ts[c], nc.nc_params_default(window=512, slide=128, n_chunks=n,
                                                                       flags=flags))
        enc = AnsEncoder()
        for a, f in zip(cum, freq):
            enc.encode(int(a), int(f), 1 << 24)
        ref, ref_bits = enc.finish()
        assert table[c][:2] == (len(ts[c]), ref_bits), c
        assert blob[off:off + table[c][2]] == ref, c
        off += table[c][2]


def test_ans_coder_detects_wrong_coder_and_corruption(nc, m2):
    """rANS integrity (D39): a container decoded with the other coder, and any single bit flip
    in an rANS stream (its flush words, the middle, its last word) end in NC_ERR_INTEGRITY --
    the decoder must finish in the encoder's start state 2^31 with every word read."""
    import struct
    from synth import make_text
    data = make_text("alice", 1500, 5)
    ans = nc.nc_params_default(window=256, slide=128, n_chunks=1, coder=nc._lib.CODER_ANS)
    wnc = nc.nc_params_default(window=256, slide=128, n_chunks=1)
    blob = nc.nc_compress(m2, data, ans)
    assert nc.nc_decompress(m2, blob, ans) == data
    for p_enc, p_dec in ((ans, wnc), (wnc, ans)):
        b = nc.nc_compress(m2, data, p_enc)
        with pytest.raises(nc.NcError) as ei:
            nc.nc_decompress(m2, b, p_dec)
        assert ei.value.status == nc._lib.NC_ERR_INTEGRITY
    bits = struct.unpack_from("<I", blob, 13)[0]
    assert bits % 32 == 0
    s0 = 21
    for bit in [0, 5, 31, 40, 63, bits // 3, bits // 2, bits - 33, bits - 9, bits - 1]:
        corrupt = bytearray(blob)
        corrupt[s0 + bit // 8] ^= 0x80 >> (bit % 8)
        with pytest.raises(nc.NcError) as ei:
            nc.nc_decompress(m2, bytes(corrupt), ans)
        assert ei.value.status == nc._lib.NC_ERR_INTEGRITY, bit
    with pytest.raises(nc.NcError):   # a trailing byte after the last word
        nc.nc_decompress(m2, blob[:17] + struct.pack("<I", struct.unpack_from("<I", blob, 17)[0] + 1) + blob[21:] + b"\0",
                         ans)


def test_ans_coder_with_other_paths(nc, m2):
    """NC_CODER_ANS (D39) composes with every other entry point: NC06 files, the refresh
    window variant (the re-prefill decode), the skip flag, and nc_compress_tokens (device ids)
    == nc_compress (host bytes); every container round-trips and is no more than 12 bytes
    per chunk larger than the WNC container of the same input."""
    from synth import make_text
    ans = nc._lib.CODER_ANS
    data = make_text("mixed", 12000, 91)
    for over in ({}, {"window_variant": 1}, {"flags": 7}):
        p_ans = nc.nc_params_default(window=256, slide=128, n_chunks=2, coder=ans, **over)
        p_wnc = nc.nc_params_default(window=256, slide=128, n_chunks=2, **over)
        b_ans = nc.nc_compress_file(m2, data, p_ans)
        assert nc.nc_decompress_file(m2, b_ans, p_ans) == data, over
        assert len(b_ans) <= len(nc.nc_compress_file(m2, data, p_wnc)) + 12 * 4, over
    text = make_text("alice", 9000, 92)
    prm = nc.nc_params_default(window=256, slide=128, n_chunks=3, coder=ans)
    blob = nc.nc_compress(m2, text, prm)
    cuts = nc.nc_host_split(text, 3)
    toks = [nc.nc_tokenize(m2, text[cuts[c]:cuts[c + 1]], 1)[0] for c in range(len(cuts) - 1)]
    td = torch.from_numpy(np.concatenate(toks).view(np.int32).copy()).cuda()
    s = torch.cuda.current_stream()
    blob2 = nc.nc_compress_tokens(m2, td.data_ptr(), np.array([len(t) for t in toks], np.uint32), prm, s.cuda_stream)
    torch.cuda.synchronize()
    assert blob2 == blob and nc.nc_decompress(m2, blob, prm) == text
