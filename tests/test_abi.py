"""CPU tests of the C-ABI library: it loads, exports every symbol include/nc.h
declares, refuses compute without a GPU (no CPU fallback), and its host-side
logic (chunk split, tokenizer, WNC encoder, shard plan) matches the oracle."""
import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2602_19626_b200 as nc
from oracle.chunking import split_chunks
from oracle.coder import Encoder
from oracle.tokenizer import Tokenizer

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def test_exports_every_declared_symbol():
    hdr = (ROOT / "include" / "nc.h").read_text()
    declared = set(re.findall(r"\b(nc_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(nc.EXPORTS), declared ^ set(nc.EXPORTS)
    L = nc.lib()
    for name in declared:
        assert hasattr(L, name), name


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_compute_refused_without_gpu(tmp_path):
    with pytest.raises(nc.NcError) as e:
        nc.Model(tmp_path / "none.ncw")
    assert e.value.status in (nc._lib.NC_ERR_BACKEND, nc._lib.NC_ERR_INVALID)
    with pytest.raises(nc.NcError) as e:
        nc.nc_debug_quantize(np.full(4, 0.25, np.float32), 16)
    assert e.value.status == nc._lib.NC_ERR_BACKEND


def test_host_split_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(400):
        n = int(rng.integers(0, 300))
        data = bytes(rng.choice([10, 97, 98, 32], n, p=[0.05, 0.4, 0.4, 0.15]).astype(np.uint8))
        N = int(rng.integers(1, 12))
        cuts = nc.nc_host_split(data, N)
        ours = [data[a:b] for a, b in zip(cuts, cuts[1:])]
        assert ours == split_chunks(data, N), (data, N)


def test_host_wnc_encoder_matches_oracle():
    rng = np.random.default_rng(1)
    for bits in (16, 24):
        T = 1 << bits
        for trial in range(20):
            n = int(rng.integers(0, 400))
            cum = rng.integers(0, T - 1, n)
            freq = np.array([int(rng.integers(1, T - c + 1)) if rng.random() < 0.3 else
                             int(rng.integers(1, min(64, T - c) + 1)) for c in cum], dtype=np.int64)
            enc = Encoder()
            for c, f in zip(cum, freq):
                enc.encode(int(c), int(f), T)
            ref, ref_bits = enc.finish()
            s, b = nc.nc_host_wnc_encode(cum, freq, bits)
            assert (s, b) == (ref, ref_bits)


def test_host_ans_encoder_matches_oracle():
    """NC_CODER_ANS's host encoder (D39) writes the oracle rANS encoder's bytes, and the
    oracle rANS decoder recovers the symbols from them (every renormalisation branch: tiny
    and near-T frequencies, 16 and 24 bits)."""
    from oracle.ans import AnsDecoder, AnsEncoder
    rng = np.random.default_rng(11)
    for bits in (16, 24):
        T = 1 << bits
        for trial in range(20):
            n = int(rng.integers(0, 400))
            cum = rng.integers(0, T - 1, n)
            freq = np.array([int(rng.integers(1, T - c + 1)) if rng.random() < 0.3 else
                             int(rng.integers(1, min(64, T - c) + 1)) for c in cum], dtype=np.int64)
            enc = AnsEncoder()
            for c, f in zip(cum, freq):
                enc.encode(int(c), int(f), T)
            ref, ref_bits = enc.finish()
            s, b = nc.nc_host_ans_encode(cum, freq, bits)
            assert (s, b) == (ref, ref_bits)
            dec = AnsDecoder(s)
            for c, f in zip(cum, freq):   # a two-symbol-per-step CDF around each pair
                cdf = np.array([0, int(c), int(c) + int(f), T]) if c else np.array([0, int(f), T])
                sym = dec.decode(cdf, T)
                assert int(cdf[sym]) == int(c) and int(cdf[sym + 1] - cdf[sym]) == int(f)
            assert dec.finished_ok()


def test_host_tokenizer_matches_oracle():
    from synth import make_text, make_vocab
    vocab = make_vocab(49152)
    tk = Tokenizer(vocab)
    for kind, seed in (("alice", 3), ("enwik", 4)):
        data = make_text(kind, 20000, seed)
        assert nc.nc_host_tokenize_vocab(vocab, data) == tk.encode(data)
    rng = np.random.default_rng(2)
    data = bytes(rng.integers(0, 256, 5000).astype(np.uint8))
    assert nc.nc_host_tokenize_vocab(vocab, data) == tk.encode(data)


def test_host_tokenizer_duplicate_lowest_id():
    """D30: duplicate vocabulary strings -> the lowest id (same rule as oracle/tokenizer.py)."""
    vocab = [b"<0>", b"<1>", b"<2>"] + [bytes([i]) for i in range(256)] + [b"xy", b"q", b"xy"]
    assert nc.nc_host_tokenize_vocab(vocab, b"xy") == [259]
    assert nc.nc_host_tokenize_vocab(vocab, b"q") == [ord("q") + 3]


def test_shard_range_covers():
    for n in range(0, 40):
        for world in (1, 2, 3, 8):
            ranges = [nc.nc_host_shard_range(n, world, r) for r in range(world)]
            flat = [c for a, b in ranges for c in range(a, b)]
            assert flat == list(range(n))


def test_params_default():
    p = nc.nc_params_default()
    assert (p.cdf_bits, p.flags, p.window, p.slide, p.warmup, p.ngram_orders, p.ngram_cap) == \
        (24, 3, 2048, 512, 100, 4, 500000)
    assert p.alpha == 1e-3 and p.eta == 1.0 and p.temperature == 1.0


# ------------------------------------------------------------------ NC06 host ---
def test_host_segment_equals_oracle():
    """the C++ segmenter (NC06 rules 1-4) is bit-identical with the oracle's on
    mixed files and on random short inputs"""
    from oracle import nc06
    from synth import make_text
    for seed in range(4):
        data = make_text("mixed", 40000, 900 + seed)
        assert nc.nc_host_segment(data) == nc06.segment(data)
    rng = np.random.default_rng(5)
    for _ in range(300):
        d = bytes(rng.choice([0, 1, 9, 65, 97, 200], int(rng.integers(0, 300))).astype(np.uint8))
        assert nc.nc_host_segment(d) == nc06.segment(d)
    assert nc.nc_host_segment(b"") == []


def test_host_blob_codec_interoperates_with_oracle():
    """C++ blob codec vs the oracle's (Python lzma / zlib): same method choice, the same
    DEFLATE / raw bytes (the .xz framing of liblzma's buffer encoder differs from Python's
    stream encoder by a few header bytes), and each decodes the other's payload."""
    from oracle import nc06
    rng = np.random.default_rng(6)
    cases = [b"", bytes(8192), bytes(rng.integers(0, 256, 100).astype(np.uint8)), b"\x00\x01" * 500,
             bytes(rng.integers(0, 4, 20000).astype(np.uint8)), bytes(rng.integers(0, 256, 5000).astype(np.uint8))]
    for blob in cases:
        m, c = nc.nc_host_blob_encode(blob)
        mo, co = nc06.blob_encode(blob)
        assert m == mo, (len(blob), m, mo)
        if m != 2:
            assert c == co
        else:
            assert abs(len(c) - len(co)) <= 16
        assert nc.nc_host_blob_decode(mo, co, len(blob)) == blob
        assert nc06.blob_decode(m, c) == blob
    with pytest.raises(nc.NcError) as ei:
        nc.nc_host_blob_decode(1, b"\x78\x9c garbage", 10)
    assert ei.value.status == nc._lib.NC_ERR_INTEGRITY
