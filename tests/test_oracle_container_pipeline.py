"""Oracle pins: NC05 container, chunking,
tokenizer round trip and whole-pipeline losslessness."""
import json
import os

import numpy as np
import pytest

from oracle.chunking import split_chunks
from oracle.compressor import compress, decompress
from oracle.container import FormatError, read_nc05, write_nc05
from oracle.ensemble import Params
from oracle.tokenizer import Tokenizer

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_nc05_golden_bytes():
    assert write_nc05(7, 1000, []).hex() == G["nc05_golden_header_flags7_tau1_chunks0"]["hex"]
    assert len(write_nc05(7, 1000, [])) == G["nc05_header_bytes"]["value"]
    b = write_nc05(3, 1000, [(5, 17, b"\x01\x02\x03")])
    assert b[9:21].hex() == G["nc05_golden_entry_5_17_3"]["hex"]
    assert read_nc05(b) == (3, 1000, [(5, 17, b"\x01\x02\x03")])


def test_nc05_errors():
    good = write_nc05(3, 1000, [(5, 17, b"abc")])
    with pytest.raises(FormatError):
        read_nc05(b"NC99" + good[4:])
    with pytest.raises(FormatError):
        read_nc05(good[:12])
    with pytest.raises(FormatError):
        read_nc05(good[:4] + bytes([0x08]) + good[5:])
    with pytest.raises(FormatError):
        write_nc05(3, 1000, [(5, 17, b"ab")])


def test_split_chunks_examples():
    assert split_chunks(b"abcdefghi", 3) == [b"abc", b"def", b"ghi"]      # hard split
    # target 4 -> first newline at/after index 4 is index 5 -> cut after it
    assert split_chunks(b"a\nb\nc\nd", 2) == [b"a\nb\nc\n", b"d"]
    assert split_chunks(b"hello", 1) == [b"hello"]
    assert split_chunks(b"", 4) == [b""]
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(0, 200))
        data = bytes(rng.choice([10, 97, 98], n, p=[0.1, 0.45, 0.45]).astype(np.uint8))
        N = int(rng.integers(1, 10))
        ch = split_chunks(data, N)
        assert b"".join(ch) == data and 1 <= len(ch) <= N
        assert all(len(c) > 0 for c in ch) or data == b""


def test_tokenizer_roundtrip(tiny_weights):
    tk = Tokenizer(tiny_weights.vocab)
    rng = np.random.default_rng(1)
    for _ in range(50):
        data = bytes(rng.integers(0, 256, int(rng.integers(0, 300))).astype(np.uint8))
        ids = tk.encode(data)
        assert tk.decode(ids) == data and all(i >= 3 for i in ids)
    assert tk.encode(b"") == []


def test_tokenizer_greedy_longest_match():
    vocab = [b"<0>", b"<1>", b"<2>"] + [bytes([i]) for i in range(256)] + [b"ab", b"abc", b"bcd"]
    tk = Tokenizer(vocab)
    assert [vocab[i] for i in tk.encode(b"abcd")] == [b"abc", b"d"]
    assert [vocab[i] for i in tk.encode(b"abd")] == [b"ab", b"d"]


def test_tokenizer_duplicate_string_lowest_id_wins():
    """D30: a string present under several ids tokenizes to the LOWEST id.  The
    synthetic vocabulary has no duplicates (synth/vocab.py), so this only fixes the rule
    the oracle and the C++ tokenizer share; the C++ side is checked in test_abi.py."""
    vocab = [b"<0>", b"<1>", b"<2>"] + [bytes([i]) for i in range(256)] + [b"xy", b"q", b"xy"]
    tk = Tokenizer(vocab)
    assert tk.encode(b"xy") == [259]
    assert tk.encode(b"q") == [ord("q") + 3]                     # the byte token (id 116) beats id 260
    assert tk.decode(tk.encode(b"xyqxy")) == b"xyqxy"


@pytest.mark.parametrize("flags,bits,chunks", [(3, 24, 1), (3, 24, 3), (0, 16, 2), (1, 24, 2), (2, 16, 1),
                                              (7, 24, 2), (5, 16, 1)])   # 4 = confidence skip (NEXT-1)
def test_pipeline_roundtrip(tiny_weights, flags, bits, chunks):
    from synth import make_text
    data = make_text("alice", 900, 77 + flags)
    prm = Params(window=16, slide=4, warmup=20, n_chunks=chunks, flags=flags, cdf_bits=bits)
    blob = compress(data, tiny_weights, prm)
    assert decompress(blob, tiny_weights, prm) == data
    f, tau, ents = read_nc05(blob)
    assert f == flags and tau == 1000 and len(ents) <= chunks


@pytest.mark.parametrize("refresh,lm1", [(True, False), (False, True), (True, True)])
def test_pipeline_window_variants_roundtrip(tiny_weights, refresh, lm1):
    """NEXT-4 window variants through the whole oracle pipeline: blocked compress and the
    literal incremental decompress agree (round trip), and both literal and blocked LM
    modes give the same stream."""
    from synth import make_text
    data = make_text("alice", 700, 77)
    prm = Params(window=16, slide=4, n_chunks=2, refresh=refresh, lmax_minus_one=lm1)
    blob = compress(data, tiny_weights, prm)
    assert decompress(blob, tiny_weights, prm) == data
    assert compress(data, tiny_weights, prm, lm_mode="literal") == blob
    assert blob != compress(data, tiny_weights, Params(window=16, slide=4, n_chunks=2))


@pytest.mark.parametrize("flags,bits,chunks", [(3, 24, 2), (0, 16, 1), (7, 24, 1)])
def test_pipeline_ans_roundtrip(tiny_weights, flags, bits, chunks):
    """the rANS coder through the whole oracle pipeline: round trip, and the
    same per-token counts as the arithmetic coder (only the entropy coder differs), so the
    two container sizes differ by the coders' few bytes of overhead per chunk"""
    from synth import make_text
    data = make_text("alice", 900, 31)
    pa = Params(window=16, slide=4, n_chunks=chunks, flags=flags, cdf_bits=bits, coder="ans")
    pw = Params(window=16, slide=4, n_chunks=chunks, flags=flags, cdf_bits=bits)
    blob = compress(data, tiny_weights, pa)
    assert decompress(blob, tiny_weights, pa) == data
    ra, rw = [], []
    compress(data, tiny_weights, pa, collect=ra)
    compress(data, tiny_weights, pw, collect=rw)
    assert [r["freq"] for r in ra] == [r["freq"] for r in rw]
    assert abs(len(blob) - len(compress(data, tiny_weights, pw))) <= 12 * chunks


def test_pipeline_empty_and_binary(tiny_weights):
    prm = Params(window=16, slide=4, warmup=5, n_chunks=2)
    for data in (b"", b"\x00\x01\xff" * 10, b"\n\n\n"):
        assert decompress(compress(data, tiny_weights, prm), tiny_weights, prm) == data


def test_pipeline_literal_lm_same_stream(tiny_weights):
    from synth import make_text
    data = make_text("alice", 400, 5)
    prm = Params(window=8, slide=2, warmup=10)
    assert compress(data, tiny_weights, prm) == compress(data, tiny_weights, prm, lm_mode="literal")
