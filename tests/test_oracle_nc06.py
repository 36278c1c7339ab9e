"""Oracle pins for NC06 (P:512-528 hybrid binary format).

Segmenter: SPEC's worked examples, the rule thresholds at their boundaries
(63/64-byte text runs, 8/9-byte gaps, 63/64-byte binary chunks), and an independent
implementation of the four rules as regular-expression rewrites of the byte-class label
string (a different algorithm from the oracle's region lists).  Blob codec: S:472-476's
examples and library round trips.  Container: golden bytes, read/write identity, errors.
Pipeline: round trips of mixed files with the tiny model."""
import re
import struct

import numpy as np
import pytest

from oracle import nc06
from oracle.container import FormatError
from oracle.ensemble import Params


def test_classify_examples_S387():
    assert nc06.is_text_byte(65) and nc06.is_text_byte(9) and not nc06.is_text_byte(0)
    assert nc06.is_text_byte(10) and nc06.is_text_byte(13) and nc06.is_text_byte(32) and nc06.is_text_byte(126)
    assert not nc06.is_text_byte(127) and not nc06.is_text_byte(31) and not nc06.is_text_byte(0xC3)


def test_segment_examples_S391():
    assert nc06.segment(b"a" * 200) == [(nc06.TEXT, 200)]
    assert nc06.segment(b"a" * 32) == [(nc06.BINARY, 32)]
    assert nc06.segment(b"a" * 100 + b"\x00" * 5 + b"a" * 100) == [(nc06.TEXT, 205)]
    assert nc06.segment(b"") == []


def test_segment_rule_boundaries():
    T, B = nc06.TEXT, nc06.BINARY
    big = bytes(range(128, 256)) * 4                        # 512 binary bytes
    # rule 2: 63 demoted, 64 kept
    assert nc06.segment(big + b"x" * 63 + big) == [(B, 1087)]
    assert nc06.segment(big + b"x" * 64 + big) == [(B, 512), (T, 64), (B, 512)]
    # rule 3: a gap of 8 bridged, 9 not (then rule 4 absorbs the 9 as < 64 adjacent to text)
    assert nc06.segment(b"x" * 100 + b"\x01" * 8 + b"y" * 100) == [(T, 208)]
    assert nc06.segment(big + b"x" * 100 + b"\x01" * 9 + b"y" * 100 + big) == [(B, 512), (T, 209), (B, 512)]
    # rule 4: 63 absorbed, 64 not
    assert nc06.segment(b"x" * 100 + b"\x01" * 63) == [(T, 163)]
    assert nc06.segment(b"x" * 100 + b"\x01" * 64) == [(T, 100), (B, 64)]


def _segment_regex(data: bytes):
    """the four rules as rewrites of the label string (independent of the oracle)."""
    lab = "".join("T" if (32 <= b <= 126 or b in (9, 10, 13)) else "B" for b in data)
    lab = re.sub(r"T+", lambda m: m.group(0) if len(m.group(0)) >= 64 else "B" * len(m.group(0)), lab)
    lab = re.sub(r"(?<=T)B{1,8}(?=T)", lambda m: "T" * len(m.group(0)), lab)
    lab = re.sub(r"(?<=T)B{1,63}(?!B)|(?<!B)B{1,63}(?=T)", lambda m: "T" * len(m.group(0)), lab)
    return [(nc06.TEXT if m.group(0)[0] == "T" else nc06.BINARY, len(m.group(0)))
            for m in re.finditer(r"T+|B+", lab)]


@pytest.mark.parametrize("seed", range(8))
def test_segment_equals_regex_rules_and_invariants(seed):
    from synth import make_text
    data = make_text("mixed", 30000 + 1000 * seed, 500 + seed)
    regs = nc06.segment(data)
    assert regs == _segment_regex(data)
    assert sum(ln for _, ln in regs) == len(data)
    assert all(a[0] != b[0] for a, b in zip(regs, regs[1:]))            # alternate
    assert all(ln >= 64 for k, ln in regs if k == nc06.TEXT)
    assert len({k for k, _ in regs}) == 2                                # the generator gives both
    text, binary = nc06.split(data, regs)
    assert len(text) + len(binary) == len(data)
    # random short inputs, including pathological alternations
    rng = np.random.default_rng(seed)
    for _ in range(200):
        d = bytes(rng.choice([0, 1, 65, 97, 200, 10], int(rng.integers(0, 400))).astype(np.uint8))
        assert nc06.segment(d) == _segment_regex(d)


def test_blob_codec_S472():
    m, c = nc06.blob_encode(bytes(8192))
    assert m == nc06.LZMA and len(c) < 300 and nc06.blob_decode(m, c) == bytes(8192)
    r = bytes(np.random.default_rng(1).integers(0, 256, 100).astype(np.uint8))
    assert nc06.blob_encode(r) == (nc06.RAW, r)
    assert nc06.blob_encode(b"") == (nc06.RAW, b"")
    m, c = nc06.blob_encode(b"\x00\x01" * 500)                           # < 4 KB: DEFLATE
    assert m == nc06.DEFLATE and nc06.blob_decode(m, c) == b"\x00\x01" * 500
    import lzma
    import zlib
    assert nc06.blob_decode(nc06.DEFLATE, zlib.compress(b"abc" * 50)) == b"abc" * 50
    assert nc06.blob_decode(nc06.LZMA, lzma.compress(b"abc" * 5000)) == b"abc" * 5000


def test_nc06_golden_bytes_and_errors():
    blob = nc06.write_nc06(7, 1000, [(1, 100), (0, 5)], nc06.RAW, b"\x00" * 5, [(5, 17, b"\xaa\xbb\xcc")])
    want = (b"NC06" + bytes([1, 7]) + bytes([0xE8, 0x03]) + bytes([2, 0]) +
            bytes([1, 100, 0, 0, 0]) + bytes([0, 5, 0, 0, 0]) + bytes([0, 5, 0, 0, 0]) + b"\x00" * 5 +
            bytes([1, 0]) + bytes([5, 0, 0, 0, 17, 0, 0, 0, 3, 0, 0, 0]) + b"\xaa\xbb\xcc")
    assert blob == want
    assert nc06.read_nc06(blob) == (7, 1000, [(1, 100), (0, 5)], nc06.RAW, b"\x00" * 5, [(5, 17, b"\xaa\xbb\xcc")])
    for bad in (b"NC05" + blob[4:], blob[:4] + b"\x02" + blob[5:], blob[:-1], blob + b"\x00", blob[:8]):
        with pytest.raises(FormatError):
            nc06.read_nc06(bad)


@pytest.mark.parametrize("kind", ["mixed", "binary", "text3"])
def test_nc06_pipeline_roundtrip(tiny_weights, kind):
    from synth import make_text
    if kind == "mixed":
        data = make_text("mixed", 6000, 71)
    elif kind == "binary":
        data = bytes(np.random.default_rng(2).integers(0, 256, 3000).astype(np.uint8))
    else:
        data = make_text("alice", 700, 3) + bytes(range(128, 256)) * 4 + make_text("alice", 500, 4)
    prm = Params(window=16, slide=4, n_chunks=2)
    blob = nc06.compress_file(data, tiny_weights, prm)
    assert nc06.decompress_file(blob, tiny_weights, prm) == data
    _, _, regs, method, payload, chunks = nc06.read_nc06(blob)
    assert sum(ln for _, ln in regs) == len(data)
    if kind == "binary":
        assert regs == [(nc06.BINARY, 3000)] and sum(n for n, _, _ in chunks) == 0
    if kind == "text3":
        assert [k for k, _ in regs] == [nc06.TEXT, nc06.BINARY, nc06.TEXT]
