"""Oracle pins for the rANS coder (the paper's future work; SURVEY NEXT-4 ANS).

Pins: exact round trips over the method's own integer CDFs (quantize of random
distributions at V in {2, 256, 49152}, T in {2^16, 2^24}) with the decoder's state back at
its start state L; the code length against the entropy of the coded counts (sum log2(T/freq)
+ 96 bits); S:42's i.i.d. example (probabilities 1/2, 1/4, 1/8, 1/8 -> 1.75 bits/symbol
within 1 %); the empty stream; and a single-word corruption detected by the end-state check."""
import numpy as np
import pytest

from oracle.ans import L, AnsDecoder, AnsEncoder, code_length_bound
from oracle.cdf import quantize


def _random_cdfs(V, T, n, rng):
    out = []
    for _ in range(n):
        z = rng.standard_normal(V) * rng.uniform(0.1, 6.0)
        p = np.exp(z - z.max())
        c = quantize((p / p.sum()).astype(np.float32), T)
        out.append(np.concatenate([[0], np.cumsum(c)]))
    return out


@pytest.mark.parametrize("V,bits", [(2, 16), (256, 16), (256, 24), (49152, 24)])
def test_ans_roundtrip_and_bound(V, bits):
    T = 1 << bits
    rng = np.random.default_rng(V + bits)
    n = 400 if V > 1000 else 3000
    cdfs = _random_cdfs(V, T, 40, rng)
    syms, freqs, enc = [], [], AnsEncoder()
    for i in range(n):
        cum = cdfs[i % len(cdfs)]
        s = int(rng.integers(V)) if rng.random() < 0.3 else int(np.argmax(np.diff(cum)))
        enc.encode(int(cum[s]), int(cum[s + 1] - cum[s]), T)
        syms.append(s)
        freqs.append(int(cum[s + 1] - cum[s]))
    stream, nbits = enc.finish()
    assert nbits == 8 * len(stream) and nbits % 32 == 0
    assert nbits <= code_length_bound(freqs, T)
    assert nbits >= np.log2(T / np.asarray(freqs, np.float64)).sum() - 64
    dec = AnsDecoder(stream)
    out = [dec.decode(cdfs[i % len(cdfs)], T) for i in range(n)]
    assert out == syms and dec.finished_ok()


def test_ans_iid_entropy_S42():
    T = 1 << 16
    cum = np.array([0, T // 2, 3 * T // 4, 7 * T // 8, T])
    rng = np.random.default_rng(42)
    syms = rng.choice(4, size=100000, p=[0.5, 0.25, 0.125, 0.125])
    enc = AnsEncoder()
    for s in syms:
        enc.encode(int(cum[s]), int(cum[s + 1] - cum[s]), T)
    stream, nbits = enc.finish()
    ideal = 1.75 * len(syms)
    assert abs(nbits - np.log2(T / np.diff(cum)[syms]).sum()) <= 96
    assert abs(nbits - ideal) <= 0.01 * ideal + 96
    dec = AnsDecoder(stream)
    assert [dec.decode(cum, T) for _ in syms] == list(syms) and dec.finished_ok()


def test_ans_empty_and_corruption():
    stream, nbits = AnsEncoder().finish()
    assert nbits == 64 and AnsDecoder(stream).x == L and AnsDecoder(stream).finished_ok()
    T = 1 << 24
    rng = np.random.default_rng(3)
    cdfs = _random_cdfs(256, T, 8, rng)
    enc, syms = AnsEncoder(), []
    for i in range(2000):
        cum = cdfs[i % 8]
        s = int(rng.integers(256))
        enc.encode(int(cum[s]), int(cum[s + 1] - cum[s]), T)
        syms.append(s)
    stream, _ = enc.finish()
    bad = bytearray(stream)
    bad[len(bad) // 2] ^= 0x10
    dec = AnsDecoder(bytes(bad))
    out = [dec.decode(cdfs[i % 8], T) for i in range(2000)]
    assert out != syms or not dec.finished_ok()
    assert not dec.finished_ok()


def test_ans_one_and_two_symbol_closed_forms():
    """hand-derived streams: one symbol from the start state L (no renormalisation, since
    L < ((L >> b) << 32) freq) is the 8-byte big-endian x = floor(L / f) T + (L mod f) + c;
    a second symbol first in coding order (encoded last) applies the same map to that x,
    renormalising once when x >= ((L >> b) << 32) f (its low word goes to the stream END)."""
    T, b = 1 << 16, 16
    c, f = 1234, 777
    x1 = (L // f) * T + L % f + c
    assert AnsEncoder().finish() == (L.to_bytes(8, "big"), 64)
    e = AnsEncoder()
    e.encode(c, f, T)
    assert e.finish() == (x1.to_bytes(8, "big"), 64)
    c, f = 1234, 1                         # x1 = 2^47 + c
    x1 = (L // f) * T + L % f + c
    c2, f2 = 5, 1                          # x1 >= ((L >> 16) << 32) * 1 = 2^47 -> one word out
    assert x1 >= ((L >> b) << 32) * f2
    y = x1 >> 32
    x2 = (y // f2) * T + y % f2 + c2
    e = AnsEncoder()
    e.encode(c2, f2, T)                    # decoded first
    e.encode(c, f, T)
    data, nbits = e.finish()
    assert data == x2.to_bytes(8, "big") + (x1 & 0xFFFFFFFF).to_bytes(4, "big") and nbits == 96
    d = AnsDecoder(data)
    assert d.decode(np.array([0, c2, c2 + f2, T]), T) == 1
    assert d.decode(np.array([0, c, c + f, T]), T) == 1 and d.finished_ok()
