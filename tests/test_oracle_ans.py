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
