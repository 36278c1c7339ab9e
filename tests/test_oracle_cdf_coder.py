"""Oracle pins: CDF-24 quantizer and the WNC coder.

Every expected value is printed in PAPER.md / SPEC.md (tests/golden/paper_values.json),
a closed form, an exact-rational recomputation, or an invariant."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle.cdf import QuantizeError, entropy_bits, floor_fraction, floor_overhead_bits, quantize
from oracle.coder import Decoder, Encoder, find_symbol

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
V = G["V"]["value"]


def test_floor_fraction_and_overhead_paper_values():
    assert floor_fraction(V, 1 << 16) == G["cdf16_floor_fraction"]["value"]
    assert (1 << 16) - V == G["cdf16_remaining"]["value"]
    assert floor_overhead_bits(V, 1 << 16) == G["cdf16_overhead_bits"]["value"]
    T24 = G["cdf24_T"]["value"]
    assert T24 == 1 << 24
    assert abs(100 * floor_fraction(V, T24) - 0.29) < G["cdf24_floor_fraction_pct"]["tol"]
    assert abs(floor_overhead_bits(V, T24) - 0.004) < G["cdf24_overhead_bits"]["tol"]
    # D1: the printed 16,727,064 is garbled; T - V is 16,728,064
    assert T24 - V == G["cdf24_remaining_reading"]["value"] != G["cdf24_remaining_printed"]["value"]


def test_quantize_worked_examples():
    c = quantize(np.full(4, 0.25), 16)
    assert c.tolist() == G["quantize_uniform_V4_T16"]["counts"]
    assert np.concatenate([[0], np.cumsum(c)]).tolist() == G["quantize_uniform_V4_T16"]["cum"]
    p = np.zeros(V)
    p[0] = 1.0
    c = quantize(p, 1 << 16)
    assert c[0] == G["quantize_onehot_V49152_T65536"]["c0"] and (c[1:] == 1).all()
    assert quantize(np.array([1.0, 0.0]), 1 << 24).tolist() == G["quantize_onehot_V2_T2p24"]["counts"]


def test_quantize_infeasible():
    with pytest.raises(QuantizeError):
        quantize(np.full(16, 1 / 16), 16)


@pytest.mark.parametrize("Vs,T", [(4, 16), (256, 1 << 16), (V, 1 << 16), (V, 1 << 24)])
def test_quantize_invariants_fuzz(Vs, T):
    rng = np.random.default_rng(Vs + T)
    for trial in range(20):
        z = rng.standard_normal(Vs) * (1 + 4 * rng.random())
        p = np.exp(z - z.max())
        p /= p.sum()
        c = quantize(p, T)
        assert c.sum() == T and (c >= 1).all()
        a = int(np.argmax(p))
        assert c[a] == c.max()


def test_quantize_exact_rational_on_fp32():
    """D5: floor(p_f32 * (T-V)) in fp64 is exact; compare with Fraction arithmetic."""
    rng = np.random.default_rng(3)
    T = 1 << 24
    p = rng.random(V).astype(np.float32)
    p /= p.sum()
    p = p.astype(np.float32)
    c = quantize(p, T)
    a = int(np.argmax(p))
    idx = rng.choice(V, 500, replace=False)
    for i in idx:
        if i == a:
            continue
        exact = math.floor(Fraction(float(p[i])) * (T - V))
        assert c[i] == max(1, exact)


def test_quantize_ties_lowest_index():
    c = quantize(np.array([0.25, 0.25, 0.25, 0.25]), 16)
    assert c[0] == 7   # residual to index 0 (D4)


def test_negative_residual():
    """D6: sum(p) slightly above 1 with floors saturated -> negative residual is applied."""
    Vs, T = 8, 64
    p = np.array([1.05] + [0.0] * 7)          # floors saturated, sum(p) > 1
    c = quantize(p, T)
    assert c.sum() == T and (c >= 1).all()
    assert c[0] == math.floor(1.05 * (T - Vs)) + (T - math.floor(1.05 * (T - Vs)) - 7) == 57
    with pytest.raises(QuantizeError):
        quantize(np.array([1.0, 1.0, 1.0]), 8)   # others alone exceed T


def test_entropy_bits():
    assert entropy_bits([1.0, 0.0]) == 0.0
    assert entropy_bits([0.5, 0.5]) == 1.0
    assert abs(entropy_bits(np.full(V, 1 / V)) - math.log2(V)) < 1e-9


# ---------------------------------------------------------------- coder -----

def test_decode_search_examples():
    g = G["decode_search"]
    for target, sym in g["cases"]:
        assert find_symbol(g["cum"], target) == sym


def _roundtrip(Vs, T, n, rng, peaked=False):
    enc = Encoder()
    syms, cdfs = [], []
    for _ in range(n):
        z = rng.standard_normal(Vs) * (6 if peaked else 1)
        p = np.exp(z - z.max())
        p /= p.sum()
        c = quantize(p, T)
        cum = np.concatenate([[0], np.cumsum(c)])
        s = int(rng.choice(Vs, p=p))
        enc.encode(int(cum[s]), int(c[s]), T)
        syms.append(s)
        cdfs.append(cum)
    stream, bits = enc.finish()
    assert len(stream) == (bits + 7) // 8
    dec = Decoder(stream)
    out = [dec.decode(cum, T) for cum in cdfs]
    assert out == syms
    return enc


@pytest.mark.parametrize("Vs", [2, 256, V])
@pytest.mark.parametrize("bits", [16, 24])
def test_coder_roundtrip_fuzz(Vs, bits):
    rng = np.random.default_rng(Vs * 31 + bits)
    n = 300 if Vs == V else 2000
    enc = _roundtrip(Vs, 1 << bits, n, rng, peaked=True)
    assert enc.min_range > (1 << 30)          # D7 invariant


def test_paper_range_claim_is_wrong_d7():
    """P:351-356 claims R >= 2^31 after renormalization; D7: only R > 2^30 holds."""
    rng = np.random.default_rng(5)
    enc = Encoder()
    T = 1 << 24
    seen_below = False
    for _ in range(20000):
        lo = int(rng.integers(0, T - 1))
        f = int(rng.integers(1, T - lo + 1))
        enc.encode(lo, f, T)
        r = enc.high - enc.low + 1
        assert r > (1 << 30)
        seen_below |= r < (1 << 31)
    assert seen_below


def test_coder_entropy_bound_S42():
    """10^5 iid symbols of [.5,.25,.125,.125] with the exact CDF -> <= n*1.75*1.01 + 64 bits."""
    rng = np.random.default_rng(42)
    n, T = 100_000, 1 << 24
    cum = [0, T // 2, 3 * T // 4, 7 * T // 8, T]
    syms = rng.choice(4, n, p=[0.5, 0.25, 0.125, 0.125])
    enc = Encoder()
    for s in syms:
        enc.encode(cum[s], cum[s + 1] - cum[s], T)
    stream, bits = enc.finish()
    ideal = sum(-math.log2((cum[s + 1] - cum[s]) / T) for s in syms)
    assert bits <= n * 1.75 * 1.01 + 64
    assert bits >= ideal - 1
    dec = Decoder(stream)
    cum_a = np.array(cum)
    assert all(dec.decode(cum_a, T) == s for s in syms[:5000])


def test_coder_hard_bound_8c():
    """bits <= sum[-log2(f/T) - log2(1 - 2^(b-30)/f)] + 64 (R > 2^30)."""
    rng = np.random.default_rng(9)
    for b in (16, 24):
        T = 1 << b
        enc = Encoder()
        bound = 0.0
        for _ in range(5000):
            lo = int(rng.integers(0, T - 1))
            f = int(rng.integers(1, min(T - lo, 1 << (b - 4)) + 1))
            enc.encode(lo, f, T)
            bound += -math.log2(f / T) - math.log2(1 - 2 ** (b - 30) / f)
        _, bits = enc.finish()
        assert bits <= bound + 64


def test_coder_empty_and_single():
    enc = Encoder()
    stream, bits = enc.finish()
    assert bits <= 16 and len(stream) == (bits + 7) // 8
    enc = Encoder()
    enc.encode(1 << 23, 1 << 23, 1 << 24)
    stream, bits = enc.finish()
    assert len(stream) <= 5
    assert Decoder(stream).decode(np.array([0, 1 << 23, 1 << 24]), 1 << 24) == 1


def test_cdf16_vs_cdf24_two_bits_S43():
    """S:43 / P:331-334: a peaked p (0.99 on one of 49,152) costs ~2 bits more per
    token at T=2^16 than at 2^24; measured through the real coder."""
    rng = np.random.default_rng(11)
    n = 3000
    p = np.full(V, 0.01 / (V - 1))
    p[123] = 0.99
    sizes = {}
    for b in (16, 24):
        T = 1 << b
        c = quantize(p, T)
        cum = np.concatenate([[0], np.cumsum(c)])
        enc = Encoder()
        rs = np.random.default_rng(1)
        for _ in range(n):
            s = 123 if rs.random() < 0.99 else int(rs.integers(V))
            enc.encode(int(cum[s]), int(c[s]), T)
        sizes[b] = enc.finish()[1]
    diff = (sizes[16] - sizes[24]) / n
    assert 1.8 <= diff <= 2.2, diff
