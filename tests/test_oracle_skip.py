"""Oracle pins for the confidence-based LLM skip (P:452-469,
alg:compress lines 5-6 and 12; reading D32 in DESIGN.md).

The skip test is H(p_ng) < 1.5 bits after the warmup; a skipped token is coded
with p = p_ng.  Under D32 (the forward still runs, every model updates on every
token) the skip changes only the emitted distribution, never the state."""
import math

import numpy as np
import pytest

from oracle.ensemble import (FLAG_HEAD, FLAG_NGRAM, FLAG_SKIP, SKIP_TAU_BITS, ChunkModel, Params,
                             encode_tokens, entropy_bits_fp64, should_skip)


def test_skip_tau_is_the_papers():
    assert SKIP_TAU_BITS == 1.5          # "H(p_ng) < tau bits, with tau = 1.5"


def test_should_skip_spec_examples_S279_281():
    V = 49152
    one_hot = np.zeros(V)
    one_hot[17] = 1.0
    assert should_skip(one_hot)                          # H = 0 < 1.5
    half = np.zeros(V)
    half[:2] = 0.5
    assert entropy_bits_fp64(half) == 1.0 and should_skip(half)
    assert not should_skip(np.full(V, 1.0 / V))          # H = log2 V = 15.585 bits


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8, 1000, 49152])
def test_entropy_uniform_closed_form(k):
    assert entropy_bits_fp64(np.full(k, 1.0 / k)) == pytest.approx(math.log2(k), abs=1e-12)


def test_entropy_binary_closed_form_and_threshold_side():
    # H([p, 1-p]) = -p log2 p - (1-p) log2 (1-p); on both sides of 1.5 bits with a third mass
    for p in (0.1, 0.25, 0.5, 0.9):
        h = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
        assert entropy_bits_fp64([p, 1 - p]) == pytest.approx(h, abs=1e-15)
    assert should_skip([0.7, 0.2, 0.1])          # 1.157 bits
    assert not should_skip([0.4, 0.3, 0.3])      # 1.571 bits


def _repetitive_stream(V, n, period, seed):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, V, period)
    toks = np.tile(base, n // period + 1)[:n]
    flip = rng.random(n) < 0.05                  # a little noise
    toks[flip] = rng.integers(0, V, flip.sum())
    return [int(t) for t in toks]


def test_skip_emits_png_and_keeps_state_identical():
    V, n = 64, 400
    prm_on = Params(flags=FLAG_NGRAM | FLAG_HEAD | FLAG_SKIP, warmup=100)
    prm_off = Params(flags=FLAG_NGRAM | FLAG_HEAD, warmup=100)
    toks = _repetitive_stream(V, n, 7, 3)
    rng = np.random.default_rng(5)
    Z = rng.standard_normal((n, V))
    on, off = ChunkModel(V, prm_on), ChunkModel(V, prm_off)
    n_skip = 0
    for j, t in enumerate(toks):
        p1, pt1, png1 = on.distribution(Z[j])
        p0, pt0, png0 = off.distribution(Z[j])
        assert np.array_equal(pt1, pt0)
        if j < prm_on.warmup:
            assert not on.last_skipped and png1 is None          # warmup: LLM alone
        if on.last_skipped:
            n_skip += 1
            assert np.array_equal(p1, png1)                      # p = p_ng
            assert entropy_bits_fp64(png1) < 1.5
        elif png1 is not None:
            assert entropy_bits_fp64(png1) >= 1.5
            assert np.array_equal(p1, p0)
        on.update(t, pt1, png1)
        off.update(t, pt0, png0)
        # D32: every model updates on every token, so the skip never changes the state
        assert np.array_equal(on.b, off.b) and np.array_equal(on.lw, off.lw)
    assert n_skip > 50                                            # the path is exercised


def test_skip_off_without_ngram_or_flag():
    V, n = 32, 200
    toks = _repetitive_stream(V, n, 3, 1)
    Z = np.random.default_rng(2).standard_normal((n, V))
    for flags in (FLAG_HEAD | FLAG_SKIP, FLAG_NGRAM | FLAG_HEAD):   # no N-gram / no skip bit
        r = encode_tokens(Z, toks, V, Params(flags=flags, warmup=10))
        assert not any(r["skipped"])


def test_skip_codes_with_png_cost():
    """A skipped token's coded interval is the quantized p_ng of that token."""
    from oracle.cdf import quantize
    V, n = 48, 300
    toks = _repetitive_stream(V, n, 5, 9)
    Z = np.random.default_rng(4).standard_normal((n, V))
    prm = Params(flags=FLAG_NGRAM | FLAG_HEAD | FLAG_SKIP, warmup=50)
    r = encode_tokens(Z, toks, V, prm)
    cm = ChunkModel(V, prm)
    for j, t in enumerate(toks):
        p, pt, png = cm.distribution(Z[j])
        if cm.last_skipped:
            c = quantize(png, prm.T)
            assert (r["cum"][j], r["freq"][j]) == (int(c[:t].sum()), int(c[t]))
        cm.update(t, pt, png)
    assert sum(r["skipped"]) > 0
