"""GPU parity of the walk's internals (SURVEY.md §8(d) "probability-parity sampling").

Through nc_debug_walk_dump (the C ABI) the walk exports p~(t) at every row and, on a
sample of rows (the first 200, around the warmup boundary, every 97th, the last), its
full fp32 p~ and p vectors and the integer counts it coded with.  Checked here:

* the walk's counts equal the oracle's quantizer (oracle.cdf.quantize) on the
  walk's own fp32 p, BIT FOR BIT (north_star: "Integer CDFs must be bit-exact given
  identical float inputs"), and every emitted (cum_t, freq_t) is (sum c[:t], c[t]) of
  those counts -- this covers the walk's own quantizer, argmax and residual combine
  (quant4 + the cluster reduction), not only the debug quantizer kernel;
* p~(t) and p(t) at every row, and the full p~ / p vectors on the sampled rows, within
  1e-4 relative of the fp64 oracle walk on the same fp32 logits (north_star bar);
* regimes: random-init-like Gaussian logits, an informative LLM (SPEC.md:364's bigram
  stub) for which the mixer keeps a non-negligible LLM weight, the head alone at V =
  49,152 over 20K tokens (SURVEY D17's f64 bias regime), and 40K-token walks (config 3/4
  chunk length) with flags 3 and 2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P_TOL = 1e-4


@pytest.fixture(scope="module")
def nc():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2602_19626_b200 as m
    return m


def sample_rows(n, warmup, extra=()):
    rows = set(range(min(200, n))) | set(range(0, n, 97)) | {n - 1}
    rows |= {r for r in range(warmup - 2, warmup + 3) if 0 <= r < n}
    rows |= {r for r in extra if 0 <= r < n}
    return sorted(rows)


def check_dump(d, ref, toks, V, bits, warmup):
    """the bit-exact and tolerance checks shared by every test (see the module docstring)."""
    from oracle.cdf import quantize
    T = 1 << bits
    cum, freq = d["cum"].astype(np.int64), d["freq"].astype(np.int64)
    assert (freq >= 1).all() and (cum + freq <= T).all()
    # every row: p(t) and p~(t) within 1e-4 of the oracle
    p_ref, pt_ref = np.array(ref["p_true"]), np.array(ref["pt_true"])
    rel_p = np.abs(d["p_true"] - p_ref) / p_ref
    rel_pt = np.abs(d["pt_true"] - pt_ref) / pt_ref
    assert rel_p.max() < P_TOL, ("p(t)", rel_p.max(), int(rel_p.argmax()))
    assert rel_pt.max() < P_TOL, ("p~(t)", rel_pt.max(), int(rel_pt.argmax()))
    # sampled rows: counts bit-identical to the oracle's quantizer on the walk's own p; the
    # emitted pair is that CDF's entry for the true token; full vectors within tolerance
    for k, r in enumerate(d["rows"]):
        c_ref = quantize(d["p_rows"][k], T)
        assert np.array_equal(d["c_rows"][k].astype(np.int64), c_ref), ("counts", r)
        t = toks[r]
        assert cum[r] == int(c_ref[:t].sum()) and freq[r] == int(c_ref[t]), ("emit", r)
        p_o, pt_o = ref["rows"][r]
        e_pt = np.abs(d["pt_rows"][k] - pt_o) / pt_o
        e_p = np.abs(d["p_rows"][k] - p_o) / p_o
        assert e_pt.max() < P_TOL, ("p~ vector", r, e_pt.max())
        assert e_p.max() < P_TOL, ("p vector", r, e_p.max())
        if r < warmup or ref["w_llm"][r] is None:
            assert np.array_equal(d["p_rows"][k], d["pt_rows"][k])      # p = p~ before mixing
    # code length: the ideal bits of the GPU's (cum, freq) within 0.5 % of the oracle's
    ideal = -np.log2(freq / T).sum()
    ideal_ref = -np.log2(np.array(ref["freq"], np.float64) / T).sum()
    assert abs(ideal - ideal_ref) <= 0.005 * ideal_ref + 1, (ideal, ideal_ref)


def run(nc, Z, toks, V, flags, bits, warmup, rows, cyclic=False, **over):
    from oracle.ensemble import Params, encode_tokens
    from synth.logits import CyclicRows
    prm = nc.nc_params_default(flags=flags, cdf_bits=bits, warmup=warmup, **over)
    d = nc.nc_debug_walk_dump(Z, toks, prm, rows)
    Zo = CyclicRows(Z) if cyclic else Z
    ref = encode_tokens(Zo, toks, V, Params(flags=flags, cdf_bits=bits, warmup=warmup, **over), keep_rows=rows)
    return d, ref


@pytest.mark.parametrize("V,n,flags,bits", [(49152, 1200, 3, 24), (49152, 700, 1, 16), (49152, 600, 2, 24),
                                            (8192, 900, 3, 24), (256, 1500, 3, 24), (16, 600, 3, 24),
                                            (4, 300, 3, 16), (16, 800, 7, 24), (49152, 500, 0, 24)])
def test_walk_dump_gaussian(nc, V, n, flags, bits):
    from synth.logits import markov_tokens
    rng = np.random.default_rng(V + n + flags)
    Z = (rng.standard_normal((n, V)) * (1.0 + rng.random((n, 1)) * 2)).astype(np.float32)
    toks = markov_tokens(V, n, V + 3, k=1, p_follow=0.95) if flags & 4 else markov_tokens(V, n, V + 3)
    warm = 50
    rows = sample_rows(n, warm)
    d, ref = run(nc, Z, toks, V, flags, bits, warm, rows)
    if flags & 4:     # skip: fp32 vs fp64 entropy may decide differently within 1e-3 bit of 1.5
        assert all(h is None or abs(h - 1.5) > 1e-3 for h in ref["h_ng"])
        assert sum(ref["skipped"]) > 300                                   # the skip path runs
    check_dump(d, ref, toks, V, bits, warm)


@pytest.mark.parametrize("n_chunks", [1, 8, 64])
def test_walk_dump_cluster_sizes(nc, n_chunks):
    """V = 49,152 with the walk's three large-vocabulary cluster sizes: 16 CTAs (a container of
    1-2 chunks), 8 (up to 18 chunks: one wave of clusters on 148 SMs) and 4 (more chunks) --
    the cluster reductions differ, the bars do not."""
    from oracle.ensemble import Params, encode_tokens
    from synth.logits import markov_tokens
    V, n = 49152, 900
    assert nc.nc_host_walk_ctas(V, n_chunks) == (16 if n_chunks <= 2 else 8 if 8 * n_chunks <= 148 else 4)
    rng = np.random.default_rng(n_chunks)
    Z = (rng.standard_normal((n, V)) * 1.5).astype(np.float32)
    toks = markov_tokens(V, n, 5)
    rows = sample_rows(n, 50)
    prm = nc.nc_params_default(flags=3, cdf_bits=24, warmup=50, n_chunks=n_chunks)
    d = nc.nc_debug_walk_dump(Z, toks, prm, rows)
    ref = encode_tokens(Z, toks, V, Params(flags=3, cdf_bits=24, warmup=50), keep_rows=rows)
    check_dump(d, ref, toks, V, 24, 50)


def test_walk_dump_llm_competitive(nc):
    """An informative LLM (SPEC.md:364's bigram stub over a Markov token source): after the
    warmup the oracle's mixer keeps w_llm inside (1e-3, 0.999) on every row and inside
    (0.05, 0.95) on most, so p = w_l p~ + w_n p_ng mixes two live experts and parity covers
    the mixer (f64, D24) and the mixed branch."""
    from synth.logits import bigram_stub_logits, markov_tokens
    V, n = 49152, 2000
    toks = markov_tokens(V, n, 11, k=32, p_follow=0.7)
    Z = bigram_stub_logits(toks, V)
    rows = sample_rows(n, 100)
    d, ref = run(nc, Z, toks, V, 3, 24, 100, rows)
    w = np.array([x for x in ref["w_llm"] if x is not None])
    assert len(w) == n - 100
    assert w.min() > 1e-3 and w.max() < 0.999, (w.min(), w.max())
    assert ((w > 0.05) & (w < 0.95)).mean() > 0.7
    check_dump(d, ref, toks, V, 24, 100)


@pytest.mark.slow
def test_walk_dump_head_only_20k(nc):
    """flags = 2 (the adaptive head alone) at V = 49,152 over 20,480 tokens: SURVEY D17's
    regime, where an fp32 bias drifts past 1e-4 at ~18K tokens; b is f64 here."""
    from synth.logits import gaussian_logits, zipf_tokens
    V, n, R = 49152, 20480, 2048
    Z = gaussian_logits(R, V, 17)
    toks = zipf_tokens(V, n, 18)
    rows = sample_rows(n, 100, extra=range(n - 5, n))
    d, ref = run(nc, Z, toks, V, 2, 24, 100, rows, cyclic=True)
    check_dump(d, ref, toks, V, 24, 100)


@pytest.mark.slow
@pytest.mark.parametrize("flags", [3, 2])
def test_walk_dump_40k_tokens(nc, flags):
    """A config 3/4-length chunk (40,960 tokens) at V = 49,152: the f64 head and mixer and
    the N-gram tables over the full length stay within 1e-4 of the oracle at every row."""
    from synth.logits import gaussian_logits, markov_tokens
    V, n, R = 49152, 40960, 2048
    Z = gaussian_logits(R, V, 40 + flags, scale=1.5)
    toks = markov_tokens(V, n, 41, k=16, p_follow=0.7)
    rows = sorted(set(range(0, 200)) | set(range(0, n, 997)) | set(range(n - 3, n)) | {99, 100, 101})
    d, ref = run(nc, Z, toks, V, flags, 24, 100, rows, cyclic=True)
    check_dump(d, ref, toks, V, 24, 100)


def test_walk_dump_rows_validation(nc):
    V, n = 256, 50
    Z = np.zeros((n, V), np.float32)
    toks = list(range(n))
    with pytest.raises(nc.NcError):
        nc.nc_debug_walk_dump(Z, toks, nc.nc_params_default(), [n])          # row out of range
