"""Oracle pins: N-gram, mixer, adaptive head.

Pins: SPEC/PAPER worked examples, FNV-1a published vectors, closed forms, and a
brute-force batch recount of N-gram statistics straight from the token history
(an algorithm independent of the oracle's online tables)."""
import json
import math
import os
from collections import Counter

import numpy as np
import pytest

from oracle.ensemble import ChunkModel, Params, logsumexp, softmax
from oracle.ngram import NGram, context_key, fnv1a64

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_fnv_vectors():
    v = G["fnv1a64_vectors"]
    for s in ("", "a", "foobar"):
        assert fnv1a64(s.encode()) == int(v[s], 16)


def test_context_key_mixes_order():
    assert context_key(1, [5]) != context_key(2, [5, 5])
    assert context_key(3, [1, 2, 3]) == context_key(3, [1, 2, 3])


def test_ngram_fresh_uniform_and_one_update():
    ng = NGram(4)
    assert np.allclose(ng.predict(), 0.25)
    ng.update(2)
    g = G["unigram_after_one_update"]
    assert abs(((ng.cu + 1) / (ng.N + 4))[g["tok"]] - g["p"]) < 1e-15
    # order-1 context (2) has never been seen -> prediction is the unigram
    assert abs(ng.predict()[2] - g["p"]) < 1e-15


def test_lambda_half_at_n5():
    """n_k = 5 -> lambda = 5/(5+5) = 0.5.  Sequence 0,1 x5 then 0: context (0)
    seen 5 times always followed by 1; P_1(1) = 0.5*1 + 0.5*P_uni(1) = 0.5 + 0.5*6/15."""
    ng = NGram(4, orders=1)
    for t in [0, 1] * 5 + [0]:
        ng.update(t)
    assert abs(ng.predict()[1] - (0.5 + 0.5 * 6 / 15)) < 1e-15


def test_eviction_65_successors_S185():
    ng = NGram(200, orders=1)
    for s in range(65):
        ng.hist = [7]               # fixed context (7) for every update
        ng.update(100 + s if s else 100)
    r = ng.tables[1][context_key(1, [7])]
    assert len(r.toks) == 64 and r.n == 65
    assert 100 not in r.toks          # first inserted, count 1, lowest slot -> evicted
    assert 164 in r.toks


def test_abab_S186():
    ng = NGram(2)
    for i in range(1000):
        ng.update(i % 2)
    assert ng.predict()[0] > 0.95     # next after ...,0,1 is 0


def test_capacity_freeze_d22():
    ng = NGram(50, orders=1, cap=3)
    for t in range(20):
        ng.update(t)
    assert len(ng.tables[1]) == 3
    ng.hist = [0]
    ng.update(9)                      # existing contexts still update
    assert ng.tables[1][context_key(1, [0])].n == 2


def _brute_predict(hist, V, K, eps=5.0):
    """Recount everything from the history (no eviction: fewer than 64 successors)."""
    cu = Counter(hist)
    P = np.array([(cu[v] + 1) / (len(hist) + V) for v in range(V)])
    i = len(hist)
    for k in range(1, K + 1):
        if i < k:
            continue
        ctx = tuple(hist[i - k:i])
        succ = Counter(hist[j + k] for j in range(0, i - k) if tuple(hist[j:j + k]) == ctx)
        n = sum(succ.values())
        if n == 0:
            continue
        lam = n / (n + eps)
        P = lam * np.array([succ[v] / n for v in range(V)]) + (1 - lam) * P
    return P


@pytest.mark.parametrize("V", [2, 4, 16])
def test_ngram_brute_force(V):
    rng = np.random.default_rng(V)
    ng = NGram(V)
    hist = []
    for step in range(300):
        P = ng.predict()
        assert abs(P.sum() - 1) < 1e-9
        Q = _brute_predict(hist, V, 4)
        assert np.allclose(P, Q, rtol=1e-12, atol=1e-15), step
        t = int(rng.integers(V)) if rng.random() < 0.5 else (hist[-2] if len(hist) > 1 else 0)
        ng.update(t)
        hist.append(t)


def test_closed_form_equals_recursion_8c():
    """SURVEY §8(c) closed form used by the GPU walker: p_ng = a0*P_uni + sum a_k cnt_k."""
    V = 300
    rng = np.random.default_rng(7)
    ng = NGram(V, cap=40)
    for step in range(3000):
        t = int(rng.integers(V)) if rng.random() < 0.3 else int(rng.integers(20))
        ng.update(t)
        if step % 97 == 0:
            mu = np.ones(5)
            beta = np.zeros(5)
            cnt = np.zeros((5, V))
            for k in range(1, 5):
                r = ng._record(k)
                if r is None:
                    continue
                lam = r.n / (r.n + 5.0)
                mu[k] = 1 - lam * sum(r.cnts) / r.n
                beta[k] = lam / r.n
                for tok, c in zip(r.toks, r.cnts):
                    cnt[k, tok] += c
            a0 = np.prod(mu[1:])
            P = a0 * (ng.cu + 1) / (ng.N + V)
            for k in range(1, 5):
                P += beta[k] * np.prod(mu[k + 1:]) * cnt[k]
            assert np.allclose(P, ng.predict(), rtol=1e-12, atol=1e-16)


# ------------------------------------------------------------------ mixer ---

def test_mixer_paper_example():
    g = G["mixer_example"]
    w = np.array(G["mixer_w0"]["value"])
    assert abs(w[0] * g["p_llm"] + w[1] * 0.0 - g["p_mix_min"]) < 1e-15


class _FixedNGram:
    """stands in for the N-gram inside ChunkModel: predict() returns a fixed vector."""

    def __init__(self, png):
        self.png = np.asarray(png, dtype=np.float64)

    def predict(self):
        return self.png

    def update(self, tok):
        pass


def _mixed(lw, z, b, png):
    cm = ChunkModel(4, Params(warmup=0))
    cm.ng = _FixedNGram(png)
    cm.lw = np.log(np.asarray(lw, dtype=np.float64))
    cm.b = np.asarray(b, dtype=np.float64)
    return cm.distribution(np.log(np.asarray(z, dtype=np.float64)))


def test_mixer_distribution_paper_0765():
    """ChunkModel.distribution's post-warmup branch on P:403-406's example: initial weights
    (0.85, 0.15), p_llm(t) = 0.90, p_ng(t) = 0 -> p_mix(t) = 0.765 exactly
    (written out, not recomputed from the oracle's formula)."""
    p, pt, png = _mixed([0.85, 0.15], [0.9, 0.05, 0.03, 0.02], [0, 0, 0, 0], [0.0, 0.5, 0.25, 0.25])
    assert abs(pt[0] - 0.9) < 1e-15
    assert abs(p[0] - 0.765) < 1e-15
    assert np.allclose(p, [0.765, 0.1175, 0.063, 0.0545], atol=1e-15, rtol=0)


def test_mixer_distribution_hand_mixture():
    """Weights (0.3, 0.7) given as unnormalised log-weights, a non-zero head bias b and a
    known p_ng: p = w_l * p~ + w_n * p_ng with p~ = softmax(log p_llm + b) (D25: the head is
    applied BEFORE mixing).  p_llm = (1/2, 1/4, 1/8, 1/8), b = (ln 2, 0, 0, 0) -> p~ = (2/3,
    1/6, 1/12, 1/12); p_ng = (0.1, 0.2, 0.3, 0.4) -> p = (0.27, 0.19, 0.235, 0.305).  A swapped
    w_l/w_n gives (0.5367, ...), mixing p_llm instead of p~ gives (0.22, ...)."""
    lw = np.array([0.3, 0.7]) * math.e ** 5                      # unnormalised: renormalised inside
    p, pt, png = _mixed(lw, [0.5, 0.25, 0.125, 0.125], [math.log(2), 0, 0, 0], [0.1, 0.2, 0.3, 0.4])
    assert np.allclose(pt, [2 / 3, 1 / 6, 1 / 12, 1 / 12], atol=1e-15, rtol=0)
    assert np.allclose(p, [0.27, 0.19, 0.235, 0.305], atol=1e-15, rtol=0)


def test_mixer_warmup_branch_ignores_ngram():
    """i < W: p = p~ and no N-gram prediction is taken."""
    cm = ChunkModel(4, Params(warmup=5))
    cm.ng = _FixedNGram([0.1, 0.2, 0.3, 0.4])
    p, pt, png = cm.distribution(np.log(np.array([0.5, 0.25, 0.125, 0.125])))
    assert png is None and np.allclose(p, [0.5, 0.25, 0.125, 0.125], atol=1e-15, rtol=0)


def _mixer_after(p1, p2, eta, steps=1):
    prm = Params(eta=eta, warmup=0)
    cm = ChunkModel(4, prm)
    lw0 = cm.lw.copy()
    for _ in range(steps):
        pt = np.array([p1, 1 - p1, 0, 0])
        png = np.array([p2, 1 - p2, 0, 0])
        cm.update(0, pt, png)
    return lw0, cm.lw


def test_mixer_equal_probs_unchanged():
    lw0, lw = _mixer_after(0.3, 0.3, 1.0)
    assert np.allclose(lw, lw0, atol=1e-15)


def test_mixer_gap_grows_eta_ln2():
    lw0, lw = _mixer_after(1.0, 0.5, 0.1)
    assert abs((lw[0] - lw[1]) - (lw0[0] - lw0[1]) - 0.1 * math.log(2)) < 1e-12
    assert abs(logsumexp(lw)) < 1e-12


def test_mixer_converges_S256():
    V = 1000
    prm = Params(eta=1.0, warmup=0)
    cm = ChunkModel(V, prm)
    for _ in range(500):
        pt = np.full(V, 0.1 / (V - 1))
        pt[0] = 0.9
        png = np.full(V, 1.0 / V)
        cm.update(0, pt, png)
    assert math.exp(cm.lw[0] - logsumexp(cm.lw)) > 0.999


# ------------------------------------------------------------------- head ---

def test_head_identity_at_zero_bias():
    rng = np.random.default_rng(1)
    z = rng.standard_normal(50)
    cm = ChunkModel(50, Params(flags=2))
    p, pt, png = cm.distribution(z)
    assert np.allclose(pt, softmax(z), rtol=1e-12) and png is None


def test_head_examples_S264_S272():
    g = G["head_identity_and_examples"]
    cm = ChunkModel(2, Params(flags=2))
    cm.b = np.array(g["b"])
    _, pt, _ = cm.distribution(np.log(np.array(g["p"])))
    assert np.allclose(pt, g["out"], atol=1e-12)
    cm = ChunkModel(2, Params(flags=2))
    cm.update(g["observed"], np.array(g["update_pt"]), None)
    assert np.allclose(cm.b, g["b_after"], atol=1e-15)


def test_head_gradient_finite_difference():
    """b update is one SGD step on L = -log pt(t*)."""
    rng = np.random.default_rng(2)
    V = 20
    z = rng.standard_normal(V)
    b = rng.standard_normal(V) * 0.1
    t = 3

    def loss(bb):
        return -(z + bb - logsumexp(z + bb))[t]
    pt = softmax(z + b)
    g = pt.copy()
    g[t] -= 1
    for v in range(V):
        e = np.zeros(V)
        e[v] = 1e-6
        fd = (loss(b + e) - loss(b - e)) / 2e-6
        assert abs(fd - g[v]) < 1e-8


def test_temperature_S348():
    g = G["temperature_example"]
    cm = ChunkModel(2, Params(flags=0, temperature=g["tau"]))
    p, _, _ = cm.distribution(np.array(g["logits"]))
    assert np.allclose(p, g["p"], atol=1e-4)


def test_warmup_uses_llm_alone():
    V = 30
    prm = Params(warmup=100)
    cm = ChunkModel(V, prm)
    rng = np.random.default_rng(0)
    for i in range(130):
        z = rng.standard_normal(V)
        p, pt, png = cm.distribution(z)
        if i < 100:
            assert png is None and np.array_equal(p, pt)
        else:
            assert png is not None
        cm.update(int(rng.integers(V)), pt, png)
