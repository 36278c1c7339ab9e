"""Per-chunk ensemble state machine: adaptive bias head, mixer, N-gram, quantizer,
coder (alg:compress P:246-267).

Per token i of a chunk (canonical algorithm of SURVEY.md §8(c)):
  log p_llm = log_softmax(z / tau)                       (eq:lm)
  pt  = softmax(log p_llm + b)                           (head)
  if i < W (warmup) or N-gram off:  p = pt
  else: p_ng = NGram.predict()
        if skip on and H(p_ng) < 1.5 bits:  p = p_ng   (confidence skip, alg:compress lines 5-6,
                                                        P:452-469; reading D32)
        else: w = exp(lw - logsumexp(lw));  p = w_l pt + w_n p_ng
  c = quantize(p, T)
  emit (cum_t, freq_t) to the WNC coder
  b -= alpha (pt - onehot(t))                            (uses pt, D25)
  if i >= W and N-gram on: lw += eta [log max(pt_t,1e-12), log max(png_t,1e-12)]; lw -= lse(lw)
                                                         (D24-D26)
  NGram.update(t)

Reading D32 (the skip): the LLM forward still runs for a skipped token
(its retained K/V are needed by later tokens), so pt exists and, per alg:compress line 12
("Update: N-gram, Mixer, AdaptiveHead with t_i"), all three update on every token.
"""
from dataclasses import dataclass

import numpy as np

from .ans import AnsDecoder, AnsEncoder
from .cdf import quantize
from .coder import Decoder, Encoder
from .ngram import NGram

FLAG_NGRAM = 1
FLAG_HEAD = 2
FLAG_SKIP = 4          # confidence-based LLM skip, container flags bit 2
SKIP_TAU_BITS = 1.5    # "H(p_ng) < tau bits, with tau = 1.5"


def entropy_bits_fp64(p):
    """Shannon entropy in bits, -sum p log2 p over p > 0 (the skip test's H)."""
    p = np.asarray(p, dtype=np.float64)
    nz = p[p > 0]
    return float(-(nz * np.log2(nz)).sum())


def should_skip(p_ng, tau=SKIP_TAU_BITS):
    """true iff entropy_bits(p_ng) < tau."""
    return entropy_bits_fp64(p_ng) < tau


@dataclass
class Params:
    cdf_bits: int = 24
    flags: int = FLAG_NGRAM | FLAG_HEAD
    temperature: float = 1.0
    window: int = 2048
    slide: int = 512
    warmup: int = 100
    eta: float = 1.0
    alpha: float = 1e-3
    ngram_orders: int = 4
    ngram_cap: int = 500_000
    n_chunks: int = 1
    w_llm0: float = 0.85
    lmax_minus_one: bool = False    # NEXT-4 / D10: L_max = L - 1 instead of L
    refresh: bool = False           # NEXT-4: refresh window semantics (naive re-evaluation)
    coder: str = "wnc"              # "wnc": 32-bit arithmetic coder; "ans": rANS

    @property
    def lmax(self):
        return self.window - 1 if self.lmax_minus_one else self.window

    @property
    def tau_milli(self):
        return int(round(self.temperature * 1000))

    @property
    def tau(self):
        """effective temperature = the value the header can carry (D29)."""
        return self.tau_milli / 1000.0

    @property
    def T(self):
        return 1 << self.cdf_bits


def logsumexp(x):
    m = np.max(x)
    return m + np.log(np.sum(np.exp(x - m)))


def softmax(x):
    e = np.exp(x - np.max(x))
    return e / e.sum()


class ChunkModel:
    def __init__(self, V, prm: Params):
        self.V, self.prm = V, prm
        self.use_ng = bool(prm.flags & FLAG_NGRAM)
        self.use_head = bool(prm.flags & FLAG_HEAD)
        self.use_skip = bool(prm.flags & FLAG_SKIP) and self.use_ng
        self.last_skipped = False
        self.n_skipped = 0
        self.b = np.zeros(V)
        self.ng = NGram(V, prm.ngram_orders, cap=prm.ngram_cap) if self.use_ng else None
        self.lw = np.log(np.array([prm.w_llm0, 1.0 - prm.w_llm0]))
        self.i = 0

    def distribution(self, z):
        """returns (p, pt, png or None) for the current token."""
        zt = np.asarray(z, dtype=np.float64) / self.prm.tau
        logp = zt - logsumexp(zt)
        pt = softmax(logp + self.b) if self.use_head else softmax(logp)
        self.last_skipped = False
        if self.use_ng and self.i >= self.prm.warmup:
            png = self.ng.predict()
            if self.use_skip and should_skip(png):
                self.last_skipped = True
                self.n_skipped += 1
                return png, pt, png
            w = np.exp(self.lw - logsumexp(self.lw))
            return w[0] * pt + w[1] * png, pt, png
        return pt, pt, None

    def update(self, tok, pt, png):
        if self.use_head:
            onehot = np.zeros(self.V)
            onehot[tok] = 1.0
            self.b -= self.prm.alpha * (pt - onehot)
        if png is not None:
            self.lw = self.lw + self.prm.eta * np.array(
                [np.log(max(pt[tok], 1e-12)), np.log(max(png[tok], 1e-12))])
            self.lw = self.lw - logsumexp(self.lw)
        if self.use_ng:
            self.ng.update(tok)
        self.i += 1


def encode_tokens(Z, toks, V, prm: Params, keep_rows=()):
    """Walk one chunk given its logits rows Z[j] (row j predicts toks[j]).

    Returns dict(stream, bits, cum, freq, p_true, pt_true, rows={j: (p, pt)}, w_llm) -- w_llm[j] is
    the mixer's LLM weight used for row j (None where no mix happens)."""
    cm = ChunkModel(V, prm)
    enc = AnsEncoder() if prm.coder == "ans" else Encoder()
    cum, freq, p_true, pt_true, rows, skipped, h_ng, w_llm = [], [], [], [], {}, [], [], []
    keep = set(keep_rows)
    for j, t in enumerate(toks):
        p, pt, png = cm.distribution(Z[j])
        w_llm.append(float(np.exp(cm.lw[0] - logsumexp(cm.lw))) if png is not None else None)
        skipped.append(cm.last_skipped)
        h_ng.append(entropy_bits_fp64(png) if (png is not None and cm.use_skip) else None)
        c = quantize(p, prm.T)
        lo = int(c[:t].sum())
        enc.encode(lo, int(c[t]), prm.T)
        cum.append(lo)
        freq.append(int(c[t]))
        p_true.append(float(p[t]))
        pt_true.append(float(pt[t]))
        if j in keep:
            rows[j] = (p.copy(), pt.copy())
        cm.update(t, pt, png)
    stream, bits = enc.finish()
    return dict(stream=stream, bits=bits, cum=cum, freq=freq, p_true=p_true,
                pt_true=pt_true, rows=rows, min_range=getattr(enc, "min_range", None), skipped=skipped,
                h_ng=h_ng, w_llm=w_llm)


def decode_tokens(step, n, stream, V, prm: Params):
    """step(x) -> logits row for LM input token x (BOS first).  Returns tokens."""
    cm = ChunkModel(V, prm)
    dec = AnsDecoder(stream) if prm.coder == "ans" else Decoder(stream)
    out = []
    x = None
    for j in range(n):
        z = step(x)
        p, pt, png = cm.distribution(z)
        c = quantize(p, prm.T)
        cum = np.concatenate([[0], np.cumsum(c)])
        t = dec.decode(cum, prm.T)
        out.append(t)
        cm.update(t, pt, png)
        x = t
    if prm.coder == "ans" and not dec.finished_ok():
        raise ValueError("rANS stream does not end in the start state (corrupt stream or wrong params)")
    return out
