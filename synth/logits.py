"""Seeded synthetic token streams and logit rows for the walk tests.

Like the rest of ``synth/`` this holds no arithmetic of the compression method: it
draws token sequences and LLM-logit rows that the CPU oracle and the CUDA walk both
consume as *inputs*.

* ``markov_tokens``: a token-level Markov source (each token has ``k`` fixed successors,
  followed with probability ``p_follow``, otherwise a uniform token) -- the repetitive
  structure the N-gram learns (the regime of the paper's text).
* ``zipf_tokens``: i.i.d. Zipf(s) token ids (SURVEY D17's bias-drift simulation).
* ``gaussian_logits``: rows z ~ N(0, scale^2) (random-init LM logits are roughly
  Gaussian with std ~1).
* ``bigram_stub_logits``: the stub LM of SPEC.md:364 -- "normalized mixture of (a) a fixed
  uniform prior weight 1, and (b) a count table over (previous token -> next token)
  bigrams accumulated ... within the session": row j (predicting token j) is
  log((1/V + cnt[t_{j-1} -> v]) / (1 + n[t_{j-1}])) from tokens 0..j-1.  Unlike
  random-init weights it is informative, so after the warmup the mixer keeps a
  non-negligible LLM weight and parity covers the mixed branch p = w_l p~ + w_n p_ng.
"""
import numpy as np


def markov_tokens(V, n, seed, k=8, p_follow=0.7):
    rng = np.random.default_rng(seed)
    succ = rng.integers(0, V, (V, k))
    t = [int(rng.integers(V))]
    for _ in range(n - 1):
        t.append(int(succ[t[-1], rng.integers(k)]) if rng.random() < p_follow else int(rng.integers(V)))
    return t


def zipf_tokens(V, n, seed, s=1.07):
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, V + 1) ** s
    perm = rng.permutation(V)
    return [int(perm[i]) for i in rng.choice(V, size=n, p=w / w.sum())]


def gaussian_logits(n, V, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, V)) * scale).astype(np.float32)


def bigram_stub_logits(toks, V):
    """[n, V] float32; row j uses only toks[:j] (row 0: uniform)."""
    n = len(toks)
    Z = np.empty((n, V), np.float32)
    counts = {}
    totals = {}
    prev = None
    for j in range(n):
        row = np.full(V, 1.0 / V)
        if prev is not None:
            c = counts.get(prev)
            if c is not None:
                for v, cnt in c.items():
                    row[v] += cnt
            row /= 1.0 + totals.get(prev, 0)
        Z[j] = np.log(row).astype(np.float32)
        t = toks[j]
        if prev is not None:
            counts.setdefault(prev, {})
            counts[prev][t] = counts[prev].get(t, 0) + 1
            totals[prev] = totals.get(prev, 0) + 1
        prev = t
    return Z


class CyclicRows:
    """Row j of a long walk = table[j % R] (nc_debug_walk_dump's n_logit_rows): long
    sequential walks without an n_tok x V host array."""

    def __init__(self, table):
        self.table = table

    def __getitem__(self, j):
        return self.table[j % len(self.table)]

    def __len__(self):
        return len(self.table)
