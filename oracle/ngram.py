"""Token-level interpolated N-gram.

  P_uni(t) = (c(t) + 1) / (N + V)
  P_k = lambda_k * Phat_k(.|c_k) + (1 - lambda_k) * P_{k-1},
        lambda_k = n_k / (n_k + eps), eps = 5

Readings: four context tables k = 1..4 with k-token contexts (D18); after
eviction Phat_k(v) = cnt(v)/n_k over surviving slots and the missing mass goes to
P_{k-1}: P_k = lambda*cnt/n_k + (1 - lambda*S/n_k) * P_{k-1}, S = sum of surviving
counts (D19); contexts keyed by FNV-1a-64 over [k as u8] ++ tokens as u32
LE, key 0 -> 1 (D20); 64 continuation slots, lowest-count eviction,
ties -> lowest slot, replaced in place with count 1 (D21); per-order
capacity freeze at CAP contexts (D22).  An unavailable context
(i < k, unseen, or frozen out) leaves P_k = P_{k-1}.
"""
import struct

import numpy as np

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
MASK64 = (1 << 64) - 1


def fnv1a64(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & MASK64
    return h


def context_key(k: int, ctx) -> int:
    """D20: FNV-1a-64 over bytes [k as u8] ++ each context token as u32 LE; 0 -> 1."""
    h = fnv1a64(bytes([k]) + b"".join(struct.pack("<I", t) for t in ctx))
    return h if h != 0 else 1


class Record:
    __slots__ = ("n", "toks", "cnts")

    def __init__(self):
        self.n = 0
        self.toks = []
        self.cnts = []


class NGram:
    def __init__(self, V, orders=4, eps=5.0, slots=64, cap=500_000):
        self.V, self.K, self.eps, self.slots, self.cap = V, orders, float(eps), slots, cap
        self.cu = np.zeros(V, dtype=np.int64)     # unigram counts c(t)
        self.N = 0                                # total tokens seen
        self.tables = [None] + [dict() for _ in range(orders)]
        self.hist = []                            # tokens of this chunk so far

    def _record(self, k):
        i = len(self.hist)
        if i < k:
            return None
        return self.tables[k].get(context_key(k, self.hist[i - k:i]))

    def predict(self):
        """Dense P_K over V, literal recursion from the Laplace unigram."""
        P = (self.cu + 1.0) / (self.N + self.V)
        for k in range(1, self.K + 1):
            r = self._record(k)
            if r is None:
                continue
            lam = r.n / (r.n + self.eps)
            cnt = np.zeros(self.V)
            for t, c in zip(r.toks, r.cnts):
                cnt[t] += c
            S = float(sum(r.cnts))
            P = lam * cnt / r.n + (1.0 - lam * S / r.n) * P
        return P

    def update(self, tok):
        """Online count update after every token (D21-D22)."""
        i = len(self.hist)
        self.cu[tok] += 1
        self.N += 1
        for k in range(1, self.K + 1):
            if i < k:
                continue
            key = context_key(k, self.hist[i - k:i])
            tab = self.tables[k]
            r = tab.get(key)
            if r is None:
                if len(tab) >= self.cap:
                    continue
                r = tab[key] = Record()
            r.n += 1
            if tok in r.toks:
                r.cnts[r.toks.index(tok)] += 1
            elif len(r.toks) < self.slots:
                r.toks.append(tok)
                r.cnts.append(1)
            else:
                j = int(np.argmin(r.cnts))   # lowest count, ties -> lowest slot index
                r.toks[j] = tok
                r.cnts[j] = 1
        self.hist.append(tok)
