"""LLM next-token logits, fp64 (P:269-282 Eq. eq:lm; P:482-502 sliding window).

Model (SURVEY.md D16 reading; the paper names only SmolLM2-135M): Llama block
  a = rmsnorm(h) * g1 ; q,k,v = a Wq^T, a Wk^T, a Wv^T ; RoPE(q,k) (theta, rotate-half)
  attention of q head h on kv head h // (H/KV), scale 1/sqrt(dh), softmax over the window
  h += o Wo^T ; a = rmsnorm(h) * g2 ; h += (silu(a Wg^T) * (a Wu^T)) Wd^T
  z = (rmsnorm(h) * gf) E^T        (tied head; the bias b of eq:lm is 0)

Window: the KV cache holds at most L entries; when
adding a token would exceed L the C oldest entries are removed
(kv_cache_seq_rm) and the rest are kept with their positions shifted
(kv_cache_seq_shift); only the new token is evaluated.  Retained K/V keep the
values computed when their token was processed (D9).

Two implementations:
* ``forward_literal``: the paper's incremental loop, token by token, with an
  explicit rm + shift of a relative-position KV cache (K re-rotated by -C on
  shift, as llama.cpp's K-shift does).
* ``forward_blocked``: the same result computed as one masked pass with absolute
  positions: row j attends keys [w(j), j], w(j) = C*ceil(max(0, j+1-L)/C)
  (D10).  Pinned equal to ``forward_literal`` and to HF LlamaForCausalLM with a
  4-D window mask in tests/test_oracle_lm.py.

Window variants:
* ``lmax`` (D10's other reading): the cache holds at most L_max entries, the slide
  trigger is "adding a token would exceed L_max" and w(j) = C*ceil(max(0, j+1-L_max)/C).
  L_max = L (default) or L - 1 ("slide when full, then re-evaluate the final token").
* refresh semantics (``refresh=True``): the naive re-evaluation of P:489-492 -- on a slide
  the cache is cleared and the surviving L_max - C tokens are re-evaluated from scratch
  (fresh positions 0..), so every retained K/V is recomputed with the new window as its
  whole context; SPEC's "window equivalence" holds by construction: row j's logits
  are those of a fresh evaluation of x[w(j) .. j].  ``forward_refresh_blocked`` computes
  the same as one fresh causal pass per window block.
"""
import numpy as np


def window_start(j: int, L: int, C: int) -> int:
    """w(j) = C * ceil(max(0, j+1-L) / C)   (L here is L_max, = L by default)."""
    over = j + 1 - L
    if over <= 0:
        return 0
    return C * (-(-over // C))


def rmsnorm(x, g, eps):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def silu(x):
    return x / (1.0 + np.exp(-x))


def rope_tables(positions, dh, theta):
    """cos/sin [n, dh] for HF rotate-half pairing (i, i+dh/2), fp64 angles (D12)."""
    inv = theta ** (-np.arange(0, dh, 2, dtype=np.float64) / dh)       # [dh/2]
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv[None, :]
    ang = np.concatenate([ang, ang], axis=1)
    return np.cos(ang), np.sin(ang)


def apply_rope(x, cos, sin):
    """x [n, heads, dh]; rotate_half(x) = cat(-x2, x1)."""
    half = x.shape[-1] // 2
    rot = np.concatenate([-x[..., half:], x[..., :half]], axis=-1)
    return x * cos[:, None, :] + rot * sin[:, None, :]


class LM:
    def __init__(self, w):
        self.w = w
        self.rep = w.H // w.KV

    # ---- one transformer layer's projections for a batch of rows -------------
    def _qkv(self, lw, h, pos):
        w = self.w
        a = rmsnorm(h, lw["attn_norm"], w.eps)
        q = (a @ lw["wq"].T).reshape(-1, w.H, w.dh)
        k = (a @ lw["wk"].T).reshape(-1, w.KV, w.dh)
        v = (a @ lw["wv"].T).reshape(-1, w.KV, w.dh)
        cos, sin = rope_tables(pos, w.dh, w.rope_theta)
        return apply_rope(q, cos, sin), apply_rope(k, cos, sin), v

    def _mlp(self, lw, h):
        w = self.w
        a = rmsnorm(h, lw["mlp_norm"], w.eps)
        return h + (silu(a @ lw["wg"].T) * (a @ lw["wu"].T)) @ lw["wd"].T

    def _head(self, h):
        w = self.w
        return rmsnorm(h, w.final_norm, w.eps) @ w.embed.T

    # ---- blocked (masked) evaluation, absolute positions ---------------------
    def forward_blocked(self, x, L, C, rows_per_block=256):
        """logits [n, V] for rows j = 0..n-1 of token ids x (x[0] is BOS, D13)."""
        w = self.w
        x = np.asarray(x, dtype=np.int64)
        n = len(x)
        if n == 0:
            return np.zeros((0, w.V))
        pos = np.arange(n)
        ws = np.array([window_start(j, L, C) for j in range(n)])
        h = w.embed[x].copy()
        scale = 1.0 / np.sqrt(w.dh)
        for lw in w.layers:
            q, k, v = self._qkv(lw, h, pos)
            o = np.empty((n, w.H, w.dh))
            for r0 in range(0, n, rows_per_block):
                r1 = min(n, r0 + rows_per_block)
                k0 = ws[r0]
                rows = np.arange(r0, r1)
                keys = np.arange(k0, r1)
                mask = (keys[None, :] >= ws[rows][:, None]) & (keys[None, :] <= rows[:, None])
                for hq in range(w.H):
                    g = hq // self.rep
                    s = (q[r0:r1, hq, :] @ k[k0:r1, g, :].T) * scale
                    s = np.where(mask, s, -np.inf)
                    s = s - s.max(axis=1, keepdims=True)
                    p = np.exp(s)
                    p /= p.sum(axis=1, keepdims=True)
                    o[r0:r1, hq, :] = p @ v[k0:r1, g, :]
            h = h + o.reshape(n, w.H * w.dh) @ lw["wo"].T
            h = self._mlp(lw, h)
        return self._head(h)

    # ---- refresh semantics, blocked (NEXT-4) ----------------------------------
    def forward_refresh_blocked(self, x, L, C, lmax=None):
        """logits [n, V] under refresh semantics: the rows sharing window start w are
        computed by ONE fresh causal pass over x[w .. last row of the block] at fresh
        positions 0.. (the naive re-evaluation of P:489-492); lmax as in window_start."""
        lmax = L if lmax is None else lmax
        x = np.asarray(x, dtype=np.int64)
        n = len(x)
        out = np.zeros((n, self.w.V))
        ws = [window_start(j, lmax, C) for j in range(n)]
        j = 0
        while j < n:
            w0 = ws[j]
            j1 = j
            while j1 < n and ws[j1] == w0:
                j1 += 1
            z = self.forward_blocked(x[w0:j1], 10 ** 9, 1)     # no window inside one block
            out[j:j1] = z[j - w0:j1 - w0]
            j = j1
        return out

    # ---- literal incremental evaluation (paper's llama.cpp loop) -------------
    def incremental(self, L, C, lmax=None, refresh=False):
        return _Incremental(self, L, C, lmax, refresh)

    def forward_literal(self, x, L, C, lmax=None, refresh=False):
        inc = self.incremental(L, C, lmax, refresh)
        return np.stack([inc.step(t) for t in x]) if len(x) else np.zeros((0, self.w.V))


class _Incremental:
    """Token-by-token KV-cache evaluation with llama.cpp-style rm/shift.

    Positions are RELATIVE to the cache (they restart after every shift), and the
    cached keys are re-rotated by -C on shift, so this is an independent check of
    the absolute-position reading D12 used by forward_blocked and the GPU.
    """

    def __init__(self, lm, L, C, lmax=None, refresh=False):
        self.lm, self.L, self.C = lm, L, C
        self.lmax = L if lmax is None else lmax      # D10: slide when adding would exceed L_max
        self.refresh = refresh                       # NEXT-4: re-evaluate the survivors on a slide
        w = lm.w
        self.K = [np.zeros((0, w.KV, w.dh)) for _ in w.layers]
        self.V = [np.zeros((0, w.KV, w.dh)) for _ in w.layers]
        self.toks = []                               # tokens whose K/V are in the cache

    def _shift(self):
        """kv_cache_seq_rm(0, 0, C) then kv_cache_seq_shift(0, C, -1, -C)."""
        w = self.lm.w
        C = self.C
        n_keep = self.K[0].shape[0] - C
        cos, sin = rope_tables(np.full(n_keep, -C), w.dh, w.rope_theta)
        for i in range(len(self.K)):
            self.K[i] = apply_rope(self.K[i][C:], cos, sin)   # K-shift: rotate by -C
            self.V[i] = self.V[i][C:]

    def _refresh(self):
        """naive slide: drop the C oldest tokens, clear the cache and
        re-evaluate the survivors from scratch at positions 0.."""
        w = self.lm.w
        keep = self.toks[self.C:]
        self.K = [np.zeros((0, w.KV, w.dh)) for _ in w.layers]
        self.V = [np.zeros((0, w.KV, w.dh)) for _ in w.layers]
        self.toks = []
        for t in keep:
            self._eval(t)

    def step(self, tok):
        if self.K[0].shape[0] + 1 > self.lmax:
            if self.refresh:
                self._refresh()
            else:
                self._shift()
                self.toks = self.toks[self.C:]
        return self._eval(tok)

    def _eval(self, tok):
        lm, w = self.lm, self.lm.w
        self.toks.append(tok)
        p = self.K[0].shape[0]                 # relative position of the new token
        h = w.embed[[tok]].copy()
        scale = 1.0 / np.sqrt(w.dh)
        for li, lw in enumerate(w.layers):
            q, k, v = lm._qkv(lw, h, [p])
            self.K[li] = np.concatenate([self.K[li], k], axis=0)
            self.V[li] = np.concatenate([self.V[li], v], axis=0)
            o = np.empty((1, w.H, w.dh))
            for hq in range(w.H):
                g = hq // lm.rep
                s = (self.K[li][:, g, :] @ q[0, hq, :]) * scale
                s = np.exp(s - s.max())
                o[0, hq, :] = (s / s.sum()) @ self.V[li][:, g, :]
            h = h + o.reshape(1, -1) @ lw["wo"].T
            h = lm._mlp(lw, h)
        return lm._head(h)[0]
