"""Whole-file oracle compress / decompress (alg:compress P:246-267; P:530-570;
S:501-538).  Each chunk: tokenize, x = [BOS] ++ tokens (D13), LM logits for rows
0..n-1 with the retained-KV window (D9-D10), ensemble walk, WNC encode; then the
NC05 container.  Decompression mirrors it with the literal
incremental LM, so the token being decoded is never seen in advance.  The window
variants of NEXT-4 (Params.refresh, Params.lmax_minus_one; oracle/lm.py) apply to both.

bpb on the paper's real data is *parity unpinned* here (needs the real weights
and datasets); the synthetic pipeline is pinned by round trip and by the
per-step pins of the modules it composes.
"""
import numpy as np

from .chunking import split_chunks
from .container import read_nc05, write_nc05
from .ensemble import Params, decode_tokens, encode_tokens
from .lm import LM
from .tokenizer import Tokenizer


def _tokenizer(weights):
    """the model's own tokenizer (HF checkpoints, oracle/hf.py) or the synthetic greedy one (D30)"""
    return getattr(weights, "tokenizer", None) or Tokenizer(weights.vocab, weights.n_special)


def compress(data: bytes, weights, prm: Params, lm_mode="blocked", collect=None):
    tok = _tokenizer(weights)
    lm = LM(weights)
    entries = []
    for ch in split_chunks(data, prm.n_chunks):
        t = tok.encode(ch)
        n = len(t)
        x = [weights.bos] + t[:-1] if n else []
        if prm.refresh:
            Z = lm.forward_refresh_blocked(x, prm.window, prm.slide, prm.lmax) if lm_mode == "blocked" else \
                lm.forward_literal(x, prm.window, prm.slide, prm.lmax, refresh=True)
        elif lm_mode == "blocked":
            Z = lm.forward_blocked(x, prm.lmax, prm.slide)
        else:
            Z = lm.forward_literal(x, prm.window, prm.slide, prm.lmax)
        r = encode_tokens(Z, t, weights.V, prm)
        if collect is not None:
            collect.append(dict(tokens=t, **r))
        entries.append((n, r["bits"], r["stream"]))
    return write_nc05(prm.flags, prm.tau_milli, entries)


def decompress(blob: bytes, weights, prm: Params):
    flags, tau_milli, chunks = read_nc05(blob)
    prm = Params(**{**prm.__dict__, "flags": flags, "temperature": tau_milli / 1000.0})
    tok = _tokenizer(weights)
    lm = LM(weights)
    out = []
    for n, bits, stream in chunks:
        inc = lm.incremental(prm.window, prm.slide, prm.lmax, prm.refresh)

        def step(x, inc=inc):
            return inc.step(weights.bos if x is None else x)

        toks = decode_tokens(step, n, stream, weights.V, prm)
        out.append(tok.decode(toks))
    return b"".join(out)


def bits_per_byte(blob: bytes, n_in: int) -> float:
    return 8.0 * len(blob) / max(1, n_in)


__all__ = ["compress", "decompress", "Params", "bits_per_byte", "np"]
