"""rANS coder, the paper's future-work replacement for arithmetic coding (P:1023-1024
"Replacing arithmetic coding with Asymmetric Numeral Systems [Duda 2009] would improve
encoding speed").  CPU ORACLE -- test infrastructure only.

Range ANS over the same integer CDFs (T = 2^b, counts c_v >= 1 summing to T),
64-bit state x in [L, 2^64) with L = 2^31, 32-bit renormalisation words (reading D39):

  encode (symbols in REVERSE order):  if x >= ((L >> b) << 32) * freq: emit the low word, x >>= 32
                                      x = (x // freq) * T + x % freq + cum
  finish: emit x as two words (high first in the decoder's order)
  decode (forward):  slot = x mod T;  s = the symbol with cum[s] <= slot < cum[s+1]
                     x = freq * (x >> b) + slot - cum;  while x < L: x = (x << 32) | next word
  integrity: after the last symbol the decoder's state is L again (the encoder's start state)

Words are big-endian in the byte stream, in the decoder's reading order (the encoder builds
them back to front).  bit_count = 32 x words.
"""
import numpy as np

from .coder import find_symbol

L = 1 << 31
MASK64 = (1 << 64) - 1


class AnsEncoder:
    """collects (cum, freq) pairs in coding order; finish() encodes them in reverse."""

    def __init__(self):
        self.pairs = []

    def encode(self, cum_lo, freq, T):
        if freq < 1:
            raise ValueError("zero-width symbol interval")
        self.pairs.append((int(cum_lo), int(freq), int(T)))

    def finish(self):
        x = L
        words = []                                  # emitted in encoding order (reversed later)
        for cum, freq, T in reversed(self.pairs):
            b = T.bit_length() - 1
            x_max = ((L >> b) << 32) * freq
            if x >= x_max:
                words.append(x & 0xFFFFFFFF)
                x >>= 32
            x = (x // freq) * T + x % freq + cum
            assert L <= x <= MASK64
        words.append(x & 0xFFFFFFFF)                # flush: low word, then high word
        words.append(x >> 32)
        words.reverse()                             # decoder order: high, low, then the rest
        data = b"".join(int(w).to_bytes(4, "big") for w in words)
        return data, 32 * len(words)


class AnsDecoder:
    def __init__(self, stream: bytes):
        self.words = [int.from_bytes(stream[i:i + 4], "big") for i in range(0, len(stream) - len(stream) % 4, 4)]
        self.pos = 0
        hi, lo = self._word(), self._word()
        self.x = (hi << 32) | lo

    def _word(self):
        w = self.words[self.pos] if self.pos < len(self.words) else 0
        self.pos += 1
        return w

    def decode(self, cum, T):
        """cum: int array of length V+1 (cum[0] = 0, cum[V] = T). Returns the symbol."""
        b = T.bit_length() - 1
        slot = self.x & (T - 1)
        s = find_symbol(cum, slot)
        lo, freq = int(cum[s]), int(cum[s + 1] - cum[s])
        self.x = freq * (self.x >> b) + slot - lo
        while self.x < L:
            self.x = (self.x << 32) | self._word()
        return s

    def finished_ok(self):
        """the integrity condition: every word consumed and the state back at L."""
        return self.x == L and self.pos == len(self.words)


def code_length_bound(freqs, T):
    """bits <= sum log2(T / freq) + 64 (flush) + 32 (the last partial word): rANS loses
    at most ~log2(e) * 2^-31 per symbol to the floor in x // freq (x >= L = 2^31)."""
    f = np.asarray(freqs, dtype=np.float64)
    return float(np.log2(T / f).sum()) + 64 + 32 + len(f) * 1e-6


__all__ = ["AnsEncoder", "AnsDecoder", "code_length_bound", "L"]
