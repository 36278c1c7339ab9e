"""32-bit arithmetic coder after Witten, Neal & Cleary.

Constants HALF = 2^31, QUARTER = 2^30; E1/E2 emit on half convergence, E3 counts
underflow on quarter straddle.  Narrowing with R = high - low + 1 (64-bit
intermediates): high = low + floor(R*cum_hi/T) - 1, low += floor(R*cum_lo/T).
Finish: underflow += 1, then one bit choosing the quarter that holds low followed
by `underflow` complement bits; the stream is padded with zeros to a byte; bits
are MSB-first.  The decoder primes value with 32 bits and reads zeros past the
end.  Decode target = floor(((value - low + 1) * T - 1) / R), then binary search
for the symbol with cum[s] <= target < cum[s+1].

Reading D7: after renormalization R > 2^30 (not >= 2^31 as P:351-356 claims).
"""
import numpy as np

TOP = 1 << 32
HALF = 1 << 31
QUARTER = 1 << 30
THREE_Q = 3 << 30


class Encoder:
    def __init__(self):
        self.low, self.high, self.pending = 0, TOP - 1, 0
        self.bits = []
        self.min_range = TOP

    def _emit(self, b):
        self.bits.append(b)
        self.bits.extend([1 - b] * self.pending)
        self.pending = 0

    def encode(self, cum_lo, freq, T):
        if freq < 1:
            raise ValueError("zero-width symbol interval")
        R = self.high - self.low + 1
        self.high = self.low + (R * (cum_lo + freq)) // T - 1
        self.low = self.low + (R * cum_lo) // T
        while True:
            if self.high < HALF:
                self._emit(0)
            elif self.low >= HALF:
                self._emit(1)
                self.low -= HALF
                self.high -= HALF
            elif self.low >= QUARTER and self.high < THREE_Q:
                self.pending += 1
                self.low -= QUARTER
                self.high -= QUARTER
            else:
                break
            self.low = 2 * self.low
            self.high = 2 * self.high + 1
        self.min_range = min(self.min_range, self.high - self.low + 1)

    def finish(self):
        """returns (stream bytes, bit_count)."""
        self.pending += 1
        self._emit(0 if self.low < QUARTER else 1)
        nbits = len(self.bits)
        bits = self.bits + [0] * (-nbits % 8)
        arr = np.array(bits, dtype=np.uint8).reshape(-1, 8) if bits else np.zeros((0, 8), np.uint8)
        return np.packbits(arr, axis=1).reshape(-1).tobytes(), nbits


class Decoder:
    def __init__(self, stream: bytes):
        self.bits = np.unpackbits(np.frombuffer(stream, dtype=np.uint8)) if stream else np.zeros(0, np.uint8)
        self.pos = 0
        self.low, self.high, self.value = 0, TOP - 1, 0
        for _ in range(32):
            self.value = 2 * self.value + self._bit()

    def _bit(self):
        b = int(self.bits[self.pos]) if self.pos < len(self.bits) else 0
        self.pos += 1
        return b

    def target(self, T):
        R = self.high - self.low + 1
        return ((self.value - self.low + 1) * T - 1) // R

    def consume(self, cum_lo, freq, T):
        R = self.high - self.low + 1
        self.high = self.low + (R * (cum_lo + freq)) // T - 1
        self.low = self.low + (R * cum_lo) // T
        while True:
            if self.high < HALF:
                pass
            elif self.low >= HALF:
                self.low -= HALF
                self.high -= HALF
                self.value -= HALF
            elif self.low >= QUARTER and self.high < THREE_Q:
                self.low -= QUARTER
                self.high -= QUARTER
                self.value -= QUARTER
            else:
                break
            self.low = 2 * self.low
            self.high = 2 * self.high + 1
            self.value = 2 * self.value + self._bit()

    def decode(self, cum, T):
        """cum: int array of length V+1 (cum[0]=0, cum[V]=T). Returns the symbol."""
        s = find_symbol(cum, self.target(T))
        self.consume(int(cum[s]), int(cum[s + 1] - cum[s]), T)
        return s


def find_symbol(cum, target):
    """binary search: the s with cum[s] <= target < cum[s+1]."""
    lo, hi = 0, len(cum) - 1          # invariant cum[lo] <= target < cum[hi]
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if cum[mid] <= target:
            lo = mid
        else:
            hi = mid
    return lo
