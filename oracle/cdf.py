"""CDF quantization ("CDF-24").

  c_i = max(1, floor(p_i * (T - V)))      ; residual T - sum(c) added to c_{argmax p}

Readings: argmax ties -> lowest index (D4); the product p_i*(T-V) is
taken in fp64 (exact for fp32 p, D5); a negative residual is also added and is
an error if c_argmax would drop below 1 (D6).
"""
import math

import numpy as np


class QuantizeError(ValueError):
    pass


def quantize(p, T):
    """counts c (int64, length V) with sum == T and every c >= 1."""
    p = np.asarray(p)
    V = p.shape[0]
    if T <= V:
        raise QuantizeError("precision-infeasible: T <= V")
    c = np.maximum(1, np.floor(p.astype(np.float64) * float(T - V))).astype(np.int64)
    a = int(np.argmax(p))                  # first maximum = lowest index
    c[a] += T - int(c.sum())
    if c[a] < 1:
        raise QuantizeError("negative residual exceeds argmax count")
    return c


def floor_fraction(V, T):
    """V * MIN_PROB / T."""
    return V / T


def floor_overhead_bits(V, T):
    """Delta H ~= log2(T / (T - V))."""
    return math.log2(T / (T - V)) if V else 0.0


def entropy_bits(p):
    p = np.asarray(p, dtype=np.float64)
    nz = p[p > 0]
    return float(-(nz * np.log2(nz)).sum())
