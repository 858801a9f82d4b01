"""Exact rational arithmetic helpers for pinning the oracle (no float arithmetic of the
method here): correctly rounded Fraction -> binary32, ULP distance, bf16 bits."""
from fractions import Fraction

import numpy as np


def fraction_to_f32(fr: Fraction) -> np.float32:
    """Round an exact rational to the nearest binary32, ties to even (normal and
    subnormal range; no overflow handling -- test values stay far from FLT_MAX)."""
    fr = Fraction(fr)
    if fr == 0:
        return np.float32(0.0)
    sign = -1 if fr < 0 else 1
    a = abs(fr)
    # exponent e with 2^e <= a < 2^(e+1)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                      # subnormals share the 2^-149 quantum
    quantum = Fraction(2) ** (e - 23)
    q = a / quantum
    n = q.numerator // q.denominator
    rem = q - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    val = np.float32(float(n) * float(quantum))   # exact: n <= 2^24, power-of-two scale
    return np.float32(sign * val)


def exact(x) -> Fraction:
    """Exact rational value of a finite float32/float64."""
    return Fraction(float(x))


def f32_bits(x) -> int:
    return int(np.asarray(x, dtype=np.float32).view(np.uint32))


def ulp_dist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """ULP distance between float32 arrays (monotone integer mapping)."""
    def key(x):
        i = np.ascontiguousarray(x, dtype=np.float32).view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    return np.abs(key(a) - key(b))
