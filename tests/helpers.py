"""Exact-arithmetic helpers for the oracle pins (tests only)."""
from fractions import Fraction
import math

import numpy as np

U = 2.0 ** -53


def F(x) -> Fraction:
    return Fraction(float(x))


def exact_sqrt(q: Fraction, bits: int = 200) -> Fraction:
    """sqrt(q) to ~2^-bits relative (floor of the scaled integer square root)."""
    if q <= 0:
        return Fraction(0)
    k = bits + max(0, -(q.numerator.bit_length() - q.denominator.bit_length()) // 2 + 2)
    return Fraction(math.isqrt(q.numerator * q.denominator * 4 ** k), q.denominator * 2 ** k)


def rn(q) -> float:
    """Round an exact rational (or mpmath value) to the nearest double."""
    if isinstance(q, Fraction):
        return q.numerator / q.denominator
    return float(q)


def random_doubles(rng: np.random.Generator, n: int, emin: int = -40, emax: int = 40) -> np.ndarray:
    """Random-sign doubles with log-uniform exponents in [2^emin, 2^emax] and full mantissas."""
    m = rng.uniform(1.0, 2.0, n)
    e = rng.integers(emin, emax + 1, n)
    s = rng.choice([-1.0, 1.0], n)
    return s * np.ldexp(m, e)


def random_unit(rng: np.random.Generator, n: int) -> np.ndarray:
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)
