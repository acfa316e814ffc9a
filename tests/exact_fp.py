"""Exact-rational references for the requantization step (test infrastructure).

Nothing here calls the oracle or the CUDA path.  ``f32_rne`` rounds an exact
rational to the nearest IEEE binary32 value (ties to even), written out from
the format definition (24-bit significand, exponent >= -126, subnormal
quantum 2^-149).  ``requant_exact`` is DESIGN.md readings 4-5 (PAPER.md:200
section 3.2.2) evaluated with exact rationals and ONE rounding of
(float)acc * scale + shift -- the single-FMA form -- so a two-rounding
implementation (mul then add) disagrees with it on the adversarial inputs
``near_tie_cases`` builds.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def f32_rne(v: Fraction) -> float:
    """Nearest binary32 to the exact rational v (ties to even); +-inf past the
    largest finite value.  Returned as a Python float (exactly representable)."""
    if v == 0:
        return 0.0
    sign = -1.0 if v < 0 else 1.0
    a = abs(v)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while a >= Fraction(2) ** (e + 1):
        e += 1
    while a < Fraction(2) ** e:
        e -= 1
    q = max(e, -126) - 23                       # quantum of the binade (or of the subnormals)
    m = a / Fraction(2) ** q
    n = m.numerator // m.denominator
    rem = m - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    if n * Fraction(2) ** q >= Fraction(2) ** 128:
        return sign * math.inf
    return sign * math.ldexp(n, q)


def requant_exact(acc: int, scale: float, shift: float, relu: bool, bits: int, uns: bool = False) -> int:
    """clamp(rne(RN32((float)acc * scale + shift))) with one rounding of the
    multiply-add (readings 4-5); (float)acc is itself RN to binary32.  uns:
    unsigned output codes, clamp to [0, 2^b - 1] (reading 16)."""
    f = f32_rne(Fraction(int(acc)))
    v = f32_rne(Fraction(f) * Fraction(float(scale)) + Fraction(float(shift)))
    lo = 0 if (relu or uns) else -(1 << (bits - 1))
    hi = (1 << bits) - 1 if uns else (1 << (bits - 1)) - 1
    if math.isnan(v):
        return lo
    if math.isinf(v):
        return hi if v > 0 else lo
    r = round(Fraction(v))                      # Fraction rounding: half to even
    return min(max(r, lo), hi)


def requant_two_roundings(acc, scale, shift, relu: bool, bits: int) -> np.ndarray:
    """The plausible mistake: fp32 multiply, then fp32 add (two roundings).
    numpy float32 arithmetic rounds every operation once (no contraction)."""
    f = np.asarray(acc, dtype=np.int64).astype(np.float32)
    v = np.asarray(f * np.asarray(scale, np.float32), np.float32) + np.asarray(shift, np.float32)
    r = np.rint(v.astype(np.float64))           # exact for binary32 inputs; half to even
    lo = 0 if relu else -(1 << (bits - 1))
    hi = (1 << (bits - 1)) - 1
    return np.clip(r, lo, hi).astype(np.int64)


def near_tie_cases(g: np.random.Generator, n: int, bits: int = 8, k_lo: int | None = None, k_hi: int | None = None):
    """n (acc, scale, shift) triples whose exact (float)acc*scale + shift lies
    within half a binary32 ulp of shift from a half-integer inside the code
    range: the rounding of a separate product decides the code there.
    Every fourth case is an exact tie (product + shift == k + 1/2 exactly
    representable), where only round-half-even decides."""
    hi = (1 << (bits - 1)) - 1
    accs = g.integers(-(1 << 22), 1 << 22, size=n)
    exps = g.integers(-22, -6, size=n)
    mants = g.integers(1 << 23, 1 << 24, size=n)
    ks = g.integers(-hi if k_lo is None else k_lo, hi if k_hi is None else k_hi, size=n)
    out_acc, out_scale, out_shift = [], [], []
    for i in range(n):
        acc = int(accs[i])
        scale = math.ldexp(int(mants[i]), int(exps[i]) - 23)     # a binary32 value, non-trivial significand
        if i % 4 == 0:
            # exact tie: short operands make the product and k + 1/2 - product
            # exactly representable, so the exact sum IS the half-integer
            acc = acc >> 13                                        # |acc| < 2^9
            scale = math.ldexp(int(mants[i]) >> 10, -16 - int(exps[i]) % 3)   # 14-bit significand, ~2^-3..2^-5
        f = f32_rne(Fraction(acc))
        prod = Fraction(f) * Fraction(scale)                       # exact
        target = Fraction(2 * int(ks[i]) + 1, 2)                    # k + 1/2
        shift = f32_rne(target - prod)
        out_acc.append(acc)
        out_scale.append(scale)
        out_shift.append(shift)
    return (np.array(out_acc, np.int64), np.array(out_scale, np.float32), np.array(out_shift, np.float32))


def requant_res_exact(acc: int, scale: float, shift: float, skip: int, res_scale: float, relu: bool,
                      bits: int, uns: bool = False) -> int:
    """Reading 15 with exact rationals: u = RN32(acc*scale + shift), v = RN32(skip*res_scale + u),
    then round half to even and clamp (uns: to [0, 2^b - 1], reading 16)."""
    f = f32_rne(Fraction(int(acc)))
    u = f32_rne(Fraction(f) * Fraction(float(scale)) + Fraction(float(shift)))
    v = f32_rne(Fraction(int(skip)) * Fraction(float(res_scale)) + Fraction(u))
    lo = 0 if (relu or uns) else -(1 << (bits - 1))
    hi = (1 << bits) - 1 if uns else (1 << (bits - 1)) - 1
    if math.isinf(v):
        return hi if v > 0 else lo
    return min(max(round(Fraction(v)), lo), hi)
