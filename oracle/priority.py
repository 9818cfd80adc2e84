"""Oracle: priority transform for prioritized replay, |delta| -> fixed-point leaf q.

Paper: "prioritized replay (sum tree)" [EXT: PER, Schaul et al. 2016].
SPEC: p = |delta| + eps_p, eps_p = 1e-3; sampling
probability P(i) = p_i^alpha / sum p^alpha.

Reading §8c #7 (precision that makes the tree bit-exact):
    p = RN64(|delta| + eps_p)          (|delta| is an fp32 value, eps_p a double)
    v = RN32(p ** alpha)               (the REAL power, correctly rounded to fp32,
                                        round-half-even)
    q = RNE(v * 2**F), clamped to q_cap = floor((2**63 - 1) / n_leaves)

Here p ** alpha is evaluated by mpmath at 256 bits and rounded to a 24-bit
significand by explicit integer arithmetic, so nothing depends on a libm.
"""
from __future__ import annotations

import math
from fractions import Fraction

import mpmath

_C = mpmath.MPContext()
_C.prec = 256

F_DEFAULT = 32
INT64_MAX = (1 << 63) - 1


def q_cap(n_leaves: int) -> int:
    """Largest leaf value such that the root of n_leaves leaves fits in int64."""
    return INT64_MAX // max(1, int(n_leaves))


def _rne_shift(man: int, shift: int) -> int:
    """Round man * 2**shift to the nearest integer, ties to even (man >= 0)."""
    if shift >= 0:
        return man << shift
    s = -shift
    q, rem = divmod(man, 1 << s)
    half = 1 << (s - 1)
    if rem > half or (rem == half and (q & 1)):
        q += 1
    return q


def rn32_of_mpf(y) -> tuple[int, int]:
    """Correctly rounded fp32 (round-half-even) of a positive mpf y.

    Returns (M, E) with fp32 value M * 2**E, M < 2**24 (M == 0 for zero);
    E = None signals overflow to +inf.
    """
    if y == 0:
        return 0, 0
    man, exp = int(y.man), int(y.exp)           # y == man * 2**exp exactly
    e = man.bit_length() - 1 + exp               # floor(log2 y)
    e = max(e, -126)                             # subnormal range: fixed quantum 2**-149
    qexp = e - 23                                # quantum of the fp32 binade
    M = _rne_shift(man, exp - qexp)
    if M == (1 << 24):                           # rounded up into the next binade
        M >>= 1
        qexp += 1
    if qexp + 23 > 127:
        return 0, None
    return M, qexp


def rn32(x: float) -> float:
    """fp32 rounding of a double, via the same integer path (used by pins)."""
    M, E = rn32_of_mpf(_C.mpf(x))
    return math.inf if E is None else math.ldexp(M, E)


def priority_value(td_abs: float, alpha: float, eps_p: float = 1e-3) -> tuple[int, int]:
    """v = RN32((RN64(|delta| + eps_p)) ** alpha) as (M, E). S:624, §8c #7."""
    p = abs(float(td_abs)) + float(eps_p)        # IEEE double add: RN64
    if math.isnan(p) or math.isinf(p):
        return 0, None                           # non-finite priority: saturates (header rpl.h)
    if alpha == 0.0:
        return 1 << 23, -23                      # p**0 == 1 exactly
    y = _C.power(_C.mpf(p), _C.mpf(float(alpha)))
    return rn32_of_mpf(y)


def quantise(M: int, E, frac_bits: int, cap: int) -> tuple[int, bool]:
    """q = RNE(v * 2**F) for v = M * 2**E, clamped to cap. Returns (q, saturated)."""
    if E is None:
        return cap, True
    q = _rne_shift(M, E + frac_bits)
    if q > cap:
        return cap, True
    return q, False


def priority_q(td_abs: float, alpha: float, eps_p: float = 1e-3,
               frac_bits: int = F_DEFAULT, n_leaves: int = 1 << 20) -> int:
    """Full transform |delta| -> q (int), saturating at q_cap(n_leaves)."""
    M, E = priority_value(td_abs, alpha, eps_p)
    return quantise(M, E, frac_bits, q_cap(n_leaves))[0]


def value_float(M: int, E) -> float:
    return math.inf if E is None else math.ldexp(M, E)


def sequence_sum(vals) -> float:
    """S = RN64(sum of |v|) with the sum taken EXACTLY (rational arithmetic) and rounded
    once; NaN if any entry is NaN, else +inf if any is infinite (reading R26)."""
    vals = [abs(float(x)) for x in vals]
    if any(math.isnan(v) for v in vals):
        return math.nan
    if any(math.isinf(v) for v in vals):
        return math.inf
    exact = sum((Fraction(v) for v in vals), Fraction(0))
    return float(exact)                          # int / int true division: correctly rounded


def sequence_td(td_steps, eta: float) -> float:
    """R2D2 sequence priority (§8f NEXT-1, "eta = 0.9 mix of max and mean";
    [EXT: R2D2 eq. p = eta max_i |delta_i| + (1 - eta) mean |delta|]), reading R26:

        mx   = max_t |d_t|                          (NaN entries never win the max)
        S    = RN64(sum_t |d_t|)                    the EXACT sum (rational arithmetic),
                                                    rounded once to fp64 — no summation order
        mean = RN64(S / T)                          (IEEE division)
        mix  = RN64(RN64(eta * mx) + RN64(RN64(1 - eta) * mean))   (no fused multiply-add)
        td   = RN32(mix)

    A NaN entry makes S NaN, an infinite one +inf (the transform then saturates).
    `td` then enters the ordinary priority transform (priority_value) as |delta|."""
    vals = [abs(float(x)) for x in td_steps]
    if not vals:
        raise ValueError("empty sequence")
    mx = 0.0
    for v in vals:
        if v > mx:
            mx = v
    mean = sequence_sum(vals) / float(len(vals))
    mix = (float(eta) * mx) + ((1.0 - float(eta)) * mean)
    return rn32(mix) if math.isfinite(mix) else mix
