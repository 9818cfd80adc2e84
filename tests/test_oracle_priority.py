"""Pins for oracle.priority: the correctly rounded fp32 power and quantisation.

Special cases reduce to exactly computable values: alpha=1 (fp32 rounding of a
double, done by numpy), alpha=0.5 (integer square root), alpha=2 and 3 (exact
rational powers).  The test's own round-to-fp32 of an exact rational is plain
integer arithmetic written independently of the oracle's mpf path."""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import priority as P


def rn32_fraction(x: Fraction) -> Fraction:
    """Independent round-half-even of a positive rational to 24 significant bits."""
    assert x > 0
    e = x.numerator.bit_length() - x.denominator.bit_length()
    while Fraction(2) ** e > x:
        e -= 1
    while Fraction(2) ** (e + 1) <= x:
        e += 1
    e = max(e, -126)
    quantum = Fraction(2) ** (e - 23)
    k = x / quantum
    fl = k.numerator // k.denominator
    rem = k - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return fl * quantum


def val(td, alpha, eps=1e-3):
    M, E = P.priority_value(td, alpha, eps)
    return Fraction(M) * Fraction(2) ** E


def p_of(td, eps=1e-3):
    return abs(float(td)) + eps


TDS = np.concatenate([np.abs(np.random.default_rng(0).normal(0, 1, 300)),
                      np.random.default_rng(1).lognormal(0, 2, 200),
                      [0.0, 1e-8, 0.999, 1.0, 2.0, 1e6]]).astype(np.float32)


def test_alpha_one_is_fp32_rounding():
    for td in TDS:
        p = p_of(td)
        assert val(td, 1.0) == Fraction(float(np.float32(p)))


def test_alpha_zero_is_one():
    for td in TDS[:50]:
        assert val(td, 0.0) == 1


def test_alpha_half_is_rounded_isqrt():
    for td in TDS:
        p = Fraction(p_of(td))
        # sqrt(p) to 80 fractional bits via isqrt, then exact rounding; ties are
        # impossible (sqrt of a double is never an fp32 midpoint) so the 80-bit
        # truncation decides the rounding unless the remainder is exactly 0.
        num = p.numerator << 400
        s = math.isqrt(num * p.denominator)          # floor(sqrt(p) * 2^200 * den)
        approx = Fraction(s, p.denominator << 200)
        exact_sq = (s * s == num * p.denominator)
        v = rn32_fraction(approx if exact_sq else approx + Fraction(1, p.denominator << 201))
        assert val(td, 0.5) == v


@pytest.mark.parametrize("alpha", [2.0, 3.0])
def test_integer_alpha_exact(alpha):
    for td in TDS[:200]:
        p = Fraction(p_of(td))
        assert val(td, alpha) == rn32_fraction(p ** int(alpha))


@pytest.mark.parametrize("alpha", [0.6, 0.9, 0.4, 0.123456789])
def test_general_alpha_within_half_ulp(alpha):
    for td in TDS:
        p = p_of(td)
        ref = math.pow(p, alpha)                      # libm double, <= 1 ulp64
        v = float(val(td, alpha))
        e = math.frexp(v)[1] - 1
        ulp32 = 2.0 ** (max(e, -126) - 23)
        assert abs(v - ref) <= 0.5 * ulp32 * (1 + 1e-9) + 4 * abs(ref) * 2 ** -53


def test_quantise_ties_to_even():
    cap = P.q_cap(16)
    F = 32
    assert P.quantise(1, -33, F, cap) == (0, False)       # 0.5 -> 0
    assert P.quantise(3, -33, F, cap) == (2, False)       # 1.5 -> 2
    assert P.quantise(5, -33, F, cap) == (2, False)       # 2.5 -> 2
    assert P.quantise(3, -34, F, cap) == (1, False)       # 0.75 -> 1
    assert P.quantise(1 << 23, -23, F, cap) == (1 << 32, False)   # 1.0 -> 2^32
    assert P.quantise(1, 100, F, cap) == (cap, True)      # saturation
    assert P.quantise(0, None, F, cap) == (cap, True)     # +inf


def test_q_cap_root_fits():
    for n in [1, 16, 25600, 1 << 17, 1 << 20]:
        assert P.q_cap(n) * n <= (1 << 63) - 1
        assert (P.q_cap(n) + 1) * n > (1 << 63) - 1


def test_rn32_helper_matches_numpy():
    g = np.random.default_rng(5)
    for x in np.concatenate([g.normal(0, 1e3, 500) ** 2, 10.0 ** g.uniform(-40, 38, 500)]):
        assert P.rn32(float(x)) == float(np.float32(x))


# ---- R2D2 sequence priority (reading R26) ----
def test_sequence_td_eta_one_is_max_and_zero_is_mean():
    col = [0.5, 3.25, 1.0, 0.0]
    assert P.sequence_td(col, 1.0) == 3.25                      # eta = 1: the max (already fp32)
    assert P.sequence_td(col, 0.0) == (0.5 + 3.25 + 1.0) / 4    # eta = 0: the mean, exact here


def test_sequence_td_worked_example_and_constant():
    # [1, 2, 3], eta = 0.9: 0.9*3 + 0.1*2 = 2.9 -> the fp32 nearest 2.9
    assert P.sequence_td([1.0, 2.0, 3.0], 0.9) == float(np.float32(2.9))
    c = float(np.float32(0.37))
    assert P.sequence_td([c] * 80, 0.9) == c                    # constant column -> itself


def test_sequence_td_order_of_max_and_abs():
    a = P.sequence_td([-4.0, 1.0, 2.0], 0.5)
    b = P.sequence_td([2.0, 1.0, 4.0], 0.5)
    assert a == b == float(np.float32(0.5 * 4 + 0.5 * (7 / 3)))


def _order_sensitive_column():
    # 31 x 2^40, then 2^20, then 32 x 2^-10 (T = 64, all fp32-exact).  The exact sum is
    # 31*2^40 + 2^20 + 2^-5 (50 significant bits: representable, so S is exactly that); any
    # fp64 accumulation that adds a 2^-10 to the ~2^45 partial sum loses it (ulp there is
    # 2^-8, half-ulp 2^-9), giving 31*2^40 + 2^20.  The mean then straddles an fp32 tie:
    # exact 31*2^34 + 2^14 + 2^-11 -> 31*2^34 + 2^15; lossy 31*2^34 + 2^14 (a tie) -> 31*2^34.
    return [2.0 ** 40] * 31 + [2.0 ** 20] + [2.0 ** -10] * 32


def test_sequence_sum_exact_hand_value_and_order_independence():
    col = _order_sensitive_column()
    assert P.sequence_sum(col) == 31 * 2.0 ** 40 + 2.0 ** 20 + 2.0 ** -5
    naive = 0.0
    for v in col:                    # sequential fp64 (what a loop in increasing t would give)
        naive += v
    assert naive == 31 * 2.0 ** 40 + 2.0 ** 20          # the small terms are lost
    # eta = 0: td is RN32 of the mean; hand-derived values above
    assert P.sequence_td(col, 0.0) == 31 * 2.0 ** 34 + 2.0 ** 15
    assert float(np.float32(naive / 64)) == 31 * 2.0 ** 34  # the lossy sum would round down
    g = np.random.default_rng(3)
    for _ in range(20):              # any order of the same multiset: identical result
        perm = list(g.permutation(col))
        assert P.sequence_sum(perm) == P.sequence_sum(col)
        assert P.sequence_td(perm, 0.9) == P.sequence_td(col, 0.9)


def test_sequence_sum_matches_fsum_on_wide_columns():
    # math.fsum (Shewchuk's algorithm, correctly rounded) is an independent exact-sum routine
    import math
    g = np.random.default_rng(4)
    for trial in range(200):
        T = int(g.integers(1, 200))
        if trial % 2:
            col = np.exp(g.normal(0, 6, T)).astype(np.float32)        # heavy-tailed
        else:
            col = (10.0 ** g.uniform(-38, 38, T)).astype(np.float32)    # every fp32 binade
        col[g.random(T) < 0.1] = 0.0
        vals = [float(x) for x in col]
        assert P.sequence_sum(vals) == math.fsum(vals)
    assert math.isnan(P.sequence_sum([1.0, float("nan"), float("inf")]))
    assert P.sequence_sum([1.0, float("inf")]) == float("inf")
    assert P.sequence_sum([0.0] * 7) == 0.0
