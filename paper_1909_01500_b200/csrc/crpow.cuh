// Correctly rounded fp32 power and fixed-point quantisation for the priority
// transform:
//
//   p = RN64(|delta| + eps_p);  v = RN32(p^alpha);  q = RNE(v * 2^F) clamped to q_cap.
//
// Fast path: fp64 pow (<= 2 ulp64 per the CUDA math library) rounded to fp32 is
// accepted when it lies more than 8 ulp64 from the fp32 rounding midpoint on its
// side (Ziv's test).  Otherwise p^alpha is re-evaluated as exp(alpha log p) in
// double-double arithmetic (~2^-100 relative) and compared with that midpoint.
// fp32 midpoints are 2^29 ulp64 apart, so the slow path runs for ~2^-25 of inputs.
#pragma once
#include <math.h>
#include <stdint.h>

namespace rpl {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_ldexp(dd a, int e) { return {ldexp(a.hi, e), ldexp(a.lo, e)}; }

// ln 2 to ~107 bits
#define RPL_LN2_HI 6.93147180559945286227e-01
#define RPL_LN2_LO 2.31904681384629955842e-17

// exp of a double-double argument, |z| < 700, relative error ~1e-30.
static __device__ __noinline__ dd dd_exp(dd z) {
  const double k = rint(z.hi * 1.44269504088896338700);  // 1/ln2
  // r = z - k ln2 (k is an integer < 2^11: k*LN2_HI is exact up to the fma remainder)
  dd kl = two_prod(k, RPL_LN2_HI);
  kl.lo = fma(k, RPL_LN2_LO, kl.lo);
  dd r = dd_add(z, dd{-kl.hi, -kl.lo});
  r = dd_ldexp(r, -10);  // |r| < 2^-10 * 0.35
  // Taylor: e^r = sum r^i / i!, i <= 12  (r^13/13! < 1e-50)
  dd term = {1.0, 0.0};
  dd sum = {1.0, 0.0};
#pragma unroll 1
  for (int i = 1; i <= 12; ++i) {
    term = dd_mul(term, r);
    // divide by i: term / i  (dd / double)
    double q1 = term.hi / (double)i;
    dd pq = two_prod(q1, (double)i);
    double rem = ((term.hi - pq.hi) - pq.lo + term.lo) / (double)i;
    term = quick_two_sum(q1, rem);
    sum = dd_add(sum, term);
  }
#pragma unroll 1
  for (int i = 0; i < 10; ++i) sum = dd_mul(sum, sum);
  return dd_ldexp(sum, (int)k);
}

// natural log of a positive double as double-double: one Newton step
// y1 = y0 + x e^{-y0} - 1 from the libm value y0 (error squares: ~1e-32).
static __device__ __noinline__ dd dd_log(double x) {
  const double y0 = log(x);
  dd e = dd_exp(dd{-y0, 0.0});
  dd xe = dd_mul_d(e, x);
  dd t = dd_add(xe, dd{-1.0, 0.0});
  return dd_add(dd{y0, 0.0}, t);
}

// Fast p^alpha for p > 0 finite: exp(alpha * ln p) in plain fp64 — ln m = 2 atanh(s),
// s = (m-1)/(m+1) with m in [sqrt(1/2), sqrt(2)) (|s| <= 0.1716, odd series to s^21), ln p =
// e ln2 + ln m with ln2 split hi (32 bits, so e ln2_hi is exact) / lo; exp(t) = 2^k exp(r),
// |r| <= ln2 / 2, Taylor to r^13.  Every step is a few fp64 roundings, so the relative error
// is below (|t| + 3) * 3e-16 (ln m to ~3 ulp absolute 1.2e-16, t = alpha ln p to |t| * 2^-52,
// exp(r) to ~3 ulp); *mrel returns a bound 20-50x larger, (|t| + 8) * 2^-47, for the Ziv
// test.  Returns -1 outside t in [-103, 88] (fp32 underflow / overflow region: the caller
// uses the libm path there).  ~45 dependent fp64 operations instead of libm pow's double-
// double log / exp (the update kernel's power stage: ~1 us).
__device__ __forceinline__ double fast_pow(double p, double alpha, double* mrel) {
  long long bits = __double_as_longlong(p);
  int ex = (int)((bits >> 52) & 0x7ff);
  int e = 0;
  if (ex == 0) {  // subnormal: scale by 2^54
    p *= 18014398509481984.0;
    bits = __double_as_longlong(p);
    ex = (int)((bits >> 52) & 0x7ff);
    e = -54;
  }
  e += ex - 1023;
  double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);  // [1, 2)
  if (m > 1.4142135623730951) {
    m *= 0.5;
    e += 1;
  }
  const double f = m - 1.0;  // exact (m in [0.70, 1.42))
  double rd;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(2.0 + f));
  const double den = 2.0 + f;
  double er = fma(-den, rd, 1.0);
  rd = fma(rd, er, rd);
  er = fma(-den, rd, 1.0);
  rd = fma(rd, er, rd);
  const double s = f * rd;
  const double z = s * s;
  double P = 1.0 / 21.0;
  P = fma(P, z, 1.0 / 19.0);
  P = fma(P, z, 1.0 / 17.0);
  P = fma(P, z, 1.0 / 15.0);
  P = fma(P, z, 1.0 / 13.0);
  P = fma(P, z, 1.0 / 11.0);
  P = fma(P, z, 1.0 / 9.0);
  P = fma(P, z, 1.0 / 7.0);
  P = fma(P, z, 1.0 / 5.0);
  P = fma(P, z, 1.0 / 3.0);
  P = fma(P, z, 1.0);
  const double lnm = 2.0 * s * P;
  constexpr double LN2_HI = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000: 32 significant bits
  constexpr double LN2_LO = 1.90821492927058770002e-10;
  const double lp = fma((double)e, LN2_HI, fma((double)e, LN2_LO, lnm));
  const double t = alpha * lp;
  *mrel = (fabs(t) + 8.0) * 7.105427357601002e-15;  // 2^-47
  if (!(t >= -103.0 && t <= 88.0)) return -1.0;
  const double k = rint(t * 1.4426950408889634);
  double r = fma(-k, LN2_HI, t);
  r = fma(-k, LN2_LO, r);
  double q = 1.0 / 6227020800.0;  // 1/13!
  q = fma(q, r, 1.0 / 479001600.0);
  q = fma(q, r, 1.0 / 39916800.0);
  q = fma(q, r, 1.0 / 3628800.0);
  q = fma(q, r, 1.0 / 362880.0);
  q = fma(q, r, 1.0 / 40320.0);
  q = fma(q, r, 1.0 / 5040.0);
  q = fma(q, r, 1.0 / 720.0);
  q = fma(q, r, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  return q * __longlong_as_double((long long)((int)k + 1023) << 52);
}

// v = RN32(p^alpha) for p > 0 (finite), alpha >= 0.  Sets *slow when the fallback ran.
__device__ __forceinline__ float cr_powf(double p, double alpha, bool force_slow, bool* slow) {
  if (alpha == 0.0) return 1.0f;
  if (alpha == 1.0) return __double2float_rn(p);
  if (!force_slow) {  // fast path: accepted when it lies beyond its error bound from the fp32 midpoint
    double mrel;
    const double yf = fast_pow(p, alpha, &mrel);
    if (yf > 0.0) {
      const float f = __double2float_rn(yf);
      const double fd = (double)f;
      const float nb = (yf >= fd) ? nextafterf(f, __int_as_float(0x7f800000)) : nextafterf(f, 0.0f);
      const double mid = 0.5 * (fd + (double)nb);
      if (fabs(yf - mid) > mrel * yf) return f;
    }
  }
  const double y = pow(p, alpha);
  if (!(y < 3.4028235677973366e38)) return __int_as_float(0x7f800000);  // overflow -> +inf
  const float f = __double2float_rn(y);
  const double fd = (double)f;
  const float nb = (y >= fd) ? nextafterf(f, __int_as_float(0x7f800000)) : nextafterf(f, 0.0f);
  const double mid = 0.5 * (fd + (double)nb);  // exact: fp32 values sum exactly in fp64
  const double ulp64 = fabs(y) * 2.220446049250313e-16;
  if (!force_slow && fabs(y - mid) > 8.0 * ulp64) return f;
  *slow = true;
  // slow path: compare p^alpha with mid using exp(alpha ln p) in double-double
  dd lnp = dd_log(p);
  dd z = dd_mul_d(lnp, alpha);
  dd yy = dd_exp(z);
  const double diff = (yy.hi - mid) + yy.lo;  // yy.hi - mid exact when close
  const double tiny = fabs(mid) * 1e-28;
  bool above;
  if (diff > tiny) above = true;
  else if (diff < -tiny) above = false;
  else {
    // indistinguishable from the midpoint: ties to even
    const float lo = fminf(f, nb), hi = fmaxf(f, nb);
    return (__float_as_uint(lo) & 1u) ? hi : lo;
  }
  const float lo = fminf(f, nb), hi = fmaxf(f, nb);
  // mid lies between lo and hi; p^alpha above mid -> hi
  return above ? hi : lo;
}

// q = RNE(v * 2^F) for v >= 0 an fp32 value; saturates at cap.
__device__ __forceinline__ int64_t quantise_q(float v, int F, int64_t cap, bool* sat) {
  const uint32_t bits = __float_as_uint(v);
  const uint32_t ex = (bits >> 23) & 0xff;
  uint32_t man = bits & 0x7fffff;
  if (ex == 0xff) {  // inf / nan
    *sat = true;
    return cap;
  }
  int E;
  if (ex == 0) {
    E = -149;
  } else {
    man |= 0x800000u;
    E = (int)ex - 150;
  }
  if (man == 0) return 0;
  const int shift = E + F;
  int64_t q;
  if (shift >= 0) {
    const int bl = 32 - __clz(man);
    if (bl + shift > 62) {
      *sat = true;
      return cap;
    }
    q = (int64_t)man << shift;
  } else {
    const int s = -shift;
    if (s >= 25) return 0;  // man * 2^-s < 1/2 (or == 1/2 with an even 0)
    uint64_t m = man;
    uint64_t qq = m >> s;
    const uint64_t rem = m & ((1ull << s) - 1);
    const uint64_t half = 1ull << (s - 1);
    if (rem > half || (rem == half && (qq & 1))) ++qq;
    q = (int64_t)qq;
  }
  if (q > cap) {
    *sat = true;
    return cap;
  }
  return q;
}

}  // namespace rpl
