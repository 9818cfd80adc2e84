// R2D2 sequence priority (§8f NEXT-1, reading R26) — shared by the update kernels (sumtree.cu)
// and the gather's fused update (gather.cu).  Included INSIDE namespace rpl { namespace { ... }
// of each translation unit (device code only; needs <stdint.h> and the CUDA intrinsics).
#pragma once

// R2D2 sequence priority (§8f NEXT-1, reading R26): column i of the time-major per-step
// |delta| [T_p, n] -> RN32(eta * max + (1 - eta) * RN64(exact sum) / T_p).  The sum is the
// EXACT sum rounded once to fp64 — the same value for any order of the inputs — computed by
// eight lanes per sequence (lane j takes rows t = j mod 8):
//   fast path  an fp64 sum, which is exact in ANY order when every non-zero |d| is a multiple
//              of the smallest one's fp32 quantum 2^(Emin-150) and the total is below
//              2^53 of those quanta: Emax - Emin + 24 + ceil(log2 T_p) <= 53 (exponents of
//              the non-zero entries; typical priority columns span far fewer binades);
//   slow path  otherwise (taken by the whole warp if any of its sequences needs it): a
//              fixed-point superaccumulator in units of 2^-149 (the fp32 quantum), nine int64
//              bins of 32-bit digits (24-bit significand << up to 253), lanes combined by
//              integer adds, carries propagated, the top 64 bits rounded once to fp64 with a
//              sticky bit.
// All 32 lanes of the warp must call (groups of 8 consecutive lanes share i).  No FMA.
constexpr int SA_DIGITS = 9;

__device__ __forceinline__ void sa_add(int64_t (&bins)[SA_DIGITS], uint32_t bits) {
  const uint32_t E = (bits >> 23) & 0xffu;
  const uint32_t M = E ? ((bits & 0x7fffffu) | 0x800000u) : (bits & 0x7fffffu);
  const int sh = E ? (int)E - 1 : 0;  // value = M << sh in units of 2^-149
  const int d = sh >> 5;
  const uint64_t part = (uint64_t)M << (sh & 31);
  const int64_t lo = (int64_t)(part & 0xffffffffull), hi = (int64_t)(part >> 32);
#pragma unroll
  for (int k = 0; k < SA_DIGITS; ++k) bins[k] += (k == d ? lo : 0) + (k == d + 1 ? hi : 0);
}

// RN64 of the superaccumulator's value (digits in base 2^32, units of 2^-149).
__device__ __forceinline__ double sa_round(const int64_t (&bins)[SA_DIGITS]) {
  uint32_t dg[SA_DIGITS + 1];
  uint64_t carry = 0;
#pragma unroll
  for (int k = 0; k < SA_DIGITS; ++k) {
    const uint64_t v = (uint64_t)bins[k] + carry;
    dg[k] = (uint32_t)v;
    carry = v >> 32;
  }
  dg[SA_DIGITS] = (uint32_t)carry;
  int h = -1;
#pragma unroll
  for (int k = 0; k <= SA_DIGITS; ++k)
    if (dg[k]) h = k;
  if (h < 0) return 0.0;
  uint32_t a = 0, b = 0, c = 0;
  bool sticky = false;
#pragma unroll
  for (int k = 0; k <= SA_DIGITS; ++k) {
    if (k == h) a = dg[k];
    if (k == h - 1) b = dg[k];
    if (k == h - 2) c = dg[k];
    if (k < h - 2 && dg[k]) sticky = true;
  }
  const int lz = __clz(a);
  const uint64_t ab = ((uint64_t)a << 32) | b;
  uint64_t top = lz ? ((ab << lz) | (c >> (32 - lz))) : ab;  // bit 63: the leading one
  const uint32_t rest = lz ? (c << lz) : c;
  if (rest) sticky = true;
  if (sticky) top |= 1ull;  // below the rounding position of 64 -> 53 bits: exact RN
  // top's bit 0 has weight 2^(32 h - 32 - lz) units of 2^-149
  return ldexp(__ull2double_rn(top), 32 * h - 32 - lz - 149);
}

// Exact sum of the |d| of rows t = j (mod 8) over the 8-lane group, rounded once (RN64).
// All 32 lanes call.  Non-finite entries are skipped (the caller handles them).
__device__ __noinline__ double seq_exact_sum(const float* __restrict__ steps, int64_t T_p, int64_t n, int64_t i,
                                             bool active) {
  int64_t bins[SA_DIGITS];
#pragma unroll
  for (int k = 0; k < SA_DIGITS; ++k) bins[k] = 0;
  if (active)
    for (int64_t t = threadIdx.x & 7; t < T_p; t += 8) {
      const uint32_t bits = __float_as_uint(__ldg(steps + t * n + i)) & 0x7fffffffu;
      if ((bits >> 23) != 255u) sa_add(bins, bits);
    }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1)
#pragma unroll
    for (int k = 0; k < SA_DIGITS; ++k)
      bins[k] += (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)bins[k], o);
  return sa_round(bins);
}

constexpr int TD8_BATCH = 16;
// The first 8 * TD8_BATCH rows of a sequence's column: every load issued before the first is
// consumed (one L2 round trip, not one per unrolled group)
__device__ __forceinline__ void sequence_td8_load(float (&vals)[TD8_BATCH], const float* __restrict__ steps,
                                                  int64_t T_p, int64_t n, int64_t i, bool active) {
  const int j = threadIdx.x & 7;
#pragma unroll
  for (int u = 0; u < TD8_BATCH; ++u) {
    const int64_t t = j + 8 * (int64_t)u;
    vals[u] = (active && t < T_p) ? __ldg(steps + t * n + i) : 0.0f;
  }
}

__device__ __forceinline__ float sequence_td8_finish(const float (&vals)[TD8_BATCH], const float* __restrict__ steps,
                                                     int64_t T_p, int64_t n, int64_t i, bool active, double eta) {
  // The exponent window and the max come from the raw bits: |d| >= 0, so the bit patterns of
  // the entries order like their values — the largest pattern is the max (and flags inf /
  // NaN), the smallest non-zero pattern (min of bits - 1, a zero wrapping to 0xffffffff) gives
  // the smallest exponent.  Three integer ops and one fp64 add per entry.
  const int j = threadIdx.x & 7;
  double sm = 0.0;
  uint32_t bmax = 0u, bmin1 = 0xffffffffu;
  auto take = [&](float x) {
    const uint32_t bits = __float_as_uint(x) & 0x7fffffffu;
    bmax = max(bmax, bits);
    bmin1 = min(bmin1, bits - 1u);
    sm = __dadd_rn(sm, (double)__uint_as_float(bits));
  };
  if (active) {
#pragma unroll
    for (int u = 0; u < TD8_BATCH; ++u)
      if (j + 8 * (int64_t)u < T_p) take(vals[u]);
    for (int64_t t = j + 8 * (int64_t)TD8_BATCH; t < T_p; t += 8) take(__ldg(steps + t * n + i));
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    const double so = __shfl_xor_sync(0xffffffffu, sm, o);
    bmax = max(bmax, (uint32_t)__shfl_xor_sync(0xffffffffu, bmax, o));
    bmin1 = min(bmin1, (uint32_t)__shfl_xor_sync(0xffffffffu, bmin1, o));
    sm = __dadd_rn(sm, so);  // IEEE addition is commutative: both partners get the same sum
  }
  const int nonfin = bmax > 0x7f800000u ? 2 : (bmax == 0x7f800000u ? 1 : 0);  // 2 NaN, 1 inf
  const int emax = bmax == 0u ? 0 : max((int)(bmax >> 23), 1);              // denormals: exponent 1
  const int emin = bmin1 == 0xffffffffu ? 255 : max((int)((bmin1 + 1u) >> 23), 1);
  const double mx = nonfin == 2 ? 0.0 : (double)__uint_as_float(bmax);       // NaN never wins
  const int lgT = T_p <= 1 ? 0 : 64 - __clzll((unsigned long long)(T_p - 1));  // ceil(log2 T_p)
  const bool exact = nonfin || emax == 0 || (emax - emin + 24 + lgT <= 53);
  if (__any_sync(0xffffffffu, active && !exact)) {
    // slow path (whole warp, out of line: it is rare and must not bloat the hot code)
    const double se = seq_exact_sum(steps, T_p, n, i, active);
    if (!exact) sm = se;
  }
  if (nonfin) sm = (nonfin & 2) ? __longlong_as_double(0x7ff8000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
  const double mean = __ddiv_rn(sm, (double)T_p);
  const double mix = __dadd_rn(__dmul_rn(eta, mx), __dmul_rn(__dadd_rn(1.0, -eta), mean));
  return __double2float_rn(mix);
}

__device__ __forceinline__ float sequence_td8(const float* __restrict__ steps, int64_t T_p, int64_t n, int64_t i,
                                              bool active, double eta) {
  float vals[TD8_BATCH];
  sequence_td8_load(vals, steps, T_p, n, i, active);
  return sequence_td8_finish(vals, steps, T_p, n, i, active, eta);
}


// The same mix with G lanes per sequence (G = 2, 4 or 8) and BATCH rows per lane in registers:
// more sequences per pass where a CTA computes a whole batch of them (the one-launch step's
// gather: 224 threads, 56 sequences per pass at G = 4 instead of 28 at G = 8).  Same result
// bits as the 8-lane form: the max and the exponent window come from bit patterns, and the
// sum is either provably exact in any order or taken from the exact accumulator.
template <int G>
__device__ __noinline__ double seq_exact_sum_g(const float* __restrict__ steps, int64_t T_p, int64_t n, int64_t i,
                                               bool active) {
  int64_t bins[SA_DIGITS];
#pragma unroll
  for (int k = 0; k < SA_DIGITS; ++k) bins[k] = 0;
  if (active)
    for (int64_t t = threadIdx.x & (G - 1); t < T_p; t += G) {
      const uint32_t bits = __float_as_uint(__ldg(steps + t * n + i)) & 0x7fffffffu;
      if ((bits >> 23) != 255u) sa_add(bins, bits);
    }
#pragma unroll
  for (int o = 1; o < G; o <<= 1)
#pragma unroll
    for (int k = 0; k < SA_DIGITS; ++k)
      bins[k] += (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)bins[k], o);
  return sa_round(bins);
}

template <int G, int BATCH>
__device__ __forceinline__ void sequence_tdg_load(float (&vals)[BATCH], const float* __restrict__ steps, int64_t T_p,
                                                  int64_t n, int64_t i, bool active) {
  const int j = threadIdx.x & (G - 1);
#pragma unroll
  for (int u = 0; u < BATCH; ++u) {
    const int64_t t = j + G * (int64_t)u;
    vals[u] = (active && t < T_p) ? __ldg(steps + t * n + i) : 0.0f;
  }
}

template <int G, int BATCH>
__device__ __forceinline__ float sequence_tdg_finish(const float (&vals)[BATCH], const float* __restrict__ steps,
                                                     int64_t T_p, int64_t n, int64_t i, bool active, double eta) {
  const int j = threadIdx.x & (G - 1);
  double sm = 0.0;
  uint32_t bmax = 0u, bmin1 = 0xffffffffu;
  auto take = [&](float x) {
    const uint32_t bits = __float_as_uint(x) & 0x7fffffffu;
    bmax = max(bmax, bits);
    bmin1 = min(bmin1, bits - 1u);
    sm = __dadd_rn(sm, (double)__uint_as_float(bits));
  };
  if (active) {
#pragma unroll
    for (int u = 0; u < BATCH; ++u)
      if (j + G * (int64_t)u < T_p) take(vals[u]);
    for (int64_t t = j + G * (int64_t)BATCH; t < T_p; t += G) take(__ldg(steps + t * n + i));
  }
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    const double so = __shfl_xor_sync(0xffffffffu, sm, o);
    bmax = max(bmax, (uint32_t)__shfl_xor_sync(0xffffffffu, bmax, o));
    bmin1 = min(bmin1, (uint32_t)__shfl_xor_sync(0xffffffffu, bmin1, o));
    sm = __dadd_rn(sm, so);
  }
  const int nonfin = bmax > 0x7f800000u ? 2 : (bmax == 0x7f800000u ? 1 : 0);
  const int emax = bmax == 0u ? 0 : max((int)(bmax >> 23), 1);
  const int emin = bmin1 == 0xffffffffu ? 255 : max((int)((bmin1 + 1u) >> 23), 1);
  const double mx = nonfin == 2 ? 0.0 : (double)__uint_as_float(bmax);
  const int lgT = T_p <= 1 ? 0 : 64 - __clzll((unsigned long long)(T_p - 1));
  const bool exact = nonfin || emax == 0 || (emax - emin + 24 + lgT <= 53);
  if (__any_sync(0xffffffffu, active && !exact)) {
    const double se = seq_exact_sum_g<G>(steps, T_p, n, i, active);
    if (!exact) sm = se;
  }
  if (nonfin) sm = (nonfin & 2) ? __longlong_as_double(0x7ff8000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
  const double mean = __ddiv_rn(sm, (double)T_p);
  const double mix = __dadd_rn(__dmul_rn(eta, mx), __dmul_rn(__dadd_rn(1.0, -eta), mean));
  return __double2float_rn(mix);
}
