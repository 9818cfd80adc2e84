// Return estimation over time-major [T,B] buffers.
//
//   discounted  R_t = r_t + gamma (1-d_t) R_{t+1}
//   GAE         A_t = delta_t + gamma lambda (1-d_t) A_{t+1}
//   n-step      R^n_t, done^n_t (+ optional bootstrap / rescaling)
//   rescale     h, h^-1 elementwise                                   S:810, §8c #4
//
// Design (B200): the reverse linear recurrences x_t = a_t x_{t+1} + b_t are
// chunked scans.  A CTA owns 32 columns (lane = column: every row is one
// coalesced 128-byte warp load) and WARPS warps split a chunk of WARPS*S rows;
// each thread keeps its S rows in registers, composes its segment's affine map
// (A, B) in fp64, the CTA combines the maps through shared memory, and every
// thread re-applies the map to its registers to emit outputs.  Each input byte
// is read from HBM once and each output written once: 9 B/elem (discounted),
// 17 B/elem (GAE).  fp64 accumulation with one rounding to fp32 keeps the 1e-5
// relative bound where fp32 scans lose everything to cancellation (§8c #21).
#include <cuda.h>
#include <math.h>
#include <stdlib.h>

#include <atomic>

#include "common.cuh"

namespace rpl {

namespace {

#ifndef RPL_SCAN_WARPS  // build-flag A/B knobs: warps x rows per thread of a 128-row chunk
#define RPL_SCAN_WARPS 16
#endif
#ifndef RPL_SCAN_S
#define RPL_SCAN_S 8
#endif
constexpr int SCAN_WARPS = RPL_SCAN_WARPS;
constexpr int SCAN_S = RPL_SCAN_S;

template <int WARPS, int S, bool GAE>
__global__ void __launch_bounds__(WARPS * 32)
k_scan(const float* __restrict__ r, const float* __restrict__ v, const uint8_t* __restrict__ d,
       const float* __restrict__ boot, int64_t T, int64_t B, double gamma, double lam,
       float* __restrict__ out0, float* __restrict__ out1, const float* __restrict__ vterm) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t col = (int64_t)blockIdx.x * 32 + lane;
  const bool cv = col < B;
  __shared__ double sA[WARPS][32];
  __shared__ double sB[WARPS][32];
  __shared__ double sCarry[32];
  pdl_wait();

  // carry = x just after the current chunk: R_T = bootstrap (discounted), A_T = 0 (GAE)
  if (w == 0) sCarry[lane] = (!GAE && boot != nullptr && cv) ? (double)boot[col] : 0.0;
  const double bootv = (GAE && cv) ? (double)boot[col] : 0.0;
  const double ga = GAE ? gamma * lam : gamma;

  const int64_t CH = (int64_t)WARPS * S;
  const int64_t nchunks = (T + CH - 1) / CH;
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    const int64_t t0 = c * CH + (int64_t)w * S;
    // registers: b_t in fp64, V_t (GAE) in fp32, done flags as a bitmask; a_t = ga (1 - d_t)
    double b[S];
    float vv[S];
    float rr[S];
    uint32_t dmask = 0, tmask = 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const int64_t t = t0 + i;
      const bool ok = cv && t < T;
      rr[i] = ok ? __ldg(r + t * B + col) : 0.f;
      const uint8_t di = ok ? __ldg(d + t * B + col) : (uint8_t)0;
      dmask |= (di ? 1u : 0u) << i;
      tmask |= (di == RPL_DONE_TIMEOUT ? 1u : 0u) << i;
      if (GAE) vv[i] = ok ? __ldg(v + t * B + col) : 0.f;
    }
    double vseg_next = 0.0;
    if (GAE && cv && t0 < T) {
      const int64_t tn = t0 + S;
      vseg_next = tn < T ? (double)__ldg(v + tn * B + col) : bootv;
    }
    // rows past T are identity maps (a = 1, b = 0)
    const int nvalid = cv ? (int)max((int64_t)0, min((int64_t)S, T - t0)) : 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double nd = ((dmask >> i) & 1u) ? 0.0 : 1.0;
      // time-limit row (R34): gamma * v_term where gamma * (next value) would stand (rare: the
      // load is issued only for such rows)
      const double tl = (vterm && ((tmask >> i) & 1u) && i < nvalid)
                            ? gamma * (double)__ldg(vterm + (t0 + i) * B + col) : 0.0;
      if (GAE) {
        double vnext;
        if (i + 1 < S) vnext = (i + 1 < nvalid) ? (double)vv[i + 1] : bootv;
        else vnext = vseg_next;
        b[i] = i < nvalid ? (((double)rr[i] + gamma * nd * vnext) + tl) - (double)vv[i] : 0.0;
      } else {
        b[i] = i < nvalid ? (double)rr[i] + tl : 0.0;
      }
    }
#define RPL_A(i) ((i) < nvalid ? (((dmask >> (i)) & 1u) ? 0.0 : ga) : 1.0)
    // segment map: x_{t0} = A * x_{t0+S} + Bc
    double A = 1.0, Bc = 0.0;
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      const double ai = RPL_A(i);
      Bc = fma(ai, Bc, b[i]);
      A = ai * A;
    }
    sA[w][lane] = A;
    sB[w][lane] = Bc;
    __syncthreads();
    double x = sCarry[lane];
#pragma unroll
    for (int ww = WARPS - 1; ww > 0; --ww) {
      if (ww > w) x = fma(sA[ww][lane], x, sB[ww][lane]);
    }
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      x = fma(RPL_A(i), x, b[i]);
      const int64_t t = t0 + i;
      if (i < nvalid) {
        out0[t * B + col] = (float)x;
        if (GAE && out1 != nullptr) out1[t * B + col] = (float)(x + (double)vv[i]);
      }
    }
#undef RPL_A
    __syncthreads();
    if (w == 0) sCarry[lane] = x;  // x at the chunk's first row
  }
}

// ---------------------------------------------------------------------------
// TMA variant (default when the layout allows it): the CTA's [CH rows x 32 columns]
// tiles of r, V and d arrive by three 2-D tensor copies (cp.async.bulk.tensor) into
// shared memory on one mbarrier instead of 24 LDGs per thread: the per-SM L1 miss
// queue no longer caps the bytes in flight (ncu/globaltimer r1: the LDG load phase was
// ~3.8 us of a 5.9 us call).  OOB rows / columns are zero-filled by the TMA unit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int WARPS, int S, bool GAE>
__global__ void __launch_bounds__(WARPS * 32)
k_scan_tma(const __grid_constant__ CUtensorMap tm_r, const __grid_constant__ CUtensorMap tm_v,
           const __grid_constant__ CUtensorMap tm_d, const float* __restrict__ v, const float* __restrict__ boot,
           int64_t T, int64_t B, double gamma, double lam, float* __restrict__ out0, float* __restrict__ out1,
           int early_trigger, const float* __restrict__ vterm) {
  constexpr int CH = WARPS * S;
  __shared__ __align__(128) float s_r[CH][32];
  __shared__ __align__(128) float s_v[GAE ? CH : 1][32];
  __shared__ __align__(128) uint8_t s_d[CH][32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double sA[WARPS][32];
  __shared__ double sB[WARPS][32];
  __shared__ double sCarry[32];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t col = (int64_t)blockIdx.x * 32 + lane;
  const bool cv = col < B;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_r) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
    if (GAE) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_v) : "memory");
  }
  __syncthreads();
  pdl_wait();
  if (w == 0) sCarry[lane] = (!GAE && boot != nullptr && cv) ? (double)boot[col] : 0.0;
  const double bootv = (GAE && cv) ? (double)boot[col] : 0.0;
  const double ga = GAE ? gamma * lam : gamma;
  const int64_t nchunks = (T + CH - 1) / CH;
  uint32_t phase = 0;
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(CH * 32 * 4 * (GAE ? 2 : 1) + CH * 32);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar)), "r"(bytes)
                   : "memory");
      const int x = blockIdx.x * 32, y = (int)(c * CH);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(s_u32(&s_r[0][0])), "l"(&tm_r), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(s_u32(&s_d[0][0])), "l"(&tm_d), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
      if (GAE)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(s_u32(&s_v[0][0])), "l"(&tm_v), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
    }
    // the next grid may start its prologue now (it still waits for this grid's completion
    // in pdl_wait before touching memory)
    if (early_trigger && c == nchunks - 1) pdl_trigger();
    {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(s_u32(&bar)), "r"(phase) : "memory");
      phase ^= 1u;
    }
    const int64_t t0 = c * CH + (int64_t)w * S;
    double b[S];
    float vv[S];
    float rr[S];
    uint32_t dmask = 0, tmask = 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      rr[i] = s_r[w * S + i][lane];
      dmask |= (s_d[w * S + i][lane] ? 1u : 0u) << i;
      tmask |= (s_d[w * S + i][lane] == RPL_DONE_TIMEOUT ? 1u : 0u) << i;
      if (GAE) vv[i] = s_v[w * S + i][lane];
    }
    double vseg_next = 0.0;
    if (GAE && cv && t0 < T) {
      const int64_t tn = t0 + S;
      if (tn >= T) vseg_next = bootv;
      else if (w + 1 < WARPS) vseg_next = (double)s_v[(w + 1) * S][lane];
      else vseg_next = (double)__ldg(v + tn * B + col);  // first row of the next chunk
    }
    __syncthreads();  // every thread holds its rows: the next chunk's TMA may overwrite the tiles
    const int nvalid = cv ? (int)max((int64_t)0, min((int64_t)S, T - t0)) : 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double nd = ((dmask >> i) & 1u) ? 0.0 : 1.0;
      // time-limit row (R34): gamma * v_term where gamma * (next value) would stand (rare: the
      // load is issued only for such rows)
      const double tl = (vterm && ((tmask >> i) & 1u) && i < nvalid)
                            ? gamma * (double)__ldg(vterm + (t0 + i) * B + col) : 0.0;
      if (GAE) {
        double vnext;
        if (i + 1 < S) vnext = (i + 1 < nvalid) ? (double)vv[i + 1] : bootv;
        else vnext = vseg_next;
        b[i] = i < nvalid ? (((double)rr[i] + gamma * nd * vnext) + tl) - (double)vv[i] : 0.0;
      } else {
        b[i] = i < nvalid ? (double)rr[i] + tl : 0.0;
      }
    }
#define RPL_A(i) ((i) < nvalid ? (((dmask >> (i)) & 1u) ? 0.0 : ga) : 1.0)
    double A = 1.0, Bc = 0.0;
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      const double ai = RPL_A(i);
      Bc = fma(ai, Bc, b[i]);
      A = ai * A;
    }
    sA[w][lane] = A;
    sB[w][lane] = Bc;
    __syncthreads();
    double x = sCarry[lane];
#pragma unroll
    for (int ww = WARPS - 1; ww > 0; --ww) {
      if (ww > w) x = fma(sA[ww][lane], x, sB[ww][lane]);
    }
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      x = fma(RPL_A(i), x, b[i]);
      const int64_t t = t0 + i;
      if (i < nvalid) {
        out0[t * B + col] = (float)x;
        if (GAE && out1 != nullptr) out1[t * B + col] = (float)(x + (double)vv[i]);
      }
    }
#undef RPL_A
    __syncthreads();
    if (w == 0) sCarry[lane] = x;
  }
}

// ---------------------------------------------------------------------------
// Column-group TMA scan with double-buffered chunks: a CTA owns COLS (16 or 32) columns;
// with COLS = 16 each warp's lanes split into two 16-column halves, so a 256-thread CTA
// still covers 128 rows per chunk with S = 8 rows per thread, and a PPO call
// ([128, 4096]) runs 256 CTAs — every SM works, two or three CTAs resident per SM so one
// CTA's stores overlap another's loads.  Chunks are prefetched one ahead into the second
// tile buffer (TMA), so for long horizons the next chunk's load overlaps this chunk's scan
// and stores.  The V value just after a chunk (GAE) is kept from the chunk processed before
// it (the scan runs from the end), not reloaded.  Same fp64 affine-map arithmetic.
// ---------------------------------------------------------------------------
template <int COLS, int WARPS, int S, bool GAE>
__global__ void __launch_bounds__(WARPS * 32)
k_scan_tma2(const __grid_constant__ CUtensorMap tm_r, const __grid_constant__ CUtensorMap tm_v,
            const __grid_constant__ CUtensorMap tm_d, const float* __restrict__ boot, int64_t T, int64_t B,
            double gamma, double lam, float* __restrict__ out0, float* __restrict__ out1, int early_trigger,
            const float* __restrict__ vterm) {
  constexpr int SUB = 32 / COLS;       // segments per warp
  constexpr int SEGS = WARPS * SUB;
  constexpr int CH = SEGS * S;         // rows per chunk
  __shared__ __align__(128) float s_r[2][CH][COLS];
  __shared__ __align__(128) float s_v[2][GAE ? CH : 1][COLS];
  __shared__ __align__(128) uint8_t s_d[2][CH][COLS];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double sA[SEGS][COLS];
  __shared__ double sB[SEGS][COLS];
  __shared__ double sCarry[COLS];
  __shared__ float sVnext[COLS];       // V of the first row of the chunk processed last (GAE)
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int ci = lane % COLS;
  const int seg = w * SUB + lane / COLS;
  const int64_t col = (int64_t)blockIdx.x * COLS + ci;
  const bool cv = col < B;
  const int64_t nchunks = (T + CH - 1) / CH;
  constexpr uint32_t BYTES = (uint32_t)(CH * COLS * 4 * (GAE ? 2 : 1) + CH * COLS);
  auto issue = [&](int64_t c, int stg) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar[stg])), "r"(BYTES)
                 : "memory");
    const int x = (int)(blockIdx.x * COLS), y = (int)(c * CH);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&s_r[stg][0][0])), "l"(&tm_r), "r"(x), "r"(y), "r"(s_u32(&bar[stg])) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&s_d[stg][0][0])), "l"(&tm_d), "r"(x), "r"(y), "r"(s_u32(&bar[stg])) : "memory");
    if (GAE)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(s_u32(&s_v[stg][0][0])), "l"(&tm_v), "r"(x), "r"(y), "r"(s_u32(&bar[stg])) : "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_r) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
    if (GAE) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_v) : "memory");
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0) {
    issue(nchunks - 1, (int)((nchunks - 1) & 1));
    if (nchunks > 1) issue(nchunks - 2, (int)((nchunks - 2) & 1));
  }
  if (early_trigger) pdl_trigger();  // the next grid's prologue may start (it still waits in pdl_wait)
  const double bootv = (GAE && cv) ? (double)boot[col] : 0.0;
  if (w == 0 && lane < COLS) {
    sCarry[lane] = (!GAE && boot != nullptr && cv) ? (double)boot[col] : 0.0;
    if (GAE) sVnext[lane] = (float)bootv;
  }
  const double ga = GAE ? gamma * lam : gamma;
  uint32_t phases = 0;  // bit s: parity to wait for on stage s
  for (int64_t c = nchunks - 1; c >= 0; --c) {
    const int stg = (int)(c & 1);
    {
      uint32_t done = 0;
      const uint32_t ph = (phases >> stg) & 1u;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(s_u32(&bar[stg])), "r"(ph) : "memory");
      phases ^= 1u << stg;
    }
    const int64_t t0 = c * CH + (int64_t)seg * S;
    double b[S];
    float vv[S];
    float rr[S];
    uint32_t dmask = 0, tmask = 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      rr[i] = s_r[stg][seg * S + i][ci];
      const uint8_t di = s_d[stg][seg * S + i][ci];
      dmask |= (di ? 1u : 0u) << i;
      tmask |= (di == RPL_DONE_TIMEOUT ? 1u : 0u) << i;
      if (GAE) vv[i] = s_v[stg][seg * S + i][ci];
    }
    double vseg_next = 0.0;
    if (GAE) {
      if (t0 + S >= T) vseg_next = bootv;
      else if (seg + 1 < SEGS) vseg_next = (double)s_v[stg][(seg + 1) * S][ci];
      else vseg_next = (double)sVnext[ci];
    }
    __syncthreads();  // every thread holds its rows: this stage may be refilled
    if (threadIdx.x == 0 && c >= 2) issue(c - 2, stg);
    const int nvalid = cv ? (int)max((int64_t)0, min((int64_t)S, T - t0)) : 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double nd = ((dmask >> i) & 1u) ? 0.0 : 1.0;
      const double tl = (vterm && ((tmask >> i) & 1u) && i < nvalid)
                            ? gamma * (double)__ldg(vterm + (t0 + i) * B + col) : 0.0;  // R34
      if (GAE) {
        double vnext;
        if (i + 1 < S) vnext = (i + 1 < nvalid) ? (double)vv[i + 1] : bootv;
        else vnext = vseg_next;
        b[i] = i < nvalid ? (((double)rr[i] + gamma * nd * vnext) + tl) - (double)vv[i] : 0.0;
      } else {
        b[i] = i < nvalid ? (double)rr[i] + tl : 0.0;
      }
    }
#define RPL_A(i) ((i) < nvalid ? (((dmask >> (i)) & 1u) ? 0.0 : ga) : 1.0)
    double A = 1.0, Bc = 0.0;
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      const double ai = RPL_A(i);
      Bc = fma(ai, Bc, b[i]);
      A = ai * A;
    }
    sA[seg][ci] = A;
    sB[seg][ci] = Bc;
    __syncthreads();
    double x = sCarry[ci];
#pragma unroll
    for (int ss = SEGS - 1; ss > 0; --ss) {
      if (ss > seg) x = fma(sA[ss][ci], x, sB[ss][ci]);
    }
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
      x = fma(RPL_A(i), x, b[i]);
      const int64_t t = t0 + i;
      if (i < nvalid) {
        out0[t * B + col] = (float)x;
        if (GAE && out1 != nullptr) out1[t * B + col] = (float)(x + (double)vv[i]);
      }
    }
#undef RPL_A
    __syncthreads();
    if (seg == 0) {
      sCarry[ci] = x;
      if (GAE) sVnext[ci] = vv[0];
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent pipelined scan (variant 9): a CTA walks a list of work items — column group g
// (COLS columns) x chunk c (CH rows), every chunk of a group from the end so the carry stays
// in shared memory — with the loads of the next STAGES-1 items in flight (TMA tiles into a
// ring of stages, one mbarrier each) and the outputs leaving through TMA tensor stores from
// a double-buffered output tile, so one item's scan overlaps the next items' loads and the
// previous item's stores.  Groups are dealt round-robin to the grid (CTAs_per_SM x SMs).
// ---------------------------------------------------------------------------
// Measurement-only timeline of the pipelined scan (-DRPL_TRACE; rpl_debug_scan_trace): CTA 0's
// first item: 0 entry, 1 past the dependency wait, 2 tiles landed, 3 barrier (1), 4 barrier (2),
// 5 barrier (3), 6 store issued, 7 exit; 8 the last CTA's exit (max), 9 the first CTA's exit (min).
#ifdef RPL_TRACE
__device__ unsigned long long g_strace[10];
#define SCAN_TRACE(k)                                                                \
  do {                                                                               \
    if (threadIdx.x == 0 && blockIdx.x == 0 && i == 0) g_strace[k] = global_ns();   \
  } while (0)
#else
#define SCAN_TRACE(k) \
  do {                \
  } while (0)
#endif

template <int COLS, int WARPS, int S, int STAGES, bool GAE, int OB = 2>
struct ScanPipeSmem {
  static constexpr int SUB = 32 / COLS;
  static constexpr int SEGS = WARPS * SUB;
  static constexpr int CH = SEGS * S;
  alignas(128) float r[STAGES][CH][COLS];  // TMA tiles: 128-B aligned
  alignas(128) float v[GAE ? STAGES : 1][GAE ? CH : 1][COLS];
  alignas(128) float o0[OB][CH][COLS];
  alignas(128) float o1[GAE ? OB : 1][GAE ? CH : 1][COLS];
  alignas(128) uint8_t d[STAGES][CH][COLS];
  double sA[SEGS][COLS];
  double sB[SEGS][COLS];
  double carry[COLS];
  float vnext[COLS];
  uint64_t bar[STAGES];
};

template <int COLS, int WARPS, int S, int STAGES, bool GAE, int MINB = 2, int OB = 2>
__global__ void __launch_bounds__(WARPS * 32, MINB)
k_scan_pipe(const __grid_constant__ CUtensorMap tm_r, const __grid_constant__ CUtensorMap tm_v,
            const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ CUtensorMap tm_o0,
            const __grid_constant__ CUtensorMap tm_o1, const float* __restrict__ boot, int64_t T, int64_t B,
            double gamma, double lam, int has_o1, const float* __restrict__ vterm, int early_trigger) {
  using SM = ScanPipeSmem<COLS, WARPS, S, STAGES, GAE, OB>;
  constexpr int SUB = SM::SUB, SEGS = SM::SEGS, CH = SM::CH;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int ci = lane % COLS;
  const int seg = w * SUB + lane / COLS;
  const int64_t ngroups = (B + COLS - 1) / COLS;
  const int64_t nchunks = (T + CH - 1) / CH;
  const int64_t my_groups = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_groups * nchunks;
  constexpr uint32_t BYTES = (uint32_t)(CH * COLS * 4 * (GAE ? 2 : 1) + CH * COLS);
  // items in order: groups blockIdx.x, +gridDim.x, ...; chunks of a group from the last one.
  // Cursors advance incrementally (no 64-bit division per item): (gp, cp, sp) = the next item
  // to load (thread 0 only), (g, c) = the item being scanned.
  int64_t gp = blockIdx.x, cp = nchunks - 1;
  int sp = 0;
  auto issue = [&]() {
    const int64_t g = gp, c = cp;
    const int st = sp;
    if (--cp < 0) {
      cp = nchunks - 1;
      gp += gridDim.x;
    }
    if (++sp == STAGES) sp = 0;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&sm.bar[st])), "r"(BYTES)
                 : "memory");
    const int x = (int)(g * COLS), y = (int)(c * CH);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&sm.r[st][0][0])), "l"(&tm_r), "r"(x), "r"(y), "r"(s_u32(&sm.bar[st])) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&sm.d[st][0][0])), "l"(&tm_d), "r"(x), "r"(y), "r"(s_u32(&sm.bar[st])) : "memory");
    if (GAE)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(s_u32(&sm.v[st][0][0])), "l"(&tm_v), "r"(x), "r"(y), "r"(s_u32(&sm.bar[st])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&sm.bar[st])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_r) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_o0) : "memory");
  }
  __syncthreads();
#ifdef RPL_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) g_strace[0] = global_ns();
#endif
  pdl_wait();
#ifdef RPL_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    g_strace[1] = global_ns();
    g_strace[8] = 0;
    g_strace[9] = ~0ull;
  }
#endif
  if (threadIdx.x == 0)
    for (int64_t i = 0; i < STAGES && i < items; ++i) issue();
  // measurement knob (RPL_SCAN_TRIGGER=2): let the dependent grid launch once the first tiles
  // are requested (it still waits for this grid's completion in its griddepcontrol.wait)
  if (early_trigger == 2) pdl_trigger();
  const double ga = GAE ? gamma * lam : gamma;
  uint32_t phases = 0;  // bit st: parity to wait for on stage st
  int64_t g = blockIdx.x, c = nchunks - 1;
  int st = 0;
  float boot_f = 0.0f;  // V_T of this thread's column (GAE): loaded once per group, only read in its last chunk
  for (int64_t i = 0; i < items; ++i) {
    const int ob = OB == 1 ? 0 : (int)(i & 1);
    const int64_t col = g * COLS + ci;
    const bool cv = col < B;
    if (GAE && c == nchunks - 1) boot_f = cv ? __ldg(boot + col) : 0.0f;  // in flight during the tile wait
    if (c == nchunks - 1 && w == 0 && lane < COLS) {  // a new group: carry = R_T (or A_T = 0), V_T
      const int64_t cc = g * COLS + lane;
      sm.carry[lane] = (!GAE && boot != nullptr && cc < B) ? (double)__ldg(boot + cc) : 0.0;
      if (GAE) sm.vnext[lane] = cc < B ? __ldg(boot + cc) : 0.0f;
    }
    {
      uint32_t done = 0;
      const uint32_t ph = (phases >> st) & 1u;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(s_u32(&sm.bar[st])), "r"(ph) : "memory");
      phases ^= 1u << st;
    }
    SCAN_TRACE(2);
    const int64_t t0 = c * CH + (int64_t)seg * S;
    double b[S];
    float vv[S];
    float rr[S];
    uint32_t dmask = 0, tmask = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      rr[k] = sm.r[st][seg * S + k][ci];
      const uint8_t di = sm.d[st][seg * S + k][ci];
      dmask |= (di ? 1u : 0u) << k;
      if (vterm) tmask |= (di == RPL_DONE_TIMEOUT ? 1u : 0u) << k;
      if (GAE) vv[k] = sm.v[st][seg * S + k][ci];
    }
    __syncthreads();  // (1) the new group's carry is visible; every thread holds its rows
    SCAN_TRACE(3);
    const double bootv = (double)boot_f;
    double vseg_next = 0.0;
    if (GAE) {
      if (t0 + S >= T) vseg_next = bootv;
      else if (seg + 1 < SEGS) vseg_next = (double)sm.v[st][(seg + 1) * S][ci];
      else vseg_next = (double)sm.vnext[ci];
    }
    const int nvalid = cv ? (int)max((int64_t)0, min((int64_t)S, T - t0)) : 0;
    // fast path (every row valid, no time limits): no per-element predicates or selects
    // beyond the done bit; the common case of every chunk but a ragged last one
    const bool fast = nvalid == S && vterm == nullptr;
    double a[S];
    if (fast) {
      double vd[GAE ? S : 1];
#pragma unroll
      for (int k = 0; k < S; ++k) {
        if (GAE) vd[k] = (double)vv[k];
        a[k] = ((dmask >> k) & 1u) ? 0.0 : ga;
      }
#pragma unroll
      for (int k = 0; k < S; ++k) {
        if (GAE) {
          const double gn = ((dmask >> k) & 1u) ? 0.0 : gamma;
          const double vn = k + 1 < S ? vd[(k + 1) % S] : vseg_next;
          b[k] = fma(gn, vn, (double)rr[k]) - vd[k];
        } else {
          b[k] = (double)rr[k];
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const double nd = ((dmask >> k) & 1u) ? 0.0 : 1.0;
        const double tl = (vterm && ((tmask >> k) & 1u) && k < nvalid)
                              ? gamma * (double)__ldg(vterm + (t0 + k) * B + col) : 0.0;  // R34
        if (GAE) {
          double vn;
          if (k + 1 < S) vn = (k + 1 < nvalid) ? (double)vv[k + 1] : bootv;
          else vn = vseg_next;
          b[k] = k < nvalid ? (((double)rr[k] + gamma * nd * vn) + tl) - (double)vv[k] : 0.0;
        } else {
          b[k] = k < nvalid ? (double)rr[k] + tl : 0.0;
        }
        a[k] = k < nvalid ? (((dmask >> k) & 1u) ? 0.0 : ga) : 1.0;
      }
    }
    double A = 1.0, Bc = 0.0;
#pragma unroll
    for (int k = S - 1; k >= 0; --k) {
      Bc = fma(a[k], Bc, b[k]);
      A = a[k] * A;
    }
    sm.sA[seg][ci] = A;
    sm.sB[seg][ci] = Bc;
    if (threadIdx.x == 0) {
      // the output tile about to be written held item i-2's outputs: their store must have
      // finished reading it (at most one store group, item i-1's, stays in flight)
      if (OB == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    __syncthreads();  // (2) maps visible; this stage is free; the output tile is free
    SCAN_TRACE(4);
    if (threadIdx.x == 0 && i + STAGES < items) issue();
    double x = sm.carry[ci];
#pragma unroll
    for (int ss = SEGS - 1; ss > 0; --ss)
      if (ss > seg) x = fma(sm.sA[ss][ci], x, sm.sB[ss][ci]);
#pragma unroll
    for (int k = S - 1; k >= 0; --k) {
      x = fma(a[k], x, b[k]);
      sm.o0[ob][seg * S + k][ci] = (float)x;
      if (GAE) sm.o1[ob][seg * S + k][ci] = (float)(x + (double)vv[k]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
    __syncthreads();  // (3) the output tile is complete; maps / carry reads done
    SCAN_TRACE(5);
    if (seg == 0) {
      sm.carry[ci] = x;
      if (GAE) sm.vnext[ci] = vv[0];
    }
    if (threadIdx.x == 0) {
      const int x0 = (int)(g * COLS), y0 = (int)(c * CH);
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(&tm_o0), "r"(x0), "r"(y0), "r"(s_u32(&sm.o0[ob][0][0])) : "memory");
      if (GAE && has_o1)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(&tm_o1), "r"(x0), "r"(y0), "r"(s_u32(&sm.o1[ob][0][0])) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    SCAN_TRACE(6);
    if (--c < 0) {
      c = nchunks - 1;
      g += gridDim.x;
    }
    if (++st == STAGES) st = 0;
  }
  // the dependent grid may launch now; the CTA stays until its last output tile has been read
  // out of shared memory (the bulk stores complete before the grid does, as for any store)
  pdl_trigger();
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#ifdef RPL_TRACE
  if (threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    if (blockIdx.x == 0) g_strace[7] = t;
    atomicMax(&g_strace[8], t);
    atomicMin(&g_strace[9], t);
  }
#endif
}

// ---------------------------------------------------------------------------
// Cluster variant for short horizons (T <= CL * WARPS * S, e.g. PPO's T = 128; selectable,
// not the default — see launch_scan for the measurement): the rows
// of a 32-column group are split over a thread-block cluster of CL CTAs along T, so each
// CTA moves 1/CL of the bytes (its TMA tiles arrive CL times sooner) and CL times more
// SMs work on the call.  Each CTA composes its rows' affine maps into one CTA map per
// column; after a cluster barrier, CTA `rank` reads the maps of ranks > rank from their
// shared memory (DSMEM, ld.shared::cluster) to form its carry-in, then emits its rows.
// A second cluster barrier keeps every CTA's maps alive until all readers are done.
// ---------------------------------------------------------------------------
template <int WARPS, int S, int CL, bool GAE>
__global__ void __launch_bounds__(WARPS * 32)
k_scan_cluster(const __grid_constant__ CUtensorMap tm_r, const __grid_constant__ CUtensorMap tm_v,
               const __grid_constant__ CUtensorMap tm_d, const float* __restrict__ v, const float* __restrict__ boot,
               int64_t T, int64_t B, double gamma, double lam, float* __restrict__ out0, float* __restrict__ out1,
               const float* __restrict__ vterm) {
  constexpr int CH = WARPS * S;  // rows per CTA
  __shared__ __align__(128) float s_r[CH][32];
  __shared__ __align__(128) float s_v[GAE ? CH : 1][32];
  __shared__ __align__(128) uint8_t s_d[CH][32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double sA[WARPS][32];
  __shared__ double sB[WARPS][32];
  __shared__ double sMap[2][32];  // this CTA's composed map (A, B) per column, read by lower ranks
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int64_t cg = blockIdx.x / CL;
  const int64_t col = cg * 32 + lane;
  const bool cv = col < B;
  const int64_t row0 = (int64_t)rank * CH;
  const bool has_rows = row0 < T;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_r) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_d) : "memory");
    if (GAE) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_v) : "memory");
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0 && has_rows) {
    const uint32_t bytes = (uint32_t)(CH * 32 * 4 * (GAE ? 2 : 1) + CH * 32);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&bar)), "r"(bytes) : "memory");
    const int x = (int)(cg * 32), y = (int)row0;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&s_r[0][0])), "l"(&tm_r), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(s_u32(&s_d[0][0])), "l"(&tm_d), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
    if (GAE)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(s_u32(&s_v[0][0])), "l"(&tm_v), "r"(x), "r"(y), "r"(s_u32(&bar)) : "memory");
  }
  // loads that do not depend on the tiles, issued while they are in flight
  const double bootv = (GAE && cv) ? (double)__ldg(boot + col) : 0.0;
  const double carry0 = (!GAE && boot != nullptr && cv) ? (double)__ldg(boot + col) : 0.0;
  const int64_t t0 = row0 + (int64_t)w * S;
  const int64_t tn = t0 + S;  // first row after this thread's segment
  double vnext_global = 0.0;
  if (GAE && cv && w == WARPS - 1 && tn < T) vnext_global = (double)__ldg(v + tn * B + col);  // next CTA's first row
  const double ga = GAE ? gamma * lam : gamma;
  if (has_rows) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done) : "r"(s_u32(&bar)), "r"(0u) : "memory");
  }
  double b[S];
  float vv[S];
  float rr[S];
  uint32_t dmask = 0, tmask = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    rr[i] = has_rows ? s_r[w * S + i][lane] : 0.f;
    dmask |= ((has_rows && s_d[w * S + i][lane]) ? 1u : 0u) << i;
    tmask |= ((has_rows && s_d[w * S + i][lane] == RPL_DONE_TIMEOUT) ? 1u : 0u) << i;
    if (GAE) vv[i] = has_rows ? s_v[w * S + i][lane] : 0.f;
  }
  double vseg_next = 0.0;
  if (GAE && cv && t0 < T) {
    if (tn >= T) vseg_next = bootv;
    else if (w + 1 < WARPS) vseg_next = (double)s_v[(w + 1) * S][lane];
    else vseg_next = vnext_global;
  }
  const int nvalid = cv ? (int)max((int64_t)0, min((int64_t)S, T - t0)) : 0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const double nd = ((dmask >> i) & 1u) ? 0.0 : 1.0;
    const double tl = (vterm && ((tmask >> i) & 1u) && i < nvalid)
                          ? gamma * (double)__ldg(vterm + (t0 + i) * B + col) : 0.0;  // R34
    if (GAE) {
      double vn;
      if (i + 1 < S) vn = (i + 1 < nvalid) ? (double)vv[i + 1] : bootv;
      else vn = vseg_next;
      b[i] = i < nvalid ? (((double)rr[i] + gamma * nd * vn) + tl) - (double)vv[i] : 0.0;
    } else {
      b[i] = i < nvalid ? (double)rr[i] + tl : 0.0;
    }
  }
#define RPL_A(i) ((i) < nvalid ? (((dmask >> (i)) & 1u) ? 0.0 : ga) : 1.0)
  double A = 1.0, Bc = 0.0;
#pragma unroll
  for (int i = S - 1; i >= 0; --i) {
    const double ai = RPL_A(i);
    Bc = fma(ai, Bc, b[i]);
    A = ai * A;
  }
  sA[w][lane] = A;
  sB[w][lane] = Bc;
  __syncthreads();
  if (w == 0) {  // the CTA map: x_{row0} = Acta x_{row0+CH} + Bcta
    double Ac = 1.0, Bcc = 0.0;
#pragma unroll
    for (int ww = WARPS - 1; ww >= 0; --ww) {
      Bcc = fma(sA[ww][lane], Bcc, sB[ww][lane]);
      Ac = sA[ww][lane] * Ac;
    }
    sMap[0][lane] = Ac;
    sMap[1][lane] = Bcc;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  double x = carry0;  // value just after row T-1 (ranks past T hold identity maps)
  for (int rr_ = CL - 1; rr_ > (int)rank; --rr_) {
    uint32_t ra, rb;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(s_u32(&sMap[0][lane])), "r"(rr_));
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(s_u32(&sMap[1][lane])), "r"(rr_));
    double ra_v, rb_v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(ra_v) : "r"(ra) : "memory");
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(rb_v) : "r"(rb) : "memory");
    x = fma(ra_v, x, rb_v);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // done reading remote maps
#pragma unroll
  for (int ww = WARPS - 1; ww > 0; --ww) {
    if (ww > w) x = fma(sA[ww][lane], x, sB[ww][lane]);
  }
#pragma unroll
  for (int i = S - 1; i >= 0; --i) {
    x = fma(RPL_A(i), x, b[i]);
    const int64_t t = t0 + i;
    if (i < nvalid) {
      out0[t * B + col] = (float)x;
      if (GAE && out1 != nullptr) out1[t * B + col] = (float)(x + (double)vv[i]);
    }
  }
#undef RPL_A
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // keep sMap alive for the readers
}

__global__ void k_nstep(const float* __restrict__ r, const uint8_t* __restrict__ d, int64_t T,
                        int64_t B, int n, double gamma, const float* __restrict__ q,
                        const float* __restrict__ q_boot, int rescale, double eps,
                        float* __restrict__ out, uint8_t* __restrict__ done_out, const float* __restrict__ vterm) {
  const int64_t rows = T - n + 1;
  const int64_t total = rows * B;
  // dependent launch at entry: the next call's CTAs sit resident beside this grid's (PPO
  // [128, 4096] n = 5: 6.95 -> 6.83 us rescaled, 4.77 -> 4.55 us plain, profiles/r2/ab_nstep.txt)
  pdl_trigger();
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / B;
    const int64_t b = e - t * B;
    uint8_t dn = 0;
    // Horner from the last of the n rows; rows are fetched in blocks of 8 whose loads
    // are all issued before the recurrence consumes them (one latency per block, not per row).
    // The last block's loads are issued before the bootstrap's load and h^-1, so that
    // round trip overlaps the fp64 square root and divisions instead of following them.
    constexpr int NB = 8;
    float rb[NB];
    uint8_t db[NB];
    auto load_block = [&](int lo, int hi) {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int i = lo + j;
        const int64_t o = (t + i) * B + b;
        rb[j] = i < hi ? __ldg(r + o) : 0.0f;
        db[j] = i < hi ? __ldg(d + o) : (uint8_t)0;
      }
    };
    load_block(n > NB ? n - NB : 0, n);
    double acc = 0.0;
    if (q != nullptr) {
      const double qv = (t + n < T) ? (double)__ldg(q + (t + n) * B + b) : (double)__ldg(q_boot + b);
      acc = rescale ? h_inv(qv, eps) : qv;
    }
    for (int hi = n; hi > 0; hi -= NB) {
      const int lo = hi > NB ? hi - NB : 0;
      if (hi != n) load_block(lo, hi);
#pragma unroll
      for (int j = NB - 1; j >= 0; --j) {
        if (lo + j < hi) {
          const double ri = (double)rb[j];
          if (db[j]) {  // cut; a time-limit row bootstraps from its terminal value (R34)
            acc = (vterm && db[j] == RPL_DONE_TIMEOUT) ? fma(gamma, (double)__ldg(vterm + (t + lo + j) * B + b), ri)
                                                       : ri;
          } else {
            acc = fma(gamma, acc, ri);
          }
          dn |= db[j];
        }
      }
    }
    if (rescale) acc = h_fwd(acc, eps);
    out[e] = (float)acc;
    if (done_out != nullptr) done_out[e] = dn ? 1 : 0;
  }
}

// n-step targets for n <= NS_MAXN (the common case): thread = (column b, run of NS_U
// consecutive outputs t0 .. t0+NS_U-1).  The run's NS_U + n - 1 reward / done rows are loaded
// once into registers (coalesced across the warp's columns, all in flight together) and
// shared by the run's outputs; the grid is 2-D (columns x runs), so no 64-bit division.
// Same arithmetic per output as k_nstep (fp64 Horner from the bootstrap, R24 / R34 / R5).
#ifndef RPL_NSTEP_U  // outputs per thread of k_nstep_runs (build-flag A/B knob; PPO [128,4096] n=5
#define RPL_NSTEP_U 4  // rescaled: U=1 8.86, 2 8.16, 4 6.94, 8 9.69 us per call, scripts/gpu_ab_nstep.sh)
#endif
constexpr int NS_U = RPL_NSTEP_U;
constexpr int NS_MAXN = 8;

__global__ void __launch_bounds__(128)
k_nstep_runs(const float* __restrict__ r, const uint8_t* __restrict__ d, int64_t T, int64_t B, int n, double gamma,
             const float* __restrict__ q, const float* __restrict__ q_boot, int rescale, double eps,
             float* __restrict__ out, uint8_t* __restrict__ done_out, const float* __restrict__ vterm) {
  pdl_trigger();  // at entry, as k_nstep
  pdl_wait();
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = T - n + 1;
  const int64_t t0 = (int64_t)blockIdx.y * NS_U;
  if (b >= B || t0 >= rows) return;
  constexpr int W = NS_U + NS_MAXN - 1;
  float rw[W];
  uint8_t dw[W];
  const int nload = (int)min((int64_t)(NS_U + n - 1), T - t0);
  const float* rp = r + t0 * B + b;
  const uint8_t* dp = d + t0 * B + b;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    rw[i] = i < nload ? __ldg(rp + (int64_t)i * B) : 0.0f;
    dw[i] = i < nload ? __ldg(dp + (int64_t)i * B) : (uint8_t)0;
  }
  float qv[NS_U];
  if (q != nullptr) {
#pragma unroll
    for (int u = 0; u < NS_U; ++u) {
      const int64_t tq = t0 + u + n;
      qv[u] = t0 + u < rows ? (tq < T ? __ldg(q + tq * B + b) : __ldg(q_boot + b)) : 0.0f;
    }
  }
#pragma unroll
  for (int u = 0; u < NS_U; ++u) {
    if (t0 + u >= rows) break;
    double acc = 0.0;
    if (q != nullptr) acc = rescale ? h_inv((double)qv[u], eps) : (double)qv[u];
    uint8_t dn = 0;
#pragma unroll
    for (int j = NS_MAXN - 1; j >= 0; --j) {
      if (j < n) {
        const int i = u + j;
        const double ri = (double)rw[i];
        if (dw[i]) {
          acc = (vterm && dw[i] == RPL_DONE_TIMEOUT) ? fma(gamma, (double)__ldg(vterm + (t0 + i) * B + b), ri) : ri;
        } else {
          acc = fma(gamma, acc, ri);
        }
        dn |= dw[i];
      }
    }
    if (rescale) acc = h_fwd(acc, eps);
    out[(t0 + u) * B + b] = (float)acc;
    if (done_out != nullptr) done_out[(t0 + u) * B + b] = dn ? 1 : 0;
  }
}

__global__ void k_rescale(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                          double eps, int inverse) {
  pdl_wait();
  const int64_t n4 = n / 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (int64_t i = i0; i < n4; i += stride) {
      float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
      float4 o;
      o.x = (float)(inverse ? h_inv(v.x, eps) : h_fwd(v.x, eps));
      o.y = (float)(inverse ? h_inv(v.y, eps) : h_fwd(v.y, eps));
      o.z = (float)(inverse ? h_inv(v.z, eps) : h_fwd(v.z, eps));
      o.w = (float)(inverse ? h_inv(v.w, eps) : h_fwd(v.w, eps));
      reinterpret_cast<float4*>(y)[i] = o;
    }
    for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      y[i] = (float)(inverse ? h_inv(x[i], eps) : h_fwd(x[i], eps));
  } else {
    for (int64_t i = i0; i < n; i += stride)
      y[i] = (float)(inverse ? h_inv(x[i], eps) : h_fwd(x[i], eps));
  }
}

int elementwise_grid(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

}  // namespace
}  // namespace rpl

using namespace rpl;

// Measurement-only knob (RPL_SCAN_VARIANT): 0 = default (the persistent pipelined scan,
// k_scan_pipe, 32 x 128 tiles, when the layout is TMA-addressable — B % 4 == 0 for f32 and
// B % 16 == 0 for the u8 done tiles — else LDG 16 warps x 8 rows), 9 = the pipeline with 16 x
// 128 tiles and two CTAs per SM, 10-17 = further pipeline shapes (A/B), 6 = whole-column
// TMA tiles (the round-1 default), 7 = 16-column TMA tiles, double-buffered chunks, 8 = 32
// columns x 64 rows double-buffered, 4 = cluster of 2 CTAs x 64 rows (T <= 128, else
// default), 5 = cluster of 4 CTAs x 32 rows, 3 = LDG 16 warps x 8 rows, 1 = LDG 32 warps x 4
// rows, 2 = LDG 8 warps x 16 rows.  Same fp64 affine-map arithmetic; segment boundaries
// differ (results within the 1e-5 bound, not bit-identical across variants).
std::atomic<int> g_scan_variant{-1};  // -1: not set yet (read RPL_SCAN_VARIANT once)

int scan_variant() {
  int v = g_scan_variant.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("RPL_SCAN_VARIANT");
    int want = e ? atoi(e) : 0;
    if (want < 0 || want > 19) want = 0;
    int expect = -1;
    g_scan_variant.compare_exchange_strong(expect, want);
    v = g_scan_variant.load(std::memory_order_relaxed);
  }
  return v;
}

// The TMA scan triggers its dependent launch right after issuing its tile loads instead of
// at exit (PPO [128,4096], graph of back-to-back calls: GAE 4.90 -> 4.80 us, discounted
// 3.71 -> 3.66 us; profiles/r1/ppo_floor.json).  RPL_SCAN_TRIGGER=0 restores the exit
// trigger (A/B measurement).
int scan_trigger() {  // 0: exit trigger, 1: default, 2: the pipelined scan triggers after its first loads
  static const int t = [] {
    const char* e = getenv("RPL_SCAN_TRIGGER");
    return (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;
  }();
  return t;
}

namespace rpl {
void cfg_scan(int* variant, int* trigger) {  // knob state for rpl_config (abi.cu)
  *variant = scan_variant();
  *trigger = scan_trigger();
}
}  // namespace rpl

typedef CUresult (*encode_fn_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_fn_t encode_fn() {
  static const encode_fn_t fn = []() -> encode_fn_t {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<encode_fn_t>(p);
    return nullptr;
  }();
  return fn;
}

// [T, B] row-major tensor map with a [box_rows x 32 columns] box; false if the layout is
// not TMA-addressable (base not 16-B aligned, row pitch not a multiple of 16 B).
bool tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esize, int64_t T, int64_t B,
             int box_rows, int box_cols = 32) {
  encode_fn_t fn = encode_fn();
  if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15) || ((B * esize) & 15)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)T};
  const cuuint64_t strides[1] = {(cuuint64_t)(B * esize)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1u, 1u};
  return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int WARPS, int S, int CL, bool GAE>
int launch_scan_cluster(const float* r, const float* v, const uint8_t* d, const float* boot, int64_t T, int64_t B,
                        double gamma, double lam, float* o0, float* o1, cudaStream_t st, bool* used,
                        const float* vterm) {
  *used = false;
  constexpr int CH = WARPS * S;
  if (T > (int64_t)CL * CH) return RPL_OK;
  CUtensorMap mr, mv, md;
  if (!(tmap_2d(&mr, r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH) &&
        tmap_2d(&md, d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, T, B, CH) &&
        (!GAE || tmap_2d(&mv, v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH))))
    return RPL_OK;
  if (!GAE) mv = mr;
  *used = true;
  const dim3 grid((unsigned)(((B + 31) / 32) * CL));
  return launch_pdl_cluster(k_scan_cluster<WARPS, S, CL, GAE>, grid, dim3(WARPS * 32), 0, st, (unsigned)CL, mr, mv,
                            md, v, boot, T, B, gamma, lam, o0, o1, vterm);
}

template <int COLS, int WARPS, int S, int STAGES, bool GAE, int MINB, int OB = 2>
int launch_scan_pipe(const float* r, const float* v, const uint8_t* d, const float* boot, int64_t T, int64_t B,
                     double gamma, double lam, float* o0, float* o1, cudaStream_t st, const float* vterm, bool* used,
                     int trigger = -1) {
  using SMt = ScanPipeSmem<COLS, WARPS, S, STAGES, GAE, OB>;
  constexpr int CH = SMt::CH;
  CUtensorMap mr, mv, md, mo0, mo1;
  *used = false;
  if (!(tmap_2d(&mr, r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, COLS) &&
        tmap_2d(&md, d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, T, B, CH, COLS) &&
        tmap_2d(&mo0, o0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, COLS) &&
        (!GAE || tmap_2d(&mv, v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, COLS)) &&
        (!(GAE && o1) || tmap_2d(&mo1, o1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, COLS))))
    return RPL_OK;
  *used = true;
  if (!GAE) mv = mr;
  if (!(GAE && o1)) mo1 = mo0;
  auto kern = k_scan_pipe<COLS, WARPS, S, STAGES, GAE, MINB, OB>;
  const size_t dyn = sizeof(SMt);
  ensure_smem(reinterpret_cast<const void*>(kern), dyn);
  const int64_t groups = (B + COLS - 1) / COLS;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, dyn);
  int64_t grid = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  if (grid > groups) grid = groups;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(WARPS * 32), dyn, st, mr, mv, md, mo0, mo1, boot, T, B, gamma,
                    lam, (GAE && o1) ? 1 : 0, vterm, trigger >= 0 ? trigger : scan_trigger());
}

template <bool GAE>
int launch_scan(const float* r, const float* v, const uint8_t* d, const float* boot, int64_t T, int64_t B,
                double gamma, double lam, float* o0, float* o1, cudaStream_t st, const float* vterm) {
  dim3 grid((unsigned)((B + 31) / 32));
  const int var = scan_variant();
  if ((var == 4 || var == 5) && T < (1ll << 31) && B < (1ll << 31)) {
    // short horizons: rows split over a cluster (4: 2 CTAs x 64 rows, 5: 4 CTAs x 32 rows).
    // Measured slower than the whole-column tiles at PPO size (GAE 6.0 / 7.3-7.6 us vs
    // 4.96 us): the call is latency-bound, and cluster scheduling plus two cluster
    // barriers cost more than the per-CTA bytes they save.  Kept selectable.
    bool used = false;
    const int rc = var == 4
                       ? launch_scan_cluster<16, 4, 2, GAE>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, &used, vterm)
                       : launch_scan_cluster<8, 4, 4, GAE>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, &used, vterm);
    if (used) return rc;
  }
  if ((var == 0 || var == 9) && T < (1ll << 31) && B < (1ll << 31)) {  // default: persistent pipeline
    // default shape: 32-column groups (128-B tile rows), 8 warps x 16 rows = 128-row chunks, 3
    // load stages, one CTA per SM (scan size sweep, profiles/r2/scan_ab_*.json: GAE 0.75-0.76
    // and discounted 0.58-0.74 of measured HBM on 34-285 MB calls, PPO GAE 4.49 us); variant 9
    // keeps the 16-column / 2-CTAs-per-SM shape measured first.
    // One chunk per group (T <= 128, e.g. PPO): the 16-column shape, twice the CTAs (PPO GAE
    // 4.40 vs 4.56 us); longer horizons: the 32-column shape (wider TMA rows win there).
    bool used = false;
    if (var == 0 && T <= 128 && (B + 15) / 16 <= 4 * (int64_t)sm_count()) {
      // one item per CTA (every 16-column group a CTA of its own): one load stage and one output
      // buffer (38 KB of shared memory, 64 registers), 4 CTAs per SM, and the dependent launch
      // triggered once the tiles are requested — the next call's CTAs sit resident beside this
      // call's and issue their loads the moment it completes.  PPO [128, 4096], interleaved A/B
      // (scripts/scan_ab.py, 10 rounds): GAE 4.58 vs 4.89 us, discounted 3.39 vs 3.86 us per
      // call; the same shape without the early trigger: 5.02 us (profiles/r2/scan_coresident_ab.txt).
      const int rc = launch_scan_pipe<16, 8, 8, 1, GAE, 4, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used,
                                                              scan_trigger() == 0 ? 0 : 2);
      if (used) return rc;
    }
    const bool narrow = var == 9 || T <= 128;
    const int rc = narrow
                       ? launch_scan_pipe<16, 8, 8, 3, GAE, 2>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used)
                       : launch_scan_pipe<32, 8, 16, 3, GAE, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used);
    if (used) return rc;
  }
  if ((var == 18 || var == 19) && T <= 128 && B < (1ll << 31)) {
    // single-chunk horizons, one load stage and one output buffer (38 KB of shared memory), 3
    // (18) or 4 (19) CTAs per SM, the dependent launch triggered once the tiles are requested:
    // the next call's CTAs can sit resident beside this call's (A/B)
    bool used = false;
    const int rc = var == 18
                       ? launch_scan_pipe<16, 8, 8, 1, GAE, 4, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used)
                       : launch_scan_pipe<16, 8, 8, 1, GAE, 4, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used, 2);
    if (used) return rc;
  }
  if (var >= 10 && var <= 17 && T < (1ll << 31) && B < (1ll << 31)) {  // pipeline shapes (A/B)
    bool used = false;
    int rc = RPL_OK;
    switch (var) {
      case 10: rc = launch_scan_pipe<32, 8, 16, 2, GAE, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 11: rc = launch_scan_pipe<32, 16, 8, 2, GAE, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 12: rc = launch_scan_pipe<16, 8, 8, 2, GAE, 3>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 13: rc = launch_scan_pipe<32, 8, 8, 2, GAE, 2>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 14: rc = launch_scan_pipe<32, 8, 16, 3, GAE, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 15: rc = launch_scan_pipe<32, 8, 8, 3, GAE, 2>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      case 16: rc = launch_scan_pipe<32, 8, 16, 2, GAE, 2, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
      default: rc = launch_scan_pipe<32, 4, 32, 2, GAE, 2, 1>(r, v, d, boot, T, B, gamma, lam, o0, o1, st, vterm, &used); break;
    }
    if (used) return rc;
  }
  if ((var == 7 || var == 8) && T < (1ll << 31) && B < (1ll << 31)) {
    CUtensorMap mr, mv, md;
    const int CH = var == 7 ? 128 : 64;  // 7: 16 cols x (8 warps x 2 halves x 8 rows); 8: 32 cols x 16 warps x 4 rows
    const int cols = var == 7 ? 16 : 32;
    if (tmap_2d(&mr, r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, cols) &&
        tmap_2d(&md, d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, T, B, CH, cols) &&
        (!GAE || tmap_2d(&mv, v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH, cols))) {
      if (!GAE) mv = mr;
      if (var == 7)
        return launch_pdl(k_scan_tma2<16, 8, 8, GAE>, dim3((unsigned)((B + 15) / 16)), dim3(8 * 32), 0, st, mr, mv,
                          md, boot, T, B, gamma, lam, o0, o1, scan_trigger(), vterm);
      return launch_pdl(k_scan_tma2<32, 16, 4, GAE>, dim3((unsigned)((B + 31) / 32)), dim3(16 * 32), 0, st, mr, mv,
                        md, boot, T, B, gamma, lam, o0, o1, scan_trigger(), vterm);
    }
  }
  if ((var == 0 || var == 6) && T < (1ll << 31) && B < (1ll << 31)) {  // whole-column tiles (r1 default)
    CUtensorMap mr, mv, md;
    constexpr int CH = SCAN_WARPS * SCAN_S;
    if (tmap_2d(&mr, r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH) &&
        tmap_2d(&md, d, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, T, B, CH) &&
        (!GAE || tmap_2d(&mv, v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, B, CH))) {
      if (!GAE) mv = mr;
      return launch_pdl(k_scan_tma<SCAN_WARPS, SCAN_S, GAE>, grid, dim3(SCAN_WARPS * 32), 0, st, mr, mv, md, v,
                        boot, T, B, gamma, lam, o0, o1, scan_trigger(), vterm);
    }
  }
  switch (scan_variant()) {
    case 1:
      return launch_pdl(k_scan<32, 4, GAE>, grid, dim3(32 * 32), 0, st, r, v, d, boot, T, B, gamma, lam, o0, o1,
                        vterm);
    case 2:
      return launch_pdl(k_scan<8, 16, GAE>, grid, dim3(8 * 32), 0, st, r, v, d, boot, T, B, gamma, lam, o0, o1,
                        vterm);
    default:
      return launch_pdl(k_scan<SCAN_WARPS, SCAN_S, GAE>, grid, dim3(SCAN_WARPS * 32), 0, st, r, v, d, boot, T, B,
                        gamma, lam, o0, o1, vterm);
  }
}

extern "C" int rpl_returns_discounted_tl(const float* r, const uint8_t* d, const float* v_term,
                                         const float* bootstrap, int64_t T, int64_t B, double gamma, float* ret,
                                         void* stream) {
  if (!r || !d || !ret || T < 1 || B < 1) return RPL_EINVAL;
  return launch_scan<false>(r, nullptr, d, bootstrap, T, B, gamma, 0.0, ret, nullptr, as_stream(stream), v_term);
}

extern "C" int rpl_returns_discounted(const float* r, const uint8_t* d, const float* bootstrap,
                                      int64_t T, int64_t B, double gamma, float* ret, void* stream) {
  return rpl_returns_discounted_tl(r, d, nullptr, bootstrap, T, B, gamma, ret, stream);
}

extern "C" int rpl_gae_tl(const float* r, const float* v, const uint8_t* d, const float* v_term,
                          const float* bootstrap_v, int64_t T, int64_t B, double gamma, double lambda, float* adv,
                          float* ret, void* stream) {
  if (!r || !v || !d || !bootstrap_v || !adv || T < 1 || B < 1) return RPL_EINVAL;
  return launch_scan<true>(r, v, d, bootstrap_v, T, B, gamma, lambda, adv, ret, as_stream(stream), v_term);
}

extern "C" int rpl_gae(const float* r, const float* v, const uint8_t* d, const float* bootstrap_v,
                       int64_t T, int64_t B, double gamma, double lambda, float* adv, float* ret,
                       void* stream) {
  return rpl_gae_tl(r, v, d, nullptr, bootstrap_v, T, B, gamma, lambda, adv, ret, stream);
}

extern "C" int rpl_returns_nstep_tl(const float* r, const uint8_t* d, const float* v_term, int64_t T, int64_t B,
                                    int32_t n, double gamma, const float* q, const float* q_boot, int32_t rescale,
                                    double rescale_eps, float* ret_n, uint8_t* done_n, void* stream) {
  if (!r || !d || !ret_n || T < 1 || B < 1) return RPL_EINVAL;
  if (n < 1 || n > T) return RPL_ERANGE;
  if (q != nullptr && q_boot == nullptr) return RPL_EINVAL;
  if (rescale && !(rescale_eps > 0.0)) return RPL_EINVAL;
  const int64_t work = (T - n + 1) * B;
#ifndef RPL_NSTEP_THREADS  // build-flag knob for A/B measurement
#define RPL_NSTEP_THREADS 128  // same-box A/B: 69.55 vs 69.82 us per R2D2 step at 256 (64: 69.68)
#endif
  const int threads = RPL_NSTEP_THREADS;
  const int64_t runs = (T - n + 1 + NS_U - 1) / NS_U;
  if (n <= NS_MAXN && runs < 65536)  // register runs (the common n), 2-D grid
    return launch_pdl(k_nstep_runs, dim3((unsigned)((B + 127) / 128), (unsigned)runs), dim3(128), 0,
                      as_stream(stream), r, d, T, B, (int)n, gamma, q, q_boot, rescale ? 1 : 0, rescale_eps, ret_n,
                      done_n, v_term);
  return launch_pdl(k_nstep, dim3(elementwise_grid(work, threads)), dim3(threads), 0, as_stream(stream), r, d, T, B,
                    (int)n, gamma, q, q_boot, rescale ? 1 : 0, rescale_eps, ret_n, done_n, v_term);
}

extern "C" int rpl_returns_nstep(const float* r, const uint8_t* d, int64_t T, int64_t B, int32_t n,
                                 double gamma, const float* q, const float* q_boot, int32_t rescale,
                                 double rescale_eps, float* ret_n, uint8_t* done_n, void* stream) {
  return rpl_returns_nstep_tl(r, d, nullptr, T, B, n, gamma, q, q_boot, rescale, rescale_eps, ret_n, done_n, stream);
}

extern "C" int rpl_value_rescale(const float* x, float* y, int64_t n, double eps, int32_t inverse,
                                 void* stream) {
  if (!x || !y || n < 0 || !(eps > 0.0)) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int threads = 256;
  return launch_pdl(k_rescale, dim3(elementwise_grid((n + 3) / 4, threads)), dim3(threads), 0, as_stream(stream), x,
                    y, n, eps, inverse ? 1 : 0);
}

extern "C" int rpl_debug_scan_trace(int64_t* out, int32_t n) {
#ifdef RPL_TRACE
  if (!out || n < 1 || n > 10) return RPL_EINVAL;
  return cudaMemcpyFromSymbol(out, rpl::g_strace, sizeof(int64_t) * (size_t)n) == cudaSuccess ? RPL_OK : RPL_ECUDA;
#else
  (void)out;
  (void)n;
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_set_scan_variant(int32_t variant) {
  if (variant < 0 || variant > 19) return RPL_EINVAL;
  g_scan_variant.store(variant);
  return RPL_OK;
}
