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
#include <math.h>

#include "common.cuh"

namespace rpl {

namespace {

constexpr int SCAN_WARPS = 16;
constexpr int SCAN_S = 8;

template <int WARPS, int S, bool GAE>
__global__ void __launch_bounds__(WARPS * 32)
k_scan(const float* __restrict__ r, const float* __restrict__ v, const uint8_t* __restrict__ d,
       const float* __restrict__ boot, int64_t T, int64_t B, double gamma, double lam,
       float* __restrict__ out0, float* __restrict__ out1) {
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
    uint32_t dmask = 0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const int64_t t = t0 + i;
      const bool ok = cv && t < T;
      rr[i] = ok ? __ldg(r + t * B + col) : 0.f;
      const uint8_t di = ok ? __ldg(d + t * B + col) : (uint8_t)0;
      dmask |= (di ? 1u : 0u) << i;
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
      if (GAE) {
        double vnext;
        if (i + 1 < S) vnext = (i + 1 < nvalid) ? (double)vv[i + 1] : bootv;
        else vnext = vseg_next;
        b[i] = i < nvalid ? ((double)rr[i] + gamma * nd * vnext) - (double)vv[i] : 0.0;
      } else {
        b[i] = i < nvalid ? (double)rr[i] : 0.0;
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

__device__ __forceinline__ double h_fwd(double x, double eps) {
  // h(x) = x (1/(sqrt(|x|+1)+1) + eps)  ==  sign(x)(sqrt(|x|+1)-1) + eps x   (§8c #4)
  return x * (1.0 / (sqrt(fabs(x) + 1.0) + 1.0) + eps);
}

__device__ __forceinline__ double h_inv(double y, double eps) {
  // s = sqrt(x+1) solves eps s^2 + s - (1 + eps + |y|) = 0 (rationalised root);
  // x = (s-1)(s+1) with s-1 = |y| / (1 + eps (s+1))            (§8c #4)
  const double a = fabs(y);
  const double c = a + 1.0 + eps;
  const double s = 2.0 * c / (1.0 + sqrt(1.0 + 4.0 * eps * c));
  const double x = a * (s + 1.0) / (1.0 + eps * (s + 1.0));
  return copysign(x, y);
}

__global__ void k_nstep(const float* __restrict__ r, const uint8_t* __restrict__ d, int64_t T,
                        int64_t B, int n, double gamma, const float* __restrict__ q,
                        const float* __restrict__ q_boot, int rescale, double eps,
                        float* __restrict__ out, uint8_t* __restrict__ done_out) {
  const int64_t rows = T - n + 1;
  const int64_t total = rows * B;
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / B;
    const int64_t b = e - t * B;
    double acc = 0.0;
    if (q != nullptr) {
      const double qv = (t + n < T) ? (double)__ldg(q + (t + n) * B + b) : (double)__ldg(q_boot + b);
      acc = rescale ? h_inv(qv, eps) : qv;
    }
    uint8_t dn = 0;
    for (int i = n - 1; i >= 0; --i) {
      const int64_t o = (t + i) * B + b;
      const uint8_t di = __ldg(d + o);
      const double ri = (double)__ldg(r + o);
      acc = di ? ri : fma(gamma, acc, ri);
      dn |= di;
    }
    if (rescale) acc = h_fwd(acc, eps);
    out[e] = (float)acc;
    if (done_out != nullptr) done_out[e] = dn ? 1 : 0;
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

extern "C" int rpl_returns_discounted(const float* r, const uint8_t* d, const float* bootstrap,
                                      int64_t T, int64_t B, double gamma, float* ret, void* stream) {
  if (!r || !d || !ret || T < 1 || B < 1) return RPL_EINVAL;
  dim3 grid((unsigned)((B + 31) / 32));
  return launch_pdl(k_scan<SCAN_WARPS, SCAN_S, false>, grid, dim3(SCAN_WARPS * 32), 0, as_stream(stream), r,
                    (const float*)nullptr, d, bootstrap, T, B, gamma, 0.0, ret, (float*)nullptr);
}

extern "C" int rpl_gae(const float* r, const float* v, const uint8_t* d, const float* bootstrap_v,
                       int64_t T, int64_t B, double gamma, double lambda, float* adv, float* ret,
                       void* stream) {
  if (!r || !v || !d || !bootstrap_v || !adv || T < 1 || B < 1) return RPL_EINVAL;
  dim3 grid((unsigned)((B + 31) / 32));
  return launch_pdl(k_scan<SCAN_WARPS, SCAN_S, true>, grid, dim3(SCAN_WARPS * 32), 0, as_stream(stream), r, v, d,
                    bootstrap_v, T, B, gamma, lambda, adv, ret);
}

extern "C" int rpl_returns_nstep(const float* r, const uint8_t* d, int64_t T, int64_t B, int32_t n,
                                 double gamma, const float* q, const float* q_boot, int32_t rescale,
                                 double rescale_eps, float* ret_n, uint8_t* done_n, void* stream) {
  if (!r || !d || !ret_n || T < 1 || B < 1) return RPL_EINVAL;
  if (n < 1 || n > T) return RPL_ERANGE;
  if (q != nullptr && q_boot == nullptr) return RPL_EINVAL;
  if (rescale && !(rescale_eps > 0.0)) return RPL_EINVAL;
  const int64_t work = (T - n + 1) * B;
  const int threads = 256;
  return launch_pdl(k_nstep, dim3(elementwise_grid(work, threads)), dim3(threads), 0, as_stream(stream), r, d, T, B,
                    (int)n, gamma, q, q_boot, rescale ? 1 : 0, rescale_eps, ret_n, done_n);
}

extern "C" int rpl_value_rescale(const float* x, float* y, int64_t n, double eps, int32_t inverse,
                                 void* stream) {
  if (!x || !y || n < 0 || !(eps > 0.0)) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int threads = 256;
  return launch_pdl(k_rescale, dim3(elementwise_grid((n + 3) / 4, threads)), dim3(threads), 0, as_stream(stream), x,
                    y, n, eps, inverse ? 1 : 0);
}
