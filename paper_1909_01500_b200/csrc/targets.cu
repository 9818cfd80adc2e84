// Learning targets right after the gather.
//
//   rpl_returns_nstep_dq   double-Q bootstrap selection (argmax of the online net, value of
//                          the target net; [EXT: Double DQN]) fused with the n-step return
//                          and R2D2 value rescaling
//   rpl_c51_project        categorical (C51) projection of the target net's next-state
//                          distribution at the online argmax onto the fixed atoms
//                          [EXT: Bellemare et al. 2017, Algorithm 1] ("Categorical")
//
// Both are tiny, latency-bound epilogues of the learner's target forward pass: one thread
// per output (n-step) / one warp per sample (C51), fp64 arithmetic, one rounding to fp32.
// Readings: R27 (argmax = first maximum, NaN never wins), R28 (the projection is evaluated
// in its equivalent triangular-kernel form m_i = sum_j p_j max(0, 1 - |b_j - i|), a
// deterministic gather instead of the algorithm's scatter).
#include <math.h>

#include "common.cuh"

namespace rpl {
namespace {

// first maximum over A values (stride 1); NaN never wins; all NaN -> 0 (R27)
__device__ __forceinline__ int argmax_first(const float* __restrict__ v, int A) {
  int bi = 0;
  float best = 0.0f;
  bool have = false;
  for (int a = 0; a < A; ++a) {
    const float x = __ldg(v + a);
    if (x != x) continue;
    if (!have || x > best) {
      best = x;
      bi = a;
      have = true;
    }
  }
  return bi;
}

__device__ __forceinline__ double h_fwd_t(double x, double eps) {
  return x * (1.0 / (sqrt(fabs(x) + 1.0) + 1.0) + eps);  // R4 stable form
}
__device__ __forceinline__ double h_inv_t(double y, double eps) {
  const double a = fabs(y);
  const double c = a + 1.0 + eps;
  const double s = 2.0 * c / (1.0 + sqrt(1.0 + 4.0 * eps * c));
  return copysign(a * (s + 1.0) / (1.0 + eps * (s + 1.0)), y);
}

__global__ void k_nstep_dq(const float* __restrict__ r, const uint8_t* __restrict__ d, int64_t T, int64_t B, int n,
                           double gamma, const float* __restrict__ q_online, const float* __restrict__ q_target,
                           int A, int rescale, double eps, float* __restrict__ out, uint8_t* __restrict__ done_out,
                           int32_t* __restrict__ a_out) {
  pdl_wait();
  const int64_t rows = T - n + 1;
  const int64_t total = rows * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / B;
    const int64_t b = e - t * B;
    const int64_t qb = ((t + n) * B + b) * A;  // bootstrap row t+n of [T+1, B, A]
    const int a = argmax_first(q_online + qb, A);
    const double qv = (double)__ldg(q_target + qb + a);
    double acc = rescale ? h_inv_t(qv, eps) : qv;
    uint8_t dn = 0;
    for (int i = n - 1; i >= 0; --i) {  // Horner from the last row (R24)
      const int64_t o = (t + i) * B + b;
      const uint8_t di = __ldg(d + o);
      const double ri = (double)__ldg(r + o);
      acc = di ? ri : fma(gamma, acc, ri);
      dn |= di;
    }
    if (rescale) acc = h_fwd_t(acc, eps);
    out[e] = (float)acc;
    if (done_out) done_out[e] = dn ? 1 : 0;
    if (a_out) a_out[e] = a;
  }
}

// Per-step n-step TD error straight from the ring (NEXT-1 initial priorities, R33): one
// thread per output (t, b); ring rows modulo cap_T; the same target arithmetic as k_nstep_dq.
__global__ void k_ring_td_abs(const float* __restrict__ r, const uint8_t* __restrict__ d,
                              const float* __restrict__ q_taken, const float* __restrict__ q_boot, int64_t cap,
                              int64_t B, int64_t row0, int64_t T_out, int n, double gamma, int rescale, double eps,
                              float* __restrict__ out) {
  pdl_wait();
  const int64_t total = T_out * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / B;
    const int64_t b = e - t * B;
    const int64_t row = (row0 + t) % cap;
    int64_t rb = row + n;  // bootstrap row
    if (rb >= cap) rb -= cap;
    const double qv = (double)__ldg(q_boot + rb * B + b);
    double acc = rescale ? h_inv_t(qv, eps) : qv;
    for (int i = n - 1; i >= 0; --i) {  // Horner from the last row (R24)
      int64_t ri = row + i;
      if (ri >= cap) ri -= cap;
      const uint8_t di = __ldg(d + ri * B + b);
      const double rv = (double)__ldg(r + ri * B + b);
      acc = di ? rv : fma(gamma, acc, rv);
    }
    if (rescale) acc = h_fwd_t(acc, eps);
    out[e] = (float)fabs(acc - (double)__ldg(q_taken + row * B + b));
  }
}

constexpr int C51_WARPS = 4;

__global__ void __launch_bounds__(C51_WARPS * 32)
k_c51_project(const float* __restrict__ p_target, const float* __restrict__ q_online, const float* __restrict__ R,
              const uint8_t* __restrict__ done_n, int64_t n, int A, int N, double v_min, double v_max,
              double gamma_n, float* __restrict__ m_out, int32_t* __restrict__ a_out) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * C51_WARPS + (threadIdx.x >> 5);
  if (s >= n) return;
  int a = 0;
  if (lane == 0 && q_online) a = argmax_first(q_online + s * A, A);
  a = __shfl_sync(0xffffffffu, a, 0);
  const float* p = p_target + (s * A + a) * N;
  const double dz = (v_max - v_min) / (double)(N - 1);
  const double g = done_n && __ldg(done_n + s) ? 0.0 : gamma_n;
  const double Rs = (double)__ldg(R + s);
  for (int i = lane; i < N; i += 32) {
    double m = 0.0;
    for (int j = 0; j < N; ++j) {
      double tz = Rs + g * (v_min + j * dz);
      tz = fmin(fmax(tz, v_min), v_max);
      const double bj = (tz - v_min) / dz;
      const double wgt = 1.0 - fabs(bj - (double)i);
      if (wgt > 0.0) m = fma((double)__ldg(p + j), wgt, m);
    }
    m_out[s * N + i] = (float)m;
  }
  if (lane == 0 && a_out) a_out[s] = a;
}

}  // namespace
}  // namespace rpl

using namespace rpl;

extern "C" int rpl_returns_nstep_dq(const float* r, const uint8_t* d, int64_t T, int64_t B, int32_t n, double gamma,
                                    const float* q_online, const float* q_target, int32_t A, int32_t rescale,
                                    double rescale_eps, float* ret_n, uint8_t* done_n, int32_t* a_star,
                                    void* stream) {
  if (!r || !d || !ret_n || !q_online || !q_target || T < 1 || B < 1 || A < 1) return RPL_EINVAL;
  if (n < 1 || n > T) return RPL_ERANGE;
  if (rescale && !(rescale_eps > 0.0)) return RPL_EINVAL;
  const int64_t work = (T - n + 1) * B;
  const int threads = 256;
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  return launch_pdl(k_nstep_dq, dim3((unsigned)blocks), dim3(threads), 0, as_stream(stream), r, d, T, B, (int)n, gamma,
                    q_online, q_target, (int)A, rescale ? 1 : 0, rescale_eps, ret_n, done_n, a_star);
}

extern "C" int rpl_c51_project(const float* p_target, const float* q_online, const float* R, const uint8_t* done_n,
                               int64_t n, int32_t A, int32_t n_atoms, double v_min, double v_max, double gamma_n,
                               float* m_out, int32_t* a_star, void* stream) {
  if (!p_target || !R || !m_out || n < 0 || A < 1 || n_atoms < 2 || !(v_max > v_min) || !(gamma_n >= 0.0))
    return RPL_EINVAL;
  if (!q_online && A != 1) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int64_t blocks = (n + C51_WARPS - 1) / C51_WARPS;
  return launch_pdl(k_c51_project, dim3((unsigned)blocks), dim3(C51_WARPS * 32), 0, as_stream(stream), p_target,
                    q_online, R, done_n, n, (int)A, (int)n_atoms, v_min, v_max, gamma_n, m_out, a_star);
}

extern "C" int rpl_ring_td_abs(const float* rew, const uint8_t* done, const float* q_taken, const float* q_boot,
                               int64_t cap_T, int64_t B, int64_t row0, int64_t T_out, int32_t n, double gamma,
                               int32_t rescale, double rescale_eps, float* out, void* stream) {
  if (!rew || !done || !q_taken || !q_boot || !out || cap_T < 1 || B < 1 || row0 < 0 || row0 >= cap_T || T_out < 0)
    return RPL_EINVAL;
  if (n < 1 || T_out + n > cap_T) return RPL_ERANGE;
  if (rescale && !(rescale_eps > 0.0)) return RPL_EINVAL;
  if (T_out == 0) return RPL_OK;
  const int threads = 256;
  int64_t blocks = (T_out * B + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (blocks > cap) blocks = cap;
  return launch_pdl(k_ring_td_abs, dim3((unsigned)blocks), dim3(threads), 0, as_stream(stream), rew, done, q_taken,
                    q_boot, cap_T, B, row0, T_out, (int)n, gamma, rescale ? 1 : 0, rescale_eps, out);
}
