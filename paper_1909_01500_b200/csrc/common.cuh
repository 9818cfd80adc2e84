// Shared device/host helpers for librpl (sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "rpl.h"

namespace rpl {

extern std::atomic<int64_t> g_launches;  // host-side launch counter (rpl_launch_count)

// Per-device attribute caches (the library's only state; thread-safe).
inline std::mutex& cache_mutex() {
  static std::mutex m;
  return m;
}

inline int sm_count() {
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(cache_mutex());
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] = (v > 0 ? v : 148);
}

// Raise a kernel's dynamic shared-memory limit to `bytes` once per (device, kernel).
inline void ensure_smem(const void* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(cache_mutex());
  size_t& cur = done[std::make_pair(dev, kernel)];
  if (bytes > cur) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cur = bytes;
  }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the last launch; map failures to RPL_ECUDA.
inline int launch_status() {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RPL_OK : RPL_ECUDA;
}

// Programmatic dependent launch (PDL).  Hot-path kernels are launched with the
// programmatic-stream-serialization attribute, so a kernel's launch and prologue
// (shared-memory / mbarrier setup) overlap the tail of the previous kernel on the
// stream; pdl_wait() — executed before the kernel's first global-memory access —
// blocks until the previous grid has completed and its writes are visible, so
// stream order (the device analogue of the paper's RW lock) is unchanged.
// pdl_trigger() lets the next grid start launching once every CTA has called it.
// RPL_PDL=0 in the environment disables the attribute (A/B measurement).
// Measurement knob (build flag, default 0): bit 1 update, 2 sampler, 4 sequence gather,
// (8, the n-step kernels: they now always trigger at entry) — that kernel triggers its
// dependent launch at entry instead of at exit.
#ifndef RPL_PDL_EARLY
#define RPL_PDL_EARLY 0
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

// Shared-memory carveout of every hot-path kernel (RPL_CARVEOUT: -1 = leave the driver's
// choice, else the percentage passed as cudaFuncAttributePreferredSharedMemoryCarveout): an
// SM whose carveout differs between consecutive kernels must be reconfigured between them.
int carveout_knob();
inline void set_carveout(const void* kernel) {
  const int c = carveout_knob();
  if (c < 0) return;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(cache_mutex());
  int& cur = done[std::make_pair(dev, kernel)];
  if (cur != c + 1) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
    cudaGetLastError();
    cur = c + 1;
  }
}

template <typename... KArgs, typename... Args>
int launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       unsigned cluster_x, Args... args) {
  set_carveout(reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 1) {  // thread-block cluster along x (distributed shared memory)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  ++g_launches;
  if (e != cudaSuccess) {
    cudaGetLastError();
    return RPL_ECUDA;
  }
  return RPL_OK;
}

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  return launch_pdl_cluster(kernel, grid, block, smem, st, 1u, args...);
}

// Cooperative launch (cudaLaunchAttributeCooperative) for kernels with a grid-wide barrier:
// the runtime guarantees every CTA is co-resident or fails the launch (never a silent
// deadlock next to other streams' work).  The grid must not exceed the occupancy-derived
// capacity (checked here: RPL_EINVAL).  PDL is added when enabled; if the runtime rejects the
// combination the launch is retried cooperative-only.
template <typename... KArgs, typename... Args>
int launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  set_carveout(reinterpret_cast<const void*>(kernel));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, (int)(block.x * block.y * block.z), smem) !=
          cudaSuccess ||
      (int64_t)grid.x * grid.y * grid.z > (int64_t)per_sm * sm_count()) {
    cudaGetLastError();
    return RPL_EINVAL;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  int na = 1;
  if (pdl_enabled()) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess && na == 2) {
    cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  }
  ++g_launches;
  if (e != cudaSuccess) {
    cudaGetLastError();
    return RPL_ECUDA;
  }
  return RPL_OK;
}

// fp64 reciprocal and square root without the IEEE slow paths: the hardware approximation
// (MUFU on the high word) refined by two Newton steps to full double precision (relative
// error ~1e-16; not always correctly rounded).  Arguments here are finite and >= 1, or
// inf / NaN which propagate.  Used by h / h^-1, whose outputs are rounded to fp32.
__device__ __forceinline__ double rcp64(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double sqrt64(double y) {  // y >= 1 (or inf / NaN)
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  const double hy = 0.5 * y;
  r = r * fma(-hy * r, r, 1.5);
  r = r * fma(-hy * r, r, 1.5);
  const double s = y * r;
  return isinf(y) ? y : fma(0.5 * r, fma(-s, s, y), s);
}

__device__ __forceinline__ double h_fwd(double x, double eps) {
  // h(x) = x (1/(sqrt(|x|+1)+1) + eps)  ==  sign(x)(sqrt(|x|+1)-1) + eps x   (§8c #4)
  return x * (rcp64(sqrt64(fabs(x) + 1.0) + 1.0) + eps);
}

__device__ __forceinline__ double h_inv(double y, double eps) {
  // s = sqrt(x+1) solves eps s^2 + s - (1 + eps + |y|) = 0 (rationalised root);
  // x = (s-1)(s+1) with s-1 = |y| / (1 + eps (s+1))            (§8c #4)
  const double a = fabs(y);
  const double c = a + 1.0 + eps;
  const double s = 2.0 * c * rcp64(1.0 + sqrt64(1.0 + 4.0 * eps * c));
  const double x = a * (s + 1.0) * rcp64(1.0 + eps * (s + 1.0));
  return copysign(x, y);
}

__device__ __forceinline__ void set_err(int32_t* err, int32_t bits) {
  if (err) atomicOr(err, bits);
}

// ---- peer exchange boards (rpl.h RPL_BOARD_WORDS; K5 / K7 over NVLink peer memory) ----
constexpr int BOARD_MAX_WORLD = 64;

// slot = {value, tag}: the value store is ordered before the tag by the release (sys scope:
// the slot may live in a peer GPU's memory).
__device__ __forceinline__ void board_publish(int64_t* slot, int64_t value, uint64_t tag) {
  asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(slot), "l"(value) : "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot + 1), "l"(tag) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until the slot carries `tag`, then read its value; false after ~2 s (peer missing).
__device__ __forceinline__ bool board_wait(const int64_t* slot, uint64_t tag, int64_t* value) {
  const uint64_t t0 = global_ns();
  while (true) {
    uint64_t t;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(t) : "l"(slot + 1) : "memory");
    if (t == tag) {
      int64_t v;
      asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
      *value = v;
      return true;
    }
    if (global_ns() - t0 > 2000000000ull) return false;
    __nanosleep(64);
  }
}

// A peer that never published within board_wait's ~2 s: the exchange failed.  Set the device
// error bit and trap, so the failure surfaces at the next synchronisation (the context reports
// a launch failure) instead of the step continuing on a default value.
__device__ __forceinline__ void board_fail(int32_t* err) {
  set_err(err, RPL_DERR_PEER);
  __threadfence_system();
  __trap();
}

// 64-bit warp shuffles (int64 payloads)
__device__ __forceinline__ int64_t shfl_up64(int64_t v, int d) {
  return (int64_t)__shfl_up_sync(0xffffffffu, (unsigned long long)v, d);
}
__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
  return (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)v, src);
}
__device__ __forceinline__ int64_t shfl_xor64(int64_t v, int m) {
  return (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)v, m);
}

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += shfl_xor64(v, m);
  return v;
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    int64_t o = shfl_xor64(v, m);
    v = o > v ? o : v;
  }
  return v;
}
__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    int64_t o = shfl_xor64(v, m);
    v = o < v ? o : v;
  }
  return v;
}

// Device-side view of the tree layout (passed by value to kernels).
struct TreeDev {
  int64_t n_leaves;
  int64_t q_cap;
  int64_t level_off[RPL_MAX_LEVELS];
  int64_t hdr_off;
  int32_t fanout, log2w, depth, frac_bits;
};

inline TreeDev tree_dev(const rpl_tree_layout* L) {
  TreeDev t;
  t.n_leaves = L->n_leaves;
  t.q_cap = L->q_cap;
  for (int i = 0; i < RPL_MAX_LEVELS; ++i) t.level_off[i] = L->level_off[i];
  t.hdr_off = L->hdr_off;
  t.fanout = L->fanout;
  int lg = 0;
  while ((1 << lg) < L->fanout) ++lg;
  t.log2w = lg;
  t.depth = L->depth;
  t.frac_bits = L->frac_bits;
  return t;
}

// Philox4x32-10 [EXT: Salmon et al. 2011]; u64 draw = x0 | x1 << 32 for
// ctr = (lo32(c), hi32(c), 0, 0), key = (lo32(seed), hi32(seed)).
__device__ __forceinline__ uint64_t philox_u64(uint64_t seed, uint64_t c) {
  uint32_t c0 = (uint32_t)c, c1 = (uint32_t)(c >> 32), c2 = 0, c3 = 0;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return (uint64_t)c0 | ((uint64_t)c1 << 32);
}

// ---- stratified sampling by descent (a8, §8c #8; shared by the samplers and the fused gather) ----
__device__ __forceinline__ uint64_t stratum_lo(uint64_t k, uint64_t Q, uint64_t n) {
  // floor(k Q / n) without 128-bit products: k*(Q/n) + floor(k*(Q%n)/n); k <= n < 2^31
  return k * (Q / n) + (k * (Q % n)) / n;
}

// Exact division by a fixed n (1 <= n < 2^31) without a 64-bit divide on the critical path:
// m = floor((2^64 - 1) / n) is computed once (it depends on n alone, so before any dependency
// wait); q = mulhi(x, m) undershoots floor(x / n) by at most 2, fixed by the remainder test.
struct DivN {
  uint64_t n, m;
};
__device__ __forceinline__ DivN divn_make(uint64_t n) { return DivN{n, ~0ull / n}; }
__device__ __forceinline__ uint64_t divn(uint64_t x, const DivN& d, uint64_t* rem) {
  uint64_t q = __umul64hi(x, d.m);
  uint64_t r = x - q * d.n;
  while (r >= d.n) {
    ++q;
    r -= d.n;
  }
  *rem = r;
  return q;
}
// Stratum bounds for a fixed Q (Qn = Q / n, Qr = Q % n): the same integers as stratum_lo.
struct Strata {
  uint64_t Q, Qn, Qr;
  DivN dn;
};
__device__ __forceinline__ Strata strata_make(uint64_t Q, const DivN& dn) {
  Strata s;
  s.Q = Q;
  s.dn = dn;
  s.Qn = divn(Q, dn, &s.Qr);
  return s;
}
__device__ __forceinline__ uint64_t strata_lo(uint64_t k, const Strata& s) {
  uint64_t r;
  return k * s.Qn + divn(k * s.Qr, s.dn, &r);  // k * Qr < n^2 <= 2^62
}
__device__ __forceinline__ uint64_t strata_prefix(int64_t k, const Strata& s, const uint64_t* draws, uint64_t seed,
                                                  uint64_t ctr0) {
  const uint64_t lo = strata_lo((uint64_t)k, s);
  const uint64_t hi = strata_lo((uint64_t)k + 1, s);
  const uint64_t u = draws ? draws[k] : philox_u64(seed, ctr0 + (uint64_t)k);
  return lo + __umul64hi(u, hi - lo);
}

// Global prefix of stratum k (a8, §8c #8): lo_k + floor(u_k (hi_k - lo_k) / 2^64).
// Non-decreasing in k (prefix_k < hi_k = lo_{k+1} <= prefix_{k+1}, or = lo_k for an
// empty stratum), so the strata a shard owns form one contiguous run.
__device__ __forceinline__ uint64_t stratum_prefix(int64_t k, uint64_t Q, int64_t n, const uint64_t* draws,
                                                   uint64_t seed, uint64_t ctr0) {
  const uint64_t lo = stratum_lo((uint64_t)k, Q, (uint64_t)n);
  const uint64_t hi = stratum_lo((uint64_t)k + 1, Q, (uint64_t)n);
  const uint64_t u = draws ? draws[k] : philox_u64(seed, ctr0 + (uint64_t)k);
  return lo + __umul64hi(u, hi - lo);
}

// Descend from the root for `prefix` (< node sum); returns leaf index, writes q.  Words
// [0, n_top) of the tree (whole top levels) may be staged in shared memory (`top`): those
// levels are read from there, the rest from global memory.
__device__ __forceinline__ int64_t descend(const TreeDev& L, const int64_t* __restrict__ tree,
                                           int64_t prefix, int64_t* q_out, int32_t* errbits,
                                           const int64_t* top = nullptr, int64_t n_top = 0) {
  const int lane = threadIdx.x & 31;
  int64_t node = 0;
  int64_t c = 0;
  for (int l = 0; l < L.depth; ++l) {
    const int64_t base = L.level_off[l + 1] + (node << L.log2w);
    c = lane < L.fanout ? (base < n_top ? top[base + lane] : tree[base + lane]) : 0;
    int64_t incl = c;
#pragma unroll
    for (int dlt = 1; dlt < 32; dlt <<= 1) {
      const int64_t o = shfl_up64(incl, dlt);
      if (lane >= dlt) incl += o;
    }
    unsigned bal = __ballot_sync(0xffffffffu, prefix < incl);
    int f;
    if (bal == 0) {  // prefix >= node sum: inconsistent tree / out of range -> clamp
      *errbits |= RPL_DERR_TREE;
      const unsigned nz = __ballot_sync(0xffffffffu, c > 0);
      f = nz ? 31 - __clz(nz) : 0;
      const int64_t inc_last = shfl64(incl, f);
      prefix = nz ? inc_last - 1 : 0;  // the last unit of the last non-empty child
    } else {
      f = __ffs(bal) - 1;
    }
    const int64_t inc_f = shfl64(incl, f);
    const int64_t c_f = shfl64(c, f);
    prefix -= inc_f - c_f;
    if (prefix < 0) prefix = 0;
    node = (node << L.log2w) + f;
    c = c_f;
  }
  *q_out = c;
  return node;
}

}  // namespace rpl
