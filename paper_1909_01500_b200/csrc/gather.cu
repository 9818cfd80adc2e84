// Gather of sampled transitions and sequences from the frame-deduplicated ring
// (P:38, P:123 fn).
//
// Design (B200): the gather is a pure HBM copy with a little index arithmetic, so
// it is built around the Tensor Memory Accelerator's bulk-copy path:
//   * one CTA per task (transition sample, or sequence sample x chunk of C rows);
//   * one elected thread issues cp.async.bulk global->shared copies of every
//     unique frame row the task needs (7056-B Atari frames, 16-B aligned) on one
//     mbarrier (expect_tx = total bytes);
//   * meanwhile the other warps resolve episode starts from the done flags
//     (frame-stack padding, §8c #13), copy the small per-row fields and compute
//     the fused n-step return (fp64 Horner);
//   * after the barrier, one lane per output stack issues a cp.async.bulk
//     shared->global store of the whole k-stack (k*7056 B contiguous in shared
//     memory when the stack has no padding, else one store per frame).
// Each unique frame is read from HBM once per task and written once per stack
// slot that uses it: the algorithmic bytes of SURVEY.md §8(d).
// Items whose size is not a multiple of 16 bytes (Mujoco vectors) use the same
// index logic with vectorised LSU copies.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "crpow.cuh"

namespace rpl {
namespace {

#include "seqprio.cuh"  // sequence_td8 (R26): the fused update's sequence priorities

#ifndef RPL_G_THREADS  // one-CTA-per-sample gathers (build-flag A/B knob)
#define RPL_G_THREADS 128
#endif
constexpr int G_THREADS = RPL_G_THREADS;
#ifndef RPL_TRANS_CONSUMERS  // consumer warps of the transition pipeline (build-flag A/B knob)
#define RPL_TRANS_CONSUMERS 4  // same-box DQN bs 512 step: 22.14 us vs 22.79 at 8 (6: 22.19, 12: 22.80)
#endif
#ifndef RPL_SEQ_SLOT_KB  // frame-slot budget of the default sequence gather (build-flag A/B knob)
#define RPL_SEQ_SLOT_KB 200
#endif
constexpr int SEQ_CHUNK = 8;  // output rows per sequence task

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// Intra-CTA flags with release / acquire semantics (the producer / consumer hand-offs of
// the persistent gathers): everything a thread did before flag_release is visible to a
// thread whose flag_acquire observes the value.
__device__ __forceinline__ void flag_release(volatile int* f, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32((const void*)f)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const int64_t* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int flag_acquire(volatile int* f) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32((const void*)f)) : "memory");
  return v;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// IS-weight normaliser (a9, §8c #10): *qmin when the caller passes it (e.g. the global
// batch min of Mode L), else the min of q over this batch's sampled entries (idx >= 0),
// computed by the calling warp (all 32 lanes must call) — this lets the sampler skip its
// grid-wide reduction.
__device__ __forceinline__ int64_t warp_batch_qmin(const int64_t* __restrict__ qmin, const int64_t* __restrict__ idx,
                                                   const int64_t* __restrict__ q, int64_t n) {
  if (qmin) return *qmin;
  int64_t m = INT64_MAX;
  // blocks of 8 loads per lane in flight before any is consumed (one latency per 256 entries)
  for (int64_t j0 = threadIdx.x & 31; j0 < n; j0 += 32 * 8) {
    int64_t iv[8], qv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t j = j0 + 32 * u;
      iv[u] = j < n ? __ldg(idx + j) : -1;
      qv[u] = j < n ? __ldg(q + j) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (iv[u] >= 0 && qv[u] < m) m = qv[u];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const int64_t x = (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)m, o);
    m = x < m ? x : m;
  }
  return m;
}

// Cooperative copy of `bytes` bytes with the widest aligned word.
__device__ __forceinline__ void coop_copy(void* dst, const void* src, int64_t bytes, int t, int nt) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src);
  if ((a & 15) == 0 && (bytes & 15) == 0) {
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    for (int64_t i = t; i < bytes / 16; i += nt) d[i] = __ldg(s + i);
  } else if ((a & 3) == 0 && (bytes & 3) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int64_t i = t; i < bytes / 4; i += nt) d[i] = __ldg(s + i);
  } else {
    const uint8_t* s = reinterpret_cast<const uint8_t*>(src);
    uint8_t* d = reinterpret_cast<uint8_t*>(dst);
    for (int64_t i = t; i < bytes; i += nt) d[i] = __ldg(s + i);
  }
}
__device__ __forceinline__ void coop_zero(void* dst, int64_t bytes, int t, int nt) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  if ((a & 15) == 0 && (bytes & 15) == 0) {
    int4* d = reinterpret_cast<int4*>(dst);
    for (int64_t i = t; i < bytes / 16; i += nt) d[i] = make_int4(0, 0, 0, 0);
  } else {
    uint8_t* d = reinterpret_cast<uint8_t*>(dst);
    for (int64_t i = t; i < bytes; i += nt) d[i] = 0;
  }
}

#ifdef RPL_DIAG
#define GDIAG(D) ((D).diag)
#else
#define GDIAG(D) 0
#endif

struct GDesc {
  int32_t kind, pad_mode, out_mode, k;
  int64_t cap_T, B, cursor, size;
  int64_t obs_bytes, act_bytes, rnn_bytes;
  int32_t n_step, seq_len, period, rnn_parts;
  double gamma;
  const uint8_t* obs;
  const uint8_t* act;
  const float* rew;
  const uint8_t* done;
  const uint8_t* rnn;
  uint8_t* o_obs;
  uint8_t* o_next_obs;
  uint8_t* o_act;
  uint8_t* o_prev_act;
  float* o_rew;
  float* o_prev_rew;
  uint8_t* o_done;
  float* o_ret;
  uint8_t* o_done_n;
  float* o_w;
  uint8_t* o_rnn;
  int use_tma;
  int diag;  // rpl_debug_set_gather_diag mask (0 in normal operation)
  const int64_t* n_active;  // device count of leading entries to gather (NULL: all n)
  const int64_t* col_offset;  // device output column offset (NULL: 0)
  int8_t* o_start;            // per-row episode-start offsets [L, n] (NULL: not produced)
  int64_t* const* peer_boards;  // K7 fused (rpl_gather_desc.peer_boards; NULL: off)
  int peer_world, peer_rank;
  const float* q_tgt;  // fused n-step targets (rpl_gather_desc.q_tgt / o_tgt / ...)
  float* o_tgt;
  uint8_t* o_tgt_done;
  int tgt_lo, tgt_T, rescale;
  double rescale_eps;
  const float* v_term;  // time-limit bootstrap values (R34; NULL: every done is terminal)
  int64_t* done_flag;   // completion signal (Mode C; NULL: off)
  int64_t* done_seq;    // [2] call counter + CTA ticket (device, this rank's memory)
  int64_t* smp_tree;    // fused stratified sampling (rpl_gather_sample; NULL: idx given)
  TreeDev smp_L;
  uint64_t smp_seed;
  int64_t* work;        // dynamic-tail unit counter + ticket (rpl_gather_desc.work; NULL: static split)
  // fused priority update before the sampling (rpl_gather_update_sample; NULL: none)
  const int64_t* upd_idx;
  const float* upd_td;
  int upd_n, upd_T, upd_live, upd_pad;
  double upd_eta, upd_alpha, upd_eps;
};

// Output column offset (rpl_gather_desc.col_offset); read after pdl_wait.
__device__ __forceinline__ int64_t col_off(const GDesc& D) { return D.col_offset ? *D.col_offset : 0; }

// Number of leading entries of idx to gather (rpl_gather_desc.n_active); read after pdl_wait.
__device__ __forceinline__ int64_t active_n(const GDesc& D, int64_t n) {
  if (!D.n_active) return n;
  const int64_t a = *D.n_active;
  return a < 0 ? 0 : (a < n ? a : n);
}

__device__ __forceinline__ int64_t wrap(int64_t r, int64_t cap) {
  r %= cap;
  return r < 0 ? r + cap : r;
}

// Source slot (window index) of stack slot j for target row index `ti` (window
// coordinates: window index w <-> ring row first + w).  Episode start s(t) is the
// latest row s in (t-k+1, t] whose previous row ended an episode, else t-k+1
// (frame-stacking wrapper semantics, §8c #13).  Returns -1 for a zero slot.
// dwin[w] = done flag of window row w-1 (dwin has one extra leading entry).
__device__ __forceinline__ int stack_src(const uint8_t* dwin, int ti, int j, int k, int pad_mode) {
  int s = ti;
  while (s > ti - k + 1 && !dwin[s]) --s;  // dwin[s] = done[row s - 1]
  const int want = ti - k + 1 + j;
  if (want >= s) return want;
  return pad_mode == RPL_PAD_ZERO ? -1 : s;
}

// n-step return over ring rows row .. row+ns-1 (mod cap_T) of column b (a2, R24): fp64
// Horner from the last row, starting from the bootstrap value `acc`; a done row cuts the
// recursion (acc = r), and with v_term given a time-limit row (done == RPL_DONE_TIMEOUT)
// bootstraps from its terminal value instead (acc = r + gamma v_term, R34).  *dn = OR of the
// done flags.  Rows are loaded in blocks of 8, all in flight before the recurrence uses them.
__device__ __forceinline__ double nstep_rows(const GDesc& D, int64_t row, int64_t b, int ns, double acc,
                                             uint8_t* dn) {
  constexpr int NB = 8;
  uint8_t d_or = 0;
  for (int hi = ns; hi > 0; hi -= NB) {
    const int lo = hi > NB ? hi - NB : 0;
    float rb[NB];
    uint8_t db[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      int64_t rr = row + lo + j;
      while (rr >= D.cap_T) rr -= D.cap_T;
      const bool in = lo + j < hi;
      rb[j] = in ? __ldg(D.rew + rr * D.B + b) : 0.0f;
      db[j] = in ? __ldg(D.done + rr * D.B + b) : (uint8_t)0;
    }
#pragma unroll
    for (int j = NB - 1; j >= 0; --j) {
      if (lo + j < hi) {
        const double ri = (double)rb[j];
        if (db[j]) {
          acc = ri;
          if (db[j] == RPL_DONE_TIMEOUT && D.v_term) {
            int64_t rr = row + lo + j;
            while (rr >= D.cap_T) rr -= D.cap_T;
            acc = fma(D.gamma, (double)__ldg(D.v_term + rr * D.B + b), ri);
          }
        } else {
          acc = fma(D.gamma, acc, ri);
        }
        d_or |= db[j];
      }
    }
  }
  *dn = d_or;
  return acc;
}

// ---------------------------------------------------------------------------
// Transitions: one CTA per sample.  Window rows r-k+1 .. r+n (NR = k+n rows).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(G_THREADS)
k_gather_transition(GDesc D, const int64_t* __restrict__ idx, int64_t n, const int64_t* __restrict__ q,
                    const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint8_t dwin[64];
  __shared__ int sslot[2][32];
  const int tid = threadIdx.x;
  const int64_t s = blockIdx.x;
  pdl_wait();
  if (s >= active_n(D, n)) return;
  const int64_t sc = s + col_off(D);  // output column (Mode C offset)
  const int64_t leaf = idx[s];
  if (leaf < 0) return;
  const int k = D.k, ns = D.n_step;
  const int NR = k + ns;
  if (leaf >= D.cap_T * D.B) {
    if (tid == 0) set_err(err, RPL_DERR_IDX);
    return;
  }
  const int64_t r = leaf / D.B, b = leaf - (leaf / D.B) * D.B;
  const int64_t first = r - (k - 1);
  const int64_t ob = D.obs_bytes;

  const bool tma = D.use_tma && (D.o_obs || D.o_next_obs);
  if (tma) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_expect_tx(&bar, (uint32_t)(NR * ob));
      for (int w = 0; w < NR; ++w) {
        const int64_t row = wrap(first + w, D.cap_T);
        bulk_g2s(smem + (int64_t)w * ob, D.obs + (row * D.B + b) * ob, (uint32_t)ob, &bar);
      }
    }
  }
  // done flags of rows first-1 .. r+n  (dwin[w] = done[first + w - 1])
  if (tid < NR + 1) dwin[tid] = __ldg(D.done + wrap(first + tid - 1, D.cap_T) * D.B + b);
  if (tid == 0) {
    const int64_t age = wrap(D.cursor - 1 - r, D.cap_T);
    if (!(age >= ns && age <= D.size - k)) set_err(err, RPL_DERR_INVALID_LEAF);
  }
  __syncthreads();
  // stack slot sources: [0] obs at window index k-1, [1] next obs at window index k-1+n
  if (tid < 2 * k) {
    const int which = tid / k, j = tid - which * k;
    sslot[which][j] = stack_src(dwin, (k - 1) + which * ns, j, k, D.pad_mode);
  }
  // scalars (warp 1): action, fused n-step return, IS weight (a9)
  if (tid >= 32 && tid < 64) {
    const int l = tid - 32;
    const int64_t qm = (D.o_w && q) ? warp_batch_qmin(qmin, idx, q, n) : 0;
    if (D.o_act) {
      const uint8_t* src = D.act + (r * D.B + b) * D.act_bytes;
      uint8_t* dst = D.o_act + sc * D.act_bytes;
      for (int64_t i = l; i < D.act_bytes; i += 32) dst[i] = src[i];
    }
    if (l == 0) {
      if (D.o_ret || D.o_done_n) {  // fused n-step return (R24, R34)
        uint8_t dn = 0;
        const double acc = nstep_rows(D, r, b, ns, 0.0, &dn);
        if (D.o_ret) D.o_ret[sc] = (float)acc;
        if (D.o_done_n) D.o_done_n[sc] = dn ? 1 : 0;
      }
      if (D.o_w && q) {
        const int64_t qs = q[s];
        D.o_w[sc] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
      }
    }
  }
  __syncthreads();

  uint8_t* outs[2] = {D.o_obs ? D.o_obs + sc * k * ob : nullptr, D.o_next_obs ? D.o_next_obs + sc * k * ob : nullptr};
  if (tma) {
    uint8_t* zrow = smem + (int64_t)NR * ob;  // zero row for RPL_PAD_ZERO
    bool needs_zero = false;
    for (int w = 0; w < 2; ++w)
      for (int j = 0; j < k; ++j) needs_zero |= (sslot[w][j] < 0);
    if (needs_zero) {
      coop_zero(zrow, ob, tid, G_THREADS);
      fence_proxy_async();
      __syncthreads();
    }
    if (tid < 32) {
      if (tid == 0) mbar_wait(&bar, 0);
      __syncwarp();
      fence_proxy_async();
      // lane 0: obs stack, lane 1: next-obs stack
      if (tid < 2 && outs[tid]) {
        const int* sl = sslot[tid];
        bool contiguous = true;
        for (int j = 1; j < k; ++j) contiguous &= (sl[j] == sl[0] + j) && sl[0] >= 0;
        if (contiguous && sl[0] >= 0) {
          bulk_s2g(outs[tid], smem + (int64_t)sl[0] * ob, (uint32_t)(k * ob));
        } else {
          for (int j = 0; j < k; ++j)
            bulk_s2g(outs[tid] + j * ob, sl[j] < 0 ? zrow : smem + (int64_t)sl[j] * ob, (uint32_t)ob);
        }
        bulk_commit();
        bulk_wait_read0();
      }
    }
  } else if (!D.use_tma) {
    for (int w = 0; w < 2; ++w) {
      if (!outs[w]) continue;
      for (int j = 0; j < k; ++j) {
        const int src = sslot[w][j];
        if (src < 0) {
          coop_zero(outs[w] + j * ob, ob, tid, G_THREADS);
        } else {
          const int64_t row = wrap(first + src, D.cap_T);
          coop_copy(outs[w] + j * ob, D.obs + (row * D.B + b) * ob, ob, tid, G_THREADS);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Sequences: grid (chunks, samples).  Stacked: output rows tau in [c*C, c*C+C) of
// L, window rows row0 + c*C - (k-1) .. row0 + c*C + C - 1.  Unique: output rows
// u in [c*C, c*C+C) of L+k-1 <-> ring rows row0 - (k-1) + u.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(G_THREADS)
k_gather_sequence(GDesc D, const int64_t* __restrict__ idx, int64_t n, const int64_t* __restrict__ q,
                  const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint8_t dwin[64];
  __shared__ int sslot[SEQ_CHUNK][8];
  const int tid = threadIdx.x;
  const int64_t s = blockIdx.y;
  if (s >= active_n(D, n)) return;
  const int64_t sc = s + col_off(D);  // output column (Mode C offset)
  const int c = blockIdx.x;
  const int64_t leaf = idx[s];
  if (leaf < 0) return;
  const int k = D.k, L = D.seq_len;
  const int64_t nblk = D.cap_T / D.period;
  if (leaf >= nblk * D.B) {
    if (tid == 0 && c == 0) set_err(err, RPL_DERR_IDX);
    return;
  }
  const int64_t blk = leaf / D.B, b = leaf - (leaf / D.B) * D.B;
  const int64_t row0 = blk * D.period;
  const int64_t ob = D.obs_bytes;
  const bool stacked = D.out_mode == RPL_OUT_STACKED;
  const int rows_out = stacked ? L : L + k - 1;
  const int o0 = c * SEQ_CHUNK;
  if (o0 >= rows_out && o0 >= L) return;
  const int Cn = max(0, min(SEQ_CHUNK, rows_out - o0));
  // window (frames to stage): stacked -> [row0+o0-(k-1), row0+o0+Cn); unique -> [row0-(k-1)+o0, +Cn)
  const int64_t first = stacked ? row0 + o0 - (k - 1) : row0 - (k - 1) + o0;
  const int NR = stacked ? (Cn > 0 ? Cn + k - 1 : 0) : Cn;

  if (D.use_tma && NR > 0 && D.o_obs) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_expect_tx(&bar, (uint32_t)(NR * ob));
      for (int w = 0; w < NR; ++w) {
        const int64_t row = wrap(first + w, D.cap_T);
        bulk_g2s(smem + (int64_t)w * ob, D.obs + (row * D.B + b) * ob, (uint32_t)ob, &bar);
      }
    }
  }
  if (tid < NR + 1) dwin[tid] = __ldg(D.done + wrap(first + tid - 1, D.cap_T) * D.B + b);
  if (tid == 0 && c == 0) {
    const int64_t age = wrap(D.cursor - 1 - row0, D.cap_T);
    const int hist = k - 1 > 1 ? k - 1 : 1;
    if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
  }
  __syncthreads();
  if (stacked && tid < Cn * k) {
    const int tau = tid / k, j = tid - (tid / k) * k;
    sslot[tau][j] = stack_src(dwin, tau + k - 1, j, k, D.pad_mode);
  }
  // per-row scalars for output rows tau in [o0, o0+C) of L (both modes)
  {
    const int t_hi = min(o0 + SEQ_CHUNK, L);
    for (int tau = o0 + (tid >> 5); tau < t_hi; tau += G_THREADS / 32) {
      const int l = tid & 31;
      const int64_t row = wrap(row0 + tau, D.cap_T);
      const int64_t prow = wrap(row0 + tau - 1, D.cap_T);
      const uint8_t pd = __ldg(D.done + prow * D.B + b);  // previous row ended an episode?
      if (D.o_act)
        for (int64_t i = l; i < D.act_bytes; i += 32)
          D.o_act[(tau * n + sc) * D.act_bytes + i] = D.act[(row * D.B + b) * D.act_bytes + i];
      if (D.o_prev_act)
        for (int64_t i = l; i < D.act_bytes; i += 32)
          D.o_prev_act[(tau * n + sc) * D.act_bytes + i] = pd ? 0 : D.act[(prow * D.B + b) * D.act_bytes + i];
      if (l == 0) {
        if (D.o_rew) D.o_rew[tau * n + sc] = __ldg(D.rew + row * D.B + b);
        if (D.o_prev_rew) D.o_prev_rew[tau * n + sc] = pd ? 0.0f : __ldg(D.rew + prow * D.B + b);
        if (D.o_done) D.o_done[tau * n + sc] = __ldg(D.done + row * D.B + b);
      }
    }
  }
  // stored recurrent state at the sequence start (chunk 0), [parts, n, rnn_bytes]
  if (c == 0 && D.o_rnn) {
    for (int p = 0; p < D.rnn_parts; ++p)
      coop_copy(D.o_rnn + (p * n + sc) * D.rnn_bytes,
                D.rnn + ((blk * D.B + b) * D.rnn_parts + p) * D.rnn_bytes, D.rnn_bytes, tid, G_THREADS);
  }
  if (c == 0 && D.o_w && q && tid < 32) {
    const int64_t qm = warp_batch_qmin(qmin, idx, q, n);
    const int64_t qs = q[s];
    if (tid == 0) D.o_w[sc] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
  }
  __syncthreads();
  if (!D.o_obs || NR == 0) return;

  if (D.use_tma) {
    uint8_t* zrow = smem + (int64_t)NR * ob;
    bool needs_zero = false;
    if (stacked)
      for (int t = 0; t < Cn; ++t)
        for (int j = 0; j < k; ++j) needs_zero |= (sslot[t][j] < 0);
    if (needs_zero) {
      coop_zero(zrow, ob, tid, G_THREADS);
      fence_proxy_async();
      __syncthreads();
    }
    if (tid < 32) {
      if (tid == 0) mbar_wait(&bar, 0);
      __syncwarp();
      fence_proxy_async();
      if (stacked) {
        if (tid < Cn) {
          const int tau = tid;
          uint8_t* dst = D.o_obs + (((int64_t)(o0 + tau) * n + sc) * k) * ob;
          const int* sl = sslot[tau];
          bool contiguous = sl[0] >= 0;
          for (int j = 1; j < k; ++j) contiguous &= (sl[j] == sl[0] + j);
          if (contiguous) {
            bulk_s2g(dst, smem + (int64_t)sl[0] * ob, (uint32_t)(k * ob));
          } else {
            for (int j = 0; j < k; ++j)
              bulk_s2g(dst + j * ob, sl[j] < 0 ? zrow : smem + (int64_t)sl[j] * ob, (uint32_t)ob);
          }
          bulk_commit();
          bulk_wait_read0();
        }
      } else {
        if (tid < Cn) {
          uint8_t* dst = D.o_obs + ((int64_t)(o0 + tid) * n + sc) * ob;
          bulk_s2g(dst, smem + (int64_t)tid * ob, (uint32_t)ob);
          bulk_commit();
          bulk_wait_read0();
        }
      }
    }
  } else {
    if (stacked) {
      for (int tau = 0; tau < Cn; ++tau) {
        uint8_t* dst = D.o_obs + (((int64_t)(o0 + tau) * n + sc) * k) * ob;
        for (int j = 0; j < k; ++j) {
          const int src = sslot[tau][j];
          if (src < 0) coop_zero(dst + j * ob, ob, tid, G_THREADS);
          else coop_copy(dst + j * ob, D.obs + (wrap(first + src, D.cap_T) * D.B + b) * ob, ob, tid, G_THREADS);
        }
      }
    } else {
      for (int u = 0; u < Cn; ++u)
        coop_copy(D.o_obs + ((int64_t)(o0 + u) * n + sc) * ob,
                  D.obs + (wrap(first + u, D.cap_T) * D.B + b) * ob, ob, tid, G_THREADS);
    }
  }
}


// ---------------------------------------------------------------------------
// Sequences, persistent TMA pipeline (stacked output).  The n*L output rows are
// split into equal contiguous ranges, one per CTA, in (sample, row) order; a
// range breaks into "pieces" (runs of rows of one sample).  A piece of R rows
// needs the R+k-1 frames rows tau0-k+1 .. tau0+R-1, each loaded ONCE into a
// ring of NS shared-memory slots:
//   warp 0 / lane 0  producer: cp.async.bulk global->shared, one mbarrier per
//                    slot; a slot is refilled once the consumer has released it;
//   warp 1 / lane 0  consumer: per output row, waits for its k frames and issues
//                    one cp.async.bulk shared->global store of the k-stack
//                    (per-frame stores when padded or wrapping the ring); keeps
//                    PIPE_G store groups in flight and releases frames whose
//                    last reader has finished (cp.async.bulk.wait_group.read);
//   warps 2-3        per-row fields, stored recurrent state, IS weights.
// Loads and stores of different rows overlap continuously, and each frame is
// read from HBM once per piece (pieces add k-1 frames at their start).
// ---------------------------------------------------------------------------
constexpr int PIPE_THREADS = 128;
constexpr int PIPE_MAX_NS = 32;
constexpr int PIPE_MAX_ROWS = 512;  // output rows per CTA
template <int G>
__device__ __forceinline__ void bulk_wait_read_G() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(G) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int PIPE_G>  // store groups (output rows) in flight per consumer
__global__ void __launch_bounds__(PIPE_THREADS)
k_gather_seq_pipe(GDesc D, const int64_t* __restrict__ idx, int64_t n, int NS, int64_t rows_per_cta,
                  const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  extern __shared__ __align__(128) uint8_t smem[];  // NS frame slots + 1 zero slot
  __shared__ __align__(8) uint64_t full[PIPE_MAX_NS];
  __shared__ int8_t start_off[PIPE_MAX_ROWS];
  __shared__ int rel_hist[64];
  __shared__ volatile int free_count;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n_eff = active_n(D, n);
  const int k = D.k, L = D.seq_len;
  const int64_t ob = D.obs_bytes;
  const int64_t total = n * (int64_t)L;
  const int64_t g0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t g1 = min(total, g0 + rows_per_cta);
  if (g0 >= g1) return;
  const int nrows = (int)(g1 - g0);
  const int64_t nblk = D.cap_T / D.period;
  uint8_t* zrow = smem + (int64_t)NS * ob;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
    free_count = 0;
  }
  // per-row episode-start offsets (frame-stack padding, §8c #13) and validity flags
  for (int c = tid; c < nrows; c += PIPE_THREADS) {
    const int64_t g = g0 + c;
    const int64_t s = g / L;
    const int tau = (int)(g - s * L);
    const int64_t leaf = s < n_eff ? idx[s] : -1;
    int8_t so = 0;
    if (leaf >= 0 && leaf < nblk * D.B) {
      const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
      const int64_t row = blk * D.period + tau;
      int st = 0;  // start offset in (tau-k+1 .. tau]: latest row whose previous row ended an episode
      for (int j = k - 1; j >= 1; --j) {
        if (__ldg(D.done + wrap(row - (k - 1) + j - 1, D.cap_T) * D.B + b)) {
          st = j;
          break;
        }
      }
      so = (int8_t)st;
      if (tau == 0) {
        const int64_t age = wrap(D.cursor - 1 - blk * D.period, D.cap_T);
        const int hist = k - 1 > 1 ? k - 1 : 1;
        if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
      }
    } else if (leaf >= nblk * D.B && tau == 0) {
      set_err(err, RPL_DERR_IDX);
    }
    start_off[c] = so;
  }
  if (D.pad_mode == RPL_PAD_ZERO) coop_zero(zrow, ob, tid, PIPE_THREADS);
  fence_proxy_async();
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer ----------------
      int64_t i = 0;  // frame position
      int64_t g = g0;
      while (g < g1) {
        const int64_t s = g / L;
        const int tau0 = (int)(g - s * L);
        const int R = (int)min((int64_t)(L - tau0), g1 - g);
        const int64_t leaf = s < n_eff ? idx[s] : -1;
        if (leaf >= 0 && leaf < nblk * D.B) {
          const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
          const int64_t first = blk * D.period + tau0 - (k - 1);
          for (int w = 0; w < R + k - 1; ++w, ++i) {
            const int slot = (int)(i % NS);
            if (i >= NS) {
              while (free_count <= i - NS) __nanosleep(20);
              fence_proxy_async();
              // observe the slot's previous phase before re-arming it, so every arrive on a
              // barrier follows the completion of its previous phase (synccheck)
              mbar_wait(&full[slot], (uint32_t)(((i / NS) - 1) & 1));
            }
            mbar_expect_tx(&full[slot], (uint32_t)ob);
            bulk_g2s(smem + (int64_t)slot * ob, D.obs + (wrap(first + w, D.cap_T) * D.B + b) * ob, (uint32_t)ob,
                     &full[slot]);
          }
        }
        g += R;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- consumer ----------------
      int64_t F = 0;   // first frame position of the current piece
      int c = 0;       // CTA-local row counter
      int64_t g = g0;
      while (g < g1) {
        const int64_t s = g / L;
        const int tau0 = (int)(g - s * L);
        const int R = (int)min((int64_t)(L - tau0), g1 - g);
        const int64_t leaf = s < n_eff ? idx[s] : -1;
        const bool ok = leaf >= 0 && leaf < nblk * D.B;
        for (int m = 0; m < R; ++m, ++c) {
          if (ok) {
            const int so = start_off[c];
            // wait for the frames of this row: window coords m .. m+k-1 (positions F+m ..)
            for (int j = (so > 0 ? so : 0); j < k; ++j) {
              const int64_t pos = F + m + j;
              mbar_wait(&full[pos % NS], (uint32_t)((pos / NS) & 1));
            }
            uint8_t* dst = D.o_obs + (((int64_t)(tau0 + m) * n + s) * k) * ob;
            const int64_t p0 = F + m;
            const int sl0 = (int)(p0 % NS);
            if (so == 0 && sl0 + k <= NS) {
              bulk_s2g(dst, smem + (int64_t)sl0 * ob, (uint32_t)(k * ob));
            } else {
              for (int j = 0; j < k; ++j) {
                const uint8_t* src;
                if (j >= so) src = smem + (int64_t)((p0 + j) % NS) * ob;
                else src = D.pad_mode == RPL_PAD_ZERO ? zrow : smem + (int64_t)((p0 + so) % NS) * ob;
                bulk_s2g(dst + j * ob, src, (uint32_t)ob);
              }
            }
          }
          bulk_commit();
          // frames released once this row's store has read them: all positions < F+m+1,
          // and at the end of the piece its whole window
          rel_hist[c & 63] = (int)(ok ? (m == R - 1 ? F + R + k - 1 : F + m + 1) : F);
          bulk_wait_read_G<PIPE_G>();
          if (c >= PIPE_G) free_count = rel_hist[(c - PIPE_G) & 63];
        }
        if (ok) F += R + k - 1;
        g += R;
      }
      bulk_wait_all();
      free_count = 0x7fffffff;
    }
  } else {
    // ---------------- per-row fields, stored state, IS weights (warps 2-3) ----------------
    const int t2 = tid - 64;
    const int64_t qm = (D.o_w && q) ? warp_batch_qmin(qmin, idx, q, n) : 0;
    for (int c = t2; c < nrows; c += PIPE_THREADS - 64) {
      const int64_t gg = g0 + c;
      const int64_t s = gg / L;
      const int tau = (int)(gg - s * L);
      const int64_t leaf = s < n_eff ? idx[s] : -1;
      if (leaf < 0 || leaf >= nblk * D.B) continue;
      const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
      const int64_t row = wrap(blk * D.period + tau, D.cap_T);
      const int64_t prow = wrap(blk * D.period + tau - 1, D.cap_T);
      const uint8_t pd = __ldg(D.done + prow * D.B + b);
      const int64_t o = (int64_t)tau * n + s;
      if (D.o_act) coop_copy(D.o_act + o * D.act_bytes, D.act + (row * D.B + b) * D.act_bytes, D.act_bytes, 0, 1);
      if (D.o_prev_act) {
        if (pd) coop_zero(D.o_prev_act + o * D.act_bytes, D.act_bytes, 0, 1);
        else coop_copy(D.o_prev_act + o * D.act_bytes, D.act + (prow * D.B + b) * D.act_bytes, D.act_bytes, 0, 1);
      }
      if (D.o_rew) D.o_rew[o] = __ldg(D.rew + row * D.B + b);
      if (D.o_prev_rew) D.o_prev_rew[o] = pd ? 0.0f : __ldg(D.rew + prow * D.B + b);
      if (D.o_done) D.o_done[o] = __ldg(D.done + row * D.B + b);
      if (tau == 0 && D.o_w && q) {
        const int64_t qs = q[s];
        D.o_w[s] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
      }
    }
    // stored recurrent state for samples whose row 0 lies in this CTA
    if (D.o_rnn) {
      for (int64_t s = (g0 + L - 1) / L; s * L < g1; ++s) {
        const int64_t leaf = s < n_eff ? idx[s] : -1;
        if (leaf < 0 || leaf >= nblk * D.B) continue;
        const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
        for (int p = 0; p < D.rnn_parts; ++p)
          coop_copy(D.o_rnn + (p * n + s) * D.rnn_bytes, D.rnn + ((blk * D.B + b) * D.rnn_parts + p) * D.rnn_bytes,
                    D.rnn_bytes, t2, PIPE_THREADS - 64);
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Sequences, frame-centric LSU variant (stacked output): one warp per unique
// frame (sample s, window row w in [-(k-1), L-1]).  The warp loads the frame
// once into registers (16-B vector loads, several in flight per lane) and stores
// it to every stack slot whose source it is: stack tau in [w, w+k-1] takes it at
// slot w-(tau-k+1) when w >= s(tau), and at the padded slots below when w is the
// episode start s(tau) (repeat mode; zero mode writes zeros there instead).
// Each frame is read from L2/HBM once; every output byte is written once.
// ---------------------------------------------------------------------------
constexpr int FC_WARPS = 4;
constexpr int FC_MAX_V4 = 16;  // 16 x 32 lanes x 16 B = 8 KB per warp pass

__device__ __forceinline__ int seq_start(const GDesc& D, int64_t row0, int64_t b, int tau, int k) {
  // s(tau) - (tau-k+1) in [0, k-1]: latest row in (tau-k+1, tau] whose previous row ended an episode
  for (int j = k - 1; j >= 1; --j)
    if (__ldg(D.done + wrap(row0 + tau - (k - 1) + j - 1, D.cap_T) * D.B + b)) return j;
  return 0;
}

__global__ void __launch_bounds__(FC_WARPS * 32)
k_gather_seq_lsu(GDesc D, const int64_t* __restrict__ idx, int64_t n, const int64_t* __restrict__ q,
                 const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int k = D.k, L = D.seq_len;
  const int W = L + k - 1;  // unique frames per sample
  const int64_t task = (int64_t)blockIdx.x * FC_WARPS + (threadIdx.x >> 5);
  if (task >= n * W) return;
  const int64_t s = task / W;
  const int w = (int)(task - s * W) - (k - 1);  // window row, -(k-1) .. L-1
  const int64_t leaf = s < active_n(D, n) ? idx[s] : -1;
  const int64_t nblk = D.cap_T / D.period;
  if (leaf < 0) return;
  if (leaf >= nblk * D.B) {
    if (lane == 0 && w == 0) set_err(err, RPL_DERR_IDX);
    return;
  }
  const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
  const int64_t row0 = blk * D.period;
  const int64_t ob = D.obs_bytes;
  const int4* src = reinterpret_cast<const int4*>(D.obs + (wrap(row0 + w, D.cap_T) * D.B + b) * ob);
  const int nv = (int)(ob / 16);
  // destinations: lane j < k*k enumerates (stack tau = w + t, slot) pairs
  // stack tau = w + t (t = 0..k-1) uses this frame at natural slot k-1-t if w >= s(tau);
  // padded slots 0..(s(tau)-(tau-k+1))-1 take the start frame when w == s(tau).
  uint32_t natural = 0, padrep = 0, padzero = 0;  // bit t: stack w+t
  int padcnt[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) padcnt[t] = 0;
  if (w == 0 && D.o_w && q) {  // warp-uniform (w is this warp's frame)
    const int64_t qm = warp_batch_qmin(qmin, idx, q, n);
    const int64_t qs = q[s];
    if (lane == 0) D.o_w[s] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
  }
  for (int t = 0; t < k; ++t) {
    const int tau = w + t;
    if (tau < 0 || tau >= L) continue;
    const int so = seq_start(D, row0, b, tau, k);  // s(tau) = tau-k+1+so
    const int stw = tau - k + 1 + so;
    if (w >= stw) natural |= 1u << t;
    if (so > 0 && w == stw) {
      padcnt[t] = so;
      if (D.pad_mode == RPL_PAD_ZERO) padzero |= 1u << t;
      else padrep |= 1u << t;
    }
  }
  if (!(natural | padrep | padzero)) return;
  for (int base = 0; base < nv; base += 32 * FC_MAX_V4) {
    int4 v[FC_MAX_V4];
#pragma unroll
    for (int u = 0; u < FC_MAX_V4; ++u) {
      const int i = base + u * 32 + lane;
      if (i < nv) v[u] = __ldg(src + i);
    }
    for (int t = 0; t < k; ++t) {
      const int tau = w + t;
      if (tau < 0 || tau >= L) continue;
      int4* stack = reinterpret_cast<int4*>(D.o_obs + (((int64_t)tau * n + s) * k) * ob);
      if (natural & (1u << t)) {
        int4* dst = stack + (int64_t)(k - 1 - t) * (ob / 16);
#pragma unroll
        for (int u = 0; u < FC_MAX_V4; ++u) {
          const int i = base + u * 32 + lane;
          if (i < nv) dst[i] = v[u];
        }
      }
      if ((padrep | padzero) & (1u << t)) {
        for (int j = 0; j < padcnt[t]; ++j) {
          int4* dst = stack + (int64_t)j * (ob / 16);
#pragma unroll
          for (int u = 0; u < FC_MAX_V4; ++u) {
            const int i = base + u * 32 + lane;
            if (i < nv) dst[i] = (padzero & (1u << t)) ? make_int4(0, 0, 0, 0) : v[u];
          }
        }
      }
    }
  }
}

// per-row fields + stored state for the LSU variant (one thread per output row)
__global__ void k_gather_seq_fields(GDesc D, const int64_t* __restrict__ idx, int64_t n, int32_t* err) {
  const int L = D.seq_len;
  const int64_t nblk = D.cap_T / D.period;
  for (int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gg < n * L; gg += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = gg / L;
    const int tau = (int)(gg - s * L);
    const int64_t leaf = s < active_n(D, n) ? idx[s] : -1;
    if (leaf < 0 || leaf >= nblk * D.B) continue;
    const int64_t blk = leaf / D.B, b = leaf - blk * D.B;
    const int64_t row = wrap(blk * D.period + tau, D.cap_T);
    const int64_t prow = wrap(blk * D.period + tau - 1, D.cap_T);
    const uint8_t pd = __ldg(D.done + prow * D.B + b);
    const int64_t o = (int64_t)tau * n + s;
    if (D.o_act) coop_copy(D.o_act + o * D.act_bytes, D.act + (row * D.B + b) * D.act_bytes, D.act_bytes, 0, 1);
    if (D.o_prev_act) {
      if (pd) coop_zero(D.o_prev_act + o * D.act_bytes, D.act_bytes, 0, 1);
      else coop_copy(D.o_prev_act + o * D.act_bytes, D.act + (prow * D.B + b) * D.act_bytes, D.act_bytes, 0, 1);
    }
    if (D.o_rew) D.o_rew[o] = __ldg(D.rew + row * D.B + b);
    if (D.o_prev_rew) D.o_prev_rew[o] = pd ? 0.0f : __ldg(D.rew + prow * D.B + b);
    if (D.o_done) D.o_done[o] = __ldg(D.done + row * D.B + b);
    if (tau == 0) {
      const int64_t age = wrap(D.cursor - 1 - blk * D.period, D.cap_T);
      const int hist = D.k - 1 > 1 ? D.k - 1 : 1;
      if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
      if (D.o_rnn)
        for (int p = 0; p < D.rnn_parts; ++p)
          coop_copy(D.o_rnn + (p * n + s) * D.rnn_bytes, D.rnn + ((blk * D.B + b) * D.rnn_parts + p) * D.rnn_bytes,
                    D.rnn_bytes, 0, 1);
    }
  }
}


// ---------------------------------------------------------------------------
// Sequences, persistent pipeline with TMA loads and LSU stores (default).
// A CTA owns a contiguous run of output rows g = s*L + tau (time-major within
// each sample s), i.e. one or a few "pieces" (runs of rows of one sample); a
// piece of R rows reads its R + k - 1 unique frames once.  Stores are issued by
// CONSUMER WARPS as 16-B st.global from shared memory rather than bulk stores:
// bulk stores and bulk loads share the SM's TMA queue, so in the all-TMA
// pipeline every frame load waits behind queued 28-KB stores.  Roles:
//   warp 0, lane 0   producer: TMA bulk loads of each piece's frames into NS
//                    slots (one mbarrier per slot); refills a slot once the
//                    contiguous done-frontier has passed every row reading it;
//   warp 1           meta: per-row fields (act, prev_act, rew, prev_rew, done),
//                    IS weights and stored recurrent state — the latency-bound
//                    scattered loads never sit on a consumer's critical path;
//   warps 2..NC+1    consumers: one k-stack (k*7056 B) per row, LDS.128 ->
//                    STG.128, then flag the row done.
// Index math is 32-bit and incremental (ring rows, slots and mbarrier parities
// are tabulated once per row in parallel): 64-bit div/mod on the producer's
// serial path cost ~19 us per launch before (ncu r1, diag 19).
// ---------------------------------------------------------------------------
constexpr int PL_MAX_ROWS = 256;  // output rows per CTA (host caps rows_per_cta)

// Measurement-only step timeline of the sequence gather (-DRPL_TRACE builds; rpl_debug_gather_trace):
// 0 CTA 0 entry, 1 CTA 0 past its dependency wait, 2 CTA 0's first frame landed
// (its first consumer row's mbarrier), 3 last CTA end (max).
#ifdef RPL_TRACE
__device__ unsigned long long g_gtrace[9];
__device__ unsigned long long g_gend[512];  // per-CTA end of the last launch
__device__ unsigned long long g_gstatic[512];  // dynamic tail: per-CTA time its static rows were stored
__device__ unsigned long long g_gunits[512];   // dynamic tail: per-CTA units taken
__device__ unsigned long long g_ggrab[512][8][2];  // dynamic tail: per-CTA first grabs: time, (rows << 32) | queued
#endif

// Fused sampling's batch reduction (one warp of the CTA that took the last ticket): the batch
// min q over the n samples (every CTA's index / q writes were released with its ticket and
// acquired by this CTA's), the IS weights (a9, R10) and the stream-position advance.
__device__ __noinline__ void smp_finish(const GDesc& D, const int64_t* idx, const int64_t* q, int64_t n, double beta,
                                        uint64_t smp_pos) {
  const int lane = threadIdx.x & 31;
  int64_t m = INT64_MAX;
  for (int64_t j = lane; j < n; j += 32) {
    const int64_t ij = __ldcg(idx + j), qj = __ldcg(q + j);
    if (ij >= 0 && qj < m) m = qj;
  }
  m = warp_min64(m);
  if (D.o_w)
    for (int64_t j = lane; j < n; j += 32) {
      const int64_t qj = __ldcg(q + j);
      D.o_w[j] = qj > 0 ? (float)pow((double)m / (double)qj, beta) : 0.0f;
    }
  if (lane == 0) {
    D.smp_tree[D.smp_L.hdr_off + 1] = 0;
    D.smp_tree[D.smp_L.hdr_off + 2] = (int64_t)(smp_pos + (uint64_t)n);
  }
}
// One warp per CTA, after a barrier that follows the CTA's index / q writes: take the ticket
// (acq_rel releases them, and the last taker acquires everyone's); the last one finishes.
// Taken by the meta warp (or warp 0 of a CTA without rows), so no copy warp waits on it.
__device__ __forceinline__ void smp_ticket_finish(const GDesc& D, const int64_t* idx, const int64_t* q, int64_t n,
                                                  double beta, uint64_t smp_pos) {
  unsigned long long t = 0;
  if ((threadIdx.x & 31) == 0)
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                 : "=l"(t) : "l"(D.smp_tree + D.smp_L.hdr_off + 1) : "memory");
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t == (unsigned long long)gridDim.x - 1) smp_finish(D, idx, q, n, beta, smp_pos);
}

template <int NC>
__global__ void __launch_bounds__((NC + 2) * 32, 1)
k_gather_seq_pipe_lsu(GDesc D, const int64_t* __restrict__ idx, int64_t n, int NS, int64_t rows_per_cta,
                      const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, double beta, int32_t* err,
                      int trig_at) {
  extern __shared__ __align__(128) uint8_t smem[];  // NS frame slots
  __shared__ __align__(8) uint64_t full[PIPE_MAX_NS];
  // per piece p (sample s = s_first + p)
  __shared__ int p_b[PL_MAX_ROWS];     // ring column, -1: skipped sample
  __shared__ int p_row0[PL_MAX_ROWS];  // ring row of the piece's first output row
  __shared__ int p_blk[PL_MAX_ROWS];   // storage block (stored RNN state)
  __shared__ int p_F[PL_MAX_ROWS];     // frame position of the piece's first frame
  // per output row c
  __shared__ int row_new[PL_MAX_ROWS];    // frame position of the row's NEWEST frame (-1: skipped)
  __shared__ int rel[PL_MAX_ROWS];        // frames released once rows <= c are done
  __shared__ int row_ring[PL_MAX_ROWS];   // ring row
  __shared__ short row_piece[PL_MAX_ROWS];
  __shared__ short row_tau[PL_MAX_ROWS];
  __shared__ int8_t start_off[PL_MAX_ROWS];
  __shared__ volatile int row_done[PL_MAX_ROWS];
  // frame positions issued so far (producer, release): a consumer waits on a slot's mbarrier
  // only once the phase it needs is armed, so a parity test can never match a phase two
  // rounds old (a consumer warp may run ahead of another warp's rows)
  __shared__ volatile int s_issued;
  __shared__ int s_npieces;
  __shared__ int64_t p_leaf[PL_MAX_ROWS];  // fused sampling: the piece's sampled leaf
  constexpr int NT = (NC + 2) * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = D.k, L = D.seq_len;
  const int ob = (int)D.obs_bytes;
  const int nv = ob / 16;
  const int cap = (int)D.cap_T, Bc = (int)D.B, period = (int)D.period;
  const int64_t nleaves = (int64_t)(cap / period) * Bc;
  // shared-memory setup that reads no global memory runs before the dependency wait, while
  // the sampler finishes
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  for (int c = tid; c < PL_MAX_ROWS; c += NT) row_done[c] = 0;
  if (tid == 0) s_issued = 0;
  if (trig_at == 0) pdl_trigger();  // A/B knob (rpl_debug_set_gather_trigger; RPL_PDL_EARLY & 4 sets 0)
#ifdef RPL_TRACE
  if (tid == 0 && blockIdx.x == 0) g_gtrace[0] = global_ns();
#endif
  pdl_wait();  // idx (and n_active) come from the sampler launched just before
#ifdef RPL_TRACE
  if (tid == 0 && blockIdx.x == 0) {  // the previous launch is complete: this launch's end slots
    g_gtrace[1] = global_ns();
    g_gtrace[3] = 0;
    g_gtrace[8] = ~0ull;
  }
#endif
  // rows g = s*L + tau of the active samples, split evenly over the grid
  const int total = (int)(active_n(D, n) * L);
  const int64_t coff = col_off(D);  // output column of entry 0 (Mode C)
  const bool unique = D.out_mode == RPL_OUT_UNIQUE;
  const int rpc = D.n_active ? (total + (int)gridDim.x - 1) / (int)gridDim.x : (int)rows_per_cta;
  const int g0 = (int)blockIdx.x * rpc;
  const int g1 = min(total, g0 + rpc);
  // (S) Fused sampling (rpl_gather_sample; the tree was updated by the kernel before).  The
  //     tree's top levels (root .. the deepest level that fits the frame-slot area, which no
  //     TMA load has touched yet) are staged in shared memory with one round of 16-B cp.async,
  //     in flight with the stream-position read, so the root and the upper levels of every
  //     descent cost one L2 round trip.  One warp per piece then descends for the piece's
  //     stratum (a8; the same strata and Philox stream as rpl_sumtree_sample_stream); the CTA
  //     owning a sample's first row writes its index and q.  Every CTA then takes a ticket
  //     (acq_rel: its index / q writes are released with it); the LAST one computes the
  //     batch-min IS weights (a9) and advances the stream position — in its meta warp, while
  //     its consumer warps stream frames, so no CTA's copy waits for the batch reduction.
  const bool smp = D.smp_tree != nullptr;
  uint64_t smp_pos = 0;
  const DivN smp_dn = divn_make(smp ? (uint64_t)n : 1ull);  // before any global read: n alone
  if (smp) {
    const int64_t* top = reinterpret_cast<const int64_t*>(smem);
    int64_t ntop = 0;
    const int64_t cap_words = (int64_t)NS * ob / 8;
    for (int l = 0; l <= D.smp_L.depth; ++l) {
      const int64_t end = l < D.smp_L.depth ? D.smp_L.level_off[l + 1] : D.smp_L.hdr_off;
      if (end > cap_words) break;
      ntop = end;
    }
    for (int64_t j = 2 * (int64_t)tid; j < ntop; j += 2 * NT)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem + j * 8)), "l"(D.smp_tree + j)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    smp_pos = (uint64_t)__ldcg(D.smp_tree + D.smp_L.hdr_off + 2);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#ifdef RPL_TRACE
    if (tid == 0 && blockIdx.x == 0) g_gtrace[4] = global_ns();
#endif
    const uint64_t smp_Q = (uint64_t)(ntop > 0 ? top[0] : __ldcg(D.smp_tree + D.smp_L.level_off[0]));
    const Strata smp_st = strata_make(smp_Q, smp_dn);
    if (g0 < g1) {
      const int s_first = g0 / L;
      const int npieces = (g1 - 1) / L - s_first + 1;
      int32_t eb = 0;
      for (int pc = warp; pc < npieces; pc += NT / 32) {
        const int sm = s_first + pc;
        int64_t leaf = -1, qv = 0;
        if (smp_Q == 0) {
          eb |= RPL_DERR_EMPTY;
        } else {
          const uint64_t prefix = strata_prefix(sm, smp_st, nullptr, D.smp_seed, smp_pos);
          leaf = descend(D.smp_L, D.smp_tree, (int64_t)prefix, &qv, &eb, top, ntop);
        }
        if (lane == 0) {
          p_leaf[pc] = leaf;
          if (sm * L >= g0) {
            const_cast<int64_t*>(idx)[sm] = leaf;
            const_cast<int64_t*>(q)[sm] = qv;
          }
        }
      }
      if (lane == 0 && eb) set_err(err, eb);
    }
    fence_proxy_async();  // the staged words were read through the generic proxy; TMA refills them
    __syncthreads();
#ifdef RPL_TRACE
    if (tid == 0 && blockIdx.x == 0) g_gtrace[5] = global_ns();
#endif
    if (g0 >= g1 && warp == 0) smp_ticket_finish(D, idx, q, n, beta, smp_pos);  // no rows: take the ticket now
  }
  // K7 fused (peer boards): the step's tag comes from this rank's own board (its sampler's
  // K5 slot); CTA 0 publishes this rank's batch-min q over its owned entries to every rank
  // — before any early exit, so a rank that owns nothing still publishes (INT64_MAX)
  const bool peer = D.peer_boards != nullptr && D.o_w != nullptr && q != nullptr;
  uint64_t ptag = 0;
  if (peer) {
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];"
                 : "=l"(ptag) : "l"(D.peer_boards[D.peer_rank] + 2 * D.peer_rank + 1) : "memory");
    if (blockIdx.x == 0 && warp == 1) {
      const int64_t qm_local = warp_batch_qmin(nullptr, idx, q, n);
      if (lane < D.peer_world)
        board_publish(D.peer_boards[lane] + 2 * D.peer_world + 2 * D.peer_rank, qm_local, ptag);
    }
  }
  do {  // (break = this CTA has no rows; the completion epilogue below still runs)
  if (g0 >= g1) break;
  const int nrows = g1 - g0;
  const int s_first = g0 / L;
  const int npieces = (g1 - 1) / L - s_first + 1;

  if (tid == 0) s_npieces = npieces;
  // (A) pieces, in parallel: one sampled leaf each
  for (int pc = tid; pc < npieces; pc += NT) {
    const int sm = s_first + pc;
    const int tau0 = max(g0 - sm * L, 0);
    const int64_t leaf = smp ? p_leaf[pc] : idx[sm];
    int bcol = -1, row0 = 0, blk = 0;
    if (leaf >= 0 && leaf < nleaves) {
      if (nleaves < (1ll << 31)) {  // 32-bit division (every value below fits)
        blk = (int)((uint32_t)leaf / (uint32_t)Bc);
        bcol = (int)leaf - blk * Bc;
        row0 = (int)((uint32_t)(blk * period + tau0) % (uint32_t)cap);
      } else {
        blk = (int)(leaf / Bc);
        bcol = (int)(leaf - (int64_t)blk * Bc);
        row0 = (int)(((int64_t)blk * period + tau0) % cap);
      }
      if (tau0 == 0) {
        // cursor, blk * period < cap_T < 2^30 (host-checked): 32-bit modulo
        int age = ((int)D.cursor - 1 - blk * period) % cap;
        if (age < 0) age += cap;
        const int hist = k - 1 > 1 ? k - 1 : 1;
        if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
      }
    } else if (leaf >= nleaves && tau0 == 0) {
      set_err(err, RPL_DERR_IDX);
    }
    p_b[pc] = bcol;
    p_row0[pc] = row0;
    p_blk[pc] = blk;
  }
  __syncthreads();
#ifdef RPL_TRACE
  if (tid == 0 && blockIdx.x == 0) g_gtrace[7] = global_ns();
#endif
  // (B) frame positions: exclusive scan over pieces (serial: a CTA holds one to a few pieces).
  //     A piece loads window rows tau0-(k-1) .. tau0+R-1, except in RPL_OUT_UNIQUE mode when it
  //     starts mid-sample (tau0 > 0, only a CTA's first piece): its rows store only their newest
  //     frame, so the k-1 history rows are not loaded (`skip`).
  const int skip0 = (unique && g0 > s_first * L) ? k - 1 : 0;
  if (tid == 0) {
    int F = 0;
    for (int pc = 0; pc < npieces; ++pc) {
      p_F[pc] = F;
      if (p_b[pc] >= 0) {
        const int sm = s_first + pc;
        const int R = min(g1, (sm + 1) * L) - max(g0, sm * L);
        F += R + k - 1 - (pc == 0 ? skip0 : 0);
      }
    }
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: TMA loads only ----------------
      int frontier = 0;  // rows [0, frontier) are done
      int released = 0;  // frames < released may be overwritten
      int i = 0, slot = 0;
      for (int pc = 0; pc < npieces; ++pc) {
        const int bcol = p_b[pc];
        if (bcol < 0) continue;
        const int sm = s_first + pc;
        const int R = min(g1, (sm + 1) * L) - max(g0, sm * L);
        const int skip = pc == 0 ? skip0 : 0;
        int row = p_row0[pc] - (k - 1) + skip;
        while (row < 0) row += cap;
        const uint8_t* col = D.obs + (int64_t)bcol * ob;
        const int64_t rstride = (int64_t)Bc * ob;
        for (int w = skip; w < R + k - 1; ++w, ++i) {
          if (i >= NS) {
            while (released <= i - NS) {
              if (frontier < nrows && flag_acquire(&row_done[frontier])) {
                released = rel[frontier];
                ++frontier;
              } else {
                __nanosleep(20);
              }
            }
            fence_proxy_async();
            // the slot's previous phase completed before its readers finished: observe it, so
            // every arrive on a barrier follows the completion of its previous phase
            if (!(GDIAG(D) & 2)) mbar_wait(&full[slot], (uint32_t)(((i / NS) - 1) & 1));
          }
          if (!(GDIAG(D) & 2)) {
#ifdef RPL_TRACE
            if (i == 0 && blockIdx.x == 0) g_gtrace[6] = global_ns();
#endif
            mbar_expect_tx(&full[slot], (uint32_t)ob);
            const uint8_t* src = col + (int64_t)row * rstride;
            // frames are streamed once: evict-first keeps the L2 for the sum tree and the
            // small per-row fields (measured: step 74.6 -> 69.8 us with the stores below)
            if (GDIAG(D) & 8) bulk_g2s(smem + slot * ob, src, (uint32_t)ob, &full[slot]);
            else bulk_g2s_evict_first(smem + slot * ob, src, (uint32_t)ob, &full[slot]);
          }
          flag_release(&s_issued, i + 1);
          if (++row == cap) row = 0;
          if (++slot == NS) slot = 0;
        }
      }
      // knob 1: the dependent grid may launch once every CTA's producer has issued its last load
      if (trig_at == 1) pdl_trigger();
      // tail: observe the last phase of every armed slot, so the CTA never exits with bulk
      // copies into its shared memory in flight (also frames no row reads)
      if (!(GDIAG(D) & 2))
        for (int p = i > NS ? i - NS : 0; p < i; ++p) mbar_wait(&full[p % NS], (uint32_t)((p / NS) & 1));
    }
  } else {
    // (C) row tables + episode-start offsets, rows spread over warps 1..NC+1; the
    //     k-1 done flags of a row are loaded together before any is inspected.
    for (int c = tid - 32; c < nrows; c += NT - 32) {
      const int g = g0 + c;
      const int sm = g / L;
      const int tau = g - sm * L;
      const int pc = sm - s_first;
      const int bcol = p_b[pc];
      const int m = g - max(g0, sm * L);
      int8_t so = 0;
      int ring = 0;
      if (bcol >= 0) {
        const int R = min(g1, (sm + 1) * L) - max(g0, sm * L);
        const int skip = pc == 0 ? skip0 : 0;
        const int F = p_F[pc];
        const int nw = F + m + (k - 1) - skip;  // window row m+k-1 (the row's newest frame)
        row_new[c] = nw;
        // stacked: the row's oldest frame is no longer needed; unique: each row reads only its
        // newest frame (and the sample's first row its history too); end of piece: all of it
        rel[c] = m == R - 1 ? F + R + k - 1 - skip : (unique ? nw + 1 : nw - (k - 1) + 1);
        ring = p_row0[pc] + m;
        if (ring >= cap) ring -= cap;
        uint8_t dw[8];
#pragma unroll
        for (int j = 1; j < 8; ++j) {
          int rr = ring - k + j;  // done flag of window row j-1 = ring row (ring - (k-1) + j - 1)
          while (rr < 0) rr += cap;
          dw[j] = j < k ? __ldg(D.done + (int64_t)rr * Bc + bcol) : (uint8_t)0;
        }
#pragma unroll
        for (int j = 1; j < 8; ++j)
          if (dw[j]) so = (int8_t)j;  // latest episode start in the window wins
      } else {
        row_new[c] = -1;
        rel[c] = p_F[pc];
      }
      row_ring[c] = ring;
      row_piece[c] = (short)pc;
      row_tau[c] = (short)tau;
      start_off[c] = so;
    }
    asm volatile("bar.sync 1, %0;" ::"n"((NC + 1) * 32) : "memory");

    if (warp == 1) {
      // ---------------- meta warp: per-row fields, IS weights ----------------
      if (smp) smp_ticket_finish(D, idx, q, n, beta, smp_pos);  // fused sampling's ticket / batch reduction
      const int64_t qm = (D.o_w && q && !peer && !smp) ? warp_batch_qmin(qmin, idx, q, n) : 0;
      const int64_t ab = D.act_bytes;
      const bool a8 = ab == 8 && ((reinterpret_cast<uintptr_t>(D.act) | reinterpret_cast<uintptr_t>(D.o_act) |
                                   reinterpret_cast<uintptr_t>(D.o_prev_act)) & 7) == 0;
      for (int c = lane; c < nrows && !(GDIAG(D) & 16); c += 32) {
        if (row_new[c] < 0) continue;
        const int pc = row_piece[c];
        const int sm = s_first + pc;
        const int tau = row_tau[c];
        const int bcol = p_b[pc];
        const int ring = row_ring[c];
        const int prow = ring == 0 ? cap - 1 : ring - 1;
        const int64_t e = (int64_t)ring * Bc + bcol, pe = (int64_t)prow * Bc + bcol;
        const uint8_t pd = __ldg(D.done + pe);
        const uint8_t dd = __ldg(D.done + e);
        const float rw = D.o_rew ? __ldg(D.rew + e) : 0.0f;
        const float prw = D.o_prev_rew ? __ldg(D.rew + pe) : 0.0f;
        const int64_t o = (int64_t)tau * n + coff + sm;
        if (a8) {
          const uint64_t* a = reinterpret_cast<const uint64_t*>(D.act);
          const uint64_t av = D.o_act ? __ldg(a + e) : 0ull;
          const uint64_t pav = D.o_prev_act ? __ldg(a + pe) : 0ull;
          if (D.o_act) reinterpret_cast<uint64_t*>(D.o_act)[o] = av;
          if (D.o_prev_act) reinterpret_cast<uint64_t*>(D.o_prev_act)[o] = pd ? 0ull : pav;
        } else {
          if (D.o_act) coop_copy(D.o_act + o * ab, D.act + e * ab, ab, 0, 1);
          if (D.o_prev_act) {
            if (pd) coop_zero(D.o_prev_act + o * ab, ab, 0, 1);
            else coop_copy(D.o_prev_act + o * ab, D.act + pe * ab, ab, 0, 1);
          }
        }
        if (D.o_rew) D.o_rew[o] = rw;
        if (D.o_prev_rew) D.o_prev_rew[o] = pd ? 0.0f : prw;
        if (D.o_done) D.o_done[o] = dd;
        if (D.o_start) D.o_start[o] = start_off[c];
        if (tau == 0 && D.o_w && q && !peer && !smp) {
          const int64_t qs = q[sm];
          D.o_w[coff + sm] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
        }
      }
      // fused n-step targets (a2 + a4, R5 / R24 / R34) for the target rows in this CTA:
      // rows tau .. tau+n_step-1 straight from the ring, bootstrap q_tgt[tau + n_step]
      if (D.o_tgt) {
        const int ns = D.n_step;
        for (int c = lane; c < nrows; c += 32) {
          if (row_new[c] < 0) continue;
          const int t = row_tau[c] - D.tgt_lo;
          if (t < 0 || t >= D.tgt_T) continue;
          const int64_t col = coff + s_first + row_piece[c];
          double acc = 0.0;
          if (D.q_tgt) {
            const double qv = (double)__ldg(D.q_tgt + (int64_t)(row_tau[c] + ns) * n + col);
            acc = D.rescale ? h_inv(qv, D.rescale_eps) : qv;
          }
          uint8_t dn = 0;
          acc = nstep_rows(D, row_ring[c], p_b[row_piece[c]], ns, acc, &dn);
          if (D.rescale) acc = h_fwd(acc, D.rescale_eps);
          D.o_tgt[(int64_t)t * n + col] = (float)acc;
          if (D.o_tgt_done) D.o_tgt_done[(int64_t)t * n + col] = dn ? 1 : 0;
        }
      }
      if (peer) {  // global batch min over every rank's published value, then the IS weights
        int64_t v = INT64_MAX;
        if (lane < D.peer_world &&
            !board_wait(D.peer_boards[D.peer_rank] + 2 * D.peer_world + 2 * lane, ptag, &v)) {
          board_fail(err);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const int64_t x = (int64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
          v = x < v ? x : v;
        }
        for (int c = lane; c < nrows; c += 32) {
          if (row_new[c] < 0 || row_tau[c] != 0) continue;
          const int sm = s_first + row_piece[c];
          const int64_t qs = q[sm];
          D.o_w[coff + sm] = qs > 0 ? (float)pow((double)v / (double)qs, beta) : 0.0f;
        }
      }
      // stored recurrent state of every sample whose first row lives here
      if (D.o_rnn && !(GDIAG(D) & 16)) {
        const int nparts = D.rnn_parts;
        const int64_t rb = D.rnn_bytes;
        for (int pc = 0; pc < npieces; ++pc) {
          const int sm = s_first + pc;
          if (sm * L < g0 || p_b[pc] < 0) continue;  // first row not in this CTA, or skipped
          const int64_t blk = p_blk[pc], bcol = p_b[pc];
          for (int pp = 0; pp < nparts; ++pp)
            coop_copy(D.o_rnn + (pp * n + coff + sm) * rb, D.rnn + ((blk * Bc + bcol) * nparts + pp) * rb, rb, lane, 32);
        }
      }
    } else {
      // ---------------- consumers: one k-stack per row, LSU stores ----------------
      for (int c = warp - 2; c < nrows; c += NC) {
        const int pn = row_new[c];
        // slot / mbarrier parity of window index j (position pn - (k-1) + j)
        const int sn = pn % NS;
        const uint32_t parn = (uint32_t)((pn / NS) & 1);
        auto slot_of = [&](int j, uint32_t* par) {
          int sl = sn - (k - 1 - j);
          *par = parn;
          if (sl < 0) {
            sl += NS;
            *par ^= 1u;
          }
          return sl;
        };
        if (pn >= 0)  // every frame this row reads (positions <= pn) has its phase armed
          while (flag_acquire(&s_issued) <= pn) __nanosleep(20);
        if (pn >= 0 && unique) {
          // RPL_OUT_UNIQUE: raw rows, each written once — row tau stores its newest frame
          // (unique row tau+k-1); the sample's first row also stores unique rows 0..k-2
          const int sm = s_first + row_piece[c];
          const int tau = row_tau[c];
          for (int j = tau == 0 ? 0 : k - 1; j < k; ++j) {
            uint32_t par;
            const int sl = slot_of(j, &par);
            if (!(GDIAG(D) & 2)) mbar_wait(&full[sl], par);
            if (GDIAG(D) & 1) continue;
            int4* d = reinterpret_cast<int4*>(D.o_obs + ((int64_t)(tau + j) * n + coff + sm) * ob);
            const int4* sp = reinterpret_cast<const int4*>(smem + sl * ob);
#pragma unroll 4
            for (int v = lane; v < nv; v += 32) __stcs(d + v, sp[v]);
          }
        } else if (pn >= 0) {
          const int so = start_off[c];
          const int sm = s_first + row_piece[c];
          const int tau = row_tau[c];
          if (!(GDIAG(D) & 2))
            for (int j = so; j < k; ++j) {
              uint32_t par;
              const int sl = slot_of(j, &par);
              mbar_wait(&full[sl], par);
            }
#ifdef RPL_TRACE
          if (c == 0 && lane == 0 && blockIdx.x == 0) g_gtrace[2] = global_ns();
#endif
          int4* dst = reinterpret_cast<int4*>(D.o_obs + ((int64_t)tau * n + coff + sm) * k * ob);
          if (!(GDIAG(D) & 1))
            for (int j = 0; j < k; ++j) {
              int4* d = dst + j * nv;
              if (j < so && D.pad_mode == RPL_PAD_ZERO) {
                for (int v = lane; v < nv; v += 32) d[v] = make_int4(0, 0, 0, 0);
              } else {
                uint32_t par;
                const int sl = slot_of(j < so ? so : j, &par);
                const int4* sp = reinterpret_cast<const int4*>(smem + sl * ob);
                if (GDIAG(D) & 4) {
#pragma unroll 4
                  for (int v = lane; v < nv; v += 32) d[v] = sp[v];
                } else {  // streaming (evict-first) stores
#pragma unroll 4
                  for (int v = lane; v < nv; v += 32) __stcs(d + v, sp[v]);
                }
              }
            }
        }
        __syncwarp();
        if (lane == 0) {
          fence_proxy_async();
          flag_release(&row_done[c], 1);
        }
      }
    }
  }
  } while (0);
  // Completion signal (rpl_gather_desc.done_flag, Mode C): every CTA publishes its stores at
  // system scope and takes a ticket; the last CTA bumps the call counter done_seq[0] and
  // writes it to done_flag with st.release.sys (peer memory over NVLink), so the learner's
  // rpl_wait_flags observes the whole batch without any collective.
  if (D.done_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned t = atomicAdd(reinterpret_cast<unsigned*>(D.done_seq + 1), 1u);
      if (t == gridDim.x - 1) {
        __threadfence_system();
        D.done_seq[1] = 0;
        const int64_t sq = D.done_seq[0] + 1;
        D.done_seq[0] = sq;
        asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(D.done_flag), "l"(sq) : "memory");
      }
    }
  }
#ifdef RPL_TRACE
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMax(&g_gtrace[3], t);
    atomicMin(&g_gtrace[8], t);
    if (blockIdx.x < 512) g_gend[blockIdx.x] = t;
  }
#endif
  pdl_trigger();
}
// Measurement knob: where the sequence gather lets its dependent grid launch (-1 at exit,
// 0 at entry, 1 once the CTA's producer has issued its last load); rpl_debug_set_gather_trigger.
std::atomic<int> g_gather_trigger{(RPL_PDL_EARLY & 4) ? 0 : -1};
// Dynamic-tail sequence gather (k_gather_seq_dyn): the static share of the rows (percent of
// an even split, 0 = every row dynamic; -1 = the static kernel), the rows per dynamic unit, and the look-ahead (rows
// published but not yet stored below which the meta warp grabs the next unit).
// rpl_debug_set_gather_dyn.
// in-process sweeps (scripts/ab_dyn_sweep.py, profiles/r2/dyn_sweep.txt): 88 / 16 / 12 until the
// default gather got its own instantiation; since then 80 / 16 / 16 (-1.0 us per R2D2 step; the
// in-process harness then preferred 78 % by 0.27 us, bench.py itself 80 % by 0.2 us)
std::atomic<int> g_dyn_pct{80};
std::atomic<int> g_dyn_rows{16};
std::atomic<int> g_dyn_look{16};
// fused sampling: warp 0 issues up to this many of piece 0's first frame loads right after its
// descent (0: the producer starts once every table is built); rpl_debug_set_gather_dyn's
// pct = 1000 + count sets it (measured neutral at 2-8 and +1.5 us at 28 with the shared
// instantiation; with the default gather's own instantiation and the 80 / 16 / 16 schedule 10
// is -0.4 us per R2D2 step: profiles/r2/dyn_sweep.txt)
std::atomic<int> g_dyn_early{10};
// measurement: 1 = every dynamic-tail launch takes the fused-update instantiation (the
// default gather's code before it had its own); rpl_debug_set_gather_dyn's pct = 2000 + on
std::atomic<int> g_dyn_updk{0};  // measured neutral at 2-8 and +1.5 us at 28 (profiles/r2/dyn_sweep.txt)

template <int NC>
int launch_seq_lsu(const GDesc& g, const int64_t* idx, int64_t n, int NS, int64_t rows_per_cta, const int64_t* q,
                   const int64_t* qmin, double beta, int32_t* dev_err, size_t dyn, int64_t grid, cudaStream_t st) {
  ensure_smem(reinterpret_cast<const void*>(k_gather_seq_pipe_lsu<NC>), dyn);
  return launch_pdl(k_gather_seq_pipe_lsu<NC>, dim3((unsigned)grid), dim3((NC + 2) * 32), dyn, st, g, idx, n, NS,
                    rows_per_cta, q, qmin, beta, dev_err, g_gather_trigger.load(std::memory_order_relaxed));
}

// ---------------------------------------------------------------------------
// Sequences with a DYNAMIC TAIL (default when rpl_gather_desc.work is given and the call is a
// single learner's batch: no col_offset / n_active / peer boards / completion flag / fused
// sampling).  Same pipeline and roles as k_gather_seq_pipe_lsu, but the rows are not all split
// statically: measured with the step timeline (-DRPL_TRACE, scripts/step_trace.py), the 146
// CTAs of the static split finish between 44 and 63 us for the same 55 rows — the SMs do not
// all see the same memory throughput — so the launch ended ~8 us after its median CTA.  Here
// CTA c takes the static rows [c*rs, (c+1)*rs) (rs = a fraction of the even share) and the
// remaining rows are handed out at run time through an atomic row counter (work[0]), GUIDED:
// a grab takes ~1/(2 grid) of the rows still left, between 2 and `dyn_rows`, so the early
// grabs are long and the last ones short.  The meta warp grabs when fewer than `lookahead` of
// the CTA's published rows are not yet stored, publishes the grab's pieces and row tables
// (the producer and the consumers pick them up through release/acquire counters), then
// writes their per-row fields.  A piece that starts mid-sample reloads its k-1 history frames.
// The last CTA to leave (ticket work[1]) re-zeroes the counters.
// ---------------------------------------------------------------------------
constexpr int DY_MAX_ROWS = 256;
constexpr int DY_MAX_PIECES = 96;

// Fused update (rpl_gather_update_sample): the new q of the batch's winning leaves, looked up
// by leaf in a per-CTA open-addressing table.
constexpr int UF_MAX = 128;   // update entries per call
constexpr int UF_SLOTS = 256;  // table slots (>= 2 UF_MAX, a power of two)
__device__ __forceinline__ int uf_slot(int64_t leaf) {
  return (int)(((unsigned long long)leaf * 0x9E3779B97F4A7C15ull) >> 56) & (UF_SLOTS - 1);
}
// descend() with every internal level staged in shared memory (already carrying the update's
// deltas) and the leaf level read from global memory with the update's new values overlaid
__device__ __forceinline__ int64_t descend_overlay(const TreeDev& L, const int64_t* __restrict__ tree, int64_t prefix,
                                                   int64_t* q_out, int32_t* errbits, const int64_t* top,
                                                   const unsigned long long* ukey, const long long* uval) {
  const int lane = threadIdx.x & 31;
  int64_t node = 0;
  int64_t c = 0;
  for (int l = 0; l < L.depth; ++l) {
    const int64_t base = L.level_off[l + 1] + (node << L.log2w);
    if (lane < L.fanout) {
      if (l + 1 < L.depth) {
        c = top[base + lane];
      } else {
        const int64_t leaf = (node << L.log2w) + lane;
        c = tree[base + lane];
        int sl = uf_slot(leaf);
        while (ukey[sl] != ~0ull) {
          if (ukey[sl] == (unsigned long long)leaf) {
            c = uval[sl];
            break;
          }
          sl = (sl + 1) & (UF_SLOTS - 1);
        }
      }
    } else {
      c = 0;
    }
    int64_t incl = c;
#pragma unroll
    for (int dlt = 1; dlt < 32; dlt <<= 1) {
      const int64_t o = shfl_up64(incl, dlt);
      if (lane >= dlt) incl += o;
    }
    unsigned bal = __ballot_sync(0xffffffffu, prefix < incl);
    int f;
    if (bal == 0) {
      *errbits |= RPL_DERR_TREE;
      const unsigned nz = __ballot_sync(0xffffffffu, c > 0);
      f = nz ? 31 - __clz(nz) : 0;
      const int64_t inc_last = shfl64(incl, f);
      prefix = nz ? inc_last - 1 : 0;
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

template <int NC, bool UPD>
__global__ void __launch_bounds__((NC + 3) * 32, 1)
k_gather_seq_dyn(GDesc D, const int64_t* __restrict__ idx, int64_t n, int NS, int rs, int dyn_rows,
                 int lookahead, const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, double beta,
                 int32_t* err, int trig_at, int early_frames) {
  extern __shared__ __align__(128) uint8_t smem[];  // NS frame slots
  __shared__ __align__(8) uint64_t full[PIPE_MAX_NS];
  // per piece (a run of rows of one sample)
  __shared__ int p_s[DY_MAX_PIECES];        // sample (batch position)
  __shared__ int p_b[DY_MAX_PIECES];        // ring column, -1: skipped sample
  __shared__ int p_row0[DY_MAX_PIECES];     // ring row of the piece's first output row
  __shared__ int p_blk[DY_MAX_PIECES];      // storage block (stored RNN state)
  __shared__ int p_F[DY_MAX_PIECES];        // frame position of the piece's first loaded frame
  __shared__ short p_tau0[DY_MAX_PIECES];   // tau of the piece's first row
  __shared__ short p_R[DY_MAX_PIECES];      // rows
  __shared__ int8_t p_skip[DY_MAX_PIECES];  // leading history frames not loaded (unique mode)
  // per output row c
  __shared__ int row_new[DY_MAX_ROWS];  // frame position of the row's NEWEST frame (-1: skipped)
  __shared__ int rel[DY_MAX_ROWS];      // frames released once rows <= c are done
  __shared__ int row_ring[DY_MAX_ROWS];
  __shared__ short row_piece[DY_MAX_ROWS];
  __shared__ short row_tau[DY_MAX_ROWS];
  __shared__ int8_t start_off[DY_MAX_ROWS];
  __shared__ volatile int row_done[DY_MAX_ROWS];
  __shared__ volatile int s_issued;      // frame positions issued (producer, release)
  __shared__ volatile int s_pieces_pub;  // pieces whose tables are complete (release)
  __shared__ volatile int s_rows_pub;    // rows whose tables are complete (release)
  __shared__ volatile int s_frontier;    // rows [0, s_frontier) stored (producer's view)
  __shared__ volatile int s_more;        // 0 once no further piece will be published
  constexpr int NT = (NC + 3) * 32;  // producer, meta, fields, NC consumers
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = D.k, L = D.seq_len;
  const int ob = (int)D.obs_bytes;
  const int nv = ob / 16;
  const int cap = (int)D.cap_T, Bc = (int)D.B, period = (int)D.period;
  const int64_t nleaves = (int64_t)(cap / period) * Bc;
  const bool unique = D.out_mode == RPL_OUT_UNIQUE;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
    s_issued = 0;
    s_frontier = 0;
    s_more = 1;
  }
  for (int c = tid; c < DY_MAX_ROWS; c += NT) row_done[c] = 0;
  if (trig_at == 0) pdl_trigger();
#ifdef RPL_TRACE
  if (tid == 0 && blockIdx.x == 0) g_gtrace[0] = global_ns();
  if (tid == 0) atomicMin(&g_gtrace[4], (unsigned long long)global_ns());  // earliest CTA entry
#endif
  // one warp waits for the previous grid (a grid launched early by PDL sits here; the other
  // warps wait at the CTA barrier, which orders their reads after the wait)
  if (warp == 0) pdl_wait();  // idx / q come from the kernel launched just before
  __syncthreads();
#ifdef RPL_TRACE
  if (tid == 0 && blockIdx.x == 0) {
    g_gtrace[1] = global_ns();
    g_gtrace[3] = 0;
    g_gtrace[8] = ~0ull;
  }
  if (tid == 0) {
    atomicMin(&g_gtrace[5], (unsigned long long)global_ns());  // earliest past the wait
    atomicMax(&g_gtrace[6], (unsigned long long)global_ns());  // latest past the wait
  }
#endif
  const int total = (int)(n * L);
  const int g0 = min(total, (int)blockIdx.x * rs);
  const int g1 = min(total, g0 + rs);
  // dynamic units over rows [gridDim.x * rs, total): a partial first sample, then whole samples
  const int r0 = min(total, (int)gridDim.x * rs);
  const int su0 = r0 / L, tu0 = r0 - su0 * L;
  const int sfull = su0 + (tu0 > 0 ? 1 : 0);  // the first wholly dynamic sample
  const int s_first = g0 / L;
  const int np0 = g1 > g0 ? (g1 - 1) / L - s_first + 1 : 0;
  // (S) fused sampling (rpl_gather_sample), as in k_gather_seq_pipe_lsu: top levels staged in
  //     the frame-slot area, one warp per static piece descends; CTA c also descends the
  //     wholly dynamic samples sfull + c + j * grid (their units may run on any CTA: they read the index from
  //     global memory once every CTA has counted itself into work[2]).  Each sample's index /
  //     q is written once (its first row's static owner, or its assigned CTA); the ticket /
  //     batch-min weights / stream advance follow in the meta warp.
  const bool smp = D.smp_tree != nullptr;
  __shared__ int64_t p_leaf[DY_MAX_PIECES];
  // the fused update's tables (UPD: the rpl_gather_update_sample instantiation only)
  constexpr int UFM = UPD ? UF_MAX : 1, UFS = UPD ? UF_SLOTS : 1;
  __shared__ int64_t u_leaf[UFM], u_old[UFM], u_q[UFM];
  __shared__ float u_td[UFM];
  __shared__ int8_t u_win[UFM];
  __shared__ unsigned long long uf_key[UFS];
  __shared__ long long uf_val[UFS];
  __shared__ int uf_pos[UFS];
  __shared__ int s_pre;  // frames of piece 0 issued by warp 0 right after its descent
  if (tid == 0) s_pre = 0;
  uint64_t smp_pos = 0;
  const DivN smp_dn = divn_make(smp ? (uint64_t)n : 1ull);
  if (smp) {
    // the top levels are staged at the END of the frame-slot area, so warp 0 can start piece
    // 0's frame loads into the first slots while the other warps still descend
    int64_t ntop = 0;
    const int64_t cap_words = (int64_t)(NS - 1) * ob / 8;
    for (int l = 0; l <= D.smp_L.depth; ++l) {
      const int64_t end = l < D.smp_L.depth ? D.smp_L.level_off[l + 1] : D.smp_L.hdr_off;
      if (end > cap_words) break;
      ntop = end;
    }
    const int64_t top_off = (((int64_t)NS * ob - ntop * 8) / 128) * 128;  // 128-B aligned
    const int pre_cap = (int)(top_off / ob);                                // slots wholly below it
    const int64_t* top = reinterpret_cast<const int64_t*>(smem + top_off);
    for (int64_t j = 2 * (int64_t)tid; j < ntop; j += 2 * NT)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem + top_off + j * 8)),
                   "l"(D.smp_tree + j) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    smp_pos = (uint64_t)__ldcg(D.smp_tree + D.smp_L.hdr_off + 2);
    // (U) fused priority update (rpl_gather_update_sample, a5-a7 + R26): every CTA computes the
    //     batch's sequence priorities, winners and deltas itself, applies the deltas to its
    //     staged copy of the internal levels and overlays the winners' new q on the leaf level
    //     it reads — so it samples the UPDATED tree without waiting for anyone; CTA 0 writes
    //     the update to global memory once every CTA has finished reading the old tree
    //     (work[3] counts the readers).  Same tree and draws as rpl_sumtree_update_seq
    //     followed by rpl_gather_sample.
    const bool upd = UPD && D.upd_td != nullptr;
    const int nu = upd ? D.upd_n : 0;
    if (upd) {
      for (int s2 = tid; s2 < UF_SLOTS; s2 += NT) {
        uf_key[s2] = ~0ull;
        uf_pos[s2] = -1;
      }
      if (tid < nu) {
        int64_t lf = D.upd_idx[tid];
        if (lf < 0 || lf >= nleaves) lf = -1;
        u_leaf[tid] = lf;
        u_old[tid] = lf >= 0 ? __ldcg(D.smp_tree + D.smp_L.level_off[D.smp_L.depth] + lf) : 0;
      }
      // sequence priorities: UG lanes per sequence, NT / UG sequences per pass (56: a 64-entry
      // batch in two passes, where eight lanes took three); the next pass's loads are in flight
      // while this pass reduces
      constexpr int UG = 4, UB = 20;
      float va[UB], vb[UB];
      sequence_tdg_load<UG, UB>(va, D.upd_td, D.upd_T, nu, tid / UG, (tid / UG) < nu);
      for (int p0 = 0; p0 < nu; p0 += NT / UG) {
        const int jj = p0 + tid / UG, jn = jj + NT / UG;
        if (p0 + NT / UG < nu) sequence_tdg_load<UG, UB>(vb, D.upd_td, D.upd_T, nu, jn, jn < nu);
        const float v = sequence_tdg_finish<UG, UB>(va, D.upd_td, D.upd_T, nu, jj, jj < nu, D.upd_eta);
        if ((tid & (UG - 1)) == 0 && jj < nu) u_td[jj] = v;
#pragma unroll
        for (int u2 = 0; u2 < UB; ++u2) va[u2] = vb[u2];
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#ifdef RPL_TRACE
    if (tid == 0 && blockIdx.x == 0) g_gtrace[2] = global_ns();  // staged (+ the update's priorities)
#endif
    if (upd) {
      // winners (the batch's last position of each leaf: a hash of the indices keeps the
      // largest position), new q, deltas
      int64_t* topw = reinterpret_cast<int64_t*>(smem + top_off);
      int usl = -1;
      if (tid < nu && u_leaf[tid] >= 0) {
        const int64_t lf = u_leaf[tid];
        usl = uf_slot(lf);
        while (true) {
          const unsigned long long prev = atomicCAS(&uf_key[usl], ~0ull, (unsigned long long)lf);
          if (prev == ~0ull || prev == (unsigned long long)lf) break;
          usl = (usl + 1) & (UF_SLOTS - 1);
        }
        atomicMax(&uf_pos[usl], tid);
      }
      __syncthreads();
      int64_t root_delta = 0;
      if (tid < nu) {
        const int64_t lf = u_leaf[tid];
        bool win = lf >= 0 && uf_pos[usl] == tid;
        int64_t q = 0;
        if (lf >= 0) {
          const double p = (double)fabsf(u_td[tid]) + D.upd_eps;
          float v;
          if (!isfinite(p)) {
            v = __int_as_float(0x7f800000);
          } else {
            bool slow = false;
            v = cr_powf(p, D.upd_alpha, false, &slow);
          }
          bool sat = false;
          q = quantise_q(v, D.smp_L.frac_bits, D.smp_L.q_cap, &sat);
          if (D.upd_live && u_old[tid] == 0) win = false;  // R30: a zero leaf is left alone
        }
        u_win[tid] = win ? 1 : 0;
        u_q[tid] = q;
        // the leaf's value after the update, written once per leaf by its last batch position
        if (lf >= 0 && uf_pos[usl] == tid) uf_val[usl] = (long long)(win ? q : u_old[tid]);
        if (win) {
          const int64_t delta = q - u_old[tid];
          root_delta = delta;
          if (delta != 0) {  // levels below the root: few entries per node
            int64_t node = lf;
            for (int l = D.smp_L.depth - 1; l >= 1; --l) {
              node >>= D.smp_L.log2w;
              atomicAdd(reinterpret_cast<unsigned long long*>(topw + D.smp_L.level_off[l] + node),
                        (unsigned long long)delta);
            }
          }
        }
      }
      // the root takes every delta: a warp sum, then one shared add per warp
      root_delta = warp_sum64(root_delta);
      if (lane == 0 && root_delta != 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(topw + D.smp_L.level_off[0]), (unsigned long long)root_delta);
      __syncthreads();
    }
    const uint64_t smp_Q = (uint64_t)(ntop > 0 ? top[0] : __ldcg(D.smp_tree + D.smp_L.level_off[0]));
    const Strata smp_st = strata_make(smp_Q, smp_dn);
    // wholly dynamic samples sfull + blockIdx.x + j * gridDim.x are this CTA's to descend
    const int first_x = sfull + (int)blockIdx.x;
    const int extra = (r0 < total && first_x < (int)n) ? ((int)n - first_x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    int32_t eb = 0;
    for (int pc = warp; pc < np0 + extra; pc += NT / 32) {
      const int sm = pc < np0 ? s_first + pc : first_x + (pc - np0) * (int)gridDim.x;
      int64_t leaf = -1, qv = 0;
      if (smp_Q == 0) {
        eb |= RPL_DERR_EMPTY;
      } else {
        const uint64_t prefix = strata_prefix(sm, smp_st, nullptr, D.smp_seed, smp_pos);
        leaf = upd ? descend_overlay(D.smp_L, D.smp_tree, (int64_t)prefix, &qv, &eb, top, uf_key, uf_val)
                   : descend(D.smp_L, D.smp_tree, (int64_t)prefix, &qv, &eb, top, ntop);
      }
      if (lane == 0) {
        if (pc < np0) p_leaf[pc] = leaf;
        if (pc >= np0 || sm * L >= g0) {
          const_cast<int64_t*>(idx)[sm] = leaf;
          const_cast<int64_t*>(q)[sm] = qv;
        }
        if (pc == 0 && np0 > 0 && leaf >= 0 && leaf < nleaves && early_frames) {
          // piece 0's first frames, now: slots 0 .. pre-1 (fresh, below the staged levels)
          const int tau0 = max(g0 - sm * L, 0);
          const int R = min(g1, (sm + 1) * L) - max(g0, sm * L);
          const int skip = (unique && tau0 > 0) ? k - 1 : 0;
          const int pre = min(min(R + k - 1 - skip, pre_cap), early_frames);
          const int blk = (int)(leaf / Bc);
          const int bcol = (int)(leaf - (int64_t)blk * Bc);
          int row = (int)(((int64_t)blk * period + tau0) % cap) - (k - 1) + skip;
          while (row < 0) row += cap;
          const uint8_t* colp = D.obs + (int64_t)bcol * ob;
          for (int w = 0; w < pre; ++w) {
            mbar_expect_tx(&full[w], (uint32_t)ob);
            bulk_g2s_evict_first(smem + w * ob, colp + (int64_t)row * Bc * ob, (uint32_t)ob, &full[w]);
            if (++row == cap) row = 0;
          }
          s_pre = pre;
          flag_release(&s_issued, pre);
        }
      }
    }
    if (lane == 0 && eb) set_err(err, eb);
    fence_proxy_async();  // the staged words were read through the generic proxy; TMA refills them
    __syncthreads();
#ifdef RPL_TRACE
    if (tid == 0 && blockIdx.x == 0) g_gtrace[7] = global_ns();  // descents done
#endif
    if (tid == 0) {  // this CTA's index / q writes are done, and its reads of the old tree (release)
      __threadfence();
      atomicAdd(reinterpret_cast<unsigned long long*>(D.work + 2), 1ull);
    }
    if (g1 <= g0 && warp == 0) smp_ticket_finish(D, idx, q, n, beta, smp_pos);  // no static rows: ticket now
  }
  // ---- (A) static pieces (one per sample overlapping [g0, g1)), in parallel
  for (int pc = tid; pc < np0; pc += NT) {
    const int sm = s_first + pc;
    const int tau0 = max(g0 - sm * L, 0);
    const int R = min(g1, (sm + 1) * L) - max(g0, sm * L);
    const int64_t leaf = smp ? p_leaf[pc] : idx[sm];
    int bcol = -1, row0 = 0, blk = 0;
    if (leaf >= 0 && leaf < nleaves) {
      blk = (int)(leaf / Bc);
      bcol = (int)(leaf - (int64_t)blk * Bc);
      row0 = (int)(((int64_t)blk * period + tau0) % cap);
      if (tau0 == 0) {
        int age = ((int)D.cursor - 1 - blk * period) % cap;
        if (age < 0) age += cap;
        const int hist = k - 1 > 1 ? k - 1 : 1;
        if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
      }
    } else if (leaf >= nleaves && tau0 == 0) {
      set_err(err, RPL_DERR_IDX);
    }
    p_s[pc] = sm;
    p_b[pc] = bcol;
    p_row0[pc] = row0;
    p_blk[pc] = blk;
    p_tau0[pc] = (short)tau0;
    p_R[pc] = (short)R;
    p_skip[pc] = (int8_t)((unique && tau0 > 0) ? k - 1 : 0);
  }
  __syncthreads();
  // ---- (B) frame positions of the static pieces (serial: one to a few)
  __shared__ int s_F_total;
  if (tid == 0) {
    int F = 0;
    for (int pc = 0; pc < np0; ++pc) {
      p_F[pc] = F;
      if (p_b[pc] >= 0) F += p_R[pc] + k - 1 - p_skip[pc];
    }
    s_F_total = F;
    s_pieces_pub = np0;
    s_rows_pub = g1 - g0;
  }
  __syncthreads();
  // row-table entry of row c (piece pc, m-th row of the piece); done flags loaded together
  auto row_entry = [&](int c, int pc, int m) {
    const int bcol = p_b[pc];
    const int R = p_R[pc];
    const int skip = p_skip[pc];
    const int F = p_F[pc];
    int8_t so = 0;
    int ring = 0;
    if (bcol >= 0) {
      const int nw = F + m + (k - 1) - skip;
      row_new[c] = nw;
      rel[c] = m == R - 1 ? F + R + k - 1 - skip : (unique ? nw + 1 : nw - (k - 1) + 1);
      ring = p_row0[pc] + m;
      if (ring >= cap) ring -= cap;
      uint8_t dw[8];
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        int rr = ring - k + j;
        while (rr < 0) rr += cap;
        dw[j] = j < k ? __ldg(D.done + (int64_t)rr * Bc + bcol) : (uint8_t)0;
      }
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (dw[j]) so = (int8_t)j;
    } else {
      row_new[c] = -1;
      rel[c] = F;
    }
    row_ring[c] = ring;
    row_piece[c] = (short)pc;
    row_tau[c] = (short)(p_tau0[pc] + m);
    start_off[c] = so;
  };
  // per-row fields, fused targets, IS weight and stored state of rows [ca, cb) (meta warp)
  auto row_fields = [&](int ca, int cb, int64_t qm) {
    const int64_t ab = D.act_bytes;
    const bool a8 = ab == 8 && ((reinterpret_cast<uintptr_t>(D.act) | reinterpret_cast<uintptr_t>(D.o_act) |
                                 reinterpret_cast<uintptr_t>(D.o_prev_act)) & 7) == 0;
    for (int c = ca + lane; c < cb; c += 32) {
      if (row_new[c] < 0) continue;
      const int pc = row_piece[c];
      const int sm = p_s[pc];
      const int tau = row_tau[c];
      const int bcol = p_b[pc];
      const int ring = row_ring[c];
      const int prow = ring == 0 ? cap - 1 : ring - 1;
      const int64_t e = (int64_t)ring * Bc + bcol, pe = (int64_t)prow * Bc + bcol;
      const uint8_t pd = __ldg(D.done + pe);
      const uint8_t dd = __ldg(D.done + e);
      const float rw = D.o_rew ? __ldg(D.rew + e) : 0.0f;
      const float prw = D.o_prev_rew ? __ldg(D.rew + pe) : 0.0f;
      const int64_t o = (int64_t)tau * n + sm;
      if (a8) {
        const uint64_t* a = reinterpret_cast<const uint64_t*>(D.act);
        const uint64_t av = D.o_act ? __ldg(a + e) : 0ull;
        const uint64_t pav = D.o_prev_act ? __ldg(a + pe) : 0ull;
        if (D.o_act) reinterpret_cast<uint64_t*>(D.o_act)[o] = av;
        if (D.o_prev_act) reinterpret_cast<uint64_t*>(D.o_prev_act)[o] = pd ? 0ull : pav;
      } else {
        if (D.o_act) coop_copy(D.o_act + o * ab, D.act + e * ab, ab, 0, 1);
        if (D.o_prev_act) {
          if (pd) coop_zero(D.o_prev_act + o * ab, ab, 0, 1);
          else coop_copy(D.o_prev_act + o * ab, D.act + pe * ab, ab, 0, 1);
        }
      }
      if (D.o_rew) D.o_rew[o] = rw;
      if (D.o_prev_rew) D.o_prev_rew[o] = pd ? 0.0f : prw;
      if (D.o_done) D.o_done[o] = dd;
      if (D.o_start) D.o_start[o] = start_off[c];
      if (tau == 0 && D.o_w && q && !smp) {
        const int64_t qs = q[sm];
        D.o_w[sm] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
      }
    }
    if (D.o_tgt) {  // fused n-step targets (a2 + a4, R5 / R24 / R34)
      const int ns = D.n_step;
      for (int c = ca + lane; c < cb; c += 32) {
        if (row_new[c] < 0) continue;
        const int t = row_tau[c] - D.tgt_lo;
        if (t < 0 || t >= D.tgt_T) continue;
        const int64_t col = p_s[row_piece[c]];
        double acc = 0.0;
        if (D.q_tgt) {
          const double qv = (double)__ldg(D.q_tgt + (int64_t)(row_tau[c] + ns) * n + col);
          acc = D.rescale ? h_inv(qv, D.rescale_eps) : qv;
        }
        uint8_t dn = 0;
        acc = nstep_rows(D, row_ring[c], p_b[row_piece[c]], ns, acc, &dn);
        if (D.rescale) acc = h_fwd(acc, D.rescale_eps);
        D.o_tgt[(int64_t)t * n + col] = (float)acc;
        if (D.o_tgt_done) D.o_tgt_done[(int64_t)t * n + col] = dn ? 1 : 0;
      }
    }
    if (D.o_rnn) {  // stored recurrent state of every sample whose first row is in [ca, cb)
      const int nparts = D.rnn_parts;
      const int64_t rb = D.rnn_bytes;
      for (int c = ca; c < cb; ++c) {
        if (row_tau[c] != 0 || row_new[c] < 0) continue;
        const int pc = row_piece[c];
        const int64_t blk = p_blk[pc], bcol = p_b[pc];
        const int sm = p_s[pc];
        for (int pp = 0; pp < nparts; ++pp)
          coop_copy(D.o_rnn + (pp * n + sm) * rb, D.rnn + ((blk * Bc + bcol) * nparts + pp) * rb, rb, lane, 32);
      }
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer: TMA loads of every published piece ----------------
      const int pre = s_pre;  // piece 0's frames already in flight (fused sampling)
      int frontier = 0, released = 0, i = pre, slot = pre;
      auto advance = [&]() {  // the contiguous done-frontier (also read by the meta warp)
        if (frontier < flag_acquire(&s_rows_pub) && flag_acquire(&row_done[frontier])) {
          released = rel[frontier];
          ++frontier;
          s_frontier = frontier;
#ifdef RPL_TRACE
          if (frontier == g1 - g0 && blockIdx.x < 512) g_gstatic[blockIdx.x] = global_ns();
#endif
          return true;
        }
        return false;
      };
      for (int pc = 0;; ++pc) {
        while (pc >= flag_acquire(&s_pieces_pub)) {  // wait for the next piece (or the end)
          if (!flag_acquire(&s_more) && pc >= flag_acquire(&s_pieces_pub)) goto prod_done;
          if (!advance()) __nanosleep(32);
        }
        const int bcol = p_b[pc];
        if (bcol < 0) continue;
        const int R = p_R[pc];
        const int skip = p_skip[pc];
        const int done0 = pc == 0 ? pre : 0;
        int row = p_row0[pc] - (k - 1) + skip + done0;
        while (row < 0) row += cap;
        while (row >= cap) row -= cap;
        const uint8_t* col = D.obs + (int64_t)bcol * ob;
        const int64_t rstride = (int64_t)Bc * ob;
        for (int w = skip + done0; w < R + k - 1; ++w, ++i) {
          if (i >= NS) {
            while (released <= i - NS)
              if (!advance()) __nanosleep(20);
            fence_proxy_async();
            mbar_wait(&full[slot], (uint32_t)(((i / NS) - 1) & 1));
          }
          mbar_expect_tx(&full[slot], (uint32_t)ob);
          bulk_g2s_evict_first(smem + slot * ob, col + (int64_t)row * rstride, (uint32_t)ob, &full[slot]);
          flag_release(&s_issued, i + 1);
          if (++row == cap) row = 0;
          if (++slot == NS) slot = 0;
        }
      }
    prod_done:
      if (trig_at == 1) pdl_trigger();
      // observe the last phase of every armed slot: no bulk copy into shared memory is in
      // flight when the CTA exits
      for (int p = i > NS ? i - NS : 0; p < i; ++p) mbar_wait(&full[p % NS], (uint32_t)((p / NS) & 1));
    }
  } else {
    // (C) static row tables, rows spread over warps 1..NC+2
    for (int c = tid - 32; c < g1 - g0; c += NT - 32) {
      const int g = g0 + c;
      const int pc = g / L - s_first;
      row_entry(c, pc, g - max(g0, p_s[pc] * L));
    }
    asm volatile("bar.sync 1, %0;" ::"n"((NC + 2) * 32) : "memory");
    if (UPD && warp == 2 && blockIdx.x == 0 && D.upd_td != nullptr) {
      // the fused update's global writes (a6-a7): once every CTA has read the old tree (each
      // counted itself into work[2] after its descents), the winners' leaves, the int64 deltas
      // of their ancestors, max-priority-seen and the error bits
      if (lane == 0)
        while (ld_acquire_u64(D.work + 2) < (unsigned long long)gridDim.x) __nanosleep(64);
      __syncwarp();
      int64_t* leaves = D.smp_tree + D.smp_L.level_off[D.smp_L.depth];
      int64_t lmax = INT64_MIN;
      int32_t eb = 0;
      for (int j = lane; j < D.upd_n; j += 32) {
        const int64_t raw = D.upd_idx[j];
        if (raw >= nleaves) eb |= RPL_DERR_IDX;
        const int64_t lf = u_leaf[j];
        if (lf >= 0 && !(D.upd_live && u_old[j] == 0)) lmax = u_q[j] > lmax ? u_q[j] : lmax;
        if (u_win[j]) {
          leaves[lf] = u_q[j];
          const int64_t delta = u_q[j] - u_old[j];
          if (delta != 0) {
            int64_t node = lf;
            for (int l = D.smp_L.depth - 1; l >= 0; --l) {
              node >>= D.smp_L.log2w;
              atomicAdd(reinterpret_cast<unsigned long long*>(D.smp_tree + D.smp_L.level_off[l] + node),
                        (unsigned long long)delta);
            }
          }
        }
      }
      lmax = warp_max64(lmax);
      int64_t* hdr = D.smp_tree + D.smp_L.hdr_off;
      if (lane == 0) {
        if (lmax > __ldcg(hdr)) atomicMax(reinterpret_cast<long long*>(hdr), (long long)lmax);
        if (eb) set_err(err, eb);
      }
      // an attached min-tree (R29): every winner's min path, level by level from the leaves'
      // parents up (a lane per winner; the W children loaded together)
      int64_t* mins = reinterpret_cast<int64_t*>(__ldcg(hdr + 5));
      if (mins) {
        __threadfence_block();
        __syncwarp();
        for (int l = D.smp_L.depth - 1; l >= 0; --l) {
          const int sh = D.smp_L.log2w * (D.smp_L.depth - l);
          for (int j = lane; j < D.upd_n; j += 32) {
            if (!u_win[j]) continue;
            const int64_t node = u_leaf[j] >> sh;
            const int64_t c0 = node << D.smp_L.log2w;
            int64_t m2 = INT64_MAX;
            if (l == D.smp_L.depth - 1) {
              for (int c = 0; c < D.smp_L.fanout; ++c) {
                const int64_t v = __ldcg(leaves + c0 + c);
                if (v > 0 && v < m2) m2 = v;
              }
            } else {
              for (int c = 0; c < D.smp_L.fanout; ++c) {
                const int64_t v = __ldcg(mins + D.smp_L.level_off[l + 1] + c0 + c);
                if (v < m2) m2 = v;
              }
            }
            mins[D.smp_L.level_off[l] + node] = m2;
          }
          __threadfence_block();
          __syncwarp();
        }
      }
    }
    if (warp == 2) {
      // ---------------- fields warp: per-row fields of every published row, in order ----------------
      const int64_t qm = (D.o_w && q && !smp) ? warp_batch_qmin(qmin, idx, q, n) : 0;
      int fd = 0;
      while (true) {
        const int rp = flag_acquire(&s_rows_pub);
        if (fd < rp) {
          const int fe = min(rp, fd + 32);
          row_fields(fd, fe, qm);
          fd = fe;
        } else if (!flag_acquire(&s_more) && fd >= flag_acquire(&s_rows_pub)) {
          break;
        } else {
          __nanosleep(64);
        }
      }
    } else if (warp == 1) {
      // ---------------- meta warp: the dynamic tail ----------------
      if (smp && g1 > g0) smp_ticket_finish(D, idx, q, n, beta, smp_pos);  // fused sampling's ticket / weights
      bool idx_ready = !smp;
      int F = s_F_total;
      int pcn = np0, cn = g1 - g0;
      const int ndyn = total - r0;  // dynamic rows [r0, total); work[0] counts the rows taken
      int grabs = 0;
      bool exhausted = ndyn <= 0;
      // lookahead: bits 0-7 the rows kept queued before a grab; bits 8-15 (if non-zero) the
      // queue once fewer than bits 16-30 rows are left in the pool (the end of the pool: a
      // shorter queue when it runs dry means less spread between the CTAs' ends)
      const int look_base = lookahead & 0xff;
      const int look_end = ((lookahead >> 8) & 0xff) ? ((lookahead >> 8) & 0xff) : look_base;
      const int look_thr = lookahead >> 16;
      int left = ndyn;  // rows left in the pool, as this warp last saw it
      while (!exhausted) {
        // grab only when this CTA is about to run dry (a slower SM takes less), and GUIDED: a
        // grab takes ~1/grid of what is left, between 2 and dyn_rows rows, so early grabs are
        // long (few reloaded history frames) and the last ones short (fine balance)
        if (cn - s_frontier <= (left < look_thr ? look_end : look_base)) {
          if (cn + dyn_rows > DY_MAX_ROWS || pcn + 2 > DY_MAX_PIECES) {
            exhausted = true;
            continue;
          }
          int start = 0, cnt = 0;
          if (lane == 0) {
            const int taken = (int)__ldcg(D.work);
            int sz = (ndyn - taken) / (int)gridDim.x;
            sz = sz < 2 ? 2 : (sz > dyn_rows ? dyn_rows : sz);
            if (sz > L) sz = L;  // a grab spans at most two samples (two pieces)
            start = (int)atomicAdd(reinterpret_cast<unsigned long long*>(D.work), (unsigned long long)sz);
            cnt = min(sz, ndyn - start);
          }
          start = __shfl_sync(0xffffffffu, start, 0);
          cnt = __shfl_sync(0xffffffffu, cnt, 0);
          if (cnt <= 0) {
            exhausted = true;
            continue;
          }
          left = ndyn - start - cnt;
#ifdef RPL_TRACE
          if (lane == 0 && blockIdx.x < 512 && grabs < 8) {
            g_ggrab[blockIdx.x][grabs][0] = global_ns();
            g_ggrab[blockIdx.x][grabs][1] = ((unsigned long long)cnt << 32) | (unsigned)(cn - s_frontier);
          }
#endif
          ++grabs;
          if (!idx_ready) {  // fused sampling: every CTA has written its samples' indices
            if (lane == 0)
              while (ld_acquire_u64(D.work + 2) < (unsigned long long)gridDim.x) __nanosleep(64);
            __syncwarp();
            idx_ready = true;
          }
          // the grabbed rows [ga, gb) as pieces of whole samples: tables first (published), fields later
          for (int ga = r0 + start, gb = r0 + start + cnt; ga < gb;) {
            const int sm = ga / L;
            const int tau0 = ga - sm * L;
            const int R = min(gb, (sm + 1) * L) - ga;
            if (lane == 0) {
              const int64_t leaf = __ldcg(idx + sm);
              int bcol = -1, row0 = 0, blk = 0;
              if (leaf >= 0 && leaf < nleaves) {
                blk = (int)(leaf / Bc);
                bcol = (int)(leaf - (int64_t)blk * Bc);
                row0 = (int)(((int64_t)blk * period + tau0) % cap);
                if (tau0 == 0) {
                  int age = ((int)D.cursor - 1 - blk * period) % cap;
                  if (age < 0) age += cap;
                  const int hist = k - 1 > 1 ? k - 1 : 1;
                  if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
                }
              } else if (leaf >= nleaves && tau0 == 0) {
                set_err(err, RPL_DERR_IDX);
              }
              const int skip = (unique && tau0 > 0) ? k - 1 : 0;
              p_s[pcn] = sm;
              p_b[pcn] = bcol;
              p_row0[pcn] = row0;
              p_blk[pcn] = blk;
              p_F[pcn] = F;
              p_tau0[pcn] = (short)tau0;
              p_R[pcn] = (short)R;
              p_skip[pcn] = (int8_t)skip;
            }
            __syncwarp();
            if (lane < R) row_entry(cn + lane, pcn, lane);
            __syncwarp();
            if (p_b[pcn] >= 0) F += R + k - 1 - p_skip[pcn];
            if (lane == 0) {
              flag_release(&s_rows_pub, cn + R);
              flag_release(&s_pieces_pub, pcn + 1);
            }
            cn += R;
            ++pcn;
            ga += R;
          }
        } else {
          __nanosleep(64);
        }
      }
      __syncwarp();
      if (lane == 0) flag_release(&s_more, 0);
#ifdef RPL_TRACE
      if (lane == 0 && blockIdx.x < 512) g_gunits[blockIdx.x] = (unsigned long long)grabs;
#endif
    } else {
      // ---------------- consumers: one k-stack per published row ----------------
      for (int c = warp - 3;; c += NC) {
        while (c >= flag_acquire(&s_rows_pub)) {
          if (!flag_acquire(&s_more) && c >= flag_acquire(&s_rows_pub)) goto cons_done;
          __nanosleep(32);
        }
        {
          const int pn = row_new[c];
          const int sn = pn % NS;
          const uint32_t parn = (uint32_t)((pn / NS) & 1);
          auto slot_of = [&](int j, uint32_t* par) {
            int sl = sn - (k - 1 - j);
            *par = parn;
            if (sl < 0) {
              sl += NS;
              *par ^= 1u;
            }
            return sl;
          };
          if (pn >= 0)
            while (flag_acquire(&s_issued) <= pn) __nanosleep(20);
          const int sm = p_s[row_piece[c]];
          const int tau = row_tau[c];
          if (pn >= 0 && unique) {
            for (int j = tau == 0 ? 0 : k - 1; j < k; ++j) {
              uint32_t par;
              const int sl = slot_of(j, &par);
              mbar_wait(&full[sl], par);
              int4* d = reinterpret_cast<int4*>(D.o_obs + ((int64_t)(tau + j) * n + sm) * ob);
              const int4* sp = reinterpret_cast<const int4*>(smem + sl * ob);
#pragma unroll 4
              for (int v = lane; v < nv; v += 32) __stcs(d + v, sp[v]);
            }
          } else if (pn >= 0) {
            const int so = start_off[c];
            for (int j = so; j < k; ++j) {
              uint32_t par;
              const int sl = slot_of(j, &par);
              mbar_wait(&full[sl], par);
            }
            int4* dst = reinterpret_cast<int4*>(D.o_obs + ((int64_t)tau * n + sm) * k * ob);
            for (int j = 0; j < k; ++j) {
              int4* d = dst + j * nv;
              if (j < so && D.pad_mode == RPL_PAD_ZERO) {
                for (int v = lane; v < nv; v += 32) d[v] = make_int4(0, 0, 0, 0);
              } else {
                uint32_t par;
                const int sl = slot_of(j < so ? so : j, &par);
                const int4* sp = reinterpret_cast<const int4*>(smem + sl * ob);
#pragma unroll 4
                for (int v = lane; v < nv; v += 32) __stcs(d + v, sp[v]);
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            fence_proxy_async();
            flag_release(&row_done[c], 1);
          }
        }
      }
    cons_done:;
    }
  }
  __syncthreads();
#ifdef RPL_TRACE
  if (threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMax(&g_gtrace[3], t);
    atomicMin(&g_gtrace[8], t);
    if (blockIdx.x < 512) g_gend[blockIdx.x] = t;
  }
#endif
  if (threadIdx.x == 0) {  // the last CTA out re-zeroes the unit counter and the ticket
    unsigned long long t;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(t) : "l"(D.work + 1) : "memory");
    if (t == (unsigned long long)gridDim.x - 1) {
      D.work[0] = 0;
      D.work[1] = 0;
      D.work[2] = 0;
    }
  }
  if (trig_at != 0 && trig_at != 1) pdl_trigger();
}

template <int NC>
int launch_seq_dyn(const GDesc& g, const int64_t* idx, int64_t n, int NS, int rs, int dyn_rows, int lookahead,
                   const int64_t* q, const int64_t* qmin, double beta, int32_t* dev_err, size_t dyn, int64_t grid,
                   cudaStream_t st) {
  // the fused update (rpl_gather_update_sample) has its own instantiation: the default gather
  // carries none of its code, registers or tables
  auto kern = (g.upd_td != nullptr || g_dyn_updk.load(std::memory_order_relaxed)) ? k_gather_seq_dyn<NC, true>
                                                                                  : k_gather_seq_dyn<NC, false>;
  ensure_smem(reinterpret_cast<const void*>(kern), dyn);
  // With the update fused in (rpl_gather_update_sample) the next kernel is usually the next
  // step's gather, whose CTAs only fit once this grid's CTAs leave: let it launch once each
  // CTA's producer has issued its last load, so its CTAs land (and run their prologue) on the
  // SMs as they free up.  In-process A/B: 65.45 -> 63.96 us per step (trigger at entry: 64.03;
  // profiles/r2/ab_one_launch.txt).  The two-launch step keeps the exit trigger (its update
  // is small enough to sit beside the gather; an early trigger there costs 0.4 us).
  int trig = g_gather_trigger.load(std::memory_order_relaxed);
  if (trig == -1 && g.upd_td != nullptr) trig = 1;
  return launch_pdl(kern, dim3((unsigned)grid), dim3((NC + 3) * 32), dyn, st, g, idx, n, NS, rs,
                    dyn_rows, lookahead, q, qmin, beta, dev_err, trig, g_dyn_early.load(std::memory_order_relaxed));
}

// ---------------------------------------------------------------------------
// Sequences, variant 6: LSU frame loads, TMA bulk stores.  The mirror image of the
// default kernel: loader warps stream the unique frames global -> registers ->
// shared memory (ld.global.cs, evict-first) and flag each slot; ONE thread issues
// every k-stack store as cp.async.bulk shared -> global (L2 evict-first), so the
// SM's TMA queue carries only stores (measured ceiling for 28-KB bulk stores:
// 6.3 TB/s) and the LSU only the 1-in-5 bytes that are loads.  The issuer keeps
// LB_G row groups in flight and releases frames once their group has been read.
// Same tables, meta warp and outputs as the default kernel.
// ---------------------------------------------------------------------------
constexpr int LB_G = 8;

__device__ __forceinline__ void bulk_s2g_ef(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}

template <int NL>
__global__ void __launch_bounds__((NL + 2) * 32, 1)
k_gather_seq_ldg_bulk(GDesc D, const int64_t* __restrict__ idx, int64_t n, int NS, int64_t rows_per_cta,
                      const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  extern __shared__ __align__(128) uint8_t smem[];  // NS frame slots + 1 zero slot
  __shared__ int p_b[PL_MAX_ROWS];
  __shared__ int p_row0[PL_MAX_ROWS];
  __shared__ int p_blk[PL_MAX_ROWS];
  __shared__ int p_F[PL_MAX_ROWS];
  __shared__ int p_R[PL_MAX_ROWS];
  __shared__ int row_first[PL_MAX_ROWS];
  __shared__ int rel[PL_MAX_ROWS];
  __shared__ int row_ring[PL_MAX_ROWS];
  __shared__ short row_piece[PL_MAX_ROWS];
  __shared__ short row_tau[PL_MAX_ROWS];
  __shared__ int8_t start_off[PL_MAX_ROWS];
  __shared__ volatile int frame_ready[PIPE_MAX_NS];
  __shared__ volatile int s_released;
  __shared__ int s_ftotal;
  constexpr int NT = (NL + 2) * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = D.k, L = D.seq_len;
  const int ob = (int)D.obs_bytes;
  const int nv = ob / 16;
  const int cap = (int)D.cap_T, Bc = (int)D.B, period = (int)D.period;
  const int64_t nleaves = (int64_t)(cap / period) * Bc;
  pdl_wait();  // idx (and n_active) come from the sampler launched just before
  // rows g = s*L + tau of the active samples, split evenly over the grid
  const int total = (int)(active_n(D, n) * L);
  const int64_t coff = col_off(D);  // output column of entry 0 (Mode C)
  const int rpc = D.n_active ? (total + (int)gridDim.x - 1) / (int)gridDim.x : (int)rows_per_cta;
  const int g0 = (int)blockIdx.x * rpc;
  const int g1 = min(total, g0 + rpc);
  // K7 fused (peer boards): the step's tag comes from this rank's own board (its sampler's
  // K5 slot); CTA 0 publishes this rank's batch-min q over its owned entries to every rank
  // — before any early exit, so a rank that owns nothing still publishes (INT64_MAX)
  const bool peer = D.peer_boards != nullptr && D.o_w != nullptr && q != nullptr;
  uint64_t ptag = 0;
  if (peer) {
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];"
                 : "=l"(ptag) : "l"(D.peer_boards[D.peer_rank] + 2 * D.peer_rank + 1) : "memory");
    if (blockIdx.x == 0 && warp == 1) {
      const int64_t qm_local = warp_batch_qmin(nullptr, idx, q, n);
      if (lane < D.peer_world)
        board_publish(D.peer_boards[lane] + 2 * D.peer_world + 2 * D.peer_rank, qm_local, ptag);
    }
  }
  if (g0 >= g1) return;
  const int nrows = g1 - g0;
  const int s_first = g0 / L;
  const int npieces = (g1 - 1) / L - s_first + 1;
  uint8_t* zslot = smem + NS * ob;

  for (int i = tid; i < NS; i += NT) frame_ready[i] = -1;
  if (tid == 0) s_released = 0;
  if (D.pad_mode == RPL_PAD_ZERO) {
    for (int v = tid; v < nv; v += NT) reinterpret_cast<int4*>(zslot)[v] = make_int4(0, 0, 0, 0);
    fence_proxy_async();
  }
  for (int pc = tid; pc < npieces; pc += NT) {
    const int sm = s_first + pc;
    const int tau0 = max(g0 - sm * L, 0);
    const int64_t leaf = idx[sm];
    int bcol = -1, row0 = 0, blk = 0;
    if (leaf >= 0 && leaf < nleaves) {
      blk = (int)(leaf / Bc);
      bcol = (int)(leaf - (int64_t)blk * Bc);
      row0 = (int)(((int64_t)blk * period + tau0) % cap);
      if (tau0 == 0) {
        // cursor, blk * period < cap_T < 2^30 (host-checked): 32-bit modulo
        int age = ((int)D.cursor - 1 - blk * period) % cap;
        if (age < 0) age += cap;
        const int hist = k - 1 > 1 ? k - 1 : 1;
        if (!(age >= L - 1 && age + hist <= D.size - 1)) set_err(err, RPL_DERR_INVALID_LEAF);
      }
    } else if (leaf >= nleaves && tau0 == 0) {
      set_err(err, RPL_DERR_IDX);
    }
    p_b[pc] = bcol;
    p_row0[pc] = row0;
    p_blk[pc] = blk;
    p_R[pc] = min(g1, (sm + 1) * L) - max(g0, sm * L);
  }
  __syncthreads();
  if (tid == 0) {
    int F = 0;
    for (int pc = 0; pc < npieces; ++pc) {
      p_F[pc] = F;
      if (p_b[pc] >= 0) F += p_R[pc] + k - 1;
    }
    s_ftotal = F;
  }
  __syncthreads();
  // row tables + episode-start offsets (all warps)
  for (int c = tid; c < nrows; c += NT) {
    const int g = g0 + c;
    const int sm = g / L;
    const int tau = g - sm * L;
    const int pc = sm - s_first;
    const int bcol = p_b[pc];
    const int m = g - max(g0, sm * L);
    int8_t so = 0;
    int ring = 0;
    if (bcol >= 0) {
      const int R = p_R[pc];
      const int F = p_F[pc];
      row_first[c] = F + m;
      rel[c] = m == R - 1 ? F + R + k - 1 : F + m + 1;
      ring = p_row0[pc] + m;
      if (ring >= cap) ring -= cap;
      uint8_t dw[8];
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        int rr = ring - k + j;
        while (rr < 0) rr += cap;
        dw[j] = j < k ? __ldg(D.done + (int64_t)rr * Bc + bcol) : (uint8_t)0;
      }
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (dw[j]) so = (int8_t)j;
    } else {
      row_first[c] = -1;
      rel[c] = p_F[pc];
    }
    row_ring[c] = ring;
    row_piece[c] = (short)pc;
    row_tau[c] = (short)tau;
    start_off[c] = so;
  }
  __syncthreads();
  const int ftotal = s_ftotal;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- store issuer: TMA bulk stores only ----------------
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int c = 0; c < nrows; ++c) {
        const int p0 = row_first[c];
        if (p0 >= 0 && !(GDIAG(D) & 1)) {
          const int so = start_off[c];
          const int sm = s_first + row_piece[c];
          const int tau = row_tau[c];
          const int s0 = p0 % NS;
          for (int j = so; j < k; ++j) {
            int sl = s0 + j;
            if (sl >= NS) sl -= NS;
            while (flag_acquire(&frame_ready[sl]) != p0 + j + 1) __nanosleep(20);
          }
          fence_proxy_async();
          uint8_t* dst = D.o_obs + ((int64_t)tau * n + coff + sm) * k * ob;
          if (so == 0 && s0 + k <= NS) {
            bulk_s2g_ef(dst, smem + s0 * ob, (uint32_t)(k * ob), pol);
          } else {
            for (int j = 0; j < k; ++j) {
              const uint8_t* src;
              if (j < so && D.pad_mode == RPL_PAD_ZERO) {
                src = zslot;
              } else {
                int sl = s0 + (j < so ? so : j);
                if (sl >= NS) sl -= NS;
                src = smem + sl * ob;
              }
              bulk_s2g_ef(dst + j * ob, src, (uint32_t)ob, pol);
            }
          }
        }
        bulk_commit();
        bulk_wait_read_G<LB_G>();
        if (c >= LB_G) flag_release(&s_released, rel[c - LB_G]);
      }
      bulk_wait_all();
    }
  } else if (warp == 1) {
    // ---------------- meta warp (as in the default kernel) ----------------
    const int64_t qm = (D.o_w && q) ? warp_batch_qmin(qmin, idx, q, n) : 0;
    const int64_t ab = D.act_bytes;
    const bool a8 = ab == 8 && ((reinterpret_cast<uintptr_t>(D.act) | reinterpret_cast<uintptr_t>(D.o_act) |
                                 reinterpret_cast<uintptr_t>(D.o_prev_act)) & 7) == 0;
    for (int c = lane; c < nrows && !(GDIAG(D) & 16); c += 32) {
      if (row_first[c] < 0) continue;
      const int pc = row_piece[c];
      const int sm = s_first + pc;
      const int tau = row_tau[c];
      const int bcol = p_b[pc];
      const int ring = row_ring[c];
      const int prow = ring == 0 ? cap - 1 : ring - 1;
      const int64_t e = (int64_t)ring * Bc + bcol, pe = (int64_t)prow * Bc + bcol;
      const uint8_t pd = __ldg(D.done + pe);
      const uint8_t dd = __ldg(D.done + e);
      const float rw = D.o_rew ? __ldg(D.rew + e) : 0.0f;
      const float prw = D.o_prev_rew ? __ldg(D.rew + pe) : 0.0f;
      const int64_t o = (int64_t)tau * n + coff + sm;
      if (a8) {
        const uint64_t* a = reinterpret_cast<const uint64_t*>(D.act);
        const uint64_t av = D.o_act ? __ldg(a + e) : 0ull;
        const uint64_t pav = D.o_prev_act ? __ldg(a + pe) : 0ull;
        if (D.o_act) reinterpret_cast<uint64_t*>(D.o_act)[o] = av;
        if (D.o_prev_act) reinterpret_cast<uint64_t*>(D.o_prev_act)[o] = pd ? 0ull : pav;
      } else {
        if (D.o_act) coop_copy(D.o_act + o * ab, D.act + e * ab, ab, 0, 1);
        if (D.o_prev_act) {
          if (pd) coop_zero(D.o_prev_act + o * ab, ab, 0, 1);
          else coop_copy(D.o_prev_act + o * ab, D.act + pe * ab, ab, 0, 1);
        }
      }
      if (D.o_rew) D.o_rew[o] = rw;
      if (D.o_prev_rew) D.o_prev_rew[o] = pd ? 0.0f : prw;
      if (D.o_done) D.o_done[o] = dd;
      if (tau == 0 && D.o_w && q) {
        const int64_t qs = q[sm];
        D.o_w[coff + sm] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
      }
    }
    if (D.o_rnn && !(GDIAG(D) & 16)) {
      const int nparts = D.rnn_parts;
      const int64_t rb = D.rnn_bytes;
      for (int pc = 0; pc < npieces; ++pc) {
        const int sm = s_first + pc;
        if (sm * L < g0 || p_b[pc] < 0) continue;
        const int64_t blk = p_blk[pc], bcol = p_b[pc];
        for (int pp = 0; pp < nparts; ++pp)
          coop_copy(D.o_rnn + (pp * n + coff + sm) * rb, D.rnn + ((blk * Bc + bcol) * nparts + pp) * rb, rb, lane, 32);
      }
    }
  } else {
    // ---------------- loaders: frames global -> registers -> shared memory ----------------
    const int64_t rstride = (int64_t)Bc * ob;
    int pc = 0;  // piece cursor (frame positions increase monotonically per warp)
    for (int f = warp - 2; f < ftotal; f += NL) {
      while (p_b[pc] < 0 || f >= p_F[pc] + p_R[pc] + k - 1) ++pc;
      int row = p_row0[pc] - (k - 1) + (f - p_F[pc]);
      while (row < 0) row += cap;
      while (row >= cap) row -= cap;
      const int4* src = reinterpret_cast<const int4*>(D.obs + (int64_t)p_b[pc] * ob + (int64_t)row * rstride);
      while (f >= flag_acquire(&s_released) + NS) __nanosleep(20);
      const int sl = f % NS;
      int4* dst = reinterpret_cast<int4*>(smem + sl * ob);
      if (!(GDIAG(D) & 2)) {
        constexpr int U = 8;
        for (int v0 = lane; v0 < nv; v0 += 32 * U) {
          int4 r[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (v0 + 32 * u < nv) r[u] = __ldcs(src + v0 + 32 * u);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (v0 + 32 * u < nv) dst[v0 + 32 * u] = r[u];
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) flag_release(&frame_ready[sl], f + 1);
    }
  }
  pdl_trigger();
}

template <int NL>
int launch_seq_ldg_bulk(const GDesc& g, const int64_t* idx, int64_t n, int NS, int64_t rows_per_cta,
                        const int64_t* q, const int64_t* qmin, double beta, int32_t* dev_err, size_t dyn,
                        int64_t grid, cudaStream_t st) {
  ensure_smem(reinterpret_cast<const void*>(k_gather_seq_ldg_bulk<NL>), dyn);
  return launch_pdl(k_gather_seq_ldg_bulk<NL>, dim3((unsigned)grid), dim3((NL + 2) * 32), dyn, st, g, idx, n, NS,
                    rows_per_cta, q, qmin, beta, dev_err);
}

// ---------------------------------------------------------------------------
// Transitions, persistent pipeline (large batches, n >= 2 x SMs): a CTA owns a run of
// samples; warp 0 lane 0 streams each sample's k+n unique frames (TMA, evict-first) into
// one of SPF slot groups (one mbarrier per group), warp 1 resolves every sample's stack
// sources (episode starts, §8c #13) and writes the scalars (action, fused n-step return,
// done_n, IS weight), and the consumer warps expand the two k-stacks of each sample
// (obs at window k-1, next obs at k-1+n, §8c #14) with 16-B streaming stores.  A sample's
// slot group is refilled once both of its stacks are written.  Same outputs as
// k_gather_transition (which keeps small batches: one latency chain per sample).
// ---------------------------------------------------------------------------
constexpr int TP_MAX_S = 64;  // samples per CTA
constexpr int TP_MAX_G = 8;   // slot groups (samples in flight)

template <int NC>
__global__ void __launch_bounds__((NC + 2) * 32, 1)
k_gather_trans_pipe(GDesc D, const int64_t* __restrict__ idx, int64_t n, int SPF, int spc,
                    const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, double beta, int32_t* err) {
  extern __shared__ __align__(128) uint8_t smem[];  // SPF groups of NR frame slots
  __shared__ __align__(8) uint64_t full[TP_MAX_G];
  __shared__ int s_b[TP_MAX_S];            // ring column, -1: skipped sample
  __shared__ int s_r[TP_MAX_S];            // ring row of the transition
  __shared__ int8_t ssl[TP_MAX_S][2][8];   // stack slot -> window index (-1: zero)
  __shared__ volatile int sdone[TP_MAX_S]; // stacks written (0..2)
  __shared__ int s_arm[TP_MAX_S];          // armed (loaded) samples before this one (-1: skipped)
  __shared__ int s_of_arm[TP_MAX_S];       // sample of armed index a
  __shared__ volatile int s_armed;         // armed samples issued so far (producer, release)
  constexpr int NT = (NC + 2) * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = D.k, ns = D.n_step, NR = k + ns;
  const int ob = (int)D.obs_bytes;
  const int nv = ob / 16;
  const int cap = (int)D.cap_T, Bc = (int)D.B;
  pdl_wait();
  const int64_t n_eff = active_n(D, n);
  const int64_t coff = col_off(D);
  const int64_t s0 = (int64_t)blockIdx.x * spc;
  const int64_t s1 = min(n_eff, s0 + spc);
  if (s0 >= s1) return;
  const int nsm = (int)(s1 - s0);
  if (tid == 0) {
    for (int i = 0; i < SPF; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  for (int j = tid; j < nsm; j += NT) {
    const int64_t leaf = idx[s0 + j];
    int bcol = -1, row = 0;
    if (leaf >= 0 && leaf < (int64_t)cap * Bc) {
      row = (int)(leaf / Bc);
      bcol = (int)(leaf - (int64_t)row * Bc);
      const int64_t age = wrap(D.cursor - 1 - row, D.cap_T);
      if (!(age >= ns && age <= D.size - k)) set_err(err, RPL_DERR_INVALID_LEAF);
    } else if (leaf >= (int64_t)cap * Bc) {
      set_err(err, RPL_DERR_IDX);
    }
    s_b[j] = bcol;
    s_r[j] = row;
    sdone[j] = bcol < 0 ? 2 : 0;
  }
  if (tid == 0) s_armed = 0;
  __syncthreads();
  // Slot groups and mbarrier phases follow the ARMED samples only (skipped entries — idx < 0
  // or out of range — load nothing and must not consume a phase): armed index a of sample j
  // is the number of loaded samples before it; group a % SPF, phase (a / SPF) & 1.
  if (warp == 0) {
    int base = 0;
    for (int j0 = 0; j0 < nsm; j0 += 32) {
      const int j = j0 + lane;
      const bool ok = j < nsm && s_b[j] >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      const int a = base + __popc(m & ((1u << lane) - 1u));
      if (j < nsm) s_arm[j] = ok ? a : -1;
      if (ok) s_of_arm[a] = j;
      base += __popc(m);
    }
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer ----------------
      const int64_t rstride = (int64_t)Bc * ob;
      for (int j = 0; j < nsm; ++j) {
        const int bcol = s_b[j];
        if (bcol < 0) continue;
        const int a = s_arm[j];
        const int grp = a % SPF;
        if (a >= SPF) {  // the group's previous sample must have both stacks written
          while (flag_acquire(&sdone[s_of_arm[a - SPF]]) < 2) __nanosleep(20);
          fence_proxy_async();
          mbar_wait(&full[grp], (uint32_t)(((a / SPF) - 1) & 1));  // previous phase completed
        }
        mbar_expect_tx(&full[grp], (uint32_t)(NR * ob));
        int row = s_r[j] - (k - 1);
        while (row < 0) row += cap;
        const uint8_t* col = D.obs + (int64_t)bcol * ob;
        for (int w = 0; w < NR; ++w) {
          bulk_g2s_evict_first(smem + (grp * NR + w) * ob, col + (int64_t)row * rstride, (uint32_t)ob, &full[grp]);
          if (++row == cap) row = 0;
        }
        flag_release(&s_armed, a + 1);
      }
    }
  } else if (warp == 1) {
    // ---------------- meta: stack sources, then scalars ----------------
    for (int j = lane; j < nsm; j += 32) {
      const int bcol = s_b[j];
      if (bcol < 0) continue;
      uint8_t dw[32];  // dw[w] = done[first + w - 1], w = 0..NR
      int rr = s_r[j] - k;
      while (rr < 0) rr += cap;
      for (int w = 0; w <= NR; ++w) {
        dw[w] = __ldg(D.done + (int64_t)rr * Bc + bcol);
        if (++rr == cap) rr = 0;
      }
      for (int which = 0; which < 2; ++which)
        for (int jj = 0; jj < k; ++jj) ssl[j][which][jj] = (int8_t)stack_src(dw, (k - 1) + which * ns, jj, k, D.pad_mode);
    }
    __threadfence_block();
    asm volatile("bar.arrive 1, %0;" ::"n"((NC + 1) * 32) : "memory");
    const int64_t qm = (D.o_w && q) ? warp_batch_qmin(qmin, idx, q, n) : 0;
    for (int j = lane; j < nsm; j += 32) {
      const int bcol = s_b[j];
      if (bcol < 0) continue;
      const int64_t sc = coff + s0 + j;
      const int64_t r = s_r[j];
      if (D.o_act) coop_copy(D.o_act + sc * D.act_bytes, D.act + (r * Bc + bcol) * D.act_bytes, D.act_bytes, 0, 1);
      if (D.o_ret || D.o_done_n) {  // fused n-step return (R24, R34)
        uint8_t dn = 0;
        const double acc = nstep_rows(D, r, bcol, ns, 0.0, &dn);
        if (D.o_ret) D.o_ret[sc] = (float)acc;
        if (D.o_done_n) D.o_done_n[sc] = dn ? 1 : 0;
      }
      if (D.o_w && q) {
        const int64_t qs = q[s0 + j];
        D.o_w[sc] = qs > 0 ? (float)pow((double)qm / (double)qs, beta) : 0.0f;
      }
    }
  } else {
    // ---------------- consumers: one k-stack per item (sample, which) ----------------
    asm volatile("bar.sync 1, %0;" ::"n"((NC + 1) * 32) : "memory");
    for (int it = warp - 2; it < 2 * nsm; it += NC) {
      const int j = it >> 1, which = it & 1;
      if (s_b[j] < 0) continue;
      uint8_t* outb = which ? D.o_next_obs : D.o_obs;
      const int a = s_arm[j];
      const int grp = a % SPF;
      // wait until this sample's phase is armed (a consumer warp may run ahead of the warps
      // still on the group's previous sample: a bare parity test could then match the phase
      // two rounds old), then observe it — even without an output, so no CTA exits with
      // bulk copies into its shared memory still in flight
      while (flag_acquire(&s_armed) <= a) __nanosleep(20);
      mbar_wait(&full[grp], (uint32_t)((a / SPF) & 1));
      if (outb) {
        int4* dst = reinterpret_cast<int4*>(outb + (coff + s0 + j) * (int64_t)k * ob);
        for (int jj = 0; jj < k; ++jj) {
          int4* d = dst + jj * nv;
          const int src = ssl[j][which][jj];
          if (src < 0) {
            for (int v = lane; v < nv; v += 32) __stcs(d + v, make_int4(0, 0, 0, 0));
          } else {
            const int4* sp = reinterpret_cast<const int4*>(smem + (grp * NR + src) * ob);
#pragma unroll 4
            for (int v = lane; v < nv; v += 32) __stcs(d + v, sp[v]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        asm volatile("red.release.cta.shared::cta.add.s32 [%0], 1;" ::"r"(smem_u32((const void*)&sdone[j]))
                     : "memory");
      }
    }
  }
  pdl_trigger();
}

// Work-skipping diagnostics (rpl_debug_set_gather_diag, RPL_GATHER_DIAG) exist only in a
// -DRPL_DIAG build; in the default build GDIAG() is the constant 0 and the branches compile out.
#ifdef RPL_DIAG
int env_diag() {
  const char* v = getenv("RPL_GATHER_DIAG");  // measurement only (rpl_debug_set_gather_diag)
  return v ? atoi(v) : 0;
}
int g_seq_diag = env_diag();
#else
int g_seq_diag = 0;
#endif

GDesc to_dev(const rpl_gather_desc* d) {
  GDesc g;
  g.kind = d->kind;
  g.pad_mode = d->pad_mode;
  g.out_mode = d->out_mode;
  g.k = d->k;
  g.cap_T = d->cap_T;
  g.B = d->B;
  g.cursor = d->cursor;
  g.size = d->size;
  g.obs_bytes = d->obs_bytes;
  g.act_bytes = d->act_bytes;
  g.rnn_bytes = d->rnn_bytes;
  g.n_step = d->n_step;
  g.seq_len = d->seq_len;
  g.period = d->period;
  g.rnn_parts = d->rnn_parts;
  g.gamma = d->gamma;
  g.obs = static_cast<const uint8_t*>(d->obs);
  g.act = static_cast<const uint8_t*>(d->act);
  g.rew = d->rew;
  g.done = d->done;
  g.rnn = static_cast<const uint8_t*>(d->rnn);
  g.o_obs = static_cast<uint8_t*>(d->o_obs);
  g.o_next_obs = static_cast<uint8_t*>(d->o_next_obs);
  g.o_act = static_cast<uint8_t*>(d->o_act);
  g.o_prev_act = static_cast<uint8_t*>(d->o_prev_act);
  g.o_rew = d->o_rew;
  g.o_prev_rew = d->o_prev_rew;
  g.o_done = d->o_done;
  g.o_ret = d->o_ret;
  g.o_done_n = d->o_done_n;
  g.o_w = d->o_w;
  g.o_rnn = static_cast<uint8_t*>(d->o_rnn);
  g.use_tma = 0;
  g.diag = g_seq_diag;
  g.n_active = d->n_active;
  g.col_offset = d->col_offset;
  g.o_start = d->o_start;
  g.peer_boards = d->peer_boards;
  g.peer_world = d->peer_world;
  g.peer_rank = d->peer_rank;
  g.q_tgt = d->q_tgt;
  g.o_tgt = d->o_tgt;
  g.o_tgt_done = d->o_tgt_done;
  g.tgt_lo = d->tgt_lo;
  g.tgt_T = d->tgt_T;
  g.rescale = d->rescale;
  g.rescale_eps = d->rescale_eps;
  g.v_term = d->v_term;
  g.done_flag = d->done_flag;
  g.done_seq = d->done_seq;
  g.work = d->work;
  g.upd_idx = nullptr;
  g.upd_td = nullptr;
  g.upd_n = g.upd_T = g.upd_live = g.upd_pad = 0;
  g.upd_eta = g.upd_alpha = g.upd_eps = 0.0;
  g.smp_tree = nullptr;
  g.smp_seed = 0;
  return g;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }


// 0: TMA-load / LSU-store pipeline (default, RPL_SEQ_CONSUMERS = 4 consumer warps; 4: 14, 5: 8), 1: chunked all-TMA kernel, 2: frame-centric
// LSU, 3: all-TMA pipeline
int g_seq_variant = 0;
// Consumer warps of the default sequence gather (build-flag A/B knob).  Same-box A/B of the
// R2D2 step (scripts/ab_flags.sh, 3 rounds; profiles/r1/README.md): 4 -> 68.88 us, 6 -> 69.04,
// 8 -> 69.29, 5 -> 69.77; back to back the gather alone prefers 8, inside the step 4 wins.
#ifndef RPL_SEQ_CONSUMERS
#define RPL_SEQ_CONSUMERS 4
#endif

}  // namespace
}  // namespace rpl

using namespace rpl;

extern "C" int rpl_debug_gather_trace_reset(void) {
#ifdef RPL_TRACE
  unsigned long long z[9] = {0, 0, 0, 0, ~0ull, ~0ull, 0, 0, ~0ull};
  return cudaMemcpyToSymbol(rpl::g_gtrace, z, sizeof(z)) == cudaSuccess ? RPL_OK : RPL_ECUDA;
#else
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_gather_cta_ends(int64_t* out, int32_t n) {
#ifdef RPL_TRACE
  if (!out || n < 1 || n > 512) return RPL_EINVAL;
  // out[0..n): CTA ends; out[n..2n): static-rows-stored times; out[2n..3n): dynamic units taken
  return (cudaMemcpyFromSymbol(out, rpl::g_gend, sizeof(int64_t) * (size_t)n) == cudaSuccess &&
          cudaMemcpyFromSymbol(out + n, rpl::g_gstatic, sizeof(int64_t) * (size_t)n) == cudaSuccess &&
          cudaMemcpyFromSymbol(out + 2 * n, rpl::g_gunits, sizeof(int64_t) * (size_t)n) == cudaSuccess)
             ? RPL_OK : RPL_ECUDA;
#else
  (void)out;
  (void)n;
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_gather_grabs(int64_t* out, int32_t n) {
#ifdef RPL_TRACE
  if (!out || n < 1 || n > 512) return RPL_EINVAL;
  return cudaMemcpyFromSymbol(out, rpl::g_ggrab, sizeof(int64_t) * 16 * (size_t)n) == cudaSuccess ? RPL_OK : RPL_ECUDA;
#else
  (void)out;
  (void)n;
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_gather_trace(int64_t* out, int32_t n) {
#ifdef RPL_TRACE
  if (!out || n < 1 || n > 9) return RPL_EINVAL;
  return cudaMemcpyFromSymbol(out, rpl::g_gtrace, sizeof(int64_t) * (size_t)n) == cudaSuccess ? RPL_OK : RPL_ECUDA;
#else
  (void)out;
  (void)n;
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_set_gather_dyn(int32_t pct, int32_t rows, int32_t lookahead) {
  if (pct == 2000 || pct == 2001) {  // measurement: the fused-update instantiation for every launch
    g_dyn_updk.store(pct - 2000);
    return RPL_OK;
  }
  if (pct >= 1000 && pct <= 1000 + PIPE_MAX_NS) {  // measurement: early first-frame loads (count, 0 = off)
    g_dyn_early.store(pct - 1000);
    return RPL_OK;
  }
  // lookahead: the queue (1-200), optionally | (end-of-pool queue << 8) | (its threshold in rows << 16)
  if (pct < -1 || pct > 100 || rows < 1 || rows > 32 || (lookahead & 0xff) < 1 || (lookahead & 0xff) > 200 ||
      ((lookahead >> 8) & 0xff) > 200 || lookahead < 0)
    return RPL_EINVAL;
  g_dyn_pct.store(pct);
  g_dyn_rows.store(rows);
  g_dyn_look.store(lookahead);
  return RPL_OK;
}

extern "C" int rpl_debug_set_gather_trigger(int32_t at) {
  if (at < -1 || at > 1) return RPL_EINVAL;
  g_gather_trigger.store(at);
  return RPL_OK;
}

extern "C" int rpl_debug_set_gather_variant(int32_t variant) {
  if (variant < 0 || variant > 6) return RPL_EINVAL;
  g_seq_variant = variant;
  return RPL_OK;
}

extern "C" int rpl_debug_set_gather_diag(int32_t mask) {
  if (mask < 0 || mask > 31) return RPL_EINVAL;
#ifdef RPL_DIAG
  g_seq_diag = mask;
  return RPL_OK;
#else
  return mask == 0 ? RPL_OK : RPL_EUNSUPPORTED;  // default build: diagnostics compiled out
#endif
}

namespace rpl {
void cfg_gather(int* variant, int* diag, int* diag_build, int* seq_consumers, int* trans_consumers, int* slot_kb,
                int* g_threads) {  // knob state for rpl_config (abi.cu)
  *variant = g_seq_variant;
  *diag = g_seq_diag;
#ifdef RPL_DIAG
  *diag_build = 1;
#else
  *diag_build = 0;
#endif
  *seq_consumers = RPL_SEQ_CONSUMERS;
  *trans_consumers = RPL_TRANS_CONSUMERS;
  *slot_kb = RPL_SEQ_SLOT_KB;
  *g_threads = G_THREADS;
}
}  // namespace rpl

namespace rpl {
namespace {
struct SmpArgs {
  int64_t* tree;
  TreeDev L;
  uint64_t seed;
  // fused update (rpl_gather_update_sample; upd_td NULL: none)
  const int64_t* upd_idx = nullptr;
  const float* upd_td = nullptr;
  int upd_n = 0, upd_T = 0, upd_live = 0;
  double upd_eta = 0.0, upd_alpha = 0.0, upd_eps = 0.0;
};
int gather_run(const rpl_gather_desc* desc, const int64_t* idx, const int64_t* q, const int64_t* qmin, double beta,
               int64_t n, int32_t* dev_err, void* stream, const SmpArgs* smp);
}  // namespace
}  // namespace rpl

extern "C" int rpl_gather(const rpl_gather_desc* desc, const int64_t* idx, const int64_t* q, const int64_t* qmin,
                          double beta, int64_t n, int32_t* dev_err, void* stream) {
  return gather_run(desc, idx, q, qmin, beta, n, dev_err, stream, nullptr);
}

extern "C" int rpl_sumtree_update_seq(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                                      const float* td_steps, int64_t T_p, int64_t n, double eta, double alpha,
                                      double eps_p, int32_t flags, int32_t* dev_err, void* stream);

extern "C" int rpl_gather_update_sample(const rpl_gather_desc* desc, const rpl_tree_layout* L, int64_t* tree,
                                        const int64_t* upd_idx, const float* upd_td, int64_t T_p, int64_t n_upd,
                                        double eta, double alpha, double eps_p, int32_t flags, uint64_t seed,
                                        int64_t* idx_out, int64_t* q_out, double beta, int64_t n, int32_t* dev_err,
                                        void* stream) {
  if (!desc || !L || !tree || !idx_out || !q_out || n < 1 || n > (1ll << 30) || n_upd < 0) return RPL_EINVAL;
  if (n_upd > 0 && (!upd_idx || !upd_td || T_p < 1 || T_p > (1ll << 30))) return RPL_EINVAL;
  if (!(alpha >= 0.0) || !(eps_p >= 0.0) || !(eta >= 0.0 && eta <= 1.0) || (flags & ~RPL_UPD_LIVE_ONLY))
    return RPL_EINVAL;
  if (desc->kind != RPL_GATHER_SEQUENCE || desc->n_active || desc->col_offset || desc->peer_boards || desc->done_flag)
    return RPL_EINVAL;
  if (desc->period < 1 || desc->cap_T % desc->period != 0 || L->n_leaves != (desc->cap_T / desc->period) * desc->B)
    return RPL_EINVAL;
  SmpArgs a;
  a.tree = tree;
  a.L = tree_dev(L);
  a.seed = seed;
  // one launch when the dynamic-tail kernel runs, the batch fits its tables and every internal
  // level fits the staging area (alpha 0 / 1 and an empty batch: the two-launch form)
  int NS = (int)(RPL_SEQ_SLOT_KB * 1024 / (desc->obs_bytes > 0 ? desc->obs_bytes : 1));
  if (NS > PIPE_MAX_NS) NS = PIPE_MAX_NS;
  const bool fits = n_upd >= 1 && n_upd <= UF_MAX && L->depth >= 1 &&
                    L->level_off[L->depth] <= (int64_t)(NS - 1) * desc->obs_bytes / 8;
  if (fits) {
    a.upd_idx = upd_idx;
    a.upd_td = upd_td;
    a.upd_n = (int)n_upd;
    a.upd_T = (int)T_p;
    a.upd_live = (flags & RPL_UPD_LIVE_ONLY) ? 1 : 0;
    a.upd_eta = eta;
    a.upd_alpha = alpha;
    a.upd_eps = eps_p;
    const int rc = gather_run(desc, idx_out, q_out, nullptr, beta, n, dev_err, stream, &a);
    if (rc != RPL_EUNSUPPORTED) return rc;  // RPL_EUNSUPPORTED: nothing was enqueued
    a.upd_td = nullptr;
  }
  const int rc = rpl_sumtree_update_seq(L, tree, upd_idx, upd_td, T_p, n_upd, eta, alpha, eps_p, flags, dev_err,
                                        stream);
  if (rc != RPL_OK) return rc;
  return gather_run(desc, idx_out, q_out, nullptr, beta, n, dev_err, stream, &a);
}

extern "C" int rpl_gather_sample(const rpl_gather_desc* desc, const rpl_tree_layout* L, int64_t* tree, uint64_t seed,
                                 int64_t* idx_out, int64_t* q_out, double beta, int64_t n, int32_t* dev_err,
                                 void* stream) {
  if (!desc || !L || !tree || !idx_out || !q_out || n < 1 || n > (1ll << 30)) return RPL_EINVAL;
  if (desc->kind != RPL_GATHER_SEQUENCE || desc->n_active || desc->col_offset || desc->peer_boards || desc->done_flag)
    return RPL_EINVAL;
  if (desc->period < 1 || desc->cap_T % desc->period != 0 || L->n_leaves != (desc->cap_T / desc->period) * desc->B)
    return RPL_EINVAL;
  SmpArgs a;
  a.tree = tree;
  a.L = tree_dev(L);
  a.seed = seed;
  return gather_run(desc, idx_out, q_out, nullptr, beta, n, dev_err, stream, &a);
}

namespace rpl {
namespace {
int gather_run(const rpl_gather_desc* desc, const int64_t* idx, const int64_t* q, const int64_t* qmin, double beta,
               int64_t n, int32_t* dev_err, void* stream, const SmpArgs* smp) {
  if (!desc || n < 0) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  if (!idx || !desc->done || !desc->obs || desc->cap_T < 1 || desc->B < 1 || desc->k < 1 || desc->k > 8 ||
      desc->obs_bytes < 1 || desc->size < 0 || desc->size > desc->cap_T || desc->cursor < 0 ||
      desc->cursor >= desc->cap_T)
    return RPL_EINVAL;
  if (desc->pad_mode != RPL_PAD_REPEAT && desc->pad_mode != RPL_PAD_ZERO) return RPL_EINVAL;
  if ((desc->o_act || desc->o_prev_act) && (!desc->act || desc->act_bytes < 1)) return RPL_EINVAL;
  if (desc->o_w && !(beta >= 0.0)) return RPL_EINVAL;
  if (desc->peer_boards && (desc->kind != RPL_GATHER_SEQUENCE || qmin || !q || !desc->o_w || desc->peer_world < 1 ||
                            desc->peer_world > BOARD_MAX_WORLD || desc->peer_rank < 0 ||
                            desc->peer_rank >= desc->peer_world))
    return RPL_EINVAL;
  if (desc->o_tgt && (desc->kind != RPL_GATHER_SEQUENCE || !desc->rew || desc->n_step < 1 || desc->n_step > 64 ||
                      desc->tgt_lo < 0 || desc->tgt_T < 1 ||
                      (int64_t)desc->tgt_lo + desc->tgt_T + desc->n_step > desc->seq_len ||
                      !(desc->rescale_eps >= 0.0) || (desc->rescale != 0 && desc->rescale != 1)))
    return RPL_EINVAL;
  GDesc g = to_dev(desc);
  if (smp) {
    g.smp_tree = smp->tree;
    g.smp_L = smp->L;
    g.smp_seed = smp->seed;
    g.upd_idx = smp->upd_idx;
    g.upd_td = smp->upd_td;
    g.upd_n = smp->upd_n;
    g.upd_T = smp->upd_T;
    g.upd_live = smp->upd_live;
    g.upd_eta = smp->upd_eta;
    g.upd_alpha = smp->upd_alpha;
    g.upd_eps = smp->upd_eps;
  }
  const bool fused_upd = smp && smp->upd_td != nullptr;
  // col_offset / o_start / peer boards / fused targets / fused sampling: default kernels only
  if ((desc->done_flag != nullptr) != (desc->done_seq != nullptr)) return RPL_EINVAL;
  const int seq_variant =
      (desc->col_offset || desc->o_start || desc->peer_boards || desc->o_tgt || desc->done_flag || smp)
          ? 0
          : g_seq_variant;
  const bool tma_ok = (desc->obs_bytes % 16 == 0) && aligned16(desc->obs) && aligned16(desc->o_obs) &&
                      aligned16(desc->o_next_obs) && desc->obs_bytes <= 32768;
  cudaStream_t st = as_stream(stream);
  if (desc->kind == RPL_GATHER_TRANSITION) {
    if (desc->n_step < 1 || desc->k + desc->n_step > 31) return RPL_EINVAL;
    if ((desc->o_ret || desc->o_done_n) && !desc->rew) return RPL_EINVAL;
    const int NR = desc->k + desc->n_step;
    // large batches: persistent pipeline (several samples per CTA, loads overlapping stores)
    if (tma_ok && (desc->o_obs || desc->o_next_obs) && seq_variant != 1 && n >= 2 * (int64_t)sm_count() &&
        NR <= 30 && desc->k <= 8) {
      int SPF = (int)(200 * 1024 / ((int64_t)NR * desc->obs_bytes));
      if (SPF > TP_MAX_G) SPF = TP_MAX_G;
      int64_t spc = (n + sm_count() - 1) / sm_count();
      if (SPF >= 2 && spc <= TP_MAX_S) {
        const size_t dyn = (size_t)SPF * NR * desc->obs_bytes;
        ensure_smem(reinterpret_cast<const void*>(k_gather_trans_pipe<RPL_TRANS_CONSUMERS>), dyn);
        const int64_t grid = (n + spc - 1) / spc;
        g.use_tma = 1;
        return launch_pdl(k_gather_trans_pipe<RPL_TRANS_CONSUMERS>, dim3((unsigned)grid),
                          dim3((RPL_TRANS_CONSUMERS + 2) * 32), dyn, st, g, idx, n, SPF,
                          (int)spc, q, qmin, beta, dev_err);
      }
    }
    const int64_t smem = (int64_t)(NR + 1) * desc->obs_bytes;
    g.use_tma = (tma_ok && smem <= 200 * 1024) ? 1 : 0;
    const size_t dyn = g.use_tma ? (size_t)smem : 0;
    ensure_smem(reinterpret_cast<const void*>(k_gather_transition), dyn);
    if (n > 0x7fffffff) return RPL_EINVAL;
    return launch_pdl(k_gather_transition, dim3((unsigned)n), dim3(G_THREADS), dyn, st, g, idx, n, q, qmin, beta,
                      dev_err);
  }
  if (desc->kind == RPL_GATHER_SEQUENCE) {
    if (desc->seq_len < 1 || desc->period < 1 || desc->cap_T % desc->period != 0) return RPL_EINVAL;
    if (desc->o_rnn && (!desc->rnn || desc->rnn_parts < 1 || desc->rnn_bytes < 1)) return RPL_EINVAL;
    if ((desc->o_rew || desc->o_prev_rew) && !desc->rew) return RPL_EINVAL;
    if (desc->out_mode != RPL_OUT_STACKED && desc->out_mode != RPL_OUT_UNIQUE) return RPL_EINVAL;
    if (SEQ_CHUNK + desc->k > 32) return RPL_EINVAL;
    if (tma_ok && desc->out_mode == RPL_OUT_STACKED && desc->o_obs && seq_variant == 2 &&
        desc->obs_bytes <= 16 * 32 * FC_MAX_V4 * 4) {
      const int64_t tasks = n * (int64_t)(desc->seq_len + desc->k - 1);
      k_gather_seq_lsu<<<(unsigned)((tasks + FC_WARPS - 1) / FC_WARPS), FC_WARPS * 32, 0, st>>>(g, idx, n, q, qmin,
                                                                                               beta, dev_err);
      int r = launch_status();
      if (r != RPL_OK) return r;
      const int64_t rows = n * (int64_t)desc->seq_len;
      k_gather_seq_fields<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(g, idx, n, dev_err);
      return launch_status();
    }
    if (tma_ok && desc->out_mode == RPL_OUT_STACKED && desc->o_obs && seq_variant == 6) {
      int NS = (int)(200 * 1024 / desc->obs_bytes) - 1;  // + one zero slot
      if (NS > PIPE_MAX_NS) NS = PIPE_MAX_NS;
      const int k = desc->k;
      const int64_t total = n * (int64_t)desc->seq_len;
      if (NS >= LB_G + 3 * k && total < (1ll << 30) && desc->cap_T < (1ll << 30) && desc->B < (1ll << 30)) {
        const size_t dyn = (size_t)(NS + 1) * desc->obs_bytes;
        int64_t grid = (int64_t)sm_count();
        int64_t rows_per_cta = (total + grid - 1) / grid;
        if (rows_per_cta > PL_MAX_ROWS) rows_per_cta = PL_MAX_ROWS;
        grid = (total + rows_per_cta - 1) / rows_per_cta;
        g.use_tma = 1;
        return launch_seq_ldg_bulk<8>(g, idx, n, NS, rows_per_cta, q, qmin, beta, dev_err, dyn, grid, st);
      }
    }
    if (tma_ok && desc->o_obs && (seq_variant == 0 || seq_variant == 4 || seq_variant == 5)) {
      // default: TMA-load / LSU-store pipeline.  The producer runs up to NS frames past the
      // release point of the done-frontier row f, whose own window starts exactly there, so
      // NS >= k guarantees progress; more slots let the other consumers run ahead.
      int NS = (int)(RPL_SEQ_SLOT_KB * 1024 / desc->obs_bytes);
      if (NS > PIPE_MAX_NS) NS = PIPE_MAX_NS;
      const int k = desc->k;
      const int64_t total = n * (int64_t)desc->seq_len;
      if (NS >= 2 * k && total < (1ll << 30) && desc->cap_T < (1ll << 30) && desc->B < (1ll << 30) &&
          desc->cap_T * desc->B < (1ll << 40)) {
        const size_t dyn = (size_t)NS * desc->obs_bytes;
        int64_t grid = (int64_t)sm_count();
        // dynamic tail (rpl_gather_desc.work): one learner's whole batch only
        const int dpct = g_dyn_pct.load(std::memory_order_relaxed);
        const int drows = g_dyn_rows.load(std::memory_order_relaxed);
        // (stacked output only: unique rows are 4x cheaper, and the per-grab latency then costs
        // more than the balance gains — the unique-output step measured 33.5 -> 43.4 us)
        if (desc->work && dpct >= 0 && !desc->col_offset && !desc->n_active && !desc->peer_boards &&
            !desc->done_flag && seq_variant == 0 && desc->out_mode == RPL_OUT_STACKED &&
            n <= (1 << 30) / desc->seq_len) {
          // two SMs stay free for kernels running beside the gather (the pipelined step's
          // update + sampler on a second stream), as with the static split's 146 CTAs
          const int64_t gd = grid > 8 ? grid - 2 : grid;
          int64_t rs = total * dpct / 100 / gd;
          if (rs > DY_MAX_ROWS - 4 * drows) rs = DY_MAX_ROWS - 4 * drows;
          // capacity: a CTA holds at most DY_MAX_ROWS rows and DY_MAX_PIECES pieces (its static
          // pieces, then at most two per grab of >= 2 rows), so every row is taken only if the
          // static pieces leave half the piece table and the dynamic rows fit what the grid can
          // still take; otherwise the static split (any size)
          const int64_t ldyn = total - gd * rs;
          if (rs / desc->seq_len + 2 <= DY_MAX_PIECES / 2 && ldyn <= gd * (DY_MAX_PIECES / 2 - 2) &&
              total <= gd * (DY_MAX_ROWS - 2 * drows)) {
            g.use_tma = 1;
            return launch_seq_dyn<RPL_SEQ_CONSUMERS>(g, idx, n, NS, (int)rs, drows,
                                                     g_dyn_look.load(std::memory_order_relaxed), q, qmin, beta,
                                                     dev_err, dyn, gd, st);
          }
        }
        if (fused_upd) return RPL_EUNSUPPORTED;  // the fused update needs the dynamic-tail kernel
        int64_t rows_per_cta = (total + grid - 1) / grid;
        if (rows_per_cta > PL_MAX_ROWS) rows_per_cta = PL_MAX_ROWS;
        grid = (total + rows_per_cta - 1) / rows_per_cta;
        g.use_tma = 1;
        // consumer warps: RPL_SEQ_CONSUMERS (default), 14 (variant 4), 8 (variant 5)
        if (seq_variant == 4) return launch_seq_lsu<14>(g, idx, n, NS, rows_per_cta, q, qmin, beta, dev_err, dyn,
                                                          grid, st);
        if (seq_variant == 5) return launch_seq_lsu<8>(g, idx, n, NS, rows_per_cta, q, qmin, beta, dev_err, dyn,
                                                         grid, st);
        return launch_seq_lsu<RPL_SEQ_CONSUMERS>(g, idx, n, NS, rows_per_cta, q, qmin, beta, dev_err, dyn, grid,
                                                 st);
      }
    }
    if (fused_upd) return RPL_EUNSUPPORTED;  // nothing enqueued: the caller runs the two-launch form
    if (tma_ok && desc->out_mode == RPL_OUT_STACKED && desc->o_obs &&
        (seq_variant == 3 ||
         (seq_variant == 0 && !desc->col_offset && !desc->o_start && !desc->peer_boards && !desc->o_tgt &&
          !desc->done_flag && !smp))) {
      // persistent TMA pipeline: NS frame slots (+1 zero slot); CTAs_per_SM CTAs per SM
      // Slots the consumer may need beyond the released ones: G+1 rows of advance, the
      // k-1 window, and k-1 per piece boundary crossed.  With L > G at most two boundaries
      // fall in G+1 consecutive rows (a CTA's short first and last pieces): NS >= G + 3k - 2.
      // Otherwise every row may open a piece: NS >= (G+1) k + k.
      int NS = (int)(216 * 1024 / desc->obs_bytes) - 1;
      if (NS > PIPE_MAX_NS) NS = PIPE_MAX_NS;
      const int k = desc->k, L = desc->seq_len;
      int G = 0;
      if (L > 16 && NS >= 16 + 3 * k - 2) G = 16;
      else if (NS >= 5 * k + k) G = 4;
      if (G > 0) {
        const size_t dyn = (size_t)(NS + 1) * desc->obs_bytes;
        ensure_smem(reinterpret_cast<const void*>(k_gather_seq_pipe<16>), dyn);
        ensure_smem(reinterpret_cast<const void*>(k_gather_seq_pipe<4>), dyn);
        const int64_t total = n * (int64_t)desc->seq_len;
        int64_t grid = (int64_t)sm_count();
        int64_t rows_per_cta = (total + grid - 1) / grid;
        if (rows_per_cta > PIPE_MAX_ROWS) rows_per_cta = PIPE_MAX_ROWS;
        grid = (total + rows_per_cta - 1) / rows_per_cta;
        g.use_tma = 1;
        if (G == 16)
          k_gather_seq_pipe<16><<<(unsigned)grid, PIPE_THREADS, dyn, st>>>(g, idx, n, NS, rows_per_cta, q, qmin,
                                                                             beta, dev_err);
        else
          k_gather_seq_pipe<4><<<(unsigned)grid, PIPE_THREADS, dyn, st>>>(g, idx, n, NS, rows_per_cta, q, qmin,
                                                                            beta, dev_err);
        return launch_status();
      }
    }
    if (desc->o_start || desc->peer_boards || desc->o_tgt || desc->done_flag || smp)
      return RPL_EUNSUPPORTED;  // persistent default kernel only
    const int64_t smem = (int64_t)(SEQ_CHUNK + desc->k) * desc->obs_bytes;
    g.use_tma = (tma_ok && smem <= 200 * 1024) ? 1 : 0;
    const size_t dyn = g.use_tma ? (size_t)smem : 0;
    ensure_smem(reinterpret_cast<const void*>(k_gather_sequence), dyn);
    const int rows_out = desc->out_mode == RPL_OUT_STACKED ? desc->seq_len : desc->seq_len + desc->k - 1;
    const int chunks = (rows_out + SEQ_CHUNK - 1) / SEQ_CHUNK;
    if (n > 65535) return RPL_EINVAL;
    dim3 grid((unsigned)chunks, (unsigned)n);
    k_gather_sequence<<<grid, G_THREADS, dyn, st>>>(g, idx, n, q, qmin, beta, dev_err);
    return launch_status();
  }
  return RPL_EINVAL;
}
}  // namespace
}  // namespace rpl

// ---------------------------------------------------------------------------
// k-stacks from unique rows (Mode C learner side, §8e): out[tau, s] slot j = unique row
// tau + max(j, start[tau, s]) of sample s (zero when j < start and pad_mode is ZERO) —
// the same frame-stacking-wrapper rule (§8c #13) the gather applies, with the episode
// starts computed by the owners (rpl_gather_desc.o_start).  One warp per output stack;
// its k source rows are the neighbours' too, so they come mostly from L1/L2.
// ---------------------------------------------------------------------------
namespace rpl {
namespace {
constexpr int ST_WARPS = 8;

__global__ void __launch_bounds__(ST_WARPS * 32)
k_stack_frames(const uint8_t* __restrict__ uniq, const int8_t* __restrict__ start, int L, int64_t n, int k,
               int64_t ob, int pad_mode, uint8_t* __restrict__ out, const int64_t* __restrict__ n_active) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int tau = blockIdx.x * ST_WARPS + (threadIdx.x >> 5);
  const int64_t s = blockIdx.y;
  const int64_t na = n_active ? *n_active : n;
  if (tau >= L || s >= na) return;
  const int so = start[(int64_t)tau * n + s];
  const int nv = (int)(ob / 16);
  int4* dst = reinterpret_cast<int4*>(out + (((int64_t)tau * n + s) * k) * ob);
  for (int j = 0; j < k; ++j) {
    int4* d = dst + (int64_t)j * nv;
    if (j < so && pad_mode == RPL_PAD_ZERO) {
      for (int v = lane; v < nv; v += 32) __stcs(d + v, make_int4(0, 0, 0, 0));
    } else {
      const int u = tau + (j < so ? so : j);
      const int4* src = reinterpret_cast<const int4*>(uniq + ((int64_t)u * n + s) * ob);
#pragma unroll 4
      for (int v = lane; v < nv; v += 32) __stcs(d + v, __ldg(src + v));
    }
  }
}
}  // namespace
}  // namespace rpl

extern "C" int rpl_stack_frames(const void* uniq, const int8_t* start, int64_t L, int64_t n, int32_t k,
                                int64_t obs_bytes, int32_t pad_mode, void* out, const int64_t* n_active,
                                void* stream) {
  if (!uniq || !start || !out || L < 1 || n < 0 || k < 1 || k > 8 || obs_bytes < 16 || (obs_bytes & 15) ||
      (reinterpret_cast<uintptr_t>(uniq) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) || L > (1 << 30) ||
      n > 65535 || (pad_mode != RPL_PAD_REPEAT && pad_mode != RPL_PAD_ZERO))
    return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const dim3 grid((unsigned)((L + ST_WARPS - 1) / ST_WARPS), (unsigned)n);
  return launch_pdl(k_stack_frames, grid, dim3(ST_WARPS * 32), 0, as_stream(stream),
                    static_cast<const uint8_t*>(uniq), start, (int)L, n, (int)k, obs_bytes, (int)pad_mode,
                    static_cast<uint8_t*>(out), n_active);
}

// ---------------------------------------------------------------------------
// Learner-side wait for the owners' completion signals (Mode C, §8e): lane i spins with
// ld.acquire.sys until flags[i] >= *expect (the learner's own call counter, bumped by its own
// gather earlier on this stream), then the warp issues a system-scope fence so the next
// kernel on the stream reads the owners' peer stores.  A peer that does not signal within
// ~2 s is a failed exchange: RPL_DERR_PEER is set and the kernel traps, so the error
// surfaces at the next synchronisation instead of a silently incomplete batch.
// ---------------------------------------------------------------------------
namespace rpl {
namespace {
__global__ void k_wait_flags(const int64_t* flags, int n, const int64_t* expect, int32_t* err) {
  pdl_wait();
  const int64_t want = *expect;
  for (int i = threadIdx.x; i < n; i += 32) {
    const uint64_t t0 = global_ns();
    while (true) {
      int64_t v;
      asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
      if (v >= want) break;
      if (global_ns() - t0 > 2000000000ull) {
        board_fail(err);
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence_system();
  pdl_trigger();
}
}  // namespace
}  // namespace rpl

extern "C" int rpl_wait_flags(const int64_t* flags, int32_t n, const int64_t* expect, int32_t* dev_err,
                              void* stream) {
  if (!flags || !expect || n < 1 || n > 1024) return RPL_EINVAL;
  return launch_pdl(k_wait_flags, dim3(1), dim3(32), 0, as_stream(stream), flags, (int)n, expect, dev_err);
}
