// Prioritized replay on a wide int64 fixed-point sum tree.
//
// P:38 "prioritized replay (sum tree)"; S:553-629 (tree, sampling, IS weights,
// priority updates); S:660 (max-priority-seen); readings §8c #7-#12, #17.
//
// Layout (rpl.h): levels root..leaves, fan-out W (<= 32, one warp lane per child),
// every level padded to a multiple of W; leaf q_i = RNE(RN32(p_i^alpha) 2^F).
// Integer sums make propagation order-independent and bit-exact.
//
//  update  one CTA: priority transform (crpow.cuh) -> last-writer-wins dedupe in a
//          shared-memory hash table (atomicMax of batch position per leaf) -> the
//          winner writes its leaf and adds its int64 delta to each ancestor
//          (root delta warp-aggregated).  Chunks of 512 entries (the CTA size) are applied in
//          batch order, so any batch size keeps last-write-wins.
//  sample  one warp per draw: integer stratum -> prefix -> per level the warp loads
//          the W child sums (one coalesced 256-B load), inclusive int64 warp scan,
//          ballot(prefix < incl) picks the child.  The last CTA (ticket in the tree
//          header) reduces the batch-min q and writes the IS weights (a9).
#include <math.h>
#include <stdlib.h>

#include <atomic>

#include "common.cuh"
#include "crpow.cuh"

namespace rpl {
namespace {

#ifndef RPL_UPD_THREADS  // build-flag knobs for A/B measurement (scripts/ab_flags.sh)
#define RPL_UPD_THREADS 512  // same-box A/B: 68.87 vs 69.25 us per R2D2 step at 1024 (256: two td passes, +1.1 us)
#endif
#ifndef RPL_SAMPLE_WARPS
#define RPL_SAMPLE_WARPS 4  // same-box A/B: R2D2 step 69.06 vs 69.20 us at 8; DQN bs32 / 512 step 15.67 / 22.00 vs 15.83 / 22.14
#endif
constexpr int UPD_THREADS = RPL_UPD_THREADS;
#ifndef RPL_UPD_SINGLE  // build-flag A/B knob: 0 = every batch through the chunked update
#define RPL_UPD_SINGLE 1
#endif
#ifndef RPL_HASH_SLOTS  // build-flag A/B knob (>= 2 x the update chunk, a power of two)
#define RPL_HASH_SLOTS 2048
#endif
constexpr int HASH_SLOTS = RPL_HASH_SLOTS;
constexpr unsigned long long HASH_EMPTY = ~0ull;
constexpr int SAMPLE_WARPS = RPL_SAMPLE_WARPS;
// Shared-memory staging of the tree's top levels in the sampler (34 KB): R2D2 1M-step
// (25,600 leaves) stages root + 2 levels, DQN 2^20 leaves root + 2 of 4, toy trees all.
#ifndef RPL_STAGE_WORDS  // build-flag A/B knob
#define RPL_STAGE_WORDS 4352
#endif
constexpr int STAGE_WORDS = RPL_STAGE_WORDS;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Words of the tree the sampler may stage (0 = none: base not 16-B aligned for the
// 16-B async copies, or RPL_TREE_STAGE=0 for A/B measurement).  The copy of an odd last
// word reads one word past the staged levels, which is still inside the tree (header).
std::atomic<int> g_tree_stage{-1};  // -1: not set yet (read RPL_TREE_STAGE once)

int tree_stage_on() {
  int on = g_tree_stage.load(std::memory_order_relaxed);
  if (on < 0) {
    const char* e = getenv("RPL_TREE_STAGE");
    int expect = -1;
    g_tree_stage.compare_exchange_strong(expect, (e && e[0] == '0') ? 0 : 1);
    on = g_tree_stage.load(std::memory_order_relaxed);
  }
  return on;
}

int64_t stage_cap(const int64_t* tree) {
  return (tree_stage_on() && (reinterpret_cast<uintptr_t>(tree) & 15) == 0) ? (int64_t)STAGE_WORDS - 1 : 0;
}

enum { MODE_TD = 0, MODE_Q = 1, MODE_MAXSEEN = 2, MODE_SEQ = 3 };
// Header words (rpl.h): 0 max-seen, 1 sampler ticket, 2 stream position, 3-4 grid barrier,
// 5 attached min-tree address (0: none), 6 global buffer min of the last sharded sample.
constexpr int HDR_MINTREE = 5;
// Measurement-only timeline of the update kernel (-DRPL_TRACE builds; rpl_debug_trace).
#ifdef RPL_TRACE
__device__ unsigned long long g_trace[16];
#define UPD_TRACE(k)                                          \
  do {                                                        \
    if (threadIdx.x == 0 && blockIdx.x == 0) g_trace[k] = global_ns(); \
  } while (0)
// step timeline slots: 7 update entry, 8 sampler after its dependency wait, 9 sampler end (max)
#define SMP_TRACE_END()                                                   \
  do {                                                                    \
    if (threadIdx.x == 0) atomicMax(&g_trace[9], (unsigned long long)global_ns()); \
  } while (0)
#else
#define SMP_TRACE_END() \
  do {                  \
  } while (0)
#define UPD_TRACE(k) \
  do {               \
  } while (0)
#endif
constexpr int HDR_GLOBAL_MIN = 6;
constexpr int HDR_UPD_TICKET = 7;  // multi-CTA update's ticket (scratch, 0 between calls)

#include "seqprio.cuh"  // sequence_td8 (R26), shared with the gather's fused update

__device__ __forceinline__ uint32_t hash_slot(int64_t leaf) {
  return (uint32_t)(((unsigned long long)leaf * 0x9E3779B97F4A7C15ull) >> 53) & (HASH_SLOTS - 1);
}


struct UpdSmem {
  unsigned long long hkey[HASH_SLOTS];
  int hval[HASH_SLOTS];
  int64_t sred[UPD_THREADS / 32];
  float s_td[UPD_THREADS];  // MODE_SEQ: this chunk's sequence priorities
};

// Min-tree maintenance (buffer-wide IS normaliser, R29): every internal min node on a
// written leaf's path is recomputed from its W children, level by level from the leaves'
// parents up (a barrier between levels), each distinct node by one thread (hash dedupe per
// chunk of NT entries).  A leaf's min contribution is its q when q > 0; an internal node
// holds the min of its children (INT64_MAX: no positive leaf below).  No-op without one.
template <int NT>
__device__ __forceinline__ void mintree_update(UpdSmem& S, const TreeDev& L, int64_t* __restrict__ tree,
                                               const int64_t* __restrict__ idx, int64_t n, int64_t* mins) {
  unsigned long long* hkey = S.hkey;
  const int tid = threadIdx.x;
  const int64_t* leaves = tree + L.level_off[L.depth];
  if (mins) {
    __syncthreads();
    for (int l = L.depth - 1; l >= 0; --l) {
      const int sh = L.log2w * (L.depth - l);
      for (int64_t base = 0; base < n; base += NT) {
        for (int s2 = tid; s2 < HASH_SLOTS; s2 += NT) hkey[s2] = HASH_EMPTY;
        __syncthreads();
        int64_t p = -1;
        if (base + tid < n) {
          const int64_t leaf = idx[base + tid];
          if (leaf >= 0 && leaf < L.n_leaves) p = leaf >> sh;
        }
        bool own = false;
        if (p >= 0) {
          uint32_t slot = hash_slot(p);
          while (true) {
            const unsigned long long prev = atomicCAS(&hkey[slot], HASH_EMPTY, (unsigned long long)p);
            if (prev == HASH_EMPTY) {
              own = true;
              break;
            }
            if (prev == (unsigned long long)p) break;
            slot = (slot + 1) & (HASH_SLOTS - 1);
          }
        }
        if (own) {
          const int64_t c0 = p << L.log2w;
          int64_t m2 = INT64_MAX;
          if (l == L.depth - 1) {
            for (int j = 0; j < L.fanout; ++j) {
              const int64_t v = __ldcg(leaves + c0 + j);
              if (v > 0 && v < m2) m2 = v;
            }
          } else {
            const int64_t* ch = mins + L.level_off[l + 1] + c0;
            for (int j = 0; j < L.fanout; ++j) {
              const int64_t v = __ldcg(ch + j);
              if (v < m2) m2 = v;
            }
          }
          mins[L.level_off[l] + p] = m2;
        }
        __syncthreads();
      }
    }
  }
}

// The whole batch update by ONE block of NT threads (NT <= UPD_THREADS, a multiple of 32;
// every thread must call): entries are processed in chunks of NT in batch order.
template <int NT, int mode>
__device__ __forceinline__ void tree_update_block(UpdSmem& S, const TreeDev& L, int64_t* __restrict__ tree,
                                                  const int64_t* __restrict__ idx, const float* __restrict__ td,
                                                  const int64_t* __restrict__ qin, int64_t n, double alpha,
                                                  double eps_p, int32_t* err, int force_slow, int64_t T_p, double eta,
                                                  int live_only) {
  unsigned long long* hkey = S.hkey;
  int* hval = S.hval;
  int64_t* sred = S.sred;
  float* s_td = S.s_td;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  int64_t* leaves = tree + L.level_off[L.depth];
  int64_t* hdr = tree + L.hdr_off;
  // Issue the first chunk's loads — the entry, and for a single-chunk batch the leaf's
  // current value — before the hash-table reset and the priority transform, so their
  // latency overlaps that work instead of sitting on the critical path.
  const bool single = n <= NT;
  int64_t pre_leaf = -1, pre_old = 0;
  float pre_td = 0.0f;
  if (tid < n) {
    pre_leaf = idx[tid];
    if (mode == MODE_TD) pre_td = td[tid];
  }
  if (single && pre_leaf >= 0 && pre_leaf < L.n_leaves) pre_old = __ldcg(leaves + pre_leaf);
  const int64_t maxseen_now = __ldcg(hdr);
  int64_t* mins = reinterpret_cast<int64_t*>(__ldcg(hdr + HDR_MINTREE));  // attached min-tree (R29) or NULL
  int64_t local_max = INT64_MIN;
  int32_t errbits = 0;

  for (int64_t base = 0; base < n; base += NT) {
    if (mode == MODE_SEQ) {  // this chunk's sequence priorities, 8 lanes per sequence
      const int64_t cnt = min((int64_t)NT, n - base);
      for (int64_t r0 = 0; r0 < cnt; r0 += NT / 8) {
        const int64_t jj = r0 + (tid >> 3);
        const float v = sequence_td8(td, T_p, n, base + jj, jj < cnt, eta);
        if ((tid & 7) == 0 && jj < cnt) s_td[jj] = v;
      }
      UPD_TRACE(2);
    }
    for (int s = tid; s < HASH_SLOTS; s += NT) {
      hkey[s] = HASH_EMPTY;
      hval[s] = -1;
    }
    __syncthreads();
    UPD_TRACE(3);
    const int64_t i = base + tid;
    int64_t leaf = -1, q = 0;
    if (i < n) {
      leaf = base == 0 ? pre_leaf : idx[i];
      bool ok = leaf < L.n_leaves;  // leaf < 0: padding entry, skipped silently
      if (leaf < 0) {
        leaf = -1;
      } else if (ok) {
        if (mode == MODE_TD || mode == MODE_SEQ) {
          const float tdi = mode == MODE_SEQ ? s_td[tid] : (base == 0 ? pre_td : td[i]);
          const double p = (double)fabsf(tdi) + eps_p;  // RN64(|delta| + eps_p)
          float v;
          if (!isfinite(p)) {
            v = __int_as_float(0x7f800000);
          } else {
            bool slow = false;
            v = cr_powf(p, alpha, force_slow != 0, &slow);
          }
          bool sat = false;
          q = quantise_q(v, L.frac_bits, L.q_cap, &sat);
          if (sat) errbits |= RPL_DERR_SATURATED;
        } else if (mode == MODE_Q) {
          q = qin[i];
          if (q < 0) {
            ok = false;
          } else if (q > L.q_cap) {
            q = L.q_cap;
            errbits |= RPL_DERR_SATURATED;
          }
        } else {
          q = maxseen_now;
        }
      }
      if (!ok) {
        errbits |= RPL_DERR_IDX;
        leaf = -1;
      }
      // RPL_UPD_LIVE_ONLY: a leaf that is currently 0 (invalid since it was sampled, or
      // never written) is left untouched, so a late priority cannot revive it
      if (leaf >= 0 && live_only && (single ? pre_old : __ldcg(leaves + leaf)) == 0) leaf = -1;
      if (leaf >= 0 && mode != MODE_MAXSEEN) local_max = q > local_max ? q : local_max;
    }
    uint32_t slot = 0;
    if (leaf >= 0) {
      slot = hash_slot(leaf);
      while (true) {
        unsigned long long prev = atomicCAS(&hkey[slot], HASH_EMPTY, (unsigned long long)leaf);
        if (prev == HASH_EMPTY || prev == (unsigned long long)leaf) break;
        slot = (slot + 1) & (HASH_SLOTS - 1);
      }
      atomicMax(&hval[slot], tid);  // last position in the batch wins
    }
    __syncthreads();
    UPD_TRACE(4);
    int64_t delta = 0;
    if (leaf >= 0 && hval[slot] == tid) {
      // earlier chunks may have rewritten this leaf: reload unless the batch is one chunk
      const int64_t old = single ? pre_old : __ldcg(leaves + leaf);
      leaves[leaf] = q;
      delta = q - old;
      if (delta != 0) {
        int64_t node = leaf;
        for (int l = L.depth - 1; l >= 1; --l) {
          node >>= L.log2w;
          atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[l] + node),
                    (unsigned long long)delta);
        }
      }
    }
    const int64_t rd = warp_sum64(delta);
    if (lane == 0 && rd != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[0]), (unsigned long long)rd);
    __syncthreads();
    UPD_TRACE(5);
  }
  // max-priority-seen
  int64_t m = warp_max64(local_max);
  if (lane == 0) sred[tid >> 5] = m;
  __syncthreads();
  if (tid < 32) {
    m = tid < NT / 32 ? sred[tid] : INT64_MIN;
    m = warp_max64(m);
    if (tid == 0 && m > maxseen_now) atomicMax(reinterpret_cast<long long*>(hdr), (long long)m);
  }
  if (errbits) set_err(err, errbits);
  UPD_TRACE(6);
  mintree_update<NT>(S, L, tree, idx, n, mins);
}

// The update of a batch that fits one chunk (n <= NT; MODE_SEQ: n <= NT / 8, eight lanes per
// sequence), with the kernel's round trips overlapped: the entry indices, the |delta| (or
// q / the per-step |delta| of every sequence) and the header are requested together; the
// duplicate resolution (a hash of the leaf indices alone: the last batch position of every
// distinct leaf wins, S:624 — independent of the priorities) and the leaves' current values
// follow as soon as the indices land, in flight while the priorities are computed.  The same
// result as tree_update_block (which the multi-chunk batches keep): an entry skipped by
// RPL_UPD_LIVE_ONLY shares its leaf's current value with every duplicate, so skipping after
// the hash selects the same winners.
template <int NT, int mode>
__device__ __forceinline__ void tree_update_single(UpdSmem& S, const TreeDev& L, int64_t* __restrict__ tree,
                                                   const int64_t* __restrict__ idx, const float* __restrict__ td,
                                                   const int64_t* __restrict__ qin, int64_t n, double alpha,
                                                   double eps_p, int32_t* err, int force_slow, int64_t T_p,
                                                   double eta, int live_only, int trig_at) {
  unsigned long long* hkey = S.hkey;
  int* hval = S.hval;
  int64_t* sred = S.sred;
  float* s_td = S.s_td;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  int64_t* leaves = tree + L.level_off[L.depth];
  int64_t* hdr = tree + L.hdr_off;
  // (1) every independent load in flight at once
  int64_t leaf = tid < n ? idx[tid] : -1;
  float tdi = 0.0f;
  int64_t qi = 0;
  if (mode == MODE_TD && tid < n) tdi = td[tid];
  if (mode == MODE_Q && tid < n) qi = qin[tid];
  float vals[mode == MODE_SEQ ? TD8_BATCH : 1];
  const int64_t jj = tid >> 3;  // MODE_SEQ: this lane's sequence
  if (mode == MODE_SEQ) sequence_td8_load(reinterpret_cast<float(&)[TD8_BATCH]>(vals), td, T_p, n, jj, jj < n);
  const int64_t maxseen_now = __ldcg(hdr);
  int64_t* mins = reinterpret_cast<int64_t*>(__ldcg(hdr + HDR_MINTREE));  // attached min-tree (R29) or NULL
  for (int s2 = tid; s2 < HASH_SLOTS; s2 += NT) {
    hkey[s2] = HASH_EMPTY;
    hval[s2] = -1;
  }
  __syncthreads();
  UPD_TRACE(3);
  if (trig_at == 3) pdl_trigger();  // A/B knob: the dependent launch from here
  // (2) duplicate resolution on the indices, and the leaves' current values
  int32_t errbits = 0;
  if (leaf >= L.n_leaves) {
    errbits |= RPL_DERR_IDX;
    leaf = -1;
  } else if (leaf < 0) {
    leaf = -1;  // padding entry, skipped silently
  } else if (mode == MODE_Q && qi < 0) {
    errbits |= RPL_DERR_IDX;  // an explicit q < 0 is an invalid entry: it never takes part in the dedupe
    leaf = -1;
  }
  uint32_t slot = 0;
  int64_t old = 0;
  if (leaf >= 0) {
    old = __ldcg(leaves + leaf);
    slot = hash_slot(leaf);
    while (true) {
      unsigned long long prev = atomicCAS(&hkey[slot], HASH_EMPTY, (unsigned long long)leaf);
      if (prev == HASH_EMPTY || prev == (unsigned long long)leaf) break;
      slot = (slot + 1) & (HASH_SLOTS - 1);
    }
    atomicMax(&hval[slot], tid);  // last position in the batch wins
  }
  // (3) the priorities (R26 sequence mix, R7 transform)
  if (mode == MODE_SEQ) {
    const float v = sequence_td8_finish(reinterpret_cast<const float(&)[TD8_BATCH]>(vals), td, T_p, n, jj, jj < n,
                                        eta);
    if ((tid & 7) == 0 && jj < n) s_td[jj] = v;
  }
  UPD_TRACE(2);
  if (trig_at == 2) pdl_trigger();
  __syncthreads();  // s_td and the hash table complete
  int64_t q = 0;
  if (leaf >= 0) {
    if (mode == MODE_TD || mode == MODE_SEQ) {
      const float t = mode == MODE_SEQ ? s_td[tid] : tdi;
      const double p = (double)fabsf(t) + eps_p;  // RN64(|delta| + eps_p)
      float v;
      if (!isfinite(p)) {
        v = __int_as_float(0x7f800000);
      } else {
        bool slow = false;
        v = cr_powf(p, alpha, force_slow != 0, &slow);
      }
      bool sat = false;
      q = quantise_q(v, L.frac_bits, L.q_cap, &sat);
      if (sat) errbits |= RPL_DERR_SATURATED;
    } else if (mode == MODE_Q) {
      q = qi;
      if (q > L.q_cap) {
        q = L.q_cap;
        errbits |= RPL_DERR_SATURATED;
      }
    } else {
      q = maxseen_now;
    }
  }
  // RPL_UPD_LIVE_ONLY: a leaf that is currently 0 is left untouched (R30)
  if (leaf >= 0 && live_only && old == 0) leaf = -1;
  int64_t local_max = (leaf >= 0 && mode != MODE_MAXSEEN) ? q : INT64_MIN;
  UPD_TRACE(4);
  if (trig_at == 4) pdl_trigger();
  int64_t delta = 0;
  if (leaf >= 0 && hval[slot] == tid) {
    leaves[leaf] = q;
    delta = q - old;
    if (delta != 0) {
      int64_t node = leaf;
      for (int l = L.depth - 1; l >= 1; --l) {
        node >>= L.log2w;
        atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[l] + node), (unsigned long long)delta);
      }
    }
  }
  const int64_t rd = warp_sum64(delta);
  if (lane == 0 && rd != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[0]), (unsigned long long)rd);
  UPD_TRACE(5);
  // max-priority-seen
  int64_t m = warp_max64(local_max);
  if (lane == 0) sred[tid >> 5] = m;
  __syncthreads();
  if (tid < 32) {
    m = tid < NT / 32 ? sred[tid] : INT64_MIN;
    m = warp_max64(m);
    if (tid == 0 && m > maxseen_now) atomicMax(reinterpret_cast<long long*>(hdr), (long long)m);
  }
  if (errbits) set_err(err, errbits);
  UPD_TRACE(6);
  mintree_update<NT>(S, L, tree, idx, n, mins);
}

// Multi-CTA update of a batch of n <= HASH_SLOTS / 2 entries (the default for such batches).
// One CTA is issue-bound: its 16 warps share one SM's four schedulers through ~1,500
// instructions each of loads, the sequence mix and the power transform (the update was
// ~5.5 us of the R2D2 step, scripts/step_trace.py).  Here each CTA owns UPDM_EPC entries
// (MODE_SEQ: 8 sequences, eight lanes each; else one entry per thread) and the batch is
// spread over ceil(n / UPDM_EPC) SMs.  Duplicate resolution stays exact without any
// cross-CTA exchange: every CTA inserts ALL n indices into its own shared-memory hash (the
// last valid position of every distinct leaf, S:624 — the indices alone decide it), so all
// CTAs agree on the winners and each writes only its own winning entries.  Leaf writes are
// plain stores to distinct leaves, propagation is int64 atomics (order-free, exact), max-seen
// an atomicMax per CTA.  With a min-tree attached (R29) the CTA that takes the last ticket
// (header word 7, acq_rel: it observes every CTA's leaf writes) recomputes the min paths of
// all n entries.  Same result as tree_update_single / tree_update_block.
#ifndef RPL_UPDM_THREADS  // threads per CTA of the multi-CTA update (build-flag A/B knob)
#define RPL_UPDM_THREADS 64
#endif
constexpr int UPDM_THREADS = RPL_UPDM_THREADS;
template <int mode>
__global__ void __launch_bounds__(UPDM_THREADS)
k_tree_update_multi(TreeDev L, int64_t* __restrict__ tree, const int64_t* __restrict__ idx,
                    const float* __restrict__ td, const int64_t* __restrict__ qin, int64_t n, double alpha,
                    double eps_p, int32_t* err, int force_slow, int64_t T_p, double eta, int live_only, int trig_at) {
  constexpr int EPC = mode == MODE_SEQ ? UPDM_THREADS / 8 : UPDM_THREADS;  // entries per CTA
  __shared__ UpdSmem S;
  unsigned long long* hkey = S.hkey;
  int* hval = S.hval;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  for (int s2 = tid; s2 < HASH_SLOTS; s2 += UPDM_THREADS) {  // no global access: before the wait
    hkey[s2] = HASH_EMPTY;
    hval[s2] = -1;
  }
  if (trig_at == 0) pdl_trigger();
  UPD_TRACE(7);
  if ((threadIdx.x >> 5) == 0) pdl_wait();  // one waiting warp (see g_upd_trigger)
  __syncthreads();
  UPD_TRACE(0);
  int64_t* leaves = tree + L.level_off[L.depth];
  int64_t* hdr = tree + L.hdr_off;
  const int64_t e0 = (int64_t)blockIdx.x * EPC;
  const int64_t my = e0 + tid;  // this thread's entry (tid < EPC)
  // (1) every independent load in flight at once
  int64_t leaf = (tid < EPC && my < n) ? idx[my] : -1;
  float tdi = 0.0f;
  int64_t qi = 0;
  if (mode == MODE_TD && tid < EPC && my < n) tdi = td[my];
  if (mode == MODE_Q && tid < EPC && my < n) qi = qin[my];
  float vals[mode == MODE_SEQ ? TD8_BATCH : 1];
  const int64_t jj = e0 + (tid >> 3);  // MODE_SEQ: this lane's sequence
  if (mode == MODE_SEQ) sequence_td8_load(reinterpret_cast<float(&)[TD8_BATCH]>(vals), td, T_p, n, jj, jj < n);
  const int64_t maxseen_now = __ldcg(hdr);
  const int64_t* mins = reinterpret_cast<const int64_t*>(__ldcg(hdr + HDR_MINTREE));
  __syncthreads();  // the hash reset is complete
  // (2) every index of the batch into this CTA's hash: the last valid position of each leaf
  for (int64_t j = tid; j < n; j += UPDM_THREADS) {
    const int64_t lj = idx[j];
    bool vj = lj >= 0 && lj < L.n_leaves;
    if (mode == MODE_Q && vj) vj = qin[j] >= 0;
    if (vj) {
      uint32_t slot = hash_slot(lj);
      while (true) {
        const unsigned long long prev = atomicCAS(&hkey[slot], HASH_EMPTY, (unsigned long long)lj);
        if (prev == HASH_EMPTY || prev == (unsigned long long)lj) break;
        slot = (slot + 1) & (HASH_SLOTS - 1);
      }
      atomicMax(&hval[slot], (int)j);
    }
  }
  UPD_TRACE(3);
  int32_t errbits = 0;
  if (leaf >= L.n_leaves) {
    errbits |= RPL_DERR_IDX;
    leaf = -1;
  } else if (leaf < 0) {
    leaf = -1;  // padding entry (or no entry), skipped silently
  } else if (mode == MODE_Q && qi < 0) {
    errbits |= RPL_DERR_IDX;
    leaf = -1;
  }
  const int64_t old = leaf >= 0 ? __ldcg(leaves + leaf) : 0;  // in flight during the priorities
  // (3) the priorities (R26 sequence mix, R7 transform)
  if (mode == MODE_SEQ) {
    const float v = sequence_td8_finish(reinterpret_cast<const float(&)[TD8_BATCH]>(vals), td, T_p, n, jj, jj < n,
                                        eta);
    if ((tid & 7) == 0) S.s_td[tid >> 3] = v;
  }
  UPD_TRACE(2);
  if (trig_at == 2) pdl_trigger();
  __syncthreads();  // this CTA's sequence priorities and the hash complete
  int64_t q = 0;
  if (leaf >= 0) {
    if (mode == MODE_TD || mode == MODE_SEQ) {
      const float t = mode == MODE_SEQ ? S.s_td[tid] : tdi;
      const double p = (double)fabsf(t) + eps_p;  // RN64(|delta| + eps_p)
      float v;
      if (!isfinite(p)) {
        v = __int_as_float(0x7f800000);
      } else {
        bool slow = false;
        v = cr_powf(p, alpha, force_slow != 0, &slow);
      }
      bool sat = false;
      q = quantise_q(v, L.frac_bits, L.q_cap, &sat);
      if (sat) errbits |= RPL_DERR_SATURATED;
    } else if (mode == MODE_Q) {
      q = qi;
      if (q > L.q_cap) {
        q = L.q_cap;
        errbits |= RPL_DERR_SATURATED;
      }
    } else {
      q = maxseen_now;
    }
  }
  if (leaf >= 0 && live_only && old == 0) leaf = -1;  // R30
  const int64_t local_max = (leaf >= 0 && mode != MODE_MAXSEEN) ? q : INT64_MIN;
  UPD_TRACE(4);
  if (trig_at == 4) pdl_trigger();
  int64_t delta = 0;
  if (leaf >= 0) {
    uint32_t slot = hash_slot(leaf);
    while (hkey[slot] != (unsigned long long)leaf) slot = (slot + 1) & (HASH_SLOTS - 1);
    if (hval[slot] == (int)my) {  // the batch's last position of this leaf
      leaves[leaf] = q;
      delta = q - old;
      if (delta != 0) {
        int64_t node = leaf;
        for (int l = L.depth - 1; l >= 1; --l) {
          node >>= L.log2w;
          atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[l] + node), (unsigned long long)delta);
        }
      }
    }
  }
  const int64_t rd = warp_sum64(delta);
  if (lane == 0 && rd != 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(tree + L.level_off[0]), (unsigned long long)rd);
  UPD_TRACE(5);
  int64_t m = warp_max64(local_max);  // max-priority-seen
  if (lane == 0 && m > maxseen_now) atomicMax(reinterpret_cast<long long*>(hdr), (long long)m);
  if (errbits) set_err(err, errbits);
  UPD_TRACE(6);
  if (mins) {  // R29: the last CTA recomputes every written leaf's min path
    __shared__ int s_last;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t;
      asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                   : "=l"(t) : "l"(hdr + HDR_UPD_TICKET) : "memory");
      s_last = t == (unsigned long long)gridDim.x - 1;
      if (s_last) hdr[HDR_UPD_TICKET] = 0;
    }
    __syncthreads();
    if (s_last) mintree_update<UPDM_THREADS>(S, L, tree, idx, n, const_cast<int64_t*>(mins));
  }
}

// One instantiation per mode: each kernel carries only its own path (the MODE_SEQ code in a
// shared kernel cost every launch ~1.7 us of instruction fetch, scripts/update_tp_sweep.py).
template <int mode>
__global__ void __launch_bounds__(UPD_THREADS)
k_tree_update(TreeDev L, int64_t* __restrict__ tree, const int64_t* __restrict__ idx,
              const float* __restrict__ td, const int64_t* __restrict__ qin, int64_t n,
              double alpha, double eps_p, int32_t* err, int force_slow, int64_t T_p, double eta, int live_only,
              int trig_at) {
  __shared__ UpdSmem S;
  if (trig_at == 0) pdl_trigger();  // A/B knob (rpl_debug_set_upd_trigger; RPL_PDL_EARLY & 1 sets 0)
  UPD_TRACE(7);
  pdl_wait();
  UPD_TRACE(0);
  if (RPL_UPD_SINGLE && n <= (mode == MODE_SEQ ? UPD_THREADS / 8 : UPD_THREADS))
    tree_update_single<UPD_THREADS, mode>(S, L, tree, idx, td, qin, n, alpha, eps_p, err, force_slow, T_p, eta,
                                          live_only, trig_at);
  else
    tree_update_block<UPD_THREADS, mode>(S, L, tree, idx, td, qin, n, alpha, eps_p, err, force_slow, T_p, eta,
                                   live_only);
}

// First stratum k in [0, n] whose prefix is >= x (n if none).
__device__ __forceinline__ int64_t first_stratum_at_least(uint64_t x, uint64_t Q, int64_t n, const uint64_t* draws,
                                                          uint64_t seed, uint64_t ctr0) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (stratum_prefix(mid, Q, n, draws, seed, ctr0) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <bool SHARDED>
__global__ void __launch_bounds__(SAMPLE_WARPS * 32)
k_tree_sample(TreeDev L, int64_t* __restrict__ tree, int64_t n, const uint64_t* __restrict__ draws,
              uint64_t seed, uint64_t offset, double beta, int64_t* __restrict__ out_idx,
              int64_t* __restrict__ out_q, int64_t* __restrict__ out_qmin, float* __restrict__ out_w,
              int32_t* err, int rank, int n_shards, int64_t shard_leaves,
              const int64_t* __restrict__ totals, int use_stream, int64_t* __restrict__ out_count,
              int64_t* const* boards, int64_t stage_cap, int tot_stride, int64_t* __restrict__ out_bufmin) {
  const int lane = threadIdx.x & 31;
  const DivN dn = divn_make((uint64_t)(n > 0 ? n : 1));  // n alone: before the dependency wait
  if (RPL_PDL_EARLY & 2) pdl_trigger();  // A/B knob (common.cuh)
  // one warp waits for the previous grid (launched early by PDL, the other warps wait at the
  // barrier, which orders their reads after the wait): fewer waiting warps beside the running
  // update kernel (in-process A/B of the R2D2 step with the gather: -0.85 us)
  if ((threadIdx.x >> 5) == 0) pdl_wait();
  __syncthreads();
  UPD_TRACE(8);
  // Stage the top levels (root .. the deepest level that still fits STAGE_WORDS) in shared
  // memory with one round of asynchronous 16-B copies, so the descent's first levels and Q
  // cost one L2 round trip in total instead of one each.  Levels are contiguous from word 0.
  __shared__ __align__(16) int64_t s_top[STAGE_WORDS];
  int64_t n_top = 0;
  for (int l = 0; l <= L.depth; ++l) {
    const int64_t end = l < L.depth ? L.level_off[l + 1] : L.hdr_off;
    if (end > stage_cap) break;
    n_top = end;
  }
  for (int64_t j = 2 * (int64_t)threadIdx.x; j < n_top; j += 2 * (int64_t)blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s_u32(s_top + j)), "l"(tree + j) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  // Without a batch reduction (no IS weights, no qmin requested) there is no grid-wide
  // end ticket; a stream-mode call then takes its ticket at the start instead: every CTA
  // reads the stream position (acquire: ordered before its ticket increment) and the CTA
  // that arrives last advances the position once all CTAs have read it.
  const bool reduce = out_w != nullptr || out_qmin != nullptr;
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(tree + L.hdr_off + 1);
  // Thread 0 alone reads the stream position (acquire), in flight with the staging copies,
  // and broadcasts it at the staging barrier; its ticket increment follows the read in
  // program order, so no CTA can advance the position before every CTA has read it.  The
  // ticket value stays in thread 0's register until the end, so that round trip overlaps
  // the descent.
  uint64_t spos = 0;
  __shared__ uint64_t s_spos;
  unsigned long long t0 = 0;
  if (use_stream && threadIdx.x == 0) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(spos) : "l"(tree + L.hdr_off + 2) : "memory");
    s_spos = spos;
    if (!reduce) t0 = atomicAdd(ticket, 1ull);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (use_stream) spos = s_spos;
  // Philox counter base: offset, plus the tree's stream position when use_stream
  const uint64_t ctr0 = offset + spos;
  const int64_t k = (int64_t)blockIdx.x * SAMPLE_WARPS + (threadIdx.x >> 5);
  int32_t errbits = 0;
  uint64_t Q, own_lo = 0, own_T = 0;
  __shared__ int64_t s_tot[SHARDED ? BOARD_MAX_WORLD : 1];
  if (SHARDED && boards) {
    // K5 fused (rpl_sumtree_sample_sharded_p2p): CTA 0 publishes this shard's total to every
    // rank's board, every CTA reads all totals from its own board; tag = stream position
    // after this step (identical on every rank)
    const uint64_t tag = spos + (uint64_t)n;
    // with the shard's buffer min (root of its attached min-tree, INT64_MAX without one) in
    // the board's third section, so a buffer-wide normaliser needs no second exchange (R29)
    const int64_t* mt = reinterpret_cast<const int64_t*>(__ldcg(tree + L.hdr_off + HDR_MINTREE));
    if (blockIdx.x == 0 && threadIdx.x < n_shards) {
      board_publish(boards[threadIdx.x] + 2 * rank, __ldcg(tree + L.level_off[0]), tag);
      board_publish(boards[threadIdx.x] + 4 * n_shards + 2 * rank, mt ? __ldcg(mt) : INT64_MAX, tag);
    }
    if (threadIdx.x < n_shards) {
      int64_t v = 0;
      if (!board_wait(boards[rank] + 2 * threadIdx.x, tag, &v)) board_fail(err);
      s_tot[threadIdx.x] = v;
    }
    if (mt && blockIdx.x == 0 && threadIdx.x < 32) {  // global buffer min -> header word 6
      int64_t v = INT64_MAX;
      if (lane < n_shards && !board_wait(boards[rank] + 4 * n_shards + 2 * lane, tag, &v)) board_fail(err);
      v = warp_min64(v);
      if (lane == 0) tree[L.hdr_off + HDR_GLOBAL_MIN] = v;
    }
    __syncthreads();
  }
  if (SHARDED) {
    Q = 0;
    for (int g = 0; g < n_shards; ++g) {
      const uint64_t tg = (uint64_t)(boards ? s_tot[g] : totals[(int64_t)g * tot_stride]);
      if (g < rank) own_lo += tg;
      if (g == rank) own_T = tg;
      Q += tg;
    }
  } else {
    Q = (uint64_t)(n_top > 0 ? s_top[0] : tree[L.level_off[0]]);
  }
  if (SHARDED && out_bufmin && blockIdx.x == 0 && threadIdx.x < 32) {  // {total, min} pairs: global min
    int64_t v = INT64_MAX;
    for (int g = lane; g < n_shards; g += 32) {
      const int64_t x = totals[(int64_t)g * tot_stride + 1];
      v = x < v ? x : v;
    }
    v = warp_min64(v);
    if (lane == 0) {
      *out_bufmin = v;
      tree[L.hdr_off + HDR_GLOBAL_MIN] = v;
    }
  }
  // compacted sharded output: the owned run of strata [k0, k1) goes to positions
  // 0 .. m-1 (stratum order), positions m .. n-1 get -1; *out_count = m
  const bool compact = SHARDED && out_count != nullptr;
  int64_t k0 = 0, m_own = 0;
  if (compact && Q > 0) {
    k0 = first_stratum_at_least(own_lo, Q, n, draws, seed, ctr0);
    m_own = first_stratum_at_least(own_lo + own_T, Q, n, draws, seed, ctr0) - k0;
  }
  if (k < n) {
    int64_t leaf = -1, q = 0;
    bool mine = false;
    if (Q == 0) {
      errbits |= RPL_DERR_EMPTY;
    } else {
      uint64_t prefix = strata_prefix(k, strata_make(Q, dn), draws, seed, ctr0);
      mine = true;
      if (SHARDED) {
        mine = prefix >= own_lo && prefix < own_lo + own_T;
        prefix -= own_lo;
      }
      if (mine) {
        leaf = descend(L, tree, (int64_t)prefix, &q, &errbits, s_top, n_top);
        // global index (shard-major, §8c #17); the compacted form keeps the LOCAL leaf
        // for the owner's own update / gather
        if (SHARDED && !compact) leaf += (int64_t)rank * shard_leaves;
      }
    }
    if (lane == 0) {
      if (!compact) {
        out_idx[k] = leaf;
        out_q[k] = q;
      } else {
        if (mine) {
          out_idx[k - k0] = leaf;
          out_q[k - k0] = q;
        }
        if (k >= m_own) {
          out_idx[k] = -1;
          out_q[k] = 0;
        }
        if (k == 0) {
          out_count[0] = m_own;
          out_count[1] = k0;  // global batch position of compacted entry 0 (Mode C column offset)
        }
      }
    }
  }
  if (lane == 0 && errbits) set_err(err, errbits);

  if (!reduce) {
    if (use_stream) {  // only thread 0s read the position (before their tickets): no barrier
      if (threadIdx.x == 0 && t0 == (unsigned long long)gridDim.x - 1) {
        tree[L.hdr_off + 2] = (int64_t)(spos + (uint64_t)n);  // advance the stream
        *ticket = 0ull;
      }
    }
    SMP_TRACE_END();
    return;
  }
  // last CTA: batch-min q and IS weights (§8c #10)
  __shared__ int s_last;
  __shared__ int64_t s_min[SAMPLE_WARPS];
  __syncthreads();
  if (threadIdx.x == 0) {
    // acq_rel ticket instead of __threadfence + atomicAdd: the CTA's output writes (ordered
    // before thread 0 by the barrier) are released with the arrival, and the last CTA
    // acquires every other CTA's.  A full fence.sc costs ~1 us here (measured on the
    // update+sample overlay trial, profiles/r1/README.md).
    unsigned long long t;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(t) : "l"(ticket) : "memory");
    s_last = (t == (unsigned long long)gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) {
    SMP_TRACE_END();
    return;
  }
  int64_t m = INT64_MAX;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int64_t qj = __ldcg(out_q + j);
    const int64_t ij = __ldcg(out_idx + j);
    if (ij >= 0 && qj < m) m = qj;
  }
  m = warp_min64(m);
  if (lane == 0) s_min[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = lane < SAMPLE_WARPS ? s_min[lane] : INT64_MAX;
    m = warp_min64(m);
    if (lane == 0) s_min[0] = m;
  }
  __syncthreads();
  const int64_t qmin = s_min[0];
  if (threadIdx.x == 0) {
    if (out_qmin) *out_qmin = (!SHARDED && Q == 0) ? 0 : qmin;
    *reinterpret_cast<unsigned long long*>(tree + L.hdr_off + 1) = 0ull;  // reset ticket
    if (use_stream) tree[L.hdr_off + 2] = (int64_t)(ctr0 - offset + (uint64_t)n);  // advance stream
  }
  if (out_w) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const int64_t qj = __ldcg(out_q + j);
      out_w[j] = qj > 0 ? (float)pow((double)qmin / (double)qj, beta) : 0.0f;
    }
  }
}

// Fused priority update + stream sampling (rpl_sumtree_update_sample): the two calls of a
// learner step as ONE launch.  CTA 0 runs the whole update (tree_update_block, 256 threads,
// batch order preserved); every CTA reads the stream position, then all CTAs meet at a
// grid barrier (header words 3 = arrivals, 4 = generation; sense reversal, so any grid
// size works), and each warp descends for one stratum of the UPDATED tree.  The grid is
// capped at the SM count and launched cooperatively (launch_coop), so the runtime guarantees
// that all CTAs are co-resident: the spin barrier cannot starve next to other streams' work.
// Result: identical to rpl_sumtree_update(_seq) followed by rpl_sumtree_sample_stream with
// out_qmin = out_w = NULL.  Measured (R2D2 step, B200): the pair is FASTER — 8.2 us for
// update_seq + sample_stream against 9.2 us fused, the grid barrier's atomic round trips
// costing more than the PDL kernel boundary — so bench.py keeps the pair by default
// (--tree-fused 1 selects this); the entry point is for callers launching without PDL.
__device__ __forceinline__ void grid_barrier(int64_t* hdr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(hdr + 3);
    unsigned long long* gen = reinterpret_cast<unsigned long long*>(hdr + 4);
    unsigned long long g;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(g) : "l"(gen) : "memory");
    // acq_rel arrival: this CTA's tree writes (ordered before thread 0 by the barrier) are
    // released with it, and the last arriver acquires them all (no fence.sc; see k_tree_sample)
    unsigned long long t;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(t) : "l"(cnt) : "memory");
    if (t == (unsigned long long)gridDim.x - 1) {
      *cnt = 0ull;  // ordered before the generation bump by its release
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(gen), "l"(g + 1ull) : "memory");
    } else {
      unsigned long long cur;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(gen) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

// 256 threads: measured 9.2 us for update + sample against 10.2 us with 1024-thread CTAs
constexpr int FUSED_THREADS = 256;
constexpr int FUSED_WARPS = FUSED_THREADS / 32;

__global__ void __launch_bounds__(FUSED_THREADS)
k_tree_update_sample(TreeDev L, int64_t* __restrict__ tree, const int64_t* __restrict__ idx,
                     const float* __restrict__ td, int64_t n_upd, int64_t T_p, double eta, double alpha, double eps_p,
                     int live_only, int64_t n, uint64_t seed, int64_t* __restrict__ out_idx,
                     int64_t* __restrict__ out_q, int32_t* err) {
  __shared__ UpdSmem S;
  pdl_wait();
  int64_t* hdr = tree + L.hdr_off;
  uint64_t spos = 0;
  if (threadIdx.x == 0)
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(spos) : "l"(hdr + 2) : "memory");
  if (blockIdx.x == 0 && n_upd > 0)
    (T_p > 0 ? tree_update_block<FUSED_THREADS, MODE_SEQ> : tree_update_block<FUSED_THREADS, MODE_TD>)(
        S, L, tree, idx, td, nullptr, n_upd, alpha, eps_p,
                                     err, 0, T_p, eta, live_only);
  grid_barrier(hdr);  // orders every CTA's read of hdr[2] before CTA 0 advances it below
  __shared__ uint64_t s_spos;
  if (threadIdx.x == 0) s_spos = spos;
  __syncthreads();
  spos = s_spos;
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * FUSED_WARPS + (threadIdx.x >> 5);
  int32_t errbits = 0;
  const uint64_t Q = (uint64_t)__ldcg(tree + L.level_off[0]);
  for (int64_t kk = k; kk < n; kk += (int64_t)gridDim.x * FUSED_WARPS) {
    int64_t leaf = -1, q = 0;
    if (Q == 0) {
      errbits |= RPL_DERR_EMPTY;
    } else {
      const uint64_t prefix = stratum_prefix(kk, Q, n, nullptr, seed, spos);
      leaf = descend(L, tree, (int64_t)prefix, &q, &errbits);
    }
    if (lane == 0) {
      out_idx[kk] = leaf;
      out_q[kk] = q;
    }
  }
  if (lane == 0 && errbits) set_err(err, errbits);
  if (blockIdx.x == 0 && threadIdx.x == 0) hdr[2] = (int64_t)(spos + (uint64_t)n);  // advance the stream
}

// Sampling WITHOUT replacement (§8f NEXT-4, reading R32): successive proportional draws —
// draw k takes prefix_k = floor(u_k Q_k / 2^64) on the tree with the k leaves drawn so far
// removed (their q subtracted along their root paths), then every removed leaf is put back.
// One warp, n sequential descents: exact (integer tree) but latency-bound (n x D dependent
// L2 round trips), meant for small batches.
__global__ void __launch_bounds__(32)
k_tree_sample_unique(TreeDev L, int64_t* __restrict__ tree, int64_t n, uint64_t seed, uint64_t offset,
                     int use_stream, int64_t* __restrict__ out_idx, int64_t* __restrict__ out_q, int32_t* err) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  int64_t* leaves = tree + L.level_off[L.depth];
  const uint64_t ctr0 = offset + (use_stream ? (uint64_t)__ldcg(tree + L.hdr_off + 2) : 0ull);
  int32_t errbits = 0;
  int64_t drawn = 0;
  for (int64_t k = 0; k < n; ++k) {
    const uint64_t Q = (uint64_t)__ldcg(tree + L.level_off[0]);
    if (Q == 0) {  // fewer non-zero leaves than n: the rest stay -1
      if (lane == 0) {
        out_idx[k] = -1;
        out_q[k] = 0;
      }
      errbits |= RPL_DERR_EMPTY;
      continue;
    }
    const uint64_t u = philox_u64(seed, ctr0 + (uint64_t)k);
    int64_t q = 0;
    int64_t prefix = (int64_t)__umul64hi(u, Q);
    // descent with L2-coherent loads (the removals below are plain stores of this warp)
    int64_t node = 0, c = 0;
    for (int l = 0; l < L.depth; ++l) {
      const int64_t base = L.level_off[l + 1] + (node << L.log2w);
      c = lane < L.fanout ? __ldcg(tree + base + lane) : 0;
      int64_t incl = c;
#pragma unroll
      for (int dlt = 1; dlt < 32; dlt <<= 1) {
        const int64_t o = shfl_up64(incl, dlt);
        if (lane >= dlt) incl += o;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, prefix < incl);
      const int f = bal ? __ffs(bal) - 1 : 0;
      if (!bal) errbits |= RPL_DERR_TREE;
      const int64_t inc_f = shfl64(incl, f);
      const int64_t c_f = shfl64(c, f);
      prefix -= inc_f - c_f;
      node = (node << L.log2w) + f;
      c = c_f;
    }
    q = c;
    if (lane == 0) {
      out_idx[k] = node;
      out_q[k] = q;
      // remove the leaf: subtract q along its root path
      leaves[node] = 0;
      int64_t a = node;
      for (int l = L.depth - 1; l >= 0; --l) {
        a >>= L.log2w;
        tree[L.level_off[l] + a] -= q;
      }
      __threadfence_block();
    }
    __syncwarp();
    ++drawn;
  }
  // put every drawn leaf back (integer sums: exact restore)
  if (lane == 0) {
    for (int64_t k = 0; k < drawn; ++k) {
      const int64_t leaf = out_idx[k];
      if (leaf < 0) continue;
      const int64_t q = out_q[k];
      leaves[leaf] = q;
      int64_t a = leaf;
      for (int l = L.depth - 1; l >= 0; --l) {
        a >>= L.log2w;
        tree[L.level_off[l] + a] += q;
      }
    }
    if (use_stream) tree[L.hdr_off + 2] = (int64_t)(ctr0 - offset + (uint64_t)n);
    if (errbits) set_err(err, errbits);
  }
}

__global__ void k_tree_find(TreeDev L, const int64_t* __restrict__ tree, const int64_t* __restrict__ prefix,
                            int64_t n, int64_t* __restrict__ out_idx, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * SAMPLE_WARPS + (threadIdx.x >> 5);
  if (k >= n) return;
  int32_t errbits = 0;
  const int64_t Q = tree[L.level_off[0]];
  int64_t p = prefix[k];
  if (p < 0) {
    p = 0;
    errbits |= RPL_DERR_TREE;
  }
  int64_t q;
  const int64_t leaf = Q > 0 ? descend(L, tree, p, &q, &errbits) : -1;
  if (Q == 0) errbits |= RPL_DERR_EMPTY;
  if (lane == 0) {
    out_idx[k] = leaf;
    if (errbits) set_err(err, errbits);
  }
}

// Buffer-wide IS normaliser (§8f NEXT-4, reading R29): min over the leaves with q > 0.
__global__ void k_min_init(int64_t* __restrict__ out) {
  pdl_wait();
  *out = INT64_MAX;
}
__global__ void k_leaf_min(const int64_t* __restrict__ leaves, int64_t n, int64_t* __restrict__ out) {
  pdl_wait();
  int64_t m = INT64_MAX;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = __ldcg(leaves + i);
    if (v > 0 && v < m) m = v;
  }
  m = warp_min64(m);
  if ((threadIdx.x & 31) == 0 && m != INT64_MAX) atomicMin(reinterpret_cast<long long*>(out), (long long)m);
}

__global__ void k_tree_total(const int64_t* __restrict__ tree, int64_t* __restrict__ out) {
  pdl_wait();
  *out = tree[0];
}

// {total, buffer min}: the root sum and the root of the attached min-tree (INT64_MAX without)
__global__ void k_tree_total_min(const int64_t* __restrict__ tree, int64_t hdr_off, int64_t* __restrict__ out) {
  pdl_wait();
  const int64_t* mt = reinterpret_cast<const int64_t*>(tree[hdr_off + HDR_MINTREE]);
  out[0] = tree[0];
  out[1] = mt ? mt[0] : INT64_MAX;
}

__global__ void k_set_word(int64_t* __restrict__ w, int64_t v) {
  pdl_wait();
  *w = v;
}

// Min-tree level l from level l+1 (or the leaves), one warp per node: min over the W
// children of the positive leaves / the child mins; padding nodes get INT64_MAX.  A no-op
// when no min-tree is attached (header word 5 == 0), so callers need not know.
__global__ void k_mintree_level(TreeDev L, const int64_t* __restrict__ tree, int l, int64_t len, int64_t clen) {
  pdl_wait();
  int64_t* mins = reinterpret_cast<int64_t*>(__ldcg(tree + L.hdr_off + HDR_MINTREE));
  if (!mins) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t node = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); node < len; node += warps) {
    int64_t v = INT64_MAX;
    const int64_t c = (node << L.log2w) + lane;
    if (lane < L.fanout && c < clen) {  // children of padding nodes may lie past the child level
      if (l == L.depth - 1) {
        const int64_t x = __ldcg(tree + L.level_off[L.depth] + c);
        v = x > 0 ? x : INT64_MAX;
      } else {
        v = __ldcg(mins + L.level_off[l + 1] + c);
      }
    }
    v = warp_min64(v);
    if (lane == 0) mins[L.level_off[l] + node] = v;
  }
}

__global__ void k_tree_level(TreeDev L, int64_t* __restrict__ tree, int l, int64_t len, int64_t real) {
  // node j of level l := sum of its W children on level l+1 (real nodes); padding nodes := 0.
  // A real node's children lie inside level l+1 (len(l+1) = real(l) * W), a padding
  // node's would not, so padding is never summed.
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= len) return;
  int64_t s = 0;
  if (j < real) {
    const int64_t* ch = tree + L.level_off[l + 1] + (j << L.log2w);
    for (int c = 0; c < L.fanout; ++c) s += ch[c];
  }
  tree[L.level_off[l] + j] = s;
}

__global__ void k_tree_header(int64_t* __restrict__ hdr, int64_t maxseen) {
  // [0] max-seen, [1] sampler ticket, [2] Philox stream position
  hdr[0] = maxseen;
  for (int i = 1; i < 8; ++i) hdr[i] = 0;
}

__global__ void k_is_weights(const int64_t* __restrict__ q, const int64_t* __restrict__ qmin, int64_t n,
                             double beta, float* __restrict__ w) {
  pdl_wait();
  const double m = (double)*qmin;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qj = q[j];
    w[j] = qj > 0 ? (float)pow(m / (double)qj, beta) : 0.0f;
  }
}

constexpr int UNI_THREADS = 256;
__global__ void __launch_bounds__(UNI_THREADS)
k_sample_uniform(int64_t n, uint64_t seed, uint64_t offset, uint64_t* ctr, int64_t lo_row, int64_t n_rows,
                 int64_t cap_T, int64_t B, int64_t* __restrict__ out_idx) {
  pdl_wait();
  const uint64_t base = offset + (ctr ? *ctr : 0ull);
  const uint64_t M = (uint64_t)n_rows * (uint64_t)B;
  for (int64_t k = threadIdx.x; k < n; k += UNI_THREADS) {
    const uint64_t m = __umul64hi(philox_u64(seed, base + (uint64_t)k), M);
    const int64_t row = (lo_row + (int64_t)(m / (uint64_t)B)) % cap_T;
    out_idx[k] = row * B + (int64_t)(m % (uint64_t)B);
  }
  __syncthreads();
  if (ctr && threadIdx.x == 0) *ctr = base - offset + (uint64_t)n;
}

__global__ void k_priority_values(const float* __restrict__ td, int64_t n, double alpha, double eps_p,
                                  int force_slow, float* __restrict__ v, uint8_t* __restrict__ slow_flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double p = (double)fabsf(td[j]) + eps_p;
    bool slow = false;
    float r;
    if (!isfinite(p)) r = __int_as_float(0x7f800000);
    else r = cr_powf(p, alpha, force_slow != 0, &slow);
    v[j] = r;
    if (slow_flag) slow_flag[j] = slow ? 1 : 0;
  }
}

bool layout_ok(const rpl_tree_layout* L) {
  return L && L->n_leaves >= 1 && L->fanout >= 2 && L->fanout <= 32 && (L->fanout & (L->fanout - 1)) == 0 &&
         L->depth >= 1 && L->depth < RPL_MAX_LEVELS && L->frac_bits >= 0 && L->frac_bits <= 62;
}

// Where the update kernel lets its dependent grid launch (-1 at exit, 0 at entry, 3 after its
// loads are issued, 2 after the priorities, 4 after the power transform; rpl_debug_set_upd_trigger).
// Default 0: the next kernel's launch (the sequence gather's 146 CTAs take ~3 us to become
// resident) overlaps the whole update; it still waits for the update's completion in its
// griddepcontrol.wait — which only ONE warp per CTA of the early-launched kernel executes (the
// others wait at a CTA barrier): with every warp waiting, the resident CTAs slowed the update
// and entry / after-the-priorities triggers tied; with one waiting warp the entry trigger is
// -0.85 us per R2D2 step against the trigger after the priorities, which was -1.0 us against
// the exit trigger (in-process A/Bs, scripts/ab_inproc.py; profiles/r2/ab_trigger_inproc.txt).
std::atomic<int> g_upd_trigger{0};
// Measurement knob (rpl_debug_set_upd_multi): 1 (default) = batches of n <= HASH_SLOTS / 2 take
// the multi-CTA update kernel, 0 = the single-CTA kernels only.
std::atomic<int> g_upd_multi{1};

int launch_update(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx, const float* td,
                  const int64_t* q, int mode, int64_t n, double alpha, double eps_p, int32_t* err,
                  void* stream, int force_slow, int64_t T_p = 0, double eta = 0.0, int live_only = 0) {
  if (!layout_ok(L) || !tree || n < 0) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  if (!idx) return RPL_EINVAL;
  void (*kern)(TreeDev, int64_t*, const int64_t*, const float*, const int64_t*, int64_t, double, double, int32_t*, int,
               int64_t, double, int, int) = mode == MODE_SEQ  ? k_tree_update<MODE_SEQ>
                                        : mode == MODE_Q ? k_tree_update<MODE_Q>
                                        : mode == MODE_MAXSEEN ? k_tree_update<MODE_MAXSEEN>
                                                               : k_tree_update<MODE_TD>;
  const int trig = g_upd_trigger.load(std::memory_order_relaxed);
  // multi-CTA where it wins (scripts/upd_multi_probe.py, graph of back-to-back updates): the
  // sequence mix at every n <= 1024 (n = 64: 3.9 vs 4.9 us, 512: 7.8 vs 19.8 us); the plain
  // transform only up to n = 64 (beyond, every CTA's hash of the whole batch costs more than
  // the transform it spreads: n = 512 6.4 vs 3.5 us)
  if (g_upd_multi.load(std::memory_order_relaxed) && n <= (mode == MODE_SEQ ? HASH_SLOTS / 2 : 64)) {
    void (*km)(TreeDev, int64_t*, const int64_t*, const float*, const int64_t*, int64_t, double, double, int32_t*, int,
               int64_t, double, int, int) = mode == MODE_SEQ  ? k_tree_update_multi<MODE_SEQ>
                                            : mode == MODE_Q ? k_tree_update_multi<MODE_Q>
                                            : mode == MODE_MAXSEEN ? k_tree_update_multi<MODE_MAXSEEN>
                                                                   : k_tree_update_multi<MODE_TD>;
    const int epc = mode == MODE_SEQ ? UPDM_THREADS / 8 : UPDM_THREADS;
    return launch_pdl(km, dim3((unsigned)((n + epc - 1) / epc)), dim3(UPDM_THREADS), 0, as_stream(stream), tree_dev(L),
                      tree, idx, td, q, n, alpha, eps_p, err, force_slow, T_p, eta, live_only, trig);
  }
  return launch_pdl(kern, dim3(1), dim3(UPD_THREADS), 0, as_stream(stream), tree_dev(L), tree, idx, td, q, n, alpha,
                    eps_p, err, force_slow, T_p, eta, live_only, trig);
}

}  // namespace

// Knob state for rpl_config (abi.cu).
void cfg_tree(int* stage_on, int* upd_threads, int* sample_warps, int* stage_words, int* hash_slots) {
  *stage_on = tree_stage_on();
  *upd_threads = UPD_THREADS;
  *sample_warps = SAMPLE_WARPS;
  *stage_words = STAGE_WORDS;
  *hash_slots = HASH_SLOTS;
}
}  // namespace rpl

using namespace rpl;

extern "C" int rpl_sumtree_layout(int64_t n_leaves, int32_t fanout, int32_t frac_bits, rpl_tree_layout* out) {
  if (!out || n_leaves < 1 || fanout < 2 || fanout > 32 || (fanout & (fanout - 1)) != 0 || frac_bits < 0 ||
      frac_bits > 62)
    return RPL_EINVAL;
  int depth = 1;
  int64_t capn = fanout;
  while (capn < n_leaves) {
    capn *= fanout;
    ++depth;
    if (depth + 1 > RPL_MAX_LEVELS) return RPL_EUNSUPPORTED;
  }
  rpl_tree_layout L{};
  L.n_leaves = n_leaves;
  L.fanout = fanout;
  L.depth = depth;
  L.frac_bits = frac_bits;
  L.q_cap = INT64_MAX / n_leaves;
  int64_t off = 0;
  for (int l = 0; l <= depth; ++l) {
    int64_t span = 1;
    for (int i = 0; i < depth - l; ++i) span *= fanout;
    const int64_t nodes = (n_leaves + span - 1) / span;
    const int64_t len = l == 0 ? 1 : ((nodes + fanout - 1) / fanout) * fanout;
    L.level_off[l] = off;
    L.level_len[l] = len;
    off += len;
  }
  L.hdr_off = off;
  L.n_words = off + 8;
  *out = L;
  return RPL_OK;
}

extern "C" int rpl_sumtree_init(const rpl_tree_layout* L, int64_t* tree, void* stream) {
  if (!layout_ok(L) || !tree) return RPL_EINVAL;
  if (cudaMemsetAsync(tree, 0, (size_t)L->n_words * sizeof(int64_t), as_stream(stream)) != cudaSuccess)
    return RPL_ECUDA;
  k_tree_header<<<1, 1, 0, as_stream(stream)>>>(tree + L->hdr_off, (int64_t)1 << L->frac_bits);
  return launch_status();
}

extern "C" int rpl_sumtree_update(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                                  const float* td_abs, int64_t n, double alpha, double eps_p,
                                  int32_t* dev_err, void* stream) {
  if (n > 0 && !td_abs) return RPL_EINVAL;
  if (!(alpha >= 0.0) || !(eps_p >= 0.0)) return RPL_EINVAL;
  return launch_update(L, tree, idx, td_abs, nullptr, MODE_TD, n, alpha, eps_p, dev_err, stream, 0);
}

extern "C" int rpl_sumtree_set_q(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx, const int64_t* q,
                                 int64_t n, int32_t* dev_err, void* stream) {
  return launch_update(L, tree, idx, nullptr, q, q ? MODE_Q : MODE_MAXSEEN, n, 0.0, 0.0, dev_err, stream, 0);
}

extern "C" int rpl_sumtree_sample(const rpl_tree_layout* L, int64_t* tree, int64_t n, const uint64_t* draws,
                                  uint64_t seed, uint64_t offset, double beta, int64_t* out_idx, int64_t* out_q,
                                  int64_t* out_qmin, float* out_w, int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || n < 1 || n > (1ll << 30)) return RPL_EINVAL;
  if (out_w && !(beta >= 0.0)) return RPL_EINVAL;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  return launch_pdl(k_tree_sample<false>, dim3((unsigned)blocks), dim3(SAMPLE_WARPS * 32), 0, as_stream(stream),
                    tree_dev(L), tree, n, draws, seed, offset, beta, out_idx, out_q, out_qmin, out_w, dev_err, 0, 1,
                    (int64_t)0, (const int64_t*)nullptr, 0, (int64_t*)nullptr, (int64_t* const*)nullptr, stage_cap(tree),
                    1, (int64_t*)nullptr);
}

extern "C" int rpl_sumtree_sample_stream(const rpl_tree_layout* L, int64_t* tree, int64_t n, uint64_t seed,
                                         double beta, int64_t* out_idx, int64_t* out_q, int64_t* out_qmin,
                                         float* out_w, int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || n < 1 || n > (1ll << 30)) return RPL_EINVAL;
  if (out_w && !(beta >= 0.0)) return RPL_EINVAL;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  return launch_pdl(k_tree_sample<false>, dim3((unsigned)blocks), dim3(SAMPLE_WARPS * 32), 0, as_stream(stream),
                    tree_dev(L), tree, n, (const uint64_t*)nullptr, seed, (uint64_t)0, beta, out_idx, out_q, out_qmin,
                    out_w, dev_err, 0, 1, (int64_t)0, (const int64_t*)nullptr, 1, (int64_t*)nullptr,
                    (int64_t* const*)nullptr, stage_cap(tree), 1, (int64_t*)nullptr);
}

extern "C" int rpl_sumtree_sample_sharded(const rpl_tree_layout* L, int64_t* tree, int32_t rank, int32_t n_shards,
                                          int64_t shard_leaves, const int64_t* shard_totals, int64_t n,
                                          const uint64_t* draws, uint64_t seed, uint64_t offset, int32_t use_stream,
                                          int64_t* out_idx, int64_t* out_q, int64_t* out_qmin, int64_t* out_count,
                                          int32_t* dev_err, void* stream) {
  if (draws && use_stream) return RPL_EINVAL;
  if (!layout_ok(L) || !tree || !out_idx || !out_q || !shard_totals || n < 1 || n > (1ll << 30)) return RPL_EINVAL;
  if (n_shards < 1 || rank < 0 || rank >= n_shards || shard_leaves < L->n_leaves) return RPL_EINVAL;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  return launch_pdl(k_tree_sample<true>, dim3((unsigned)blocks), dim3(SAMPLE_WARPS * 32), 0, as_stream(stream),
                    tree_dev(L), tree, n, draws, seed, offset, 0.0, out_idx, out_q, out_qmin, (float*)nullptr, dev_err,
                    (int)rank, (int)n_shards, shard_leaves, shard_totals, (int)use_stream, out_count,
                    (int64_t* const*)nullptr, stage_cap(tree), 1, (int64_t*)nullptr);
}

extern "C" int rpl_sumtree_sample_sharded_p2p(const rpl_tree_layout* L, int64_t* tree, int32_t rank,
                                              int32_t n_shards, int64_t shard_leaves, int64_t* const* boards,
                                              int64_t n, uint64_t seed, int64_t* out_idx, int64_t* out_q,
                                              int64_t* out_count, int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || !out_count || !boards || n < 1 || n > (1ll << 30))
    return RPL_EINVAL;
  if (n_shards < 1 || n_shards > BOARD_MAX_WORLD || rank < 0 || rank >= n_shards || shard_leaves < L->n_leaves)
    return RPL_EINVAL;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  return launch_pdl(k_tree_sample<true>, dim3((unsigned)blocks), dim3(SAMPLE_WARPS * 32), 0, as_stream(stream),
                    tree_dev(L), tree, n, (const uint64_t*)nullptr, seed, (uint64_t)0, 0.0, out_idx, out_q,
                    (int64_t*)nullptr, (float*)nullptr, dev_err, (int)rank, (int)n_shards, shard_leaves,
                    (const int64_t*)nullptr, 1, out_count, boards, stage_cap(tree), 1, (int64_t*)nullptr);
}

extern "C" int rpl_sumtree_find(const rpl_tree_layout* L, const int64_t* tree, const int64_t* prefix, int64_t n,
                                int64_t* out_idx, int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !prefix || !out_idx || n < 0) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  k_tree_find<<<(unsigned)blocks, SAMPLE_WARPS * 32, 0, as_stream(stream)>>>(tree_dev(L), tree, prefix, n,
                                                                              out_idx, dev_err);
  return launch_status();
}

extern "C" int rpl_sumtree_total(const rpl_tree_layout* L, const int64_t* tree, int64_t* out_total, void* stream) {
  if (!layout_ok(L) || !tree || !out_total) return RPL_EINVAL;
  return launch_pdl(k_tree_total, dim3(1), dim3(1), 0, as_stream(stream), tree, out_total);
}

extern "C" int rpl_mintree_rebuild(const rpl_tree_layout* L, const int64_t* tree, void* stream) {
  if (!layout_ok(L) || !tree) return RPL_EINVAL;
  TreeDev T = tree_dev(L);
  for (int l = L->depth - 1; l >= 0; --l) {
    const int64_t len = L->level_len[l];
    int64_t blocks = (len + 7) / 8;  // 8 warps per CTA
    if (blocks > 8 * (int64_t)sm_count()) blocks = 8 * (int64_t)sm_count();
    const int s = launch_pdl(k_mintree_level, dim3((unsigned)blocks), dim3(256), 0, as_stream(stream), T, tree, l, len,
                             (int64_t)L->level_len[l + 1]);
    if (s != RPL_OK) return s;
  }
  return RPL_OK;
}

extern "C" int rpl_mintree_attach(const rpl_tree_layout* L, int64_t* tree, int64_t* mins, void* stream) {
  if (!layout_ok(L) || !tree) return RPL_EINVAL;
  const int s = launch_pdl(k_set_word, dim3(1), dim3(1), 0, as_stream(stream), tree + L->hdr_off + HDR_MINTREE,
                           (int64_t) reinterpret_cast<uintptr_t>(mins));
  if (s != RPL_OK || !mins) return s;
  return rpl_mintree_rebuild(L, tree, stream);
}

extern "C" int rpl_sumtree_total_min(const rpl_tree_layout* L, const int64_t* tree, int64_t* out, void* stream) {
  if (!layout_ok(L) || !tree || !out) return RPL_EINVAL;
  return launch_pdl(k_tree_total_min, dim3(1), dim3(1), 0, as_stream(stream), tree, L->hdr_off, out);
}

extern "C" int rpl_sumtree_sample_sharded_pairs(const rpl_tree_layout* L, int64_t* tree, int32_t rank,
                                                int32_t n_shards, int64_t shard_leaves, const int64_t* shard_pairs,
                                                int64_t n, uint64_t seed, int64_t* out_idx, int64_t* out_q,
                                                int64_t* out_qmin, int64_t* out_count, int64_t* out_bufmin,
                                                int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || !shard_pairs || !out_count || n < 1 || n > (1ll << 30))
    return RPL_EINVAL;
  if (n_shards < 1 || rank < 0 || rank >= n_shards || shard_leaves < L->n_leaves) return RPL_EINVAL;
  const int64_t blocks = (n + SAMPLE_WARPS - 1) / SAMPLE_WARPS;
  return launch_pdl(k_tree_sample<true>, dim3((unsigned)blocks), dim3(SAMPLE_WARPS * 32), 0, as_stream(stream),
                    tree_dev(L), tree, n, (const uint64_t*)nullptr, seed, (uint64_t)0, 0.0, out_idx, out_q, out_qmin,
                    (float*)nullptr, dev_err, (int)rank, (int)n_shards, shard_leaves, shard_pairs, 1, out_count,
                    (int64_t* const*)nullptr, stage_cap(tree), 2, out_bufmin);
}

extern "C" int rpl_sumtree_rebuild(const rpl_tree_layout* L, int64_t* tree, void* stream) {
  if (!layout_ok(L) || !tree) return RPL_EINVAL;
  TreeDev T = tree_dev(L);
  for (int l = L->depth - 1; l >= 0; --l) {
    const int64_t len = L->level_len[l];
    int64_t span = 1;
    for (int i = 0; i < L->depth - l; ++i) span *= L->fanout;
    const int64_t real = (L->n_leaves + span - 1) / span;
    k_tree_level<<<(unsigned)((len + 255) / 256), 256, 0, as_stream(stream)>>>(T, tree, l, len, real);
    int s = launch_status();
    if (s != RPL_OK) return s;
  }
  return rpl_mintree_rebuild(L, tree, stream);  // the attached min-tree too (no-op without one)
}

extern "C" int rpl_is_weights(const int64_t* q, const int64_t* qmin, int64_t n, double beta, float* w,
                              void* stream) {
  if (!q || !qmin || !w || n < 0 || !(beta >= 0.0)) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  return launch_pdl(k_is_weights, dim3((unsigned)(blocks > 1024 ? 1024 : blocks)), dim3(threads), 0,
                    as_stream(stream), q, qmin, n, beta, w);
}

extern "C" int rpl_debug_priority_values(const float* td_abs, int64_t n, double alpha, double eps_p,
                                         int32_t force_slow, float* out_v, uint8_t* out_slow, void* stream) {
  if (!td_abs || !out_v || n < 0 || !(alpha >= 0.0) || !(eps_p >= 0.0)) return RPL_EINVAL;
  if (n == 0) return RPL_OK;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  k_priority_values<<<(unsigned)(blocks > 4096 ? 4096 : blocks), threads, 0, as_stream(stream)>>>(
      td_abs, n, alpha, eps_p, force_slow, out_v, out_slow);
  return launch_status();
}

extern "C" int rpl_sample_uniform(int64_t n, uint64_t seed, uint64_t offset, uint64_t* ctr, int64_t lo_row,
                                  int64_t n_rows, int64_t cap_T, int64_t B, int64_t* out_idx, void* stream) {
  if (!out_idx || n < 1 || B < 1 || cap_T < 1 || n_rows < 1 || n_rows > cap_T || lo_row < 0 || lo_row >= cap_T)
    return RPL_EINVAL;
  if ((double)n_rows * (double)B >= 4.6e18) return RPL_EINVAL;
  return launch_pdl(k_sample_uniform, dim3(1), dim3(UNI_THREADS), 0, as_stream(stream), n, seed, offset, ctr, lo_row,
                    n_rows, cap_T, B, out_idx);
}

extern "C" int rpl_sumtree_update_seq(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                                      const float* td_steps, int64_t T_p, int64_t n, double eta, double alpha,
                                      double eps_p, int32_t flags, int32_t* dev_err, void* stream) {
  if (n > 0 && (!td_steps || T_p < 1 || T_p > (1ll << 30))) return RPL_EINVAL;
  if (!(alpha >= 0.0) || !(eps_p >= 0.0) || !(eta >= 0.0 && eta <= 1.0) || (flags & ~RPL_UPD_LIVE_ONLY))
    return RPL_EINVAL;
  return launch_update(L, tree, idx, td_steps, nullptr, MODE_SEQ, n, alpha, eps_p, dev_err, stream, 0, T_p, eta,
                       (flags & RPL_UPD_LIVE_ONLY) ? 1 : 0);
}

extern "C" int rpl_sumtree_update_ex(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx, const float* td_abs,
                                     int64_t n, double alpha, double eps_p, int32_t flags, int32_t* dev_err,
                                     void* stream) {
  if (n > 0 && !td_abs) return RPL_EINVAL;
  if (!(alpha >= 0.0) || !(eps_p >= 0.0) || (flags & ~RPL_UPD_LIVE_ONLY)) return RPL_EINVAL;
  return launch_update(L, tree, idx, td_abs, nullptr, MODE_TD, n, alpha, eps_p, dev_err, stream, 0, 0, 0.0,
                       (flags & RPL_UPD_LIVE_ONLY) ? 1 : 0);
}

extern "C" int rpl_sumtree_min(const rpl_tree_layout* L, const int64_t* tree, int64_t* out_min, void* stream) {
  if (!layout_ok(L) || !tree || !out_min) return RPL_EINVAL;
  int r = launch_pdl(k_min_init, dim3(1), dim3(1), 0, as_stream(stream), out_min);
  if (r != RPL_OK) return r;
  const int threads = 256;
  int64_t blocks = (L->n_leaves + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 4;
  if (blocks > cap) blocks = cap;
  return launch_pdl(k_leaf_min, dim3((unsigned)blocks), dim3(threads), 0, as_stream(stream),
                    (const int64_t*)(tree + L->level_off[L->depth]), L->n_leaves, out_min);
}

extern "C" int rpl_sumtree_sample_unique(const rpl_tree_layout* L, int64_t* tree, int64_t n, uint64_t seed,
                                         uint64_t offset, int32_t use_stream, int64_t* out_idx, int64_t* out_q,
                                         int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || n < 1 || n > (1ll << 30)) return RPL_EINVAL;
  return launch_pdl(k_tree_sample_unique, dim3(1), dim3(32), 0, as_stream(stream), tree_dev(L), tree, n, seed, offset,
                    (int)(use_stream != 0), out_idx, out_q, dev_err);
}

extern "C" int rpl_sumtree_update_sample(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                                         const float* td, int64_t T_p, int64_t n_upd, double eta, double alpha,
                                         double eps_p, int32_t flags, int64_t n, uint64_t seed, int64_t* out_idx,
                                         int64_t* out_q, int32_t* dev_err, void* stream) {
  if (!layout_ok(L) || !tree || !out_idx || !out_q || n < 1 || n > (1ll << 30) || n_upd < 0 || T_p < 0 ||
      T_p > (1ll << 30))
    return RPL_EINVAL;
  if (n_upd > 0 && (!idx || !td)) return RPL_EINVAL;
  if (!(alpha >= 0.0) || !(eps_p >= 0.0) || !(eta >= 0.0 && eta <= 1.0) || (flags & ~RPL_UPD_LIVE_ONLY))
    return RPL_EINVAL;
  int64_t blocks = (n + FUSED_WARPS - 1) / FUSED_WARPS;
  if (blocks > sm_count()) blocks = sm_count();  // one CTA per SM at most
  // cooperative: the grid barrier's co-residency is guaranteed by the runtime, not assumed
  return launch_coop(k_tree_update_sample, dim3((unsigned)blocks), dim3(FUSED_THREADS), 0, as_stream(stream),
                    tree_dev(L), tree, idx, td, n_upd, T_p, eta, alpha, eps_p, (flags & RPL_UPD_LIVE_ONLY) ? 1 : 0, n,
                    seed, out_idx, out_q, dev_err);
}

extern "C" int rpl_debug_set_tree_stage(int32_t on) {
  if (on != 0 && on != 1) return RPL_EINVAL;
  g_tree_stage.store(on);
  return RPL_OK;
}

extern "C" int rpl_debug_set_upd_multi(int32_t on) {
  if (on != 0 && on != 1) return RPL_EINVAL;
  g_upd_multi.store(on);
  return RPL_OK;
}

extern "C" int rpl_debug_set_upd_trigger(int32_t at) {
  if (at != -1 && at != 0 && at != 2 && at != 3 && at != 4) return RPL_EINVAL;
  g_upd_trigger.store(at);
  return RPL_OK;
}

extern "C" int rpl_debug_trace_reset(void) {
#ifdef RPL_TRACE
  unsigned long long z[16] = {0};
  return cudaMemcpyToSymbol(rpl::g_trace, z, sizeof(z)) == cudaSuccess && rpl_debug_gather_trace_reset() == RPL_OK
             ? RPL_OK : RPL_ECUDA;
#else
  return RPL_EUNSUPPORTED;
#endif
}

extern "C" int rpl_debug_trace(int64_t* out, int32_t n) {
#ifdef RPL_TRACE
  if (!out || n < 1 || n > 16) return RPL_EINVAL;
  return cudaMemcpyFromSymbol(out, rpl::g_trace, sizeof(int64_t) * (size_t)n) == cudaSuccess ? RPL_OK : RPL_ECUDA;
#else
  (void)out;
  (void)n;
  return RPL_EUNSUPPORTED;  // measurement builds only (-DRPL_TRACE)
#endif
}
