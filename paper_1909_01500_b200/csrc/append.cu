// Ring append and tree validity maintenance.
//
// P:75-84 (asynchronous sampling: the sampler writes batches into the replay buffer
// while the optimiser samples from it); S:581-589 (append at the cursor, ring wrap),
// S:660 (new samples enter at max-priority-seen), S:661 (a sample is valid only once its
// n-step lookahead / sequence window is stored and while its history is not yet
// overwritten); readings §8c #2, #12, #16.
//
//  rpl_ring_append      a sampler batch of T_b rows -> ring rows cursor .. cursor+T_b-1
//                       (mod cap_T): at most two cudaMemcpyAsync per array (the copy
//                       engines, host or device source), plus the stored RNN state of
//                       every batch row that starts a storage block.
//  rpl_replay_validity  every leaf's validity before (cursor_old, size_old) and after
//                       (cursor_new, size_new) the append; a leaf that became valid gets
//                       q = max-seen, one that became invalid q = 0, each with its exact
//                       int64 delta added to its ancestors (no duplicates: one thread per
//                       leaf, so no dedupe is needed).  One thread per leaf, grid-wide.
#include "common.cuh"

namespace rpl {
namespace {

__device__ __forceinline__ int64_t age_of(int64_t row, int64_t cursor, int64_t cap) {
  int64_t a = (cursor - 1 - row) % cap;
  return a < 0 ? a + cap : a;
}

// §8c #2 / #14: transition row valid iff rows row-k+1 .. row+n are stored.
__device__ __forceinline__ bool valid_transition(int64_t row, int64_t cursor, int64_t size, int64_t cap, int k,
                                                 int n) {
  const int64_t a = age_of(row, cursor, cap);
  return size > 0 && a >= n && a <= size - k;
}

// §8c #16: sequence block valid iff rows row0-max(k-1,1) .. row0+L-1 are stored.
__device__ __forceinline__ bool valid_sequence(int64_t row0, int64_t cursor, int64_t size, int64_t cap, int k,
                                               int L) {
  const int64_t a = age_of(row0, cursor, cap);
  const int hist = k - 1 > 1 ? k - 1 : 1;
  return size > 0 && a >= L - 1 && a + hist <= size - 1;
}

__global__ void k_replay_validity(TreeDev T, int64_t* __restrict__ tree, int kind, int64_t cap, int64_t B, int k,
                                  int n_step, int L, int period, int64_t c0, int64_t s0, int64_t c1, int64_t s1) {
  pdl_wait();
  int64_t* leaves = tree + T.level_off[T.depth];
  const int64_t maxseen = __ldcg(tree + T.hdr_off);
  const int64_t nl = T.n_leaves;
  const int lane = threadIdx.x & 31;
  for (int64_t leaf = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; leaf - lane < nl;
       leaf += (int64_t)gridDim.x * blockDim.x) {
    int64_t delta = 0;
    if (leaf < nl) {
      const int64_t unit = leaf / B;  // row (transitions) or block (sequences)
      bool v0, v1;
      if (kind == RPL_GATHER_TRANSITION) {
        v0 = valid_transition(unit, c0, s0, cap, k, n_step);
        v1 = valid_transition(unit, c1, s1, cap, k, n_step);
      } else {
        v0 = valid_sequence(unit * period, c0, s0, cap, k, L);
        v1 = valid_sequence(unit * period, c1, s1, cap, k, L);
      }
      if (v0 != v1) {
        const int64_t q = v1 ? maxseen : 0;
        const int64_t old = __ldcg(leaves + leaf);
        leaves[leaf] = q;
        delta = q - old;
        if (delta != 0) {
          int64_t node = leaf;
          for (int l = T.depth - 1; l >= 1; --l) {
            node >>= T.log2w;
            atomicAdd(reinterpret_cast<unsigned long long*>(tree + T.level_off[l] + node), (unsigned long long)delta);
          }
        }
      }
    }
    const int64_t rd = warp_sum64(delta);
    if (lane == 0 && rd != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(tree + T.level_off[0]), (unsigned long long)rd);
  }
}

// Copy rows [0, T_b) of a [T_b, row_bytes] batch to ring rows cursor.. (mod cap): <= 2 copies.
int copy_rows(void* ring, const void* src, int64_t cursor, int64_t cap, int64_t T_b, int64_t row_bytes,
              cudaStream_t st) {
  if (!src || row_bytes == 0 || T_b == 0) return RPL_OK;
  const int64_t first = T_b < cap - cursor ? T_b : cap - cursor;
  uint8_t* r = static_cast<uint8_t*>(ring);
  const uint8_t* s = static_cast<const uint8_t*>(src);
  if (cudaMemcpyAsync(r + cursor * row_bytes, s, (size_t)(first * row_bytes), cudaMemcpyDefault, st) != cudaSuccess)
    return RPL_ECUDA;
  if (T_b > first &&
      cudaMemcpyAsync(r, s + first * row_bytes, (size_t)((T_b - first) * row_bytes), cudaMemcpyDefault, st) !=
          cudaSuccess)
    return RPL_ECUDA;
  return RPL_OK;
}

}  // namespace
}  // namespace rpl

using namespace rpl;

extern "C" int rpl_ring_append(const rpl_gather_desc* ring, const void* obs, const void* act, const float* rew,
                               const uint8_t* done, const void* rnn, int64_t T_b, void* stream) {
  if (!ring || T_b < 0 || T_b > ring->cap_T || ring->cap_T < 1 || ring->B < 1 || ring->cursor < 0 ||
      ring->cursor >= ring->cap_T)
    return RPL_EINVAL;
  if (T_b == 0) return RPL_OK;
  if ((obs && !ring->obs) || (act && !ring->act) || (rew && !ring->rew) || (done && !ring->done)) return RPL_EINVAL;
  cudaStream_t st = as_stream(stream);
  const int64_t cap = ring->cap_T, B = ring->B, c = ring->cursor;
  int r;
  if ((r = copy_rows(const_cast<void*>(ring->obs), obs, c, cap, T_b, B * ring->obs_bytes, st)) != RPL_OK) return r;
  if ((r = copy_rows(const_cast<void*>(ring->act), act, c, cap, T_b, B * ring->act_bytes, st)) != RPL_OK) return r;
  if ((r = copy_rows(const_cast<float*>(ring->rew), rew, c, cap, T_b, B * 4, st)) != RPL_OK) return r;
  if ((r = copy_rows(const_cast<uint8_t*>(ring->done), done, c, cap, T_b, B, st)) != RPL_OK) return r;
  if (rnn) {
    // stored state of the batch rows that start a block (row % period == 0), in batch order
    if (!ring->rnn || ring->period < 1 || cap % ring->period != 0 || ring->rnn_parts < 1 || ring->rnn_bytes < 1)
      return RPL_EINVAL;
    const int64_t P = ring->period, blk_bytes = B * ring->rnn_parts * ring->rnn_bytes;
    const int64_t first_t = (P - c % P) % P;  // first batch row that starts a block
    int64_t j = 0;
    for (int64_t t = first_t; t < T_b; t += P, ++j) {
      const int64_t blk = ((c + t) % cap) / P;
      if (cudaMemcpyAsync(static_cast<uint8_t*>(const_cast<void*>(ring->rnn)) + blk * blk_bytes,
                          static_cast<const uint8_t*>(rnn) + j * blk_bytes, (size_t)blk_bytes, cudaMemcpyDefault,
                          st) != cudaSuccess)
        return RPL_ECUDA;
    }
  }
  return RPL_OK;
}

extern "C" int rpl_ring_append_rows(void* ring_array, int64_t row_bytes, int64_t cap_T, int64_t cursor,
                                    const void* src, int64_t T_b, void* stream) {
  if (!ring_array || !src || row_bytes < 1 || cap_T < 1 || cursor < 0 || cursor >= cap_T || T_b < 0 || T_b > cap_T)
    return RPL_EINVAL;
  return copy_rows(ring_array, src, cursor, cap_T, T_b, row_bytes, as_stream(stream));
}

extern "C" int rpl_replay_validity(const rpl_tree_layout* L, int64_t* tree, int32_t kind, int64_t cap_T, int64_t B,
                                   int32_t k, int32_t n_step, int32_t seq_len, int32_t period, int64_t cursor_old,
                                   int64_t size_old, int64_t cursor_new, int64_t size_new, void* stream) {
  if (!L || !tree || cap_T < 1 || B < 1 || k < 1 || cursor_old < 0 || cursor_old >= cap_T || cursor_new < 0 ||
      cursor_new >= cap_T || size_old < 0 || size_old > cap_T || size_new < 0 || size_new > cap_T)
    return RPL_EINVAL;
  int64_t units;
  if (kind == RPL_GATHER_TRANSITION) {
    if (n_step < 1) return RPL_EINVAL;
    units = cap_T;
  } else if (kind == RPL_GATHER_SEQUENCE) {
    if (seq_len < 1 || period < 1 || cap_T % period != 0) return RPL_EINVAL;
    units = cap_T / period;
  } else {
    return RPL_EINVAL;
  }
  if (units * B != L->n_leaves) return RPL_EINVAL;
  const int threads = 256;
  int64_t blocks = (L->n_leaves + threads - 1) / threads;
  const int64_t cap_blocks = (int64_t)sm_count() * 8;
  if (blocks > cap_blocks) blocks = cap_blocks;
  const int s = launch_pdl(k_replay_validity, dim3((unsigned)blocks), dim3(threads), 0, as_stream(stream),
                           tree_dev(L), tree, (int)kind, cap_T, B, (int)k, (int)n_step, (int)seq_len, (int)period,
                           cursor_old, size_old, cursor_new, size_new);
  if (s != RPL_OK) return s;
  // an attached min-tree (R29) is rebuilt from the new leaves (device-side no-op without one)
  return rpl_mintree_rebuild(L, tree, stream);
}
