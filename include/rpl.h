/*
 * rpl.h — C ABI of librpl: the B200 (sm_100a) replay + return-estimation hot path
 * of rlpyt (arXiv 1909.01500).  SURVEY.md §8(b) lists these entry points.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = /root/reference/SPEC.md
 * line n, "§8c #k" = reading k of SURVEY.md §8(c) (restated in DESIGN.md).
 *
 * Conventions for every call
 *  - Pointers are CUDA DEVICE pointers unless the comment says (host).
 *  - `stream` is a cudaStream_t passed as an opaque pointer (NULL = legacy
 *    default stream).  Every call only ENQUEUES kernels on `stream` and returns;
 *    no call synchronises the device or allocates memory.  Torch (or any caller)
 *    owns all device buffers.
 *  - Layouts are row-major and contiguous.  [T,B] is time-major ("[Time, Batch]",
 *    P:232): element (t,b) is at t*B + b.
 *  - Return value: RPL_OK (0) or a negative rpl_status.  Argument/shape errors are
 *    detected on the host before anything is enqueued.  Data-dependent errors are
 *    OR-ed into *dev_err (a device int32, may be NULL) as RPL_DERR_* bits while the
 *    kernel still produces the defined output described per call.
 *  - Calls on the same sum tree must be stream-ordered by the caller (the device
 *    analogue of rlpyt's replay read-write lock).  No kernel uses
 *    floating-point atomics: every output is bit-deterministic for fixed inputs.
 *  - Thread safety: calls may come from several host threads / devices.  The library's
 *    only state is per-device attribute caches (SM count, raised shared-memory limits)
 *    behind a mutex, a one-time driver-entry-point lookup and an atomic launch counter;
 *    the rpl_debug_* knobs are process-global and meant for tests.
 *  - rpl_ring_append uses cudaMemcpyAsync: with pageable (non-pinned) host sources the
 *    copy is synchronous with respect to the host.
 */
#ifndef RPL_H_
#define RPL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RPL_ABI_VERSION 2  /* 2: rpl_gather_desc.work appended */
#define RPL_MAX_LEVELS 24

typedef enum {
  RPL_OK = 0,
  RPL_EINVAL = -1,       /* null pointer, bad shape or parameter */
  RPL_ERANGE = -2,       /* host-visible range error (e.g. n_step > T) */
  RPL_EEMPTY = -3,       /* sampling requested with n == 0 where not allowed */
  RPL_ECUDA = -4,        /* kernel launch / CUDA runtime failure */
  RPL_EUNSUPPORTED = -5  /* configuration not supported by this build */
} rpl_status;

/* device error word bits */
enum {
  RPL_DERR_IDX = 1,           /* a leaf index outside [0, n_leaves): entry skipped */
  RPL_DERR_SATURATED = 2,     /* a priority exceeded q_cap: clamped to q_cap */
  RPL_DERR_EMPTY = 4,         /* sampling from a tree whose total is 0: idx = -1 */
  RPL_DERR_INVALID_LEAF = 8,  /* gather window not fully inside the valid ring rows */
  RPL_DERR_TREE = 16,         /* descent found a prefix >= node sum (inconsistent tree) */
  RPL_DERR_PEER = 32          /* a peer's exchange-board value did not arrive within ~2 s */
};

const char* rpl_strerror(int status);
int rpl_abi_version(void);
/* Number of kernel launches this process has issued through librpl (host counter). */
int64_t rpl_launch_count(void);
/* The library's effective configuration as a one-line JSON object written into buf (host,
 * len bytes incl. the terminating NUL): every build-flag knob (launch shapes, RPL_PDL_EARLY,
 * whether the -DRPL_DIAG diagnostics are compiled in) and every runtime knob (RPL_PDL,
 * RPL_TREE_STAGE, RPL_SCAN_VARIANT, RPL_SCAN_TRIGGER, RPL_CARVEOUT, the debug gather variant / diag mask).
 * bench.py records it in its JSON line so that no knob can change the timed path unseen.
 * RPL_EINVAL for a NULL / empty buffer, RPL_ERANGE if it is too short (buf then holds a
 * truncated string). */
int rpl_config(char* buf, int64_t len);

/* =========================================================================
 * (1) Return estimation over time-major [T,B] buffers.  fp32 I/O, fp64
 *     accumulation, one rounding to fp32 per output (§8c #21).
 *     r: rewards f32 [T,B]; d: done u8 [T,B] (non-zero = episode ended after row t, §8c #1;
 *     2 = ended by a time limit, bootstrapped by the _tl variants below, R34).
 * ========================================================================= */

/* R_t = r_t + gamma (1 - d_t) R_{t+1},  R_T = bootstrap[b] (or 0 if bootstrap == NULL).
 * S:346 (discounted return), S:751 (returns).  ret: f32 [T,B].  T, B >= 1. */
int rpl_returns_discounted(const float* r, const uint8_t* d, const float* bootstrap,
                           int64_t T, int64_t B, double gamma, float* ret, void* stream);

/* n-step return, S:591-599, P:38:
 *   R^n_t = sum_{i<n} gamma^i r_{t+i} prod_{j<i} (1 - d_{t+j}),  done^n_t = OR_{i<n} d_{t+i},
 * for output rows t = 0 .. T-n (ret_n, done_n are [T-n+1, B]).
 * If q != NULL (value of s_tau, f32 [T,B]) then q_boot (f32 [B], the value at row T) is
 * required and ret_n holds the target  y_t = R^n_t + gamma^n (1 - done^n_t) q_{t+n}
 * (S:713-714).  If rescale != 0 the target is y_t = h(R^n_t + gamma^n (1-done^n_t) h^-1(q_{t+n}))
 * (§8c #5), or h(R^n_t) when q == NULL; eps = rescale_eps (> 0).
 * done_n may be NULL.  1 <= n <= T, else RPL_ERANGE. */
int rpl_returns_nstep(const float* r, const uint8_t* d, int64_t T, int64_t B, int32_t n,
                      double gamma, const float* q, const float* q_boot, int32_t rescale,
                      double rescale_eps, float* ret_n, uint8_t* done_n, void* stream);

/* GAE:  delta_t = r_t + gamma (1-d_t) V_{t+1} - V_t  (V_T = bootstrap_v[b]),
 * A_t = delta_t + gamma lambda (1-d_t) A_{t+1}, A_T = 0;  ret_t = A_t + V_t.
 * v: f32 [T,B]; bootstrap_v: f32 [B] (required); adv, ret: f32 [T,B] (ret may be NULL). */
int rpl_gae(const float* r, const float* v, const uint8_t* d, const float* bootstrap_v,
            int64_t T, int64_t B, double gamma, double lambda, float* adv, float* ret, void* stream);

/* Time-limit bootstrap variants (reading R34; P:95 fn "bootstrapping the value function when
 * the trajectory ends due to time limit").  d may hold RPL_DONE_TIMEOUT (2): the
 * episode ended after row t by a time limit.  Every non-zero d_t ends the episode (the
 * recursion is cut as above); with v_term (f32 [T,B], device, may be NULL) a time-limit row
 * bootstraps from the value of its final observation: the term gamma * v_term_t stands where
 * gamma * (next value) would have stood —
 *   discounted  R_t = r_t + gamma v_term_t                       at a time-limit row
 *   n-step      R^n_t gets gamma^(j+1) v_term_{t+j} when its first ended row t+j is a
 *               time-limit row (done^n_t stays 1: the learner must not bootstrap again)
 *   GAE         delta_t = r_t + gamma v_term_t - V_t             at a time-limit row
 * v_term is read only at time-limit rows.  With v_term NULL these equal the plain entries
 * (which treat d = 2 as a terminal). */
int rpl_returns_discounted_tl(const float* r, const uint8_t* d, const float* v_term, const float* bootstrap,
                              int64_t T, int64_t B, double gamma, float* ret, void* stream);
int rpl_returns_nstep_tl(const float* r, const uint8_t* d, const float* v_term, int64_t T, int64_t B, int32_t n,
                         double gamma, const float* q, const float* q_boot, int32_t rescale, double rescale_eps,
                         float* ret_n, uint8_t* done_n, void* stream);
int rpl_gae_tl(const float* r, const float* v, const uint8_t* d, const float* v_term, const float* bootstrap_v,
               int64_t T, int64_t B, double gamma, double lambda, float* adv, float* ret, void* stream);

/* Value rescaling h (inverse == 0) or h^-1 (inverse != 0), elementwise over n floats, S:810:
 *   h(x) = sign(x)(sqrt(|x|+1) - 1) + eps x, evaluated in fp64 in the cancellation-free
 *   forms of §8c #4; eps > 0.  x, y: f32 [n] (may alias). */
int rpl_value_rescale(const float* x, float* y, int64_t n, double eps, int32_t inverse, void* stream);

/* =========================================================================
 * (2) Prioritized replay on an int64 fixed-point sum tree ("prioritized replay
 *     (sum tree)").  Storage is ONE caller-owned int64 device array of
 *     layout.n_words words:
 *       [level 0 (root) | level 1 | ... | level depth (leaves)]  then  [header words]
 *     Level l holds level_len[l] nodes at word level_off[l]; node j of level l covers
 *     leaves [j*W^(depth-l), (j+1)*W^(depth-l)); its W children are nodes j*W..j*W+W-1
 *     of level l+1.  Every level is zero-padded to a multiple of W.  Leaf i is word
 *     level_off[depth] + i and holds q_i = round_half_even(RN32(p_i^alpha) * 2^F)
 *     (§8c #7).  Header: [hdr_off+0] max-priority-seen, [hdr_off+1] sampler
 *     ticket (library scratch, always 0 between calls), [hdr_off+2] Philox stream
 *     position used by rpl_sumtree_sample_stream (0 after init), [hdr_off+3] grid-barrier
 *     arrivals (scratch, 0 between calls), [hdr_off+4] grid-barrier generation (scratch),
 *     [hdr_off+5] the attached min-tree's device address (0 = none; rpl_mintree_attach),
 *     [hdr_off+6] the global buffer min written by the sharded samplers, [hdr_off+7] unused.
 * ========================================================================= */
typedef struct {
  int64_t n_leaves;
  int32_t fanout;       /* W: power of two in [2, 32] */
  int32_t depth;        /* D >= 1: smallest with W^D >= n_leaves */
  int32_t frac_bits;    /* F in [0, 62] */
  int32_t _pad;
  int64_t q_cap;        /* floor((2^63-1) / n_leaves): the root never overflows */
  int64_t level_off[RPL_MAX_LEVELS];
  int64_t level_len[RPL_MAX_LEVELS];  /* padded to a multiple of W (except the root) */
  int64_t hdr_off;
  int64_t n_words;      /* int64 words the caller must allocate */
} rpl_tree_layout;

/* The tree of n_leaves leaves ("prioritized replay (sum tree)"; S:556-557 sum tree over
 * the priorities; reading R7 for F = frac_bits, the fixed-point fraction of a leaf q, and
 * q_cap = floor((2^63-1)/n_leaves), so the root of any leaf values <= q_cap fits in int64):
 * fills *out (host POD) with the depth, every level's offset and padded length and n_words,
 * the int64 words the caller allocates (the library never allocates).  n_leaves >= 1, fanout
 * in {2,4,8,16,32}, frac_bits in [0,62]; RPL_EINVAL otherwise, RPL_EUNSUPPORTED when the depth
 * would exceed RPL_MAX_LEVELS - 1.  Host only: enqueues nothing. */
int rpl_sumtree_layout(int64_t n_leaves, int32_t fanout, int32_t frac_bits, rpl_tree_layout* out);

/* Zero every node and set max-seen to 2^F (priority 1.0, §8c #12). */
int rpl_sumtree_init(const rpl_tree_layout* L, int64_t* tree, void* stream);

/* Batched priority update (a5-a7): for k in 0..n-1, p = RN64(|td_abs[k]| + eps_p),
 * q = RNE(RN32(p^alpha) * 2^F) clamped to q_cap; leaf idx[k] := q.  Duplicate indices: the
 * LAST position in the batch wins.  Internal nodes are updated exactly (int64).
 * max-seen := max(max-seen, every valid q in the batch).  idx[k] < 0 is a padding entry (e.g. a
 * sample another shard owns) and is skipped silently; idx[k] >= n_leaves -> skipped + RPL_DERR_IDX.
 * alpha >= 0, eps_p >= 0.  n >= 0 (n == 0 is a no-op). */
int rpl_sumtree_update(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                       const float* td_abs, int64_t n, double alpha, double eps_p,
                       int32_t* dev_err, void* stream);

/* R2D2 sequence priorities (§8f NEXT-1; "eta = 0.9 mix of max and mean", reading
 * R26): td_steps [T_p, n] f32, time-major per-step |delta| of the n sampled sequences
 * (e.g. the 80 train rows).  Sequence k gets
 *   td_k = RN32(RN64(RN64(eta * max_t |d_tk|) + RN64(RN64(1 - eta) * mean_k))),
 *   mean_k = RN64(S_k / T_p),  S_k = RN64(the EXACT sum over t of |d_tk|)
 * (S_k is rounded once, so it does not depend on any summation order; NaN if a |d| is NaN,
 * +inf if one is infinite; no fused multiply-add), then exactly rpl_sumtree_update's
 * transform and write: identical to rpl_sumtree_update(idx, td, n, alpha, eps_p).
 * eta in [0, 1]; 1 <= T_p <= 2^30.  flags: 0 or RPL_UPD_LIVE_ONLY. */
int rpl_sumtree_update_seq(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                           const float* td_steps, int64_t T_p, int64_t n, double eta, double alpha,
                           double eps_p, int32_t flags, int32_t* dev_err, void* stream);

/* rpl_sumtree_update with flags.  RPL_UPD_LIVE_ONLY: entries whose leaf is currently 0 (made
 * invalid by an append since it was sampled, or never written) are skipped silently and do
 * not count toward max-seen — a learner's late priorities cannot revive a stale leaf
 * (asynchronous replay; reading R30). */
enum { RPL_UPD_LIVE_ONLY = 1 };
int rpl_sumtree_update_ex(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx, const float* td_abs,
                          int64_t n, double alpha, double eps_p, int32_t flags, int32_t* dev_err, void* stream);

/* Direct leaf write (append / validity maintenance, §8a a12): leaf idx[k] := q[k]
 * (last write wins; max-seen updated), or := current max-seen when q == NULL.
 * q values > q_cap are clamped (+ RPL_DERR_SATURATED); q < 0 is invalid (skipped + IDX). */
int rpl_sumtree_set_q(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx,
                      const int64_t* q, int64_t n, int32_t* dev_err, void* stream);

/* Stratified proportional sampling by tree descent (a8) + IS weights (a9).
 * Q = root.  Stratum k of n: lo_k = floor(k Q / n), hi_k = lo_{k+1};
 * prefix_k = lo_k + floor(u_k (hi_k - lo_k) / 2^64) with u_k = draws[k], or, when
 * draws == NULL, u_k = Philox4x32-10(ctr = offset + k, key = seed) words 0|1<<32.
 * out_idx[k] = the unique leaf i with C_i <= prefix_k < C_{i+1} (C = exclusive prefix
 * sums), out_q[k] = q_i, *out_qmin = min_k out_q[k].  If out_w != NULL:
 * out_w[k] = (N P_k)^-beta / max_j (N P_j)^-beta = (qmin / q_k)^beta  (§8c #10),
 * computed in fp64.  Q == 0 -> out_idx = -1, out_q = 0, RPL_DERR_EMPTY.  `tree` is
 * written only in its sampler-ticket header word.  n >= 1.  out_qmin and out_w may be NULL;
 * with both NULL the call needs no grid-wide reduction (one dependent round trip less) and
 * the IS weights can be produced by rpl_gather from out_q (qmin = NULL there). */
int rpl_sumtree_sample(const rpl_tree_layout* L, int64_t* tree, int64_t n, const uint64_t* draws,
                       uint64_t seed, uint64_t offset, double beta, int64_t* out_idx,
                       int64_t* out_q, int64_t* out_qmin, float* out_w, int32_t* dev_err,
                       void* stream);

/* As rpl_sumtree_sample with draws = NULL, but the Philox counter is ctr = S + k where S is
 * the tree's stream position (header word 2); the call advances S by n on the device, so a
 * captured CUDA graph draws fresh strata on every replay.  Deterministic for a fixed history. */
int rpl_sumtree_sample_stream(const rpl_tree_layout* L, int64_t* tree, int64_t n, uint64_t seed,
                              double beta, int64_t* out_idx, int64_t* out_q, int64_t* out_qmin,
                              float* out_w, int32_t* dev_err, void* stream);

/* One learner step's tree work as ONE launch: the priority update of the previous batch,
 * then stream sampling of the next — exactly rpl_sumtree_update_seq (T_p >= 1: td is the
 * time-major [T_p, n_upd] per-step |delta|, eta the max/mean mix) or rpl_sumtree_update_ex
 * (T_p == 0: td is [n_upd] |delta|; eta ignored), followed by rpl_sumtree_sample_stream
 * with out_qmin = out_w = NULL (results bit-identical to that pair).  n_upd == 0 samples
 * only.  flags: RPL_UPD_LIVE_ONLY.  The update runs on one CTA; all CTAs (at most one per
 * SM, so all co-resident) then meet at a grid barrier kept in header words 3-4.  A tree
 * must not be used by two of these calls concurrently (as for every tree write). */
int rpl_sumtree_update_sample(const rpl_tree_layout* L, int64_t* tree, const int64_t* idx, const float* td,
                              int64_t T_p, int64_t n_upd, double eta, double alpha, double eps_p, int32_t flags,
                              int64_t n, uint64_t seed, int64_t* out_idx, int64_t* out_q, int32_t* dev_err,
                              void* stream);

/* Sampling WITHOUT replacement (§8f NEXT-4, reading R32): n successive proportional draws,
 * each over the leaves not drawn yet — draw k: prefix_k = floor(u_k * Q_k / 2^64) with Q_k the
 * total after removing the k earlier leaves, u_k = Philox4x32-10(seed, offset + k [+ the tree's
 * stream position when use_stream, advanced by n]) (R23); the leaf whose half-open interval
 * holds prefix_k.  The tree is restored exactly before the call returns (integer sums).
 * Fewer than n non-zero leaves: the remaining entries are -1 (+RPL_DERR_EMPTY).  One warp,
 * n x depth dependent L2 round trips: for small batches. */
int rpl_sumtree_sample_unique(const rpl_tree_layout* L, int64_t* tree, int64_t n, uint64_t seed,
                              uint64_t offset, int32_t use_stream, int64_t* out_idx, int64_t* out_q,
                              int32_t* dev_err, void* stream);

/* Sharded sampling: rank `rank` of n_shards holds one tree; shard_totals
 * (device int64 [n_shards], e.g. all-gathered rpl_sumtree_total outputs) define the global
 * total Q and the shard-major global leaf order (global idx = rank * shard_leaves + local).
 * Every rank evaluates the same n global strata; it descends only the strata whose prefix
 * falls in its own range and writes out_idx[k] = global leaf index (or -1 when not owned),
 * out_q[k] (0 when not owned), *out_qmin = min over owned (INT64_MAX if none).  Equal to
 * rpl_sumtree_sample on the concatenation of the shards (§8c #17).  use_stream != 0 (draws
 * must be NULL) takes the Philox counter from this tree's stream position as
 * rpl_sumtree_sample_stream does; every rank's position advances by n identically.
 * out_count (device int64[2], may be NULL): when given, the output is COMPACTED — the
 * owned draws (a contiguous run of strata k0..k0+m-1, because prefixes are non-decreasing
 * in k) are written to positions 0..m-1 in stratum order as LOCAL leaf indices (this
 * shard's own tree / ring: what its update and gather take; global = rank * shard_leaves +
 * local), positions m..n-1 get idx -1 / q 0, out_count[0] = m and out_count[1] = k0.  Pass &out_count[0] as
 * rpl_gather_desc.n_active (the gather schedules only the m owned samples) and, for a
 * central learner, &out_count[1] as rpl_gather_desc.col_offset (each owner writes its
 * samples at their global batch positions).  out_qmin may be NULL (no batch reduction). */
int rpl_sumtree_sample_sharded(const rpl_tree_layout* L, int64_t* tree, int32_t rank,
                               int32_t n_shards, int64_t shard_leaves, const int64_t* shard_totals,
                               int64_t n, const uint64_t* draws, uint64_t seed, uint64_t offset,
                               int32_t use_stream, int64_t* out_idx, int64_t* out_q,
                               int64_t* out_qmin, int64_t* out_count, int32_t* dev_err,
                               void* stream);

/* Peer exchange boards (SURVEY.md §8e K5 / K7 without NCCL on the data path): every rank
 * owns one board of RPL_BOARD_WORDS(n_shards) device int64 words, zeroed before first use
 * (and again whenever the trees are re-initialised), and maps every peer's board (CUDA IPC
 * over NVLink; the rank's own board in its own slot).  `boards` is a DEVICE array of
 * n_shards pointers, boards[g] = rank g's board as seen from this process.  Board layout:
 * words [2 s, 2 s + 1] = {total, tag} published by rank s (K5), words [2 G + 2 s, +1] =
 * {batch-min q, tag} published by rank s (K7), words [4 G + 2 s, +1] = {buffer min, tag}
 * published with the K5 total (root of the shard's attached min-tree, INT64_MAX without one;
 * a sampler whose tree has a min-tree reads all G and writes the global buffer min to its
 * header word 6 — the buffer-wide normaliser with no second exchange, R29).  A value is written with a plain store and
 * its tag with st.release.sys; a reader spins on ld.acquire.sys until the tag equals the
 * step's tag = the tree's stream position after the step (identical on every rank, never
 * 0, strictly increasing).  One slot per source suffices: a rank cannot publish step j+1's
 * total before every peer has consumed step j's values (step j's gather on each rank waits
 * for every rank's K7 value, which each rank publishes after its K5 read).  A wait longer
 * than ~2 s is a failed exchange: the kernel sets RPL_DERR_PEER and traps, so the failure
 * surfaces at the next synchronisation instead of a step computed from a missing value. */
#define RPL_BOARD_WORDS(n_shards) (6 * (int64_t)(n_shards))

/* Host plumbing for the boards: lets kernels running on the calling thread's current device
 * load from / store to memory of device `peer_device` (a peer rank's board mapped through
 * CUDA IPC lives in that device's memory), i.e. cudaDeviceEnablePeerAccess from the current
 * device.  RPL_OK if access is now enabled, was already enabled, or peer_device is the
 * current device; RPL_EUNSUPPORTED if the two devices cannot access each other (no
 * NVLink / PCIe P2P path); RPL_EINVAL for a bad device index.  Synchronous, host only. */
int rpl_peer_access(int32_t peer_device);

/* rpl_sumtree_sample_sharded (stream mode, compacted) with the K5 exchange fused in: the
 * kernel publishes this tree's total to every peer's board and reads all n_shards totals
 * from its own, replacing rpl_sumtree_total + an all-gather + the sampler.  out_count
 * (device int64[2]) is required: [m, k0] as in rpl_sumtree_sample_sharded.  Give the same
 * boards to rpl_gather (rpl_gather_desc.peer_boards) for the fused K7. */
int rpl_sumtree_sample_sharded_p2p(const rpl_tree_layout* L, int64_t* tree, int32_t rank, int32_t n_shards,
                                   int64_t shard_leaves, int64_t* const* boards, int64_t n, uint64_t seed,
                                   int64_t* out_idx, int64_t* out_q, int64_t* out_count, int32_t* dev_err,
                                   void* stream);

/* Descent for explicit prefixes: out_idx[k] = leaf with C_i <= prefix[k] < C_{i+1}.
 * prefix >= total -> clamped to the last non-empty leaf + RPL_DERR_TREE. */
int rpl_sumtree_find(const rpl_tree_layout* L, const int64_t* tree, const int64_t* prefix,
                     int64_t n, int64_t* out_idx, int32_t* dev_err, void* stream);

/* Buffer-wide IS normaliser (§8f NEXT-4, R29): *out_min (device int64) = min over the
 * leaves with q > 0 (INT64_MAX when none).  Passing it as rpl_gather's qmin gives
 * w_i = (N P_i)^-beta / max_j over the WHOLE buffer (N P_j)^-beta = (q_min / q_i)^beta,
 * the PER-paper normalisation, instead of the batch max (R10).  Two launches, one
 * grid-wide read of the leaf level. */
int rpl_sumtree_min(const rpl_tree_layout* L, const int64_t* tree, int64_t* out_min, void* stream);

/* *out_total = the root, i.e. the exact total priority mass Q = sum of the leaves (S:601-603
 * "total()"; the K5 value a shard publishes, §8e).  out_total: device int64.  One thread. */
int rpl_sumtree_total(const rpl_tree_layout* L, const int64_t* tree, int64_t* out_total, void* stream);

/* Buffer-wide IS normaliser (§8f NEXT-4, reading R29; PER's "normalised by max w" over the
 * whole buffer): a MIN-TREE maintained beside the sum tree.  mins = caller-owned device int64
 * [L->level_off[L->depth]] (one word per internal node, the sum tree's internal layout):
 * node (l, j) = min of the positive leaves below it (INT64_MAX when none), so mins[0] is the
 * smallest positive leaf q_min and w_i = (q_min / q_i)^beta = (N P_i)^-beta / max over the
 * buffer.  rpl_mintree_attach records the address in header word 5 and builds every node
 * (mins == NULL detaches).  From then on every leaf write keeps it exact: the update kernels
 * (rpl_sumtree_update / _ex / _seq / set_q / update_sample) recompute the min path of each
 * written leaf level by level in the same launch; rpl_replay_validity and rpl_sumtree_rebuild
 * rebuild it.  rpl_sumtree_init clears the header (detaches).  Pass &mins[0] as rpl_gather's
 * qmin (or rpl_is_weights') for buffer-normalised weights. */
int rpl_mintree_attach(const rpl_tree_layout* L, int64_t* tree, int64_t* mins, void* stream);
/* Rebuild every node of the attached min-tree from the leaves (no-op if none attached). */
int rpl_mintree_rebuild(const rpl_tree_layout* L, const int64_t* tree, void* stream);
/* out[0] = the root sum (rpl_sumtree_total), out[1] = the attached min-tree's root
 * (INT64_MAX without one): the 16-byte per-rank record one all-gather exchanges (K5 with the
 * buffer-wide normaliser, no second collective). */
int rpl_sumtree_total_min(const rpl_tree_layout* L, const int64_t* tree, int64_t* out, void* stream);
/* rpl_sumtree_sample_sharded with the K5 record of rpl_sumtree_total_min: shard_pairs = device
 * int64 [n_shards][2] {total, buffer min} (all-gathered); stream mode, compacted output
 * (out_count required); *out_bufmin (device, may be NULL) and header word 6 := the global
 * buffer min (min over the shards).  out_qmin (may be NULL) = this rank's owned batch min. */
int rpl_sumtree_sample_sharded_pairs(const rpl_tree_layout* L, int64_t* tree, int32_t rank, int32_t n_shards,
                                     int64_t shard_leaves, const int64_t* shard_pairs, int64_t n, uint64_t seed,
                                     int64_t* out_idx, int64_t* out_q, int64_t* out_qmin, int64_t* out_count,
                                     int64_t* out_bufmin, int32_t* dev_err, void* stream);

/* Recompute every internal node from the leaves as their exact int64 range sums (the
 * sum-tree invariant; SURVEY §5 checkpoint / resume: a checkpoint stores leaves + header
 * words, and this restores the rest), and rebuild an attached min-tree (R29).  Level by level
 * from the leaves' parents to the root; padding nodes become 0. */
int rpl_sumtree_rebuild(const rpl_tree_layout* L, int64_t* tree, void* stream);

/* Uniform replay (SAC/TD3 Mujoco config, BASELINE configs[3]; "uniform
 * sampling ... with replacement"): n transition leaves drawn uniformly, with replacement,
 * from the valid window of ring rows lo_row .. lo_row+n_rows-1 (mod cap_T) x all B columns.
 *   M = n_rows * B,  m_k = floor(u_k * M / 2^64)  (u_k the k-th Philox draw, R23),
 *   out_idx[k] = ((lo_row + m_k / B) mod cap_T) * B + (m_k mod B).
 * Draw k uses counter offset + k, plus *ctr when ctr (device uint64, may be NULL) is given;
 * the call then advances *ctr by n on the device, so a captured graph draws fresh indices.
 * RPL_EINVAL: n < 1, n_rows < 1 or > cap_T, lo_row outside [0, cap_T), B < 1, M >= 2^62. */
int rpl_sample_uniform(int64_t n, uint64_t seed, uint64_t offset, uint64_t* ctr, int64_t lo_row,
                       int64_t n_rows, int64_t cap_T, int64_t B, int64_t* out_idx, void* stream);

/* w[k] = (qmin / q[k])^beta in fp64, rounded to f32 (§8c #10); q[k] <= 0 -> w = 0. */
int rpl_is_weights(const int64_t* q, const int64_t* qmin, int64_t n, double beta, float* w,
                   void* stream);

/* =========================================================================
 * (3) Gather of sampled transitions / sequences from a frame-deduplicated ring
 *     ("n-step returns; sequence replay; periodic storage of recurrent state;
 *     frame-based buffer ... storing only unique Atari frames").
 *
 * Ring: cap_T rows x B columns, time-major; obs [cap_T, B, obs_bytes] (one unique frame
 * or vector per row), act [cap_T, B, act_bytes], rew f32 [cap_T, B], done u8 [cap_T, B],
 * rnn [cap_T/period, B, rnn_parts, rnn_bytes].  `cursor` = ring row of the next append,
 * `size` = number of valid rows.  Row arithmetic wraps modulo cap_T.
 *
 * Frame stacks (k items, oldest -> newest) are rebuilt as a frame-stacking wrapper
 * would have produced them: a row tau whose previous row ended an episode
 * (done[tau-1] = 1) starts a new episode, and stack slots before the episode start
 * repeat its first frame (pad_mode RPL_PAD_REPEAT) or are zero
 * (RPL_PAD_ZERO) (§8c #13).
 *
 * TRANSITION (leaf = row*B + b): o_obs [n, k, obs_bytes] = stack at row, o_next_obs = stack
 * at row+n_step, o_act [n, act_bytes] = act[row], o_ret f32 [n] = R^n over rows
 * row..row+n_step-1, o_done_n u8 [n] (§8c #14).
 * SEQUENCE (leaf = block*B + b, row0 = block*period, §8c #15-16): L = seq_len rows from
 * row0, all outputs time-major [L, n, ...]: o_obs [L, n, k, obs_bytes] (RPL_OUT_STACKED)
 * or the raw rows row0-k+1 .. row0+L-1 as [L+k-1, n, obs_bytes] (RPL_OUT_UNIQUE);
 * o_act, o_rew, o_done at rows row0..row0+L-1; o_prev_act, o_prev_rew at rows
 * row0-1..row0+L-2, zero on an episode's first row (§8c #18); o_rnn [rnn_parts, n,
 * rnn_bytes] = rnn[block, b] (P:232 [Num_Layers, Batch, Hidden] per part, §8c #19).
 * Any output pointer may be NULL (not produced).  If o_w and q are non-NULL,
 * o_w[k] = (qmin/q[k])^beta (a9, §8c #10) with qmin = *qmin when qmin != NULL (e.g. the
 * all-reduced global batch min of sharded sampling), else the min of q[j] over this call's
 * entries with idx[j] >= 0 (the sampled batch).  idx[k] < 0 -> sample skipped (outputs untouched).
 * A window not fully inside the valid rows sets RPL_DERR_INVALID_LEAF (output still the
 * defined function of the ring contents).  obs_bytes % 16 == 0 with 16-byte aligned
 * pointers uses TMA bulk copies; other sizes use vectorised LSU copies.
 * ========================================================================= */
enum { RPL_GATHER_TRANSITION = 0, RPL_GATHER_SEQUENCE = 1 };
/* Done-flag values (u8): 0 = the episode continues; any non-zero value = the episode ended
 * after this row (frame stacks restart, prev fields zero); RPL_DONE_TIMEOUT = it ended by a
 * time limit, which the _tl / v_term paths bootstrap from the supplied terminal value (R34). */
enum { RPL_DONE_TERMINAL = 1, RPL_DONE_TIMEOUT = 2 };
enum { RPL_PAD_REPEAT = 0, RPL_PAD_ZERO = 1 };
enum { RPL_OUT_STACKED = 0, RPL_OUT_UNIQUE = 1 };

typedef struct {
  int32_t kind, pad_mode, out_mode, k;
  int64_t cap_T, B, cursor, size;
  int64_t obs_bytes, act_bytes, rnn_bytes;
  int32_t n_step, seq_len, period, rnn_parts;
  double gamma;
  const void* obs;
  const void* act;
  const float* rew;
  const uint8_t* done;
  const void* rnn;
  void* o_obs;
  void* o_next_obs;
  void* o_act;
  void* o_prev_act;
  float* o_rew;
  float* o_prev_rew;
  uint8_t* o_done;
  float* o_ret;
  uint8_t* o_done_n;
  float* o_w;
  void* o_rnn;
  /* Optional device int64 (may be NULL): only entries k < *n_active are gathered, the rest
   * are skipped as if idx[k] < 0.  With the compacted sharded sampler this lets the
   * persistent gather spread exactly the owned samples over all SMs. */
  const int64_t* n_active;
  /* Optional device int64 (may be NULL = 0): every output of entry k is written at batch
   * column *col_offset + k of the output arrays, whose column count (stride) is n.  With
   * output pointers into a central learner's buffers (CUDA IPC / peer memory over NVLink)
   * each owner's gather writes its samples straight into the learner's batch (Mode C).
   * Honoured by the default sequence pipeline, the chunked sequence kernel and the
   * transition kernel (other diagnostic variants fall back to the default when set). */
  const int64_t* col_offset;
  /* Optional int8 [L, n] output (SEQUENCE, default kernel only — RPL_EUNSUPPORTED when it
   * cannot run): the episode-start offset of each output row, i.e. how many leading stack
   * slots are padding (§8c #13).  With RPL_OUT_UNIQUE it is all a consumer needs to
   * rebuild the k-stacks (rpl_stack_frames) — Mode C ships unique rows + offsets. */
  int8_t* o_start;
  /* Optional (SEQUENCE, default kernel only; q and o_w required, qmin NULL — else
   * RPL_EINVAL): the K7 exchange fused into
   * the gather.  peer_boards = the device pointer array given to
   * rpl_sumtree_sample_sharded_p2p, peer_world = n_shards, peer_rank = this rank.  CTA 0
   * publishes this rank's batch-min q (over its owned entries; INT64_MAX if none) to every
   * board; the IS weights use the min over all ranks' values, read while the frame copy
   * runs.  The step's tag is read from this rank's own board (written by its sampler). */
  int64_t* const* peer_boards;
  int32_t peer_world;
  int32_t peer_rank;
  /* Optional fused n-step targets (SEQUENCE, default kernel only — RPL_EUNSUPPORTED when it
   * cannot run; a2 + a4 over the gathered rows, readings R5 / R24 / R34).  With o_tgt
   * non-NULL, for t in [0, tgt_T) and output row tau = tgt_lo + t of each sample:
   *   R   = Horner over the sample's rows tau .. tau+n_step-1 (fp64): acc = r + gamma acc,
   *         acc = r at a done row (and r + gamma v_term at a time-limit row, R34), starting
   *         from acc = q = q_tgt[tau + n_step, column] (h^-1(q) when rescale) or 0 without q_tgt;
   *   o_tgt[t, column]      = RN32(rescale ? h(R, rescale_eps) : R)
   *   o_tgt_done[t, column] = OR of the done flags of those rows (may be NULL)
   * — bit-identical to rpl_returns_nstep over the gathered rew / done rows tgt_lo ..
   * tgt_lo+tgt_T+n_step-2 with q = q_tgt rows tgt_lo+n_step .. and q_boot = the last one.
   * q_tgt f32 [seq_len, n] (time-major by output row, device, may be NULL), o_tgt f32
   * [tgt_T, n], o_tgt_done u8 [tgt_T, n]; column = *col_offset + k.  Requires n_step >= 1,
   * tgt_lo >= 0, tgt_T >= 1, tgt_lo + tgt_T + n_step <= seq_len (RPL_EINVAL otherwise). */
  const float* q_tgt;
  float* o_tgt;
  uint8_t* o_tgt_done;
  int32_t tgt_lo, tgt_T;
  int32_t rescale, _pad1;
  double rescale_eps;
  /* Optional time-limit bootstrap (R34; P:95 fn "bootstrapping the value function when the
   * trajectory ends due to time limit"): ring array f32 [cap_T, B] (device, may be NULL).
   * A ring row whose done flag is RPL_DONE_TIMEOUT (2) ended its episode by a time limit;
   * v_term[row] is the value of its final observation.  With v_term non-NULL every fused
   * n-step return (TRANSITION o_ret, SEQUENCE o_tgt) that stops at such a row adds
   * gamma^(j+1) v_term[row] (j = the row's offset in the n rows): the recursion is cut at the
   * episode boundary and bootstrapped from the supplied value; done_n stays 1 (the learner
   * must not bootstrap again).  With v_term NULL any non-zero done flag is a terminal. */
  const float* v_term;
  /* Optional completion signal (SEQUENCE, default kernel only; both or neither, else
   * RPL_EINVAL): done_seq = device int64 [2] in this rank's memory, zero-initialised (a call
   * counter and a CTA ticket); done_flag = a device int64 (typically another GPU's memory
   * mapped over NVLink).  When the call's last CTA has finished, every output store of the
   * call is made visible at system scope and done_flag := ++done_seq[0] (st.release.sys).
   * Mode C: each owner signals the learner this way; the learner waits with rpl_wait_flags. */
  int64_t* done_flag;
  int64_t* done_seq;
  /* Optional dynamic work distribution (SEQUENCE, stacked output; one learner's whole batch: no col_offset,
   * n_active, peer_boards or done_flag; also with rpl_gather_sample): device int64 [4],
   * zero-initialised, owned by the caller.  With it the persistent gather splits a share of
   * the rows statically and hands out the rest at run time in units of a few rows of one
   * sample through an atomic counter in work[0], so CTAs on SMs that see less memory
   * throughput take fewer rows (same outputs, bit for bit).  The call's last CTA re-zeroes
   * work[0..3]; calls sharing a buffer must be stream-ordered.  NULL: the static split. */
  int64_t* work;
} rpl_gather_desc;

int rpl_gather(const rpl_gather_desc* desc /* host */, const int64_t* idx, const int64_t* q,
               const int64_t* qmin, double beta, int64_t n, int32_t* dev_err, void* stream);

/* Sampling fused into the sequence gather (a8 + a11 in one launch; R2D2's learner step
 * becomes update -> gather): the call draws n stratified samples from `tree` exactly as
 * rpl_sumtree_sample_stream(L, tree, n, seed, ...) would (the tree's Philox stream position,
 * advanced by n on the device) and gathers them as rpl_gather(desc, idx_out, q_out, NULL,
 * beta, n, ...) would — every CTA descends the tree for the samples its rows need, the CTA
 * owning a sample's first row writes idx_out[k] / q_out[k] (device int64 [n]), and the last
 * CTA to finish writes the IS weights (batch min) into desc->o_w.  Bit-identical outputs to
 * the two calls.  SEQUENCE only; no n_active / col_offset / peer_boards / done_flag (those
 * are the sharded paths: RPL_EINVAL); L must describe cap_T/period x B leaves.  Runs on the
 * default persistent kernel (RPL_EUNSUPPORTED when it cannot: frames not TMA-addressable). */
int rpl_gather_sample(const rpl_gather_desc* desc, const rpl_tree_layout* L, int64_t* tree, uint64_t seed,
                      int64_t* idx_out, int64_t* q_out, double beta, int64_t n, int32_t* dev_err, void* stream);

/* The whole R2D2 replay step in ONE launch (a5-a7 + a8 + a9 + a11, R26; P:123 fn): exactly
 * rpl_sumtree_update_seq(L, tree, upd_idx, upd_td, T_p, n_upd, eta, alpha, eps_p, flags, ...)
 * followed by rpl_gather_sample(desc, L, tree, seed, idx_out, q_out, beta, n, ...) — same tree
 * (leaves, nodes, header, attached min-tree), same draws, same outputs bit for bit.  Every CTA
 * of the dynamic-tail gather computes the batch's sequence priorities, winners (last
 * position of each leaf) and deltas, applies them to its staged copy of the internal
 * levels and overlays the winners' new q on the leaf level it reads, so it samples the
 * updated tree at once; CTA 0 writes the update to the tree after every CTA has finished
 * reading it.  Requires desc->work, stacked output, 1 <= n_upd <= 128 and every internal tree
 * level within the frame-slot area; otherwise (or for n_upd == 0) the call enqueues the two
 * launches.  upd_idx: device int64 [n_upd] (< 0: padding, skipped; >= n_leaves:
 * RPL_DERR_IDX); upd_td: device f32 [T_p, n_upd] per-step |delta|; flags: RPL_UPD_LIVE_ONLY.
 * Argument errors as the two calls (RPL_EINVAL). */
int rpl_gather_update_sample(const rpl_gather_desc* desc, const rpl_tree_layout* L, int64_t* tree,
                             const int64_t* upd_idx, const float* upd_td, int64_t T_p, int64_t n_upd, double eta,
                             double alpha, double eps_p, int32_t flags, uint64_t seed, int64_t* idx_out,
                             int64_t* q_out, double beta, int64_t n, int32_t* dev_err, void* stream);

/* Stream-ordered wait for n completion flags (device int64 [n], e.g. the learner's flag array
 * that n owners' gathers signal through rpl_gather_desc.done_flag): returns at once, the
 * enqueued one-warp kernel spins with ld.acquire.sys until flags[i] >= *expect for every i
 * (expect: device int64, e.g. the learner's own done_seq[0]), then fences at system scope, so
 * work enqueued after it on the stream reads every owner's stores.  A flag still short after
 * ~2 s sets RPL_DERR_PEER in *dev_err and traps the kernel (the context then reports the
 * failure at the next synchronisation): an exchange never continues with a partial batch.
 * n in [1, 1024]. */
int rpl_wait_flags(const int64_t* flags, int32_t n, const int64_t* expect, int32_t* dev_err, void* stream);

/* k-stacks from unique rows (Mode C learner side, §8e): uniq [L+k-1, n, obs_bytes] as written
 * by rpl_gather with RPL_OUT_UNIQUE, start int8 [L, n] its o_start; out [L, n, k, obs_bytes]
 * gets out[tau, s, j] = uniq[tau + max(j, start[tau, s]), s] (zero when j < start and
 * pad_mode == RPL_PAD_ZERO) — bit-identical to rpl_gather's RPL_OUT_STACKED output.
 * n_active (device, may be NULL) limits the samples.  obs_bytes % 16 == 0, 16-B aligned
 * pointers, k <= 8, n <= 65535. */
int rpl_stack_frames(const void* uniq, const int8_t* start, int64_t L, int64_t n, int32_t k, int64_t obs_bytes,
                     int32_t pad_mode, void* out, const int64_t* n_active, void* stream);

/* =========================================================================
 * (4) Ring append and validity maintenance (§8a a12, §8f NEXT-2; P:75-84 the sampler
 *     writes batches while the optimiser samples).
 * ========================================================================= */

/* Copy a sampler batch of T_b rows into the ring described by `ring` (its obs / act / rew /
 * done / rnn pointers, geometry and `cursor`): batch arrays obs [T_b, B, obs_bytes],
 * act [T_b, B, act_bytes], rew f32 [T_b, B], done u8 [T_b, B] go to ring rows cursor ..
 * cursor+T_b-1 (mod cap_T) — at most two cudaMemcpyAsync each, so the source may be host
 * (pinned) or device memory.  rnn [n_blk, B, rnn_parts, rnn_bytes] holds the stored state
 * of the batch rows t with (cursor + t) % period == 0, in order (periodic storage).
 * Any source may be NULL (not written).  The caller advances cursor / size afterwards and
 * calls rpl_replay_validity.  RPL_EINVAL: T_b > cap_T, bad geometry. */
int rpl_ring_append(const rpl_gather_desc* ring, const void* obs, const void* act, const float* rew,
                    const uint8_t* done, const void* rnn, int64_t T_b, void* stream);

/* Any further per-row ring array (e.g. the actor's q_taken / q_boot for initial priorities,
 * R33): rows [0, T_b) of a [T_b, row_bytes] source -> ring rows cursor .. cursor+T_b-1
 * (mod cap_T) of ring_array [cap_T, row_bytes]; at most two cudaMemcpyAsync (host or device
 * source).  RPL_EINVAL on null pointers, cursor outside [0, cap_T), T_b > cap_T. */
int rpl_ring_append_rows(void* ring_array, int64_t row_bytes, int64_t cap_T, int64_t cursor, const void* src,
                         int64_t T_b, void* stream);

/* Tree validity maintenance after the ring moved from (cursor_old, size_old) to
 * (cursor_new, size_new): every leaf (kind TRANSITION: row*B+b with k, n_step; SEQUENCE:
 * block*B+b with k, seq_len, period) whose validity (§8c #2, #16) changed gets q = the
 * tree's max-priority-seen (became valid) or q = 0 (became invalid: never sampled),
 * with exact int64 propagation.  Leaves whose validity did not change keep their q.
 * L->n_leaves must equal (cap_T or cap_T/period) * B. */
int rpl_replay_validity(const rpl_tree_layout* L, int64_t* tree, int32_t kind, int64_t cap_T, int64_t B,
                        int32_t k, int32_t n_step, int32_t seq_len, int32_t period, int64_t cursor_old,
                        int64_t size_old, int64_t cursor_new, int64_t size_new, void* stream);

/* =========================================================================
 * (5) Learning targets right after the gather (§8f NEXT-3; P:34 Double-DQN / Categorical,
 *     P:38 n-step).
 * ========================================================================= */

/* Initial priorities of new samples (§8f NEXT-1; P:123 fn "5-step TD initial priorities";
 * S:660; reading R33): per-step |TD error| read straight from ring arrays.  For t in
 * [0, T_out), b in [0, B), ring row t' = (row0 + t) mod cap_T:
 *   y = the n-step target of row t' (rpl_returns_nstep's R24 rule: rewards rows t' .. t'+n-1
 *       cut after the first done, bootstrap q_boot[t'+n] unless done^n; rescaled per R4/R5
 *       when rescale != 0), all rows modulo cap_T, fp64;
 *   out[t, b] = RN32(|y - q_taken[t', b]|).
 * rew [cap_T, B] f32, done [cap_T, B] u8, q_taken / q_boot [cap_T, B] f32 (the actor's
 * Q(s_t, a_t) and bootstrap value of s_t, appended per row with rpl_ring_append_rows).
 * out [T_out, B] f32 is time-major with one column per env: for a sequence block it is the
 * td_steps rpl_sumtree_update_seq takes for that block's B leaves (row0 = block start +
 * burn-in, T_out = train rows); for transitions, rows row0.. are leaves row0*B .. in order.
 * RPL_ERANGE: n < 1 or T_out + n > cap_T. */
int rpl_ring_td_abs(const float* rew, const uint8_t* done, const float* q_taken, const float* q_boot,
                    int64_t cap_T, int64_t B, int64_t row0, int64_t T_out, int32_t n, double gamma,
                    int32_t rescale, double rescale_eps, float* out, void* stream);

/* n-step targets with the double-Q bootstrap: q_online, q_target [T+1, B, A] f32 (the two
 * networks' action values for rows 0..T); for output row t (0..T-n) the bootstrap is
 * q_target[t+n, b, a*] with a* = argmax_a q_online[t+n, b, a] (first maximum, NaN never
 * wins, R27) — then exactly rpl_returns_nstep's target (R24), rescaled (R4, R5) when
 * rescale != 0.  ret_n [T-n+1, B] f32, done_n (may be NULL) u8, a_star (may be NULL) int32. */
int rpl_returns_nstep_dq(const float* r, const uint8_t* d, int64_t T, int64_t B, int32_t n, double gamma,
                         const float* q_online, const float* q_target, int32_t A, int32_t rescale,
                         double rescale_eps, float* ret_n, uint8_t* done_n, int32_t* a_star, void* stream);

/* Categorical (C51) projection [EXT: Bellemare et al. 2017, Alg. 1]: for each sample s,
 * a* = argmax q_online[s, :] (R27; q_online may be NULL when A == 1), p = p_target[s, a*, :]
 * over n_atoms atoms z_j = v_min + j (v_max - v_min)/(n_atoms - 1), g = gamma_n unless
 * done_n[s] (then 0; done_n may be NULL), Tz_j = clip(R[s] + g z_j, v_min, v_max),
 * b_j = (Tz_j - v_min)/dz, and m_out[s, i] = sum_j p_j max(0, 1 - |b_j - i|) (fp64, R28:
 * the algorithm's floor/ceil split written as a gather).  p_target [n, A, n_atoms] f32,
 * m_out [n, n_atoms] f32, a_star [n] int32 (may be NULL). */
int rpl_c51_project(const float* p_target, const float* q_online, const float* R, const uint8_t* done_n,
                    int64_t n, int32_t A, int32_t n_atoms, double v_min, double v_max, double gamma_n,
                    float* m_out, int32_t* a_star, void* stream);

/* -------------------------------------------------------------------------
 * Diagnostics (tests only): v[k] = RN32(RN64(|td_abs[k]| + eps_p)^alpha) exactly as
 * rpl_sumtree_update computes it (§8c #7); force_slow != 0 runs the double-double
 * fallback for every element; out_slow[k] (may be NULL) = 1 when the fallback ran.
 * ------------------------------------------------------------------------- */
int rpl_debug_priority_values(const float* td_abs, int64_t n, double alpha, double eps_p,
                              int32_t force_slow, float* out_v, uint8_t* out_slow, void* stream);

/* Diagnostics (tests only): select the sequence-gather kernel, 0 = persistent pipeline with
 * TMA loads and LSU stores (default, 4 consumer warps), 1 = one CTA per 8-row chunk (TMA both
 * ways), 2 = frame-centric LSU copy, 3 = persistent all-TMA pipeline, 4 / 5 = variant 0 with
 * 14 / 8 consumer warps, 6 = LSU frame loads with TMA bulk stores.  All produce identical
 * outputs. */
int rpl_debug_set_gather_variant(int32_t variant);

/* Measurement / test only: kernel choice of rpl_returns_discounted and rpl_gae
 * (process-global; initial value from RPL_SCAN_VARIANT, else 0).  0 = default (whole-column
 * TMA tiles when the layout is TMA-addressable, else LDG), 4 / 5 = T <= 128: rows split over
 * a cluster of 2 / 4 CTAs (DSMEM carry exchange), 6 = TMA tiles, 3 / 1 / 2 = LDG
 * with 16x8 / 32x4 / 8x16 warps x rows.  Results agree within the fp64-accumulation bound
 * (segment boundaries differ).  RPL_EINVAL outside 0..6. */
int rpl_debug_set_scan_variant(int32_t variant);

/* Measurement / test only: 1 (default; initial value from RPL_TREE_STAGE, "0" = off) lets
 * the samplers stage the tree's top levels (whole levels, up to 4351 words from the root) in
 * shared memory before the descent; 0 descends from global memory only.  Identical outputs.
 * RPL_EINVAL for other values. */
int rpl_debug_set_tree_stage(int32_t on);

/* Diagnostics (measurement only; compiled in only with -DRPL_DIAG, see build.py
 * RPL_NVCC_EXTRA): bit mask applied to the default sequence gather.
 * 1 = skip the frame stores, 2 = skip the frame loads (outputs are then garbage),
 * 4 = normal-priority frame stores, 8 = normal L2 policy on the frame loads (the default is
 * evict-first for both: frames are streamed once),
 * 16 = skip the per-row fields and stored state.
 * 0 (default) restores normal operation.  Returns RPL_EINVAL for other values, and
 * RPL_EUNSUPPORTED for a non-zero mask in the default build (RPL_GATHER_DIAG is ignored there). */
int rpl_debug_set_gather_diag(int32_t mask);

/* Measurement builds only (-DRPL_TRACE): copies the update kernel's last globaltimer
 * timeline (n <= 16 int64 ns stamps, host out) — kernel start, staged / mixed sequence
 * priorities, hash reset, dedupe, leaf writes, end.  RPL_EUNSUPPORTED in the default build. */
int rpl_debug_trace(int64_t* out, int32_t n);
/* Measurement builds only (-DRPL_TRACE): the R2D2 step timeline.  rpl_debug_trace slots 7
 * (update kernel entry), 8 (sampler past its dependency wait), 9 (last sampler CTA end);
 * rpl_debug_gather_trace (n <= 9): 0 sequence-gather CTA 0 entry, 1 CTA 0 past its
 * dependency wait, 2 CTA 0's first frames landed, 3 last CTA end, 4-7 CTA 0's fused-sampling stages, 8 first CTA end.  The _reset calls clear
 * both (rpl_debug_trace_reset) or the gather's only.  RPL_EUNSUPPORTED in the default build. */
int rpl_debug_trace_reset(void);
/* Measurement knob (process-global, read at each update launch): where rpl_sumtree_update(_ex /
 * _seq / set_q)'s kernel lets the dependent grid launch — -1 at exit, 0 (default) at entry, 3
 * after its loads are issued, 2 after the priorities, 4 after the power transform (2-4: the
 * multi-CTA and one-chunk kernels; the chunked kernel then triggers at exit).  RPL_EINVAL
 * otherwise. */
int rpl_debug_set_upd_trigger(int32_t at);
/* Measurement builds only (-DRPL_TRACE): the last pipelined-scan launch's timeline (n <= 10
 * globaltimer ns stamps, host out): CTA 0's entry, past its wait, first tiles landed, its three
 * barriers, store issue and exit; the last and the first CTA's exits. */
int rpl_debug_scan_trace(int64_t* out, int32_t n);
/* Measurement knob (process-global): 1 (default) = rpl_sumtree_update_seq batches of n <= 1024
 * run on ceil(n / 8) CTAs, rpl_sumtree_update / _ex / set_q batches of n <= 64 on one 64-thread
 * CTA, each CTA resolving duplicates over the whole batch; 0 = the single-CTA kernels.
 * Identical results.  RPL_EINVAL for other values. */
int rpl_debug_set_upd_multi(int32_t on);
/* Measurement knob (process-global, read at each sequence-gather launch): where the default
 * sequence gather lets the dependent grid launch — -1 at exit (default), 0 at entry, 1 once
 * every CTA's producer has issued its last frame load.  RPL_EINVAL for other values. */
int rpl_debug_set_gather_trigger(int32_t at);
/* Measurement knobs of the dynamic-tail sequence gather (rpl_gather_desc.work): pct = the
 * static share of the rows in percent of an even split (0: every row dynamic; -1: the static
 * kernel; default 80), rows = the longest grab (1..32, default 16; a grab takes about
 * 1/grid of the dynamic rows left, at least 2), lookahead = rows published but not yet stored
 * below which a CTA grabs again (bits 0-7, 1..200, default 16; optionally bits 8-15 = that
 * queue once fewer than bits 16-30 rows are left in the pool, 0 = unchanged).  pct = 1000 + c
 * (rows, lookahead ignored) sets how many of its first piece's frame loads a CTA issues right
 * after its fused-sampling descent (default 10: -0.4 us per R2D2 step; 0 = none, 16 and 28 slower);
 * pct = 2001 / 2000 makes every dynamic-tail launch take / not take the fused-update kernel
 * instantiation (A/B of the default gather's own instantiation).
 * RPL_EINVAL out of range. */
int rpl_debug_set_gather_dyn(int32_t pct, int32_t rows, int32_t lookahead);
int rpl_debug_gather_trace(int64_t* out, int32_t n);
/* Measurement builds only: for the first n (<= 512) CTAs of the last sequence-gather launch
 * (host out, 3n int64): out[0, n) each CTA's globaltimer end; dynamic-tail kernel only:
 * out[n, 2n) when its static rows were stored, out[2n, 3n) the dynamic units it took. */
int rpl_debug_gather_cta_ends(int64_t* out, int32_t n);
/* Measurement builds only: the dynamic tail's first 8 grabs of each of the first n CTAs (host
 * out, 16n int64: per grab its globaltimer time and (rows << 32) | rows queued at the grab). */
int rpl_debug_gather_grabs(int64_t* out, int32_t n);
int rpl_debug_gather_trace_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* RPL_H_ */
