"""Torch-tensor binding over the librpl C ABI (include/rpl.h).

Argument marshalling only: shape/dtype/device checks, output allocation and the
current CUDA stream.  Every step of the hot path runs inside librpl's kernels.
Function names follow the ABI (rpl_<name> -> <name>).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import GatherDesc, TreeLayout, check, lib

__all__ = [
    "returns_discounted", "returns_nstep", "gae", "value_rescale", "SumTree", "is_weights", "gather",
    "GatherRing", "GatherPlan", "check_err", "launch_count", "debug_priority_values", "sample_uniform",
    "ring_append", "returns_nstep_dq", "c51_project", "stack_frames", "ring_append_rows", "ring_td_abs",
]


def _stream(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _req(t, dtype, name, shape=None):
    if t is None:
        raise ValueError(f"{name} is required")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def launch_count() -> int:
    return int(lib.rpl_launch_count())


def check_err(dev_err: torch.Tensor, allowed: int = 0):
    """Raise if any RPL_DERR_* bit outside `allowed` is set (the only host sync)."""
    v = int(dev_err.item())
    bad = v & ~allowed
    if bad:
        names = [n for b, n in _lib.DERR.items() if bad & b]
        raise _lib.RplError("device error bits: " + ", ".join(names))
    return v


# ---------------------------------------------------------------- returns
def returns_discounted(r, d, bootstrap, gamma, out=None, v_term=None):
    """rpl_returns_discounted (rpl_returns_discounted_tl with v_term [T, B]: time-limit rows,
    d == 2, bootstrap from their terminal value, R34)."""
    T, B = r.shape
    _req(r, torch.float32, "r")
    _req(d, torch.uint8, "d", (T, B))
    if bootstrap is not None:
        _req(bootstrap, torch.float32, "bootstrap", (B,))
    if v_term is not None:
        _req(v_term, torch.float32, "v_term", (T, B))
    out = torch.empty_like(r) if out is None else _req(out, torch.float32, "out", (T, B))
    check(lib.rpl_returns_discounted_tl(_ptr(r), _ptr(d), _ptr(v_term), _ptr(bootstrap), T, B, float(gamma),
                                        _ptr(out), _stream(r.device)), "rpl_returns_discounted_tl")
    return out


def returns_nstep(r, d, n, gamma, q=None, q_boot=None, rescale=False, eps=1e-3, out=None, done_out=None,
                  v_term=None):
    """rpl_returns_nstep (rpl_returns_nstep_tl with v_term [T, B], R34)."""
    T, B = r.shape
    _req(r, torch.float32, "r")
    _req(d, torch.uint8, "d", (T, B))
    if v_term is not None:
        _req(v_term, torch.float32, "v_term", (T, B))
    if q is not None:
        _req(q, torch.float32, "q", (T, B))
        _req(q_boot, torch.float32, "q_boot", (B,))
    rows = T - int(n) + 1
    if out is None:
        out = torch.empty((max(rows, 0), B), dtype=torch.float32, device=r.device)
    if done_out is None:
        done_out = torch.empty((max(rows, 0), B), dtype=torch.uint8, device=r.device)
    check(lib.rpl_returns_nstep_tl(_ptr(r), _ptr(d), _ptr(v_term), T, B, int(n), float(gamma), _ptr(q),
                                   _ptr(q_boot), 1 if rescale else 0, float(eps), _ptr(out), _ptr(done_out),
                                   _stream(r.device)), "rpl_returns_nstep_tl")
    return out, done_out


def returns_nstep_dq(r, d, n, gamma, q_online, q_target, rescale=False, eps=1e-3, out=None, done_out=None):
    """rpl_returns_nstep_dq: q_online / q_target [T+1, B, A]. Returns (y, done_n, a_star)."""
    T, B = r.shape
    _req(r, torch.float32, "r")
    _req(d, torch.uint8, "d", (T, B))
    _req(q_online, torch.float32, "q_online")
    A = int(q_online.shape[-1])
    _req(q_target, torch.float32, "q_target", (T + 1, B, A))
    if tuple(q_online.shape) != (T + 1, B, A):
        raise ValueError("q_online must be [T+1, B, A]")
    rows = T - int(n) + 1
    out = torch.empty((rows, B), dtype=torch.float32, device=r.device) if out is None else out
    done_out = torch.empty((rows, B), dtype=torch.uint8, device=r.device) if done_out is None else done_out
    a_star = torch.empty((rows, B), dtype=torch.int32, device=r.device)
    check(lib.rpl_returns_nstep_dq(_ptr(r), _ptr(d), T, B, int(n), float(gamma), _ptr(q_online), _ptr(q_target), A,
                                   1 if rescale else 0, float(eps), _ptr(out), _ptr(done_out), _ptr(a_star),
                                   _stream(r.device)), "rpl_returns_nstep_dq")
    return out, done_out, a_star


def c51_project(p_target, q_online, R, done_n, v_min, v_max, gamma_n, out=None):
    """rpl_c51_project: p_target [n, A, N], q_online [n, A] or None (A == 1). Returns (m [n, N], a_star)."""
    _req(p_target, torch.float32, "p_target")
    n, A, N = (int(x) for x in p_target.shape)
    if q_online is not None:
        _req(q_online, torch.float32, "q_online", (n, A))
    _req(R, torch.float32, "R", (n,))
    if done_n is not None:
        _req(done_n, torch.uint8, "done_n", (n,))
    out = torch.empty((n, N), dtype=torch.float32, device=p_target.device) if out is None else out
    a_star = torch.empty(n, dtype=torch.int32, device=p_target.device)
    check(lib.rpl_c51_project(_ptr(p_target), _ptr(q_online), _ptr(R), _ptr(done_n), n, A, N, float(v_min),
                              float(v_max), float(gamma_n), _ptr(out), _ptr(a_star), _stream(p_target.device)),
          "rpl_c51_project")
    return out, a_star


def gae(r, v, d, bootstrap_v, gamma, lam, adv=None, ret=None, v_term=None):
    """rpl_gae (rpl_gae_tl with v_term [T, B], R34)."""
    T, B = r.shape
    _req(r, torch.float32, "r")
    _req(v, torch.float32, "v", (T, B))
    _req(d, torch.uint8, "d", (T, B))
    _req(bootstrap_v, torch.float32, "bootstrap_v", (B,))
    if v_term is not None:
        _req(v_term, torch.float32, "v_term", (T, B))
    adv = torch.empty_like(r) if adv is None else adv
    ret = torch.empty_like(r) if ret is None else ret
    check(lib.rpl_gae_tl(_ptr(r), _ptr(v), _ptr(d), _ptr(v_term), _ptr(bootstrap_v), T, B, float(gamma), float(lam),
                         _ptr(adv), _ptr(ret), _stream(r.device)), "rpl_gae_tl")
    return adv, ret


def value_rescale(x, eps=1e-3, inverse=False, out=None):
    _req(x, torch.float32, "x")
    out = torch.empty_like(x) if out is None else out
    check(lib.rpl_value_rescale(_ptr(x), _ptr(out), x.numel(), float(eps), 1 if inverse else 0,
                                _stream(x.device)), "rpl_value_rescale")
    return out


def debug_priority_values(td_abs, alpha, eps_p=1e-3, force_slow=False):
    _req(td_abs, torch.float32, "td_abs")
    v = torch.empty_like(td_abs)
    slow = torch.empty(td_abs.shape, dtype=torch.uint8, device=td_abs.device)
    check(lib.rpl_debug_priority_values(_ptr(td_abs), td_abs.numel(), float(alpha), float(eps_p),
                                        1 if force_slow else 0, _ptr(v), _ptr(slow), _stream(td_abs.device)),
          "rpl_debug_priority_values")
    return v, slow


def is_weights(q, qmin, beta, out=None):
    _req(q, torch.int64, "q")
    _req(qmin, torch.int64, "qmin")
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device) if out is None else out
    check(lib.rpl_is_weights(_ptr(q), _ptr(qmin), q.numel(), float(beta), _ptr(out), _stream(q.device)),
          "rpl_is_weights")
    return out


def sample_uniform(n, seed, lo_row, n_rows, cap_T, B, offset=0, ctr=None, device="cuda", out=None):
    """rpl_sample_uniform: n leaves uniform over rows lo_row..lo_row+n_rows-1 (mod cap_T) x B columns.
    `ctr` (a 1-element int64 CUDA tensor) makes the draw stream advance on the device."""
    if ctr is not None:
        _req(ctr, torch.int64, "ctr", (1,))
        device = ctr.device
    out = torch.empty(int(n), dtype=torch.int64, device=device) if out is None else out
    _req(out, torch.int64, "out", (int(n),))
    check(lib.rpl_sample_uniform(int(n), int(seed) & (2**64 - 1), int(offset) & (2**64 - 1), _ptr(ctr), int(lo_row),
                                 int(n_rows), int(cap_T), int(B), _ptr(out), _stream(out.device)),
          "rpl_sample_uniform")
    return out


# ---------------------------------------------------------------- sum tree
class SumTree:
    """One int64 device array holding the whole tree (rpl.h layout)."""

    def __init__(self, n_leaves: int, fanout: int = 32, frac_bits: int = 32, device="cuda"):
        self.layout = TreeLayout()
        check(lib.rpl_sumtree_layout(int(n_leaves), int(fanout), int(frac_bits), C.byref(self.layout)),
              "rpl_sumtree_layout")
        L = self.layout
        self.n_leaves = int(n_leaves)
        self.fanout = int(fanout)
        self.frac_bits = int(frac_bits)
        self.depth = int(L.depth)
        self.q_cap = int(L.q_cap)
        self.device = torch.device(device)
        self.storage = torch.empty(int(L.n_words), dtype=torch.int64, device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._lp = C.byref(self.layout)
        self.mins = None  # attached min-tree (rpl_mintree_attach)
        self.init()

    # views
    def level(self, l: int) -> torch.Tensor:
        off, ln = int(self.layout.level_off[l]), int(self.layout.level_len[l])
        return self.storage[off:off + ln]

    @property
    def leaves(self) -> torch.Tensor:
        off = int(self.layout.level_off[self.depth])
        return self.storage[off:off + self.n_leaves]

    @property
    def header(self) -> torch.Tensor:
        off = int(self.layout.hdr_off)
        return self.storage[off:off + 8]

    def _s(self):
        return _stream(self.device)

    def init(self):
        check(lib.rpl_sumtree_init(self._lp, _ptr(self.storage), self._s()), "rpl_sumtree_init")
        self.mins = None  # init clears the header: any min-tree is detached

    def update(self, idx, td_abs, alpha, eps_p=1e-3, err=None, live_only=False):
        _req(idx, torch.int64, "idx")
        _req(td_abs, torch.float32, "td_abs", idx.shape)
        e = self.err if err is None else err
        if live_only:
            check(lib.rpl_sumtree_update_ex(self._lp, _ptr(self.storage), _ptr(idx), _ptr(td_abs), idx.numel(),
                                            float(alpha), float(eps_p), 1, _ptr(e), self._s()), "rpl_sumtree_update_ex")
            return
        check(lib.rpl_sumtree_update(self._lp, _ptr(self.storage), _ptr(idx), _ptr(td_abs), idx.numel(),
                                     float(alpha), float(eps_p), _ptr(e), self._s()), "rpl_sumtree_update")

    def update_seq(self, idx, td_steps, alpha, eta=0.9, eps_p=1e-3, err=None, live_only=False):
        """rpl_sumtree_update_seq: R2D2 eta-mix of per-step |delta| [T_p, n] per sequence, then update."""
        _req(idx, torch.int64, "idx")
        _req(td_steps, torch.float32, "td_steps")
        if td_steps.dim() != 2 or td_steps.shape[1] != idx.numel():
            raise ValueError("td_steps must be [T_p, n] with n = idx.numel()")
        e = self.err if err is None else err
        check(lib.rpl_sumtree_update_seq(self._lp, _ptr(self.storage), _ptr(idx), _ptr(td_steps),
                                         td_steps.shape[0], idx.numel(), float(eta), float(alpha), float(eps_p),
                                         1 if live_only else 0, _ptr(e), self._s()), "rpl_sumtree_update_seq")

    def validity(self, kind, cap_T, B, k, cursor_old, size_old, cursor_new, size_new, n_step=1, seq_len=1,
                 period=1):
        """rpl_replay_validity: leaves that became valid get max-seen, those that became invalid 0."""
        kind_i = _lib.GATHER_TRANSITION if kind == "transition" else _lib.GATHER_SEQUENCE
        check(lib.rpl_replay_validity(self._lp, _ptr(self.storage), kind_i, int(cap_T), int(B), int(k), int(n_step),
                                      int(seq_len), int(period), int(cursor_old), int(size_old), int(cursor_new),
                                      int(size_new), self._s()), "rpl_replay_validity")

    def set_q(self, idx, q=None, err=None):
        _req(idx, torch.int64, "idx")
        if q is not None:
            _req(q, torch.int64, "q", idx.shape)
        e = self.err if err is None else err
        check(lib.rpl_sumtree_set_q(self._lp, _ptr(self.storage), _ptr(idx), _ptr(q), idx.numel(), _ptr(e),
                                    self._s()), "rpl_sumtree_set_q")

    def sample(self, n, draws=None, seed=0, offset=0, beta=None, out=None, err=None):
        """Returns (idx, q, qmin[1], w or None)."""
        n = int(n)
        if out is None:
            idx = torch.empty(n, dtype=torch.int64, device=self.device)
            q = torch.empty(n, dtype=torch.int64, device=self.device)
            qmin = torch.empty(1, dtype=torch.int64, device=self.device)
            w = torch.empty(n, dtype=torch.float32, device=self.device) if beta is not None else None
        else:
            idx, q, qmin, w = out
        if draws is not None:  # uint64 draws carried as their int64 bit patterns
            _req(draws, torch.int64, "draws", (n,))
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample(self._lp, _ptr(self.storage), n, _ptr(draws), int(seed) & (2 ** 64 - 1),
                                     int(offset) & (2 ** 64 - 1), float(beta or 0.0), _ptr(idx), _ptr(q),
                                     _ptr(qmin), _ptr(w), _ptr(e), self._s()), "rpl_sumtree_sample")
        return idx, q, qmin, w

    def sample_stream(self, n, seed, beta=None, out=None, err=None, want_qmin=True):
        """rpl_sumtree_sample_stream: Philox draws from the tree's device-side stream position.
        want_qmin=False with beta=None skips the batch reduction (qmin returned as None)."""
        n = int(n)
        if out is None:
            idx = torch.empty(n, dtype=torch.int64, device=self.device)
            q = torch.empty(n, dtype=torch.int64, device=self.device)
            qmin = torch.empty(1, dtype=torch.int64, device=self.device) if (want_qmin or beta is not None) else None
            w = torch.empty(n, dtype=torch.float32, device=self.device) if beta is not None else None
        else:
            idx, q, qmin, w = out
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample_stream(self._lp, _ptr(self.storage), n, int(seed) & (2 ** 64 - 1),
                                            float(beta or 0.0), _ptr(idx), _ptr(q), _ptr(qmin), _ptr(w), _ptr(e),
                                            self._s()), "rpl_sumtree_sample_stream")
        return idx, q, qmin, w

    def update_sample(self, n, seed, idx=None, td=None, alpha=0.6, eta=0.9, eps_p=1e-3, out=None, err=None,
                      live_only=False):
        """rpl_sumtree_update_sample: update (td [T_p, n_upd] -> sequence priorities, or [n_upd]
        -> |delta|) then stream-sample n draws, in one launch.  idx None: sample only.
        Returns (idx, q)."""
        n = int(n)
        if out is None:
            oi = torch.empty(n, dtype=torch.int64, device=self.device)
            oq = torch.empty(n, dtype=torch.int64, device=self.device)
        else:
            oi, oq = out
        n_upd, T_p = 0, 0
        if idx is not None:
            _req(idx, torch.int64, "idx")
            _req(td, torch.float32, "td")
            n_upd = idx.numel()
            if td.dim() == 2:
                T_p = td.shape[0]
                if td.shape[1] != n_upd:
                    raise ValueError("td must be [T_p, n_upd] or [n_upd]")
            elif td.numel() != n_upd:
                raise ValueError("td must be [T_p, n_upd] or [n_upd]")
        e = self.err if err is None else err
        check(lib.rpl_sumtree_update_sample(self._lp, _ptr(self.storage), _ptr(idx), _ptr(td), T_p, n_upd,
                                            float(eta), float(alpha), float(eps_p), 1 if live_only else 0, n,
                                            int(seed) & (2 ** 64 - 1), _ptr(oi), _ptr(oq), _ptr(e), self._s()),
              "rpl_sumtree_update_sample")
        return oi, oq

    def sample_sharded(self, rank, n_shards, shard_totals, n, draws=None, seed=0, offset=0, out=None, err=None,
                       use_stream=False, count=None):
        """rpl_sumtree_sample_sharded.  count (2-element int64 CUDA tensor) selects the compacted
        output: owned draws first; count = [their number m, their first global stratum k0]."""
        n = int(n)
        _req(shard_totals, torch.int64, "shard_totals", (n_shards,))
        if count is not None:
            _req(count, torch.int64, "count", (2,))
        if out is None:
            idx = torch.empty(n, dtype=torch.int64, device=self.device)
            q = torch.empty(n, dtype=torch.int64, device=self.device)
            qmin = torch.empty(1, dtype=torch.int64, device=self.device)
        else:
            idx, q, qmin = out
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample_sharded(self._lp, _ptr(self.storage), int(rank), int(n_shards),
                                             self.n_leaves, _ptr(shard_totals), n, _ptr(draws),
                                             int(seed) & (2 ** 64 - 1), int(offset) & (2 ** 64 - 1),
                                             1 if use_stream else 0, _ptr(idx),
                                             _ptr(q), _ptr(qmin), _ptr(count), _ptr(e), self._s()),
              "rpl_sumtree_sample_sharded")
        return idx, q, qmin

    def sample_sharded_p2p(self, rank, n_shards, board_ptrs, n, seed, count, out=None, err=None):
        """rpl_sumtree_sample_sharded_p2p: compacted stream-mode sharded sampling with the
        totals exchange (K5) fused in over the peer boards (board_ptrs: device int64 [n_shards]
        of board addresses, see shard.PeerBoards).  Returns (idx, q); count = [m, k0]."""
        n = int(n)
        _req(board_ptrs, torch.int64, "board_ptrs", (n_shards,))
        _req(count, torch.int64, "count", (2,))
        if out is None:
            idx = torch.empty(n, dtype=torch.int64, device=self.device)
            q = torch.empty(n, dtype=torch.int64, device=self.device)
        else:
            idx, q = out
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample_sharded_p2p(self._lp, _ptr(self.storage), int(rank), int(n_shards),
                                                 self.n_leaves, _ptr(board_ptrs), n, int(seed) & (2 ** 64 - 1),
                                                 _ptr(idx), _ptr(q), _ptr(count), _ptr(e), self._s()),
              "rpl_sumtree_sample_sharded_p2p")
        return idx, q

    def find(self, prefix, err=None):
        _req(prefix, torch.int64, "prefix")
        out = torch.empty_like(prefix)
        e = self.err if err is None else err
        check(lib.rpl_sumtree_find(self._lp, _ptr(self.storage), _ptr(prefix), prefix.numel(), _ptr(out), _ptr(e),
                                   self._s()), "rpl_sumtree_find")
        return out

    def total(self, out=None):
        out = torch.empty(1, dtype=torch.int64, device=self.device) if out is None else out
        check(lib.rpl_sumtree_total(self._lp, _ptr(self.storage), _ptr(out), self._s()), "rpl_sumtree_total")
        return out

    def sample_unique(self, n, seed, offset=0, use_stream=False, err=None):
        """rpl_sumtree_sample_unique: n distinct leaves by successive proportional draws."""
        n = int(n)
        idx = torch.empty(n, dtype=torch.int64, device=self.device)
        q = torch.empty(n, dtype=torch.int64, device=self.device)
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample_unique(self._lp, _ptr(self.storage), n, int(seed) & (2 ** 64 - 1),
                                            int(offset) & (2 ** 64 - 1), 1 if use_stream else 0, _ptr(idx), _ptr(q),
                                            _ptr(e), self._s()), "rpl_sumtree_sample_unique")
        return idx, q

    def attach_min_tree(self):
        """rpl_mintree_attach: keep a min-tree beside the sum tree (buffer-wide IS normaliser,
        R29); `min_root` (a 1-element view) is then the buffer min after every update."""
        self.mins = torch.empty(int(self.layout.level_off[self.depth]), dtype=torch.int64, device=self.device)
        check(lib.rpl_mintree_attach(self._lp, _ptr(self.storage), _ptr(self.mins), self._s()), "rpl_mintree_attach")
        return self.mins

    def detach_min_tree(self):
        check(lib.rpl_mintree_attach(self._lp, _ptr(self.storage), None, self._s()), "rpl_mintree_attach")
        self.mins = None

    @property
    def min_root(self):
        return None if self.mins is None else self.mins[:1]

    def min_level(self, l: int) -> torch.Tensor:
        off, ln = int(self.layout.level_off[l]), int(self.layout.level_len[l])
        return self.mins[off:off + ln]

    def total_min(self, out=None):
        """rpl_sumtree_total_min: [total, buffer min] (the K5 record with the normaliser)."""
        out = torch.empty(2, dtype=torch.int64, device=self.device) if out is None else out
        check(lib.rpl_sumtree_total_min(self._lp, _ptr(self.storage), _ptr(out), self._s()), "rpl_sumtree_total_min")
        return out

    def sample_sharded_pairs(self, rank, n_shards, pairs, n, seed, count, out=None, bufmin=None, err=None):
        """rpl_sumtree_sample_sharded_pairs: pairs = all-gathered [n_shards, 2] {total, min}."""
        n = int(n)
        _req(pairs, torch.int64, "pairs", (n_shards, 2))
        _req(count, torch.int64, "count", (2,))
        if out is None:
            idx = torch.empty(n, dtype=torch.int64, device=self.device)
            q = torch.empty(n, dtype=torch.int64, device=self.device)
            qmin = torch.empty(1, dtype=torch.int64, device=self.device)
        else:
            idx, q, qmin = out
        bufmin = torch.empty(1, dtype=torch.int64, device=self.device) if bufmin is None else bufmin
        e = self.err if err is None else err
        check(lib.rpl_sumtree_sample_sharded_pairs(self._lp, _ptr(self.storage), int(rank), int(n_shards),
                                                   int(self.n_leaves), _ptr(pairs), n, int(seed) & (2 ** 64 - 1),
                                                   _ptr(idx), _ptr(q), _ptr(qmin), _ptr(count), _ptr(bufmin), _ptr(e),
                                                   self._s()), "rpl_sumtree_sample_sharded_pairs")
        return idx, q, qmin, bufmin

    def min_q(self, out=None):
        """rpl_sumtree_min: buffer-wide min q over non-zero leaves (NEXT-4 IS normaliser)."""
        out = torch.empty(1, dtype=torch.int64, device=self.device) if out is None else out
        check(lib.rpl_sumtree_min(self._lp, _ptr(self.storage), _ptr(out), self._s()), "rpl_sumtree_min")
        return out

    def rebuild(self):
        check(lib.rpl_sumtree_rebuild(self._lp, _ptr(self.storage), self._s()), "rpl_sumtree_rebuild")

    # ---- checkpoint / resume: leaves + header are the state; internal nodes are
    # recomputed exactly from the leaves (int64 sums) by rpl_sumtree_rebuild
    def state_dict(self):
        return {"n_leaves": self.n_leaves, "fanout": self.fanout, "frac_bits": self.frac_bits,
                "leaves": self.leaves.detach().cpu().clone(), "header": self.header.detach().cpu().clone()}

    def load_state_dict(self, sd):
        if (int(sd["n_leaves"]), int(sd["fanout"]), int(sd["frac_bits"])) != (self.n_leaves, self.fanout,
                                                                            self.frac_bits):
            raise ValueError("tree geometry mismatch")
        self.storage.zero_()
        self.leaves.copy_(sd["leaves"].to(self.device))
        self.header.copy_(sd["header"].to(self.device))
        # header word 5 is a device address: keep this object's own min-tree attachment
        self.header[5] = 0 if self.mins is None else self.mins.data_ptr()
        self.header[6] = 0
        self.rebuild()


# ---------------------------------------------------------------- gather
@dataclass
class GatherRing:
    """Device replay ring (time-major [cap_T, B, ...]) for rpl_gather."""
    obs: torch.Tensor            # [cap_T, B, *item] (u8 frames or f32 vectors)
    act: torch.Tensor            # [cap_T, B] int64 or [cap_T, B, A] f32
    rew: torch.Tensor            # [cap_T, B] f32
    done: torch.Tensor           # [cap_T, B] u8
    cursor: int
    size: int
    rnn: torch.Tensor | None = None  # [cap_T/period, B, parts, H] f32
    v_term: torch.Tensor | None = None  # [cap_T, B] f32 terminal values of time-limit rows (R34)

    @property
    def cap_T(self):
        return int(self.obs.shape[0])

    @property
    def B(self):
        return int(self.obs.shape[1])

    @property
    def item_shape(self):
        return tuple(self.obs.shape[2:])

    @property
    def obs_bytes(self):
        return int(self.obs[0, 0].numel() * self.obs.element_size())

    @property
    def act_shape(self):
        return tuple(self.act.shape[2:])

    @property
    def act_bytes(self):
        return int(self.act[0, 0].numel() * self.act.element_size())


def _desc(ring: GatherRing, kind, k, pad_mode, out_mode, n_step, seq_len, period, gamma):
    for name in ("obs", "act", "rew", "done"):
        t = getattr(ring, name)
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"ring.{name} must be a contiguous CUDA tensor")
    g = GatherDesc()
    g.kind, g.pad_mode, g.out_mode, g.k = kind, pad_mode, out_mode, k
    g.cap_T, g.B, g.cursor, g.size = ring.cap_T, ring.B, int(ring.cursor), int(ring.size)
    g.obs_bytes, g.act_bytes = ring.obs_bytes, ring.act_bytes
    g.n_step, g.seq_len, g.period = n_step, seq_len, period
    g.gamma = float(gamma)
    g.obs, g.act, g.rew, g.done = ring.obs.data_ptr(), ring.act.data_ptr(), ring.rew.data_ptr(), ring.done.data_ptr()
    if ring.v_term is not None:
        _req(ring.v_term, torch.float32, "ring.v_term", (ring.cap_T, ring.B))
        g.v_term = ring.v_term.data_ptr()
    if ring.rnn is not None:
        g.rnn = ring.rnn.data_ptr()
        g.rnn_parts = int(ring.rnn.shape[2])
        g.rnn_bytes = int(ring.rnn[0, 0, 0].numel() * ring.rnn.element_size())
    return g


def _set_targets(g, targets, seq_len, n, o, alloc):
    """Fused sequence n-step targets (rpl_gather_desc.q_tgt / o_tgt, R5 / R24 / R34):
    targets = dict(lo, T, n_step, gamma, rescale=False, eps=1e-3, q=None) with q f32 [L, n]."""
    lo, T = int(targets["lo"]), int(targets["T"])
    g.n_step = int(targets["n_step"])
    g.gamma = float(targets["gamma"])
    g.tgt_lo, g.tgt_T = lo, T
    g.rescale = 1 if targets.get("rescale", False) else 0
    g.rescale_eps = float(targets.get("eps", 1e-3))
    qt = targets.get("q")
    if qt is not None:
        _req(qt, torch.float32, "targets['q']", (seq_len, n))
        g.q_tgt = qt.data_ptr()
    alloc("tgt", (T, n), torch.float32, force=True)
    alloc("tgt_done", (T, n), torch.uint8, force=True)


def gather(ring: GatherRing, idx, kind="transition", k=4, n_step=1, gamma=0.99, seq_len=1, period=1,
           pad_mode=_lib.PAD_REPEAT, out_mode=_lib.OUT_STACKED, q=None, qmin=None, beta=0.0, outputs=None,
           err=None, want=None, targets=None):
    """rpl_gather.  Returns a dict of output tensors (allocated unless given in `outputs`).
    targets (SEQUENCE): fused n-step targets, see _set_targets (outputs "tgt", "tgt_done")."""
    _req(idx, torch.int64, "idx")
    n = idx.numel()
    dev = ring.obs.device
    kind_i = _lib.GATHER_TRANSITION if kind == "transition" else _lib.GATHER_SEQUENCE
    g = _desc(ring, kind_i, k, pad_mode, out_mode, n_step if kind_i == 0 else 1, seq_len, period, gamma)
    o = {} if outputs is None else dict(outputs)
    item = ring.item_shape
    od = ring.obs.dtype
    wants = set(want) if want is not None else None

    def alloc(name, shape, dtype, force=False):
        if name not in o and (force or wants is None or name in wants):
            o[name] = torch.empty(shape, dtype=dtype, device=dev)

    if kind_i == _lib.GATHER_TRANSITION:
        alloc("obs", (n, k) + item, od)
        alloc("next_obs", (n, k) + item, od)
        alloc("act", (n,) + ring.act_shape, ring.act.dtype)
        alloc("ret", (n,), torch.float32)
        alloc("done_n", (n,), torch.uint8)
    else:
        L = seq_len
        if out_mode == _lib.OUT_STACKED:
            alloc("obs", (L, n, k) + item, od)
        else:
            alloc("obs", (L + k - 1, n) + item, od)
        alloc("act", (L, n) + ring.act_shape, ring.act.dtype)
        alloc("prev_act", (L, n) + ring.act_shape, ring.act.dtype)
        alloc("rew", (L, n), torch.float32)
        alloc("prev_rew", (L, n), torch.float32)
        alloc("done", (L, n), torch.uint8)
        if ring.rnn is not None:
            alloc("rnn", (int(ring.rnn.shape[2]), n, int(ring.rnn.shape[3])), ring.rnn.dtype)
        if wants is not None and "start" in wants:  # episode-start offsets (Mode C shipping)
            alloc("start", (L, n), torch.int8)
        if targets is not None:
            _set_targets(g, targets, L, n, o, alloc)
    if q is not None:
        alloc("w", (n,), torch.float32)
    fields = {"obs": "o_obs", "next_obs": "o_next_obs", "act": "o_act", "prev_act": "o_prev_act", "rew": "o_rew",
              "prev_rew": "o_prev_rew", "done": "o_done", "ret": "o_ret", "done_n": "o_done_n", "w": "o_w",
              "rnn": "o_rnn", "start": "o_start", "tgt": "o_tgt", "tgt_done": "o_tgt_done"}
    for name, f in fields.items():
        if name in o and o[name] is not None:
            setattr(g, f, o[name].data_ptr())
    work = None
    if kind_i == _lib.GATHER_SEQUENCE:  # dynamic-tail work counter (rpl_gather_desc.work)
        work = torch.zeros(4, dtype=torch.int64, device=dev)
        g.work = work.data_ptr()
    e = err
    check(lib.rpl_gather(C.byref(g), _ptr(idx), _ptr(q), _ptr(qmin), float(beta), n, _ptr(e), _stream(dev)),
          "rpl_gather")
    return o


class GatherPlan:
    """A prepared rpl_gather call: the descriptor (ring + preallocated outputs) is
    built once, so each run() is one ctypes call (cheap enough for a hot loop and
    capturable in a CUDA graph)."""

    def __init__(self, ring: GatherRing, n, kind="transition", k=4, n_step=1, gamma=0.99, seq_len=1, period=1,
                 pad_mode=_lib.PAD_REPEAT, out_mode=_lib.OUT_STACKED, want=None, with_weights=False, outputs=None,
                 targets=None):
        """outputs: optional dict of preallocated output tensors (e.g. a central learner's
        buffers mapped over CUDA IPC, Mode C); missing ones are allocated here.
        targets: fused sequence n-step targets (see _set_targets; the bootstrap q may be
        swapped per call with run(q_tgt=...))."""
        dev = ring.obs.device
        self.n = int(n)
        dummy = torch.zeros(self.n, dtype=torch.int64, device=dev)
        # allocate via gather() on an all-skip index vector (no kernel work: idx < 0)
        self.outputs = gather(ring, torch.full_like(dummy, -1), kind=kind, k=k, n_step=n_step, gamma=gamma,
                              seq_len=seq_len, period=period, pad_mode=pad_mode, out_mode=out_mode, want=want,
                              outputs=outputs, targets=targets)
        if with_weights and "w" not in self.outputs:
            self.outputs["w"] = torch.empty(self.n, dtype=torch.float32, device=dev)
        kind_i = _lib.GATHER_TRANSITION if kind == "transition" else _lib.GATHER_SEQUENCE
        self.desc = _desc(ring, kind_i, k, pad_mode, out_mode, n_step if kind_i == 0 else 1, seq_len, period, gamma)
        fields = {"obs": "o_obs", "next_obs": "o_next_obs", "act": "o_act", "prev_act": "o_prev_act",
                  "rew": "o_rew", "prev_rew": "o_prev_rew", "done": "o_done", "ret": "o_ret", "done_n": "o_done_n",
                  "w": "o_w", "rnn": "o_rnn",
                  "start": "o_start", "tgt": "o_tgt", "tgt_done": "o_tgt_done"}
        if targets is not None:
            _set_targets(self.desc, targets, seq_len, self.n, self.outputs, lambda *a, **kw: None)
        for name, f in fields.items():
            if name in self.outputs:
                setattr(self.desc, f, self.outputs[name].data_ptr())
        if kind_i == _lib.GATHER_SEQUENCE:  # dynamic-tail work counter (rpl_gather_desc.work)
            self._work = torch.zeros(4, dtype=torch.int64, device=dev)
            self.desc.work = self._work.data_ptr()
        self._dp = C.byref(self.desc)
        self.device = dev
        self.ring = ring

    def set_cursor(self, cursor, size):
        self.desc.cursor = int(cursor)
        self.desc.size = int(size)

    def set_peers(self, board_ptrs, world, rank):
        """Fuse the batch-min exchange (K7) into the gather: board_ptrs as given to
        SumTree.sample_sharded_p2p (None: off).  Needs with_weights and q at run time."""
        self._peer_ptrs = board_ptrs  # keep the pointer array alive
        self.desc.peer_boards = None if board_ptrs is None else board_ptrs.data_ptr()
        self.desc.peer_world = int(world) if board_ptrs is not None else 0
        self.desc.peer_rank = int(rank) if board_ptrs is not None else 0

    def run_sample(self, tree, seed, idx_out, q_out, beta=0.0, err=None, stream=None, q_tgt=None):
        """rpl_gather_sample: draw this call's n stratified samples from `tree` (its stream)
        inside the gather; idx_out / q_out receive them, outputs["w"] the IS weights."""
        s = _stream(self.device) if stream is None else stream
        if q_tgt is not None:
            self.desc.q_tgt = q_tgt.data_ptr()
        check(lib.rpl_gather_sample(self._dp, tree._lp, _ptr(tree.storage), int(seed) & (2 ** 64 - 1), _ptr(idx_out),
                                    _ptr(q_out), float(beta), self.n, _ptr(err), s), "rpl_gather_sample")
        return self.outputs

    def run_update_sample(self, tree, upd_idx, upd_td, seed, idx_out, q_out, eta=0.9, alpha=0.9, eps_p=1e-3,
                          beta=0.0, live_only=False, err=None, stream=None, q_tgt=None):
        """rpl_gather_update_sample: rpl_sumtree_update_seq(upd_idx, upd_td [T_p, n_upd]) and
        rpl_gather_sample in ONE launch when the dynamic-tail kernel can run it (else the two)."""
        s = _stream(self.device) if stream is None else stream
        if q_tgt is not None:
            self.desc.q_tgt = q_tgt.data_ptr()
        T_p, n_upd = (int(upd_td.shape[0]), int(upd_td.shape[1])) if upd_td.dim() == 2 else (1, int(upd_td.numel()))
        check(lib.rpl_gather_update_sample(self._dp, tree._lp, _ptr(tree.storage), _ptr(upd_idx), _ptr(upd_td), T_p,
                                           n_upd, float(eta), float(alpha), float(eps_p),
                                           1 if live_only else 0, int(seed) & (2 ** 64 - 1), _ptr(idx_out),
                                           _ptr(q_out), float(beta), self.n, _ptr(err), s), "rpl_gather_update_sample")
        return self.outputs

    def run(self, idx, q=None, qmin=None, beta=0.0, err=None, stream=None, q_tgt=None):
        """q_tgt: this call's bootstrap values for the fused targets (f32 [L, n]; None keeps
        the one set before)."""
        s = _stream(self.device) if stream is None else stream
        if q_tgt is not None:
            self.desc.q_tgt = q_tgt.data_ptr()
        check(lib.rpl_gather(self._dp, _ptr(idx), _ptr(q), _ptr(qmin), float(beta), self.n, _ptr(err), s),
              "rpl_gather")
        return self.outputs


def ring_append(ring: GatherRing, obs=None, act=None, rew=None, done=None, rnn=None, period=1):
    """rpl_ring_append: write a [T_b, B, ...] sampler batch (host-pinned or device tensors) at
    ring.cursor, then advance ring.cursor / ring.size.  Returns (cursor_old, size_old) for
    SumTree.validity."""
    src = next(t for t in (obs, act, rew, done) if t is not None)
    T_b = int(src.shape[0])
    for name, t in (("obs", obs), ("act", act), ("rew", rew), ("done", done), ("rnn", rnn)):
        if t is not None and not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    g = _desc(ring, _lib.GATHER_SEQUENCE, 1, _lib.PAD_REPEAT, _lib.OUT_STACKED, 1, 1, period, 0.0)
    check(lib.rpl_ring_append(C.byref(g), _ptr(obs), _ptr(act), _ptr(rew), _ptr(done), _ptr(rnn), T_b,
                              _stream(ring.obs.device)), "rpl_ring_append")
    old = (ring.cursor, ring.size)
    ring.cursor = (ring.cursor + T_b) % ring.cap_T
    ring.size = min(ring.cap_T, ring.size + T_b)
    return old


def ring_append_rows(ring_array, src, cursor):
    """rpl_ring_append_rows: src [T_b, ...] (host-pinned or device) -> ring_array [cap_T, ...]
    rows cursor .. (mod cap_T).  Does not move any ring cursor."""
    if not ring_array.is_contiguous() or not src.is_contiguous() or src.dtype != ring_array.dtype \
            or tuple(src.shape[1:]) != tuple(ring_array.shape[1:]):
        raise ValueError("src must be a contiguous [T_b, ...] tensor matching ring_array's rows")
    row_bytes = int(ring_array[0].numel() * ring_array.element_size())
    check(lib.rpl_ring_append_rows(_ptr(ring_array), row_bytes, int(ring_array.shape[0]), int(cursor), _ptr(src),
                                   int(src.shape[0]), _stream(ring_array.device)), "rpl_ring_append_rows")


def ring_td_abs(rew, done, q_taken, q_boot, row0, T_out, n, gamma, rescale=False, eps=1e-3, out=None):
    """rpl_ring_td_abs: per-step |n-step TD error| of ring rows row0 .. row0+T_out-1 (mod cap_T)
    from ring arrays [cap_T, B] -> [T_out, B] f32 (R33)."""
    cap, B = (int(x) for x in rew.shape)
    _req(rew, torch.float32, "rew")
    _req(done, torch.uint8, "done", (cap, B))
    _req(q_taken, torch.float32, "q_taken", (cap, B))
    _req(q_boot, torch.float32, "q_boot", (cap, B))
    out = torch.empty((int(T_out), B), dtype=torch.float32, device=rew.device) if out is None else out
    _req(out, torch.float32, "out", (int(T_out), B))
    check(lib.rpl_ring_td_abs(_ptr(rew), _ptr(done), _ptr(q_taken), _ptr(q_boot), cap, B, int(row0), int(T_out),
                              int(n), float(gamma), 1 if rescale else 0, float(eps), _ptr(out),
                              _stream(rew.device)), "rpl_ring_td_abs")
    return out


def stack_frames(uniq, start, k, pad_mode=_lib.PAD_REPEAT, out=None, n_active=None):
    """rpl_stack_frames: uniq [L+k-1, n, *item] + start int8 [L, n] -> stacked [L, n, k, *item]."""
    _req(start, torch.int8, "start")
    L, n = (int(x) for x in start.shape)
    if uniq.shape[0] != L + k - 1 or uniq.shape[1] != n or not uniq.is_contiguous():
        raise ValueError("uniq must be a contiguous [L+k-1, n, ...] tensor")
    item = tuple(uniq.shape[2:])
    ob = int(uniq[0, 0].numel() * uniq.element_size())
    out = torch.empty((L, n, k) + item, dtype=uniq.dtype, device=uniq.device) if out is None else out
    check(lib.rpl_stack_frames(_ptr(uniq), _ptr(start), L, n, int(k), ob, int(pad_mode), _ptr(out), _ptr(n_active),
                               _stream(uniq.device)), "rpl_stack_frames")
    return out
