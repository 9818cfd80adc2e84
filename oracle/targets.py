"""Oracle: learning targets computed right after the gather.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs; never by the product package.

Paper: rlpyt's DQN family includes "Double-DQN, Dueling, Categorical (C51)"
 with n-step returns; R2D2 uses value rescaling.

  double-Q selection   a*_tau = argmax_a Qonline(s_tau, a)   (first maximum; a NaN
                       never wins, reading R27), bootstrap q_tau = Qtarget(s_tau, a*_tau)
                       [EXT: van Hasselt et al. 2016, Double DQN]
  n-step target        y_t from oracle.returns.nstep_return with q_{t+n} = that bootstrap
  C51 projection       [EXT: Bellemare et al. 2017, Algorithm 1]: atoms z_j = v_min + j dz,
                       dz = (v_max - v_min) / (N - 1); for every next-state atom j:
                       Tz_j = clip(R + g z_j, v_min, v_max) with g = gamma^n (1 - done^n);
                       b_j = (Tz_j - v_min) / dz, l = floor(b_j), u = ceil(b_j);
                       m_l += p_j (u - b_j), m_u += p_j (b_j - l); when l == u, m_l += p_j.
                       The next-state distribution p is the target net's at the action
                       the online net selects (double-Q, as above).

All arithmetic float64, loops in the algorithm's order.
"""
from __future__ import annotations

import math

import numpy as np

from . import returns as _ret


def argmax_first(values) -> int:
    """Index of the first maximum; NaN entries never win (all NaN -> 0)."""
    best, bi = None, 0
    for a, v in enumerate(values):
        v = float(v)
        if math.isnan(v):
            continue
        if best is None or v > best:
            best, bi = v, a
    return bi


def double_q_bootstrap(q_online, q_target):
    """q_online, q_target [T, B, A] -> (a* [T, B] int, q [T, B] float64 = q_target at a*)."""
    q_online = np.asarray(q_online)
    q_target = np.asarray(q_target, np.float64)
    T, B, _ = q_online.shape
    a = np.zeros((T, B), np.int64)
    q = np.zeros((T, B), np.float64)
    for t in range(T):
        for b in range(B):
            a[t, b] = argmax_first(q_online[t, b])
            q[t, b] = q_target[t, b, a[t, b]]
    return a, q


def nstep_double_q(r, d, n, gamma, q_online, q_target, rescale=False, eps=1e-3):
    """n-step targets with the double-Q bootstrap: q_online / q_target cover rows 0..T
    ([T+1, B, A]); output row t bootstraps from row t+n.  Returns (y [T-n+1, B],
    done_n [T-n+1, B], a* at rows n..T [T-n+1, B])."""
    T = np.asarray(r).shape[0]
    a, q = double_q_bootstrap(q_online, q_target)
    y, dn = _ret.nstep_return(r, d, n, gamma, q=q[:T], q_boot=q[T], rescale=rescale, eps=eps)
    return y, dn, a[n:T + 1]


def c51_project(p_next, R, g, v_min, v_max):
    """Categorical projection of one sample: p_next [N] (next-state distribution), return R,
    discount g = gamma^n (1 - done^n).  Bellemare et al. 2017, Algorithm 1."""
    p_next = [float(x) for x in p_next]
    N = len(p_next)
    dz = (v_max - v_min) / (N - 1)
    m = [0.0] * N
    for j in range(N):
        z = v_min + j * dz
        tz = min(max(R + g * z, v_min), v_max)
        b = (tz - v_min) / dz
        lo, up = math.floor(b), math.ceil(b)
        lo = min(max(lo, 0), N - 1)
        up = min(max(up, 0), N - 1)
        if lo == up:
            m[lo] += p_next[j]
        else:
            m[lo] += p_next[j] * (up - b)
            m[up] += p_next[j] * (b - lo)
    return m


def c51_targets(p_target, q_online, R, done_n, gamma_n, v_min, v_max):
    """Batch: p_target [n, A, N], q_online [n, A] (or None with A == 1), R [n], done_n [n]
    -> m [n, N] float64 (projection of the target distribution at the online argmax)."""
    p_target = np.asarray(p_target, np.float64)
    n, A, N = p_target.shape
    out = np.zeros((n, N), np.float64)
    for s in range(n):
        a = 0 if q_online is None else argmax_first(np.asarray(q_online)[s])
        g = gamma_n * (1.0 - float(done_n[s]))
        out[s] = c51_project(p_target[s, a], float(R[s]), g, v_min, v_max)
    return out


# ---- initial priorities of new samples (§8f NEXT-1; P:123 fn; reading R33) ----------
#
# P:123 fn: new samples were first prioritised with 1-step TD errors; results "improved when
# we corrected to use 5-step TD initial priorities".  SPEC S:660 makes n-step-TD initial
# priorities the recurrent algorithm's option (default n = 5).  R33: the actor stores, per
# ring row, q_taken = Q(s_t, a_t) and q_boot = its bootstrap value of s_t (max_a Q, or the
# double-Q value); the per-step TD error of row t is
#     delta_t = y_t - q_taken_t,  y_t = the n-step target of row t (R24; rescaled per §8c #5)
# with the bootstrap q_boot at row t+n; rows are taken modulo the ring capacity.  A sequence
# leaf's initial priority is the R26 mix (sequence_td) of |delta_t| over its TRAIN rows
# (block start + burn_in .. + train - 1, all stored once the leaf is valid); a transition
# leaf's is |delta_t| of its own row.


def ring_rows(a, row0, count):
    """Rows row0 .. row0+count-1 of a ring array [cap_T, ...], modulo cap_T."""
    a = np.asarray(a)
    cap = a.shape[0]
    return a[[(row0 + i) % cap for i in range(count)]]


def ring_td_abs(rew, done, q_taken, q_boot, row0, T_out, n, gamma, rescale=False, eps=1e-3):
    """|delta_t| for t = 0 .. T_out-1 (ring row row0 + t) -> float64 [T_out, B].  The n-step
    target comes from oracle.returns.nstep_return over the unrolled rows row0 .. row0+T_out+n-1
    with q = q_boot (row t+n is the bootstrap of output row t)."""
    rows = T_out + n - 1
    r = ring_rows(rew, row0, rows).astype(np.float64)
    d = ring_rows(done, row0, rows)
    qb = ring_rows(q_boot, row0, rows + 1).astype(np.float64)
    y, _ = _ret.nstep_return(r, d, n, gamma, q=qb[:rows], q_boot=qb[rows], rescale=rescale, eps=eps)
    qt = ring_rows(q_taken, row0, T_out).astype(np.float64)
    return np.abs(y - qt)


def initial_sequence_priorities(rew, done, q_taken, q_boot, block, period, burn_in, train, n, gamma, eta,
                                rescale=True, eps=1e-3):
    """Per env b: the R26 mix of fp32 |delta_t| over block `block`'s train rows -> list [B]
    of the |delta| values that then enter the priority transform (sequence_td)."""
    from . import priority as _pr
    row0 = block * period + burn_in
    td = ring_td_abs(rew, done, q_taken, q_boot, row0, train, n, gamma, rescale, eps).astype(np.float32)
    return [_pr.sequence_td(td[:, b], eta) for b in range(td.shape[1])]
