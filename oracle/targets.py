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
