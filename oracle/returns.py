"""Oracle: return estimation over time-major [T, B] sample buffers (float64).

Paper: rlpyt lists A2C/PPO, DQN variants and replay "n-step
returns"; sample buffers are time-major "[Time, Batch]".  The
paper prints no formulas; the definitions come from SPEC.md:

  * discounted return  R_t = r_t + gamma (1 - d_t) R_{t+1},  R_T = bootstrap
      (S:340-347 TrajInfo discounted return; S:751 returns = adv + values)
  * n-step return      R^n_t = sum_{i<n} gamma^i r_{t+i} prod_{j<i} (1 - d_{t+j}),
                       done^n_t = OR_{i<n} d_{t+i}
    optional target    y_t = R^n_t + gamma^n (1 - done^n_t) q_{t+n}
    rescaled target    y_t = h(R^n_t + gamma^n (1 - done^n_t) h^-1(q_{t+n}))  (§8c #5)
  * GAE                delta_t = r_t + gamma (1 - d_t) V_{t+1} - V_t,
                       A_t = delta_t + gamma lambda (1 - d_t) A_{t+1}, A_T = 0,
                       ret_t = A_t + V_t,  V_T = bootstrap

d_t = 1 means the episode ended after transition t: r_t counts, nothing after
it does and nothing is bootstrapped across it (§8c #1, pinned by S:598).

Time limits (reading R34; P:95 fn "bootstrapping the value function when the
trajectory ends due to time limit"): d_t = 2 means the episode
ended after t because of a time limit.  Any non-zero d_t ends the episode (the
recursion is cut there).  When the caller passes v_term (same [T, B] layout:
the value of the final observation of each time-limit row), a d_t = 2 row
bootstraps from it: the term gamma * v_term_t stands where gamma * (next value)
would have stood.  Without v_term, d_t = 2 is a plain terminal.

Every loop runs over t in the order the definition states and is vectorised
over the independent columns b only.  All arithmetic is float64.
"""
from __future__ import annotations

import numpy as np

from . import rescale as _rs


def _f64(x):
    return np.asarray(x, dtype=np.float64)


def _ends(d, v_term, shape):
    """(ended, tail): ended_t = 1 when d_t != 0; tail_t = v_term_t at time-limit rows
    (d_t == 2) when v_term is given, else 0 (R34)."""
    d = np.asarray(d).astype(np.int64)
    ended = (d != 0).astype(np.float64)
    tail = np.zeros(shape, np.float64)
    if v_term is not None:
        tail = np.where(d == 2, _f64(v_term), 0.0)
    return ended, tail


def discounted_return(r, d, bootstrap, gamma, v_term=None):
    """R_t = r_t + gamma*(1-e_t)*R_{t+1} + gamma*tail_t, R_T = bootstrap (or 0), with
    e_t = [d_t != 0] and tail_t = v_term_t at time-limit rows (R34). S:346."""
    r = _f64(r)
    T, B = r.shape
    e, tail = _ends(d, v_term, (T, B))
    R = np.zeros((T, B), np.float64)
    nxt = np.zeros(B, np.float64) if bootstrap is None else _f64(bootstrap).copy()
    for t in range(T - 1, -1, -1):
        nxt = r[t] + gamma * (1.0 - e[t]) * nxt + gamma * tail[t]
        R[t] = nxt
    return R


def nstep_return(r, d, n, gamma, q=None, q_boot=None, rescale=False, eps=1e-3, v_term=None):
    """n-step return by direct summation of its definition, rows 0..T-n.

    Returns (R [T-n+1, B] float64 — or the target y when q is given / rescale
    is on — and done_n [T-n+1, B] uint8).  q is [T, B] (value of s_tau), q_boot
    [B] the value at row T; the bootstrap for output row t is q_{t+n}.
    Rescaled target per §8c #5: y = h(R^n + gamma^n (1-done^n) h^-1(q_{t+n})),
    with h, h^-1 evaluated by the mpmath oracle (oracle.rescale).
    Time limits (R34): if the first ended row t+j (j < n) is a time-limit row,
    R^n also gets gamma^(j+1) v_term_{t+j}; done_n stays 1.
    """
    r = _f64(r)
    T, B = r.shape
    e, tail = _ends(d, v_term, (T, B))
    e = e.astype(np.int64)
    if n < 1 or n > T:
        raise ValueError("need 1 <= n <= T")
    rows = T - n + 1
    R = np.zeros((rows, B), np.float64)
    done_n = np.zeros((rows, B), np.uint8)
    for t in range(rows):
        acc = np.zeros(B, np.float64)
        alive = np.ones(B, np.int64)          # prod_{j<i} (1 - e_{t+j})
        for i in range(n):
            acc = acc + (gamma ** i) * r[t + i] * alive
            acc = acc + (gamma ** (i + 1)) * tail[t + i] * alive * e[t + i]   # time-limit bootstrap
            alive = alive * (1 - e[t + i])
        R[t] = acc
        done_n[t] = (1 - alive).astype(np.uint8)
    if q is None:
        if rescale:
            return _rs.h_array(R, eps), done_n
        return R, done_n
    q = _f64(q)
    qb = _f64(q_boot)
    qfull = np.concatenate([q, qb[None, :]], axis=0)  # row T = bootstrap
    gn = gamma ** n
    y = np.zeros_like(R)
    for t in range(rows):
        for b in range(B):
            boot = qfull[t + n, b]
            if rescale:
                y[t, b] = _rs.h_of_target(R[t, b], gn, int(done_n[t, b]), boot, eps)
            else:
                y[t, b] = R[t, b] + gn * (1 - int(done_n[t, b])) * boot
    return y, done_n


def gae(r, v, d, bootstrap_v, gamma, lam, v_term=None):
    """Generalised advantage estimation. Returns (adv, ret) float64.
    Time limits (R34): delta_t = r_t + gamma*(1-e_t)*V_{t+1} + gamma*tail_t - V_t."""
    r = _f64(r)
    v = _f64(v)
    T, B = r.shape
    e, tail = _ends(d, v_term, (T, B))
    adv = np.zeros((T, B), np.float64)
    v_next = _f64(bootstrap_v).copy()
    a_next = np.zeros(B, np.float64)
    for t in range(T - 1, -1, -1):
        nd = 1.0 - e[t]
        delta = r[t] + gamma * nd * v_next + gamma * tail[t] - v[t]
        a_next = delta + gamma * lam * nd * a_next
        adv[t] = a_next
        v_next = v[t]
    return adv, adv + v


def abs_scale_discounted(r, d, bootstrap, gamma, v_term=None):
    """S_t: the same recurrence on |r|, |bootstrap| and |v_term| — the magnitude scale
    used by the cancellation clause of the 1e-5 tolerance (§8c #21)."""
    return discounted_return(np.abs(_f64(r)), d, None if bootstrap is None else np.abs(_f64(bootstrap)), gamma,
                             None if v_term is None else np.abs(_f64(v_term)))


def abs_scale_gae(r, v, d, bootstrap_v, gamma, lam, v_term=None):
    """Magnitude scale for GAE outputs: the GAE recurrence on |r|, |V|, |v_term| with
    every term added (no subtraction), plus |V_t| for the returns (§8c #21)."""
    r = np.abs(_f64(r))
    v = np.abs(_f64(v))
    T, B = r.shape
    e, tail = _ends(d, None if v_term is None else np.abs(_f64(v_term)), (T, B))
    out = np.zeros((T, B), np.float64)
    v_next = np.abs(_f64(bootstrap_v)).copy()
    a_next = np.zeros(B, np.float64)
    for t in range(T - 1, -1, -1):
        nd = 1.0 - e[t]
        delta = r[t] + gamma * nd * v_next + gamma * tail[t] + v[t]
        a_next = delta + gamma * lam * nd * a_next
        out[t] = a_next + v[t]
        v_next = v[t]
    return out
