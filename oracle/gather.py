"""Oracle: gather of sampled transitions and sequences from a frame-deduplicated ring.

Paper: replay buffers with "n-step returns; sequence replay (for recurrence);
periodic storage of recurrent state (to save memory); ... frame-based buffer, to
save memory e.g. by storing only unique Atari frames"; recurrent agents
take (observation, previous_action, previous_reward); training data has
leading dims [Time, Batch] and recurrent state is [Num_Layers, Batch,
Hidden].  SPEC: frame reconstruction "equals a naive buffer that stored
full k-stacks; episode starts pad with the first frame"; sequence
replay with aligned starts and stored state.

This oracle is the NAIVE FULL-STACK reference: it rebuilds each k-stack
the way a frame-stacking environment wrapper builds it while the episode is
played — on a reset the stack is filled with copies of the first frame (or with
zeros, pad_mode "zero"); every later step shifts the new frame in — by replaying
that wrapper over the frames of rows r-k+1 .. r.  It never uses a closed form
for the padded row index.

Ring geometry: rows are ring slots 0..cap_T-1; leaf
= row * B + b for transitions and block * B + b for sequences (block = row /
period); `cursor` is the ring row the next append writes; `size` rows are valid.
d[row, b] = 1 means the episode ended after that row (§8c #1), so row+1 starts
a new episode.
"""
from __future__ import annotations

import numpy as np

from . import returns as _ret

PAD_REPEAT = 0
PAD_ZERO = 1


def _row(r, cap):
    return r % cap


def wrapper_stacks(obs, done, b, rows, k, pad_mode):
    """Replay a frame-stacking wrapper over consecutive ring rows `rows`
    (ascending, possibly wrapping) of column b; return the stack after each row.
    The wrapper is started k-1 rows before the first requested row so that its
    (unknown) earlier state has been shifted out completely."""
    cap = obs.shape[0]
    first = rows[0]
    stack = None
    out = {}
    for r in range(first - (k - 1), rows[-1] + 1):
        frame = obs[_row(r, cap), b]
        new_episode = (stack is None) or bool(done[_row(r - 1, cap), b])
        if new_episode:
            pad = frame if pad_mode == PAD_REPEAT else np.zeros_like(frame)
            stack = [pad] * (k - 1) + [frame]
        else:
            stack = stack[1:] + [frame]
        if r >= first:
            out[r] = np.stack(stack, axis=0)
    return [out[r] for r in rows]


def window_valid_transition(row, cap, cursor, size, k, n):
    """Rows row-k+1 .. row+n all stored (§8c #2, #14)."""
    age = (cursor - 1 - row) % cap
    return n <= age <= size - k


def window_valid_sequence(row0, cap, cursor, size, k, L):
    """Rows row0-max(k-1,1) .. row0+L-1 all stored (§8c #16)."""
    age = (cursor - 1 - row0) % cap
    return (L - 1) <= age and age + max(k - 1, 1) <= size - 1


def gather_transitions(idx, B, obs, act, rew, done, k, n, gamma, pad_mode=PAD_REPEAT, v_term=None):
    """DQN / Mujoco transition gather.  v_term [cap, B] (optional):
    terminal values of time-limit rows (done == 2), bootstrapped by the n-step return (R34).

    obs [cap, B, *item], act [cap, B, *a], rew [cap, B] f32, done [cap, B] u8.
    Returns dict: obs [n_s, k, *item], next_obs [n_s, k, *item], act [n_s, *a],
    ret float64 [n_s] (n-step return R^n), done_n uint8 [n_s].  idx < 0 -> skipped
    (left zero).
    """
    cap = obs.shape[0]
    ns = len(idx)
    o_obs = np.zeros((ns, k) + obs.shape[2:], obs.dtype)
    o_next = np.zeros_like(o_obs)
    o_act = np.zeros((ns,) + act.shape[2:], act.dtype)
    o_ret = np.zeros(ns, np.float64)
    o_dn = np.zeros(ns, np.uint8)
    for s, leaf in enumerate(idx):
        leaf = int(leaf)
        if leaf < 0:
            continue
        r, b = divmod(leaf, B)
        o_obs[s] = wrapper_stacks(obs, done, b, [r], k, pad_mode)[0]
        o_next[s] = wrapper_stacks(obs, done, b, [r + n], k, pad_mode)[0]
        o_act[s] = act[r, b]
        rows = [_row(r + i, cap) for i in range(n)]
        R, dn = _ret.nstep_return(rew[rows, b][:, None], done[rows, b][:, None], n, gamma,
                                  v_term=None if v_term is None else v_term[rows, b][:, None])
        o_ret[s] = R[0, 0]
        o_dn[s] = dn[0, 0]
    return dict(obs=o_obs, next_obs=o_next, act=o_act, ret=o_ret, done_n=o_dn)


def gather_sequences(idx, B, obs, act, rew, done, rnn, k, L, period, pad_mode=PAD_REPEAT,
                     stacked=True):
    """R2D2 sequence gather (S:631-639, P:123 fn).

    Leaf = block * B + b; the sequence starts at ring row row0 = block * period
    and spans L rows (burn-in + train + bootstrap tail, §8c #15).
    rnn [cap/period, B, parts, H] is the stored recurrent state (§8c #16, #19).
    Returns dict (time-major, [L, n_s, ...]):
      obs       [L, n_s, k, *item] (stacked) or [L+k-1, n_s, *item] raw rows (unique)
      act, rew, done        rows row0 .. row0+L-1
      prev_act, prev_rew    rows row0-1 .. row0+L-2, zero on an episode's first row (§8c #18)
      rnn       [parts, n_s, H]
    """
    cap = obs.shape[0]
    ns = len(idx)
    item = obs.shape[2:]
    if stacked:
        o_obs = np.zeros((L, ns, k) + item, obs.dtype)
    else:
        o_obs = np.zeros((L + k - 1, ns) + item, obs.dtype)
    o_act = np.zeros((L, ns) + act.shape[2:], act.dtype)
    o_pact = np.zeros_like(o_act)
    o_rew = np.zeros((L, ns), np.float32)
    o_prew = np.zeros((L, ns), np.float32)
    o_done = np.zeros((L, ns), np.uint8)
    parts, H = rnn.shape[2], rnn.shape[3]
    o_rnn = np.zeros((parts, ns, H), rnn.dtype)
    for s, leaf in enumerate(idx):
        leaf = int(leaf)
        if leaf < 0:
            continue
        blk, b = divmod(leaf, B)
        row0 = blk * period
        rows = list(range(row0, row0 + L))
        if stacked:
            st = wrapper_stacks(obs, done, b, rows, k, pad_mode)
            for j in range(L):
                o_obs[j, s] = st[j]
        else:
            for j in range(L + k - 1):
                o_obs[j, s] = obs[_row(row0 - (k - 1) + j, cap), b]
        for j, r in enumerate(rows):
            rr = _row(r, cap)
            o_act[j, s] = act[rr, b]
            o_rew[j, s] = rew[rr, b]
            o_done[j, s] = done[rr, b]
            prev = _row(r - 1, cap)
            if not done[prev, b]:                 # row r continues the episode of row r-1
                o_pact[j, s] = act[prev, b]
                o_prew[j, s] = rew[prev, b]
        for p in range(parts):
            o_rnn[p, s] = rnn[blk, b, p]
    return dict(obs=o_obs, act=o_act, prev_act=o_pact, rew=o_rew, prev_rew=o_prew,
                done=o_done, rnn=o_rnn)
