"""Pins for oracle.gather against a naive buffer that stored full k-stacks while
the episodes were played, SPEC's worked examples, and the
closed-form padded row index stack[j] = frame(max(t-k+1+j, s(t)))."""
import numpy as np
import pytest

from oracle import gather as G
from oracle import returns as R
from synth import rng


def play_history(seed, Ttot, B, item=(6,), k=4, p_done=0.15, pad_mode=G.PAD_REPEAT):
    """Play episodes for Ttot steps in B columns; keep frames, dones and the
    full stacks a wrapper would have produced at every absolute step."""
    g = rng(seed)
    frames = g.integers(0, 256, size=(Ttot, B) + item, dtype=np.uint8)
    done = (g.random((Ttot, B)) < p_done).astype(np.uint8)
    stacks = np.zeros((Ttot, B, k) + item, np.uint8)
    for b in range(B):
        st = None
        for t in range(Ttot):
            f = frames[t, b]
            if t == 0 or done[t - 1, b]:
                pad = f if pad_mode == G.PAD_REPEAT else np.zeros_like(f)
                st = [pad] * (k - 1) + [f]
            else:
                st = st[1:] + [f]
            stacks[t, b] = np.stack(st)
    return frames, done, stacks


def to_ring(x, cap, Ttot):
    ring = np.zeros((cap,) + x.shape[1:], x.dtype)
    for t in range(max(0, Ttot - cap), Ttot):
        ring[t % cap] = x[t]
    return ring


@pytest.mark.parametrize("pad_mode", [G.PAD_REPEAT, G.PAD_ZERO])
def test_transition_frames_equal_naive_full_stack(pad_mode):
    # S:649 / S:981: random reconstructions bit-equal a naive full-stack buffer
    k, n, cap, B, Ttot = 4, 3, 50, 3, 137
    frames, done, stacks = play_history(1, Ttot, B, k=k, pad_mode=pad_mode)
    obs = to_ring(frames, cap, Ttot)
    dn = to_ring(done, cap, Ttot)
    rew = np.zeros((cap, B), np.float32)
    act = np.zeros((cap, B), np.int64)
    cursor, size = Ttot % cap, cap
    g = rng(2)
    checked = 0
    for _ in range(3000):
        row, b = int(g.integers(0, cap)), int(g.integers(0, B))
        if not G.window_valid_transition(row, cap, cursor, size, k, n):
            continue
        age = (cursor - 1 - row) % cap
        t_abs = Ttot - 1 - age
        out = G.gather_transitions([row * B + b], B, obs, act, rew, dn, k, n, 0.99, pad_mode)
        assert np.array_equal(out["obs"][0], stacks[t_abs, b])
        assert np.array_equal(out["next_obs"][0], stacks[t_abs + n, b])
        checked += 1
    assert checked > 2000


def test_closed_form_padded_index():
    k, cap, B, Ttot = 4, 64, 4, 64
    frames, done, stacks = play_history(3, Ttot, B, k=k, p_done=0.3)
    for b in range(B):
        for t in range(k - 1, Ttot):
            s = t
            while s > t - (k - 1) and not done[s - 1, b]:
                s -= 1
            ref = np.stack([frames[max(t - k + 1 + j, s), b] for j in range(k)])
            got = G.wrapper_stacks(frames, done, b, [t], k, G.PAD_REPEAT)[0]
            assert np.array_equal(got, ref)


def test_episode_start_four_copies():
    # t = 0 of an episode -> four copies of frame 0
    frames = np.arange(10 * 1 * 2, dtype=np.uint8).reshape(10, 1, 2)
    done = np.zeros((10, 1), np.uint8)
    done[4, 0] = 1                                  # row 5 starts an episode
    st = G.wrapper_stacks(frames, done, 0, [5], 4, G.PAD_REPEAT)[0]
    assert all(np.array_equal(st[j], frames[5, 0]) for j in range(4))
    st = G.wrapper_stacks(frames, done, 0, [6], 4, G.PAD_ZERO)[0]
    assert not st[0].any() and not st[1].any()
    assert np.array_equal(st[2], frames[5, 0]) and np.array_equal(st[3], frames[6, 0])


def test_frame_dedup_memory_arithmetic():
    # k=4, T=100 per column -> 103 unique frame slots vs 400 naive
    k, T = 4, 100
    assert T + k - 1 == 103 and T * k == 400


def test_transition_scalars_and_nstep():
    k, n, cap, B = 4, 3, 40, 2
    g = rng(5)
    obs = g.integers(0, 256, (cap, B, 8), dtype=np.uint8)
    act = g.integers(0, 18, (cap, B)).astype(np.int64)
    rew = g.normal(size=(cap, B)).astype(np.float32)
    dn = (g.random((cap, B)) < 0.2).astype(np.uint8)
    idx = [5 * B + 1, 30 * B + 0, 38 * B + 1]        # last one wraps the ring for n-step
    out = G.gather_transitions(idx, B, obs, act, rew, dn, k, n, 0.99)
    for s, leaf in enumerate(idx):
        r, b = divmod(leaf, B)
        rows = [(r + i) % cap for i in range(n)]
        tot, disc, d = 0.0, 1.0, 0
        for rr in rows:
            tot += disc * float(rew[rr, b])
            if dn[rr, b]:
                d = 1
                break
            disc *= 0.99
        assert abs(out["ret"][s] - tot) < 1e-12 and out["done_n"][s] == d
        assert out["act"][s] == act[r, b]


def test_sequences_aligned_and_prev_fields():
    # m=40, warmup 40, train 80 -> starts are multiples of 40; slice 120
    k, cap, B, period, L = 4, 400, 2, 40, 120
    g = rng(6)
    obs = g.integers(0, 256, (cap, B, 4), dtype=np.uint8)
    act = g.integers(1, 18, (cap, B)).astype(np.int64)
    rew = g.normal(size=(cap, B)).astype(np.float32) + 5.0
    dn = (g.random((cap, B)) < 0.05).astype(np.uint8)
    rnn = g.normal(size=(cap // period, B, 2, 3)).astype(np.float32)
    idx = [2 * B + 1, 5 * B + 0]
    out = G.gather_sequences(idx, B, obs, act, rew, dn, rnn, k, L, period)
    assert out["obs"].shape == (L, 2, k, 4)
    for s, leaf in enumerate(idx):
        blk, b = divmod(leaf, B)
        row0 = blk * period
        assert row0 % 40 == 0
        assert np.array_equal(out["rnn"][:, s], rnn[blk, b])
        for j in range(L):
            r = (row0 + j) % cap
            assert out["act"][j, s] == act[r, b] and out["done"][j, s] == dn[r, b]
            prev = (r - 1) % cap
            if dn[prev, b]:
                assert out["prev_act"][j, s] == 0 and out["prev_rew"][j, s] == 0
            else:
                assert out["prev_act"][j, s] == act[prev, b] and out["prev_rew"][j, s] == rew[prev, b]
        st = G.wrapper_stacks(obs, dn, b, [(row0 + L - 1)], k, G.PAD_REPEAT)[0]
        assert np.array_equal(out["obs"][L - 1, s], st)
    uniq = G.gather_sequences(idx, B, obs, act, rew, dn, rnn, k, L, period, stacked=False)
    assert uniq["obs"].shape == (L + k - 1, 2, 4)
    blk, b = divmod(idx[0], B)
    assert np.array_equal(uniq["obs"][0, 0], obs[blk * period - 3, b])


def test_window_validity():
    cap = 100
    # cursor 10, size 100: newest row 9, oldest row 10
    assert not G.window_valid_transition(9, cap, 10, 100, 4, 3)     # needs rows 10..12: future
    assert G.window_valid_transition(6, cap, 10, 100, 4, 3)
    assert not G.window_valid_transition(12, cap, 10, 100, 4, 3)    # history crosses cursor
    assert G.window_valid_transition(13, cap, 10, 100, 4, 3)
    assert G.window_valid_sequence(40, 400, 0, 400, 4, 125)
    assert not G.window_valid_sequence(0, 400, 0, 400, 4, 125)
