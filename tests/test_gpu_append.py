"""GPU parity for ring append + validity maintenance (§8a a12, §8f NEXT-2): batches are
appended from pinned host memory; after every append the ring equals the host oracle ring,
every tree leaf is max-seen exactly while its window is valid (oracle window_valid_*,
§8c #2, #16) and 0 otherwise (or keeps its updated priority), internal nodes are exact
range sums, and sequences sampled from the maintained tree gather bit-exactly."""
import numpy as np
import pytest

from oracle import gather as OG
from oracle import philox as OP
from oracle import sumtree as OS
from synth import rng, td_abs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def H(t):
    return t.cpu().numpy()


def _pinned(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()


def _check_tree(tree, expected):
    leaves = [int(x) for x in H(tree.leaves)]
    assert leaves == expected
    W = tree.fanout
    pref = np.concatenate([[0], np.cumsum(np.array(expected, dtype=object))])
    for l in range(tree.depth):
        span = W ** (tree.depth - l)
        lvl = H(tree.level(l))
        for j in range(len(lvl)):
            lo, hi = min(j * span, tree.n_leaves), min((j + 1) * span, tree.n_leaves)
            assert int(lvl[j]) == int(pref[hi] - pref[lo]), (l, j)


@pytest.mark.parametrize("kind", ["sequence", "transition"])
def test_append_validity_sample_gather(rpl, kind):
    import torch
    cap, B, k, period, L, n_step = 240, 3, 4, 20, 45, 3
    H_, W_ = 8, 16
    dev = torch.device("cuda")
    ring = rpl.GatherRing(obs=torch.zeros((cap, B, H_, W_), dtype=torch.uint8, device=dev),
                          act=torch.zeros((cap, B), dtype=torch.int64, device=dev),
                          rew=torch.zeros((cap, B), dtype=torch.float32, device=dev),
                          done=torch.zeros((cap, B), dtype=torch.uint8, device=dev), cursor=0, size=0,
                          rnn=torch.zeros((cap // period, B, 2, 4), dtype=torch.float32, device=dev))
    h_obs = np.zeros((cap, B, H_, W_), np.uint8)
    h_act = np.zeros((cap, B), np.int64)
    h_rew = np.zeros((cap, B), np.float32)
    h_done = np.zeros((cap, B), np.uint8)
    h_rnn = np.zeros((cap // period, B, 2, 4), np.float32)
    units = cap // period if kind == "sequence" else cap
    N = units * B
    tree = rpl.SumTree(N, 32)
    maxseen = 1 << 32
    expected = [0] * N
    g = rng(17 if kind == "sequence" else 18)

    def valid(unit, cursor, size):
        if size == 0:
            return False
        if kind == "sequence":
            return OG.window_valid_sequence(unit * period, cap, cursor, size, k, L)
        return OG.window_valid_transition(unit, cap, cursor, size, k, n_step)

    for step, T_b in enumerate([37, 40, 40, 13, 40, 40, 40, 40, 29, 40]):
        c0, s0 = ring.cursor, ring.size
        obs = g.integers(0, 256, (T_b, B, H_, W_), dtype=np.uint8)
        act = g.integers(0, 18, (T_b, B)).astype(np.int64)
        rew = g.normal(size=(T_b, B)).astype(np.float32)
        done = (g.random((T_b, B)) < 0.05).astype(np.uint8)
        starts = [t for t in range(T_b) if (c0 + t) % period == 0]
        rnn = g.normal(size=(len(starts), B, 2, 4)).astype(np.float32)
        old = rpl.ring_append(ring, obs=_pinned(obs), act=_pinned(act), rew=_pinned(rew), done=_pinned(done),
                              rnn=_pinned(rnn) if starts else None, period=period)
        assert old == (c0, s0)
        rows = [(c0 + t) % cap for t in range(T_b)]
        h_obs[rows], h_act[rows], h_rew[rows], h_done[rows] = obs, act, rew, done
        for j, t in enumerate(starts):
            h_rnn[((c0 + t) % cap) // period] = rnn[j]
        tree.validity(kind, cap, B, k, c0, s0, ring.cursor, ring.size, n_step=n_step, seq_len=L, period=period)
        for leaf in range(N):
            v0, v1 = valid(leaf // B, c0, s0), valid(leaf // B, ring.cursor, ring.size)
            if v0 != v1:
                expected[leaf] = maxseen if v1 else 0
        torch.cuda.synchronize()
        assert np.array_equal(H(ring.obs), h_obs) and np.array_equal(H(ring.act), h_act)
        assert np.array_equal(H(ring.rew), h_rew) and np.array_equal(H(ring.done), h_done)
        assert np.array_equal(H(ring.rnn), h_rnn)
        _check_tree(tree, expected)
        # a learner update on some valid leaves: later appends must keep those priorities
        live = [i for i in range(N) if expected[i] > 0]
        if live and step % 3 == 1:
            pick = np.array(g.choice(live, min(5, len(live)), replace=False), np.int64)
            td = td_abs(g, pick.size)
            tree.update(torch.from_numpy(pick).cuda(), torch.from_numpy(td).cuda(), 0.9)
            orc = OS.SumTreeOracle(N)
            orc.update([int(x) for x in pick], [float(x) for x in td], 0.9)
            for i in pick:
                expected[int(i)] = orc.q[int(i)]
            maxseen = max(maxseen, max(orc.q[int(i)] for i in pick))
            _check_tree(tree, expected)
    # sample from the maintained tree and gather: bit-exact against the oracle ring
    idx, q, _, _ = tree.sample(16, draws=torch.from_numpy(
        np.array([x - (1 << 64) if x >= (1 << 63) else x for x in OP.draws_u64(5, 0, 16)], np.int64)).cuda())
    idx_h = H(idx)
    assert all(expected[int(i)] > 0 for i in idx_h)
    if kind == "sequence":
        out = rpl.gather(ring, idx, kind="sequence", k=k, seq_len=L, period=period)
        ref = OG.gather_sequences(idx_h, B, h_obs, h_act, h_rew, h_done, h_rnn, k, L, period)
        for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
            assert np.array_equal(H(out[name]), ref[name]), name
    else:
        out = rpl.gather(ring, idx, kind="transition", k=k, n_step=n_step, gamma=0.99)
        ref = OG.gather_transitions(idx_h, B, h_obs, h_act, h_rew, h_done, k, n_step, 0.99)
        assert np.array_equal(H(out["obs"]), ref["obs"]) and np.array_equal(H(out["next_obs"]), ref["next_obs"])
