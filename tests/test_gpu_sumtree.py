"""GPU parity: int64 sum tree (rpl_sumtree_*), priority transform and IS weights
vs the oracle.  Tree values, sampled indices and q are compared BIT-EXACTLY;
IS weights within 1e-5 relative."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import gather as OG
from oracle import philox as OP
from oracle import priority as OPR
from oracle import sumtree as OS
from synth import rng, td_abs
from tests._tol import check_rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def T_(x, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    return (t.to(dtype) if dtype is not None else t).cuda()


def H(t):
    return t.cpu().numpy()


def as_i64(u64_list):
    return np.array([x - (1 << 64) if x >= (1 << 63) else x for x in u64_list], np.int64)


def check_tree_consistent(tree, oracle):
    """Leaves bit-equal; every internal node equals the oracle's exact range sum."""
    leaves = [int(x) for x in H(tree.leaves)]
    assert leaves == oracle.q
    W = tree.fanout
    for l in range(tree.depth):
        span = W ** (tree.depth - l)
        lvl = H(tree.level(l))
        pref = [0] + list(itertools.accumulate(oracle.q))
        for j in range(len(lvl)):
            lo, hi = min(j * span, tree.n_leaves), min((j + 1) * span, tree.n_leaves)
            assert int(lvl[j]) == pref[hi] - pref[lo], (l, j)
    hdr = H(tree.header)
    assert int(hdr[0]) == oracle.max_seen
    assert int(hdr[1]) == 0  # sampler ticket reset


def test_layout(rpl):
    for n, W, depth in [(1, 32, 1), (16, 32, 1), (33, 32, 2), (25600, 32, 3), (1 << 20, 32, 4), (1 << 17, 32, 4),
                        (16, 2, 4), (1000, 4, 5)]:
        t = rpl.SumTree(n, W)
        assert t.depth == depth
        assert t.q_cap == OPR.q_cap(n)
        assert int(t.layout.level_len[0]) == 1
        assert int(t.layout.level_len[depth]) >= n


def test_toy_golden(rpl):
    import torch
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "toy.json")))
    c, I = g["config"], g["inputs"]
    tree = rpl.SumTree(16, 32, c["frac_bits"])
    tree.update(T_(np.arange(16, dtype=np.int64)), T_(np.array(I["td_init"], np.float32)), c["alpha"], c["eps_p"])
    assert [int(x) for x in H(tree.leaves)] == [int(x) for x in g["tree_q_init"]]
    tree.update(T_(np.array(I["upd_idx"], np.int64)), T_(np.array(I["upd_td"], np.float32)), c["alpha"], c["eps_p"])
    assert [int(x) for x in H(tree.leaves)] == [int(x) for x in g["tree_q"]]
    assert int(H(tree.total())[0]) == int(g["tree_total"])
    assert int(H(tree.header)[0]) == int(g["max_seen"])
    draws = T_(as_i64([int(x) for x in I["draws"]]))
    idx, q, qmin, w = tree.sample(4, draws=draws, beta=c["beta"])
    assert list(H(idx)) == g["sample_idx"]
    assert [int(x) for x in H(q)] == [int(x) for x in g["sample_q"]]
    assert int(H(qmin)[0]) == int(g["sample_qmin"])
    check_rel(H(w), g["is_weights"], what="toy IS weights")
    # the same draws from the in-kernel Philox stream (draws=NULL)
    idx2, q2, _, _ = tree.sample(4, draws=None, seed=2019, offset=0)
    assert list(H(idx2)) == g["sample_idx"]
    assert int(H(tree.err)[0]) == 0


@pytest.mark.parametrize("alpha", [0.6, 0.9, 0.5, 1.0, 0.0, 0.123])
def test_priority_values_vs_oracle(rpl, alpha):
    g = rng(int(alpha * 1000) + 3)
    td = np.concatenate([td_abs(g, 3000), td_abs(g, 3000, "heavy"), [0.0, 1e-30, 1.0, 65504.0, 3.0e38]]).astype(
        np.float32)
    for force in (False, True):
        v, slow = rpl.debug_priority_values(T_(td), alpha, 1e-3, force_slow=force)
        v = H(v)
        for i in range(td.size):
            M, E = OPR.priority_value(float(td[i]), alpha, 1e-3)
            ref = np.float32(OPR.value_float(M, E))
            assert v[i] == ref, (float(td[i]), alpha, force, float(v[i]), float(ref))


def test_priority_values_near_midpoints(rpl):
    # inputs whose p^alpha lies near an fp32 rounding midpoint exercise the Ziv
    # fallback; force the slow path on a large random set too
    g = rng(44)
    td = g.uniform(0, 4, 20000).astype(np.float32)
    v_fast, slow = rpl.debug_priority_values(T_(td), 0.6, 1e-3, force_slow=False)
    v_slow, _ = rpl.debug_priority_values(T_(td), 0.6, 1e-3, force_slow=True)
    assert np.array_equal(H(v_fast), H(v_slow))


@pytest.fixture(params=[1, 0])
def upd_multi(rpl, request):
    # 1: batches of n <= 1024 on the multi-CTA update kernel (default); 0: single-CTA kernels
    assert rpl._lib.lib.rpl_debug_set_upd_multi(request.param) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_upd_multi(1)


@pytest.fixture(params=[1, 0])
def tree_stage(rpl, request):
    # 1: the sampler stages the top levels in shared memory (all of a small tree; root +
    # 3 levels of 70000 leaves); 0: every level from global memory
    assert rpl._lib.lib.rpl_debug_set_tree_stage(request.param) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_tree_stage(1)


@pytest.mark.parametrize("n_leaves,W", [(16, 32), (100, 4), (1000, 32), (5000, 16), (70000, 32)])
def test_random_updates_vs_oracle(rpl, n_leaves, W, tree_stage, upd_multi):
    g = rng(n_leaves + W)
    tree = rpl.SumTree(n_leaves, W)
    orc = OS.SumTreeOracle(n_leaves)
    for step in range(6):
        n = int(g.integers(1, 3000))
        idx = g.integers(0, n_leaves, n).astype(np.int64)
        if step % 2 == 1:  # duplicate-heavy batch
            idx = g.integers(0, max(1, n_leaves // 50), n).astype(np.int64)
        td = td_abs(g, n, "heavy" if step % 3 == 2 else "normal")
        tree.update(T_(idx), T_(td), 0.6, 1e-3)
        orc.update(list(idx), [float(x) for x in td], 0.6, 1e-3)
    check_tree_consistent(tree, orc)
    assert int(H(tree.err)[0]) == 0
    # sampling, both draw sources
    for n, seed in [(1, 1), (32, 2), (512, 3), (4096, 4)]:
        draws = OP.draws_u64(seed, 17, n)
        idx, q, qmin, w = tree.sample(n, draws=T_(as_i64(draws)), beta=0.4)
        oi, oq, oqmin = orc.sample(n, draws)
        assert list(H(idx)) == oi
        assert [int(x) for x in H(q)] == oq
        assert int(H(qmin)[0]) == oqmin
        check_rel(H(w), OS.is_weights(oq, orc.total(), n_leaves, 0.4), what="w")
        idx2, q2, _, _ = tree.sample(n, seed=seed, offset=17)
        assert list(H(idx2)) == oi


def test_set_q_maxseen_and_find(rpl, upd_multi):
    g = rng(3)
    n_leaves = 3000
    tree = rpl.SumTree(n_leaves, 32)
    orc = OS.SumTreeOracle(n_leaves)
    idx = g.integers(0, n_leaves, 2000).astype(np.int64)
    tree.set_q(T_(idx))                      # new samples get max-seen
    orc.set_q(list(idx))
    q = g.integers(0, 1 << 40, 500).astype(np.int64)
    i2 = g.integers(0, n_leaves, 500).astype(np.int64)
    tree.set_q(T_(i2), T_(q))
    orc.set_q(list(i2), list(q))
    td = td_abs(g, 100)
    tree.update(T_(idx[:100]), T_(td), 0.6)
    orc.update(list(idx[:100]), [float(x) for x in td], 0.6)
    check_tree_consistent(tree, orc)
    Q = orc.total()
    prefixes = np.array(sorted(set([0, Q - 1] + list(g.integers(0, Q, 300)))), np.int64)
    got = H(tree.find(T_(prefixes)))
    assert [int(x) for x in got] == [orc.find(int(p)) for p in prefixes]
    # zero leaves are never returned
    assert all(orc.q[int(i)] > 0 for i in got)


def test_fanout_independence(rpl):
    g = rng(8)
    n_leaves = 4096
    td = td_abs(g, n_leaves)
    draws = T_(as_i64(OP.draws_u64(5, 0, 256)))
    res = []
    for W in (2, 4, 8, 16, 32):
        t = rpl.SumTree(n_leaves, W)
        t.update(T_(np.arange(n_leaves, dtype=np.int64)), T_(td), 0.6)
        res.append(list(H(t.sample(256, draws=draws)[0])))
    assert all(r == res[0] for r in res)


def test_empty_and_bad_index(rpl):
    import torch
    t = rpl.SumTree(64, 32)
    idx, q, qmin, w = t.sample(5, seed=1, beta=0.4)
    assert list(H(idx)) == [-1] * 5
    assert int(H(t.err)[0]) & 4
    t.err.zero_()
    t.update(T_(np.array([3, 64, -1, 5], np.int64)), T_(np.ones(4, np.float32)), 0.6)
    assert int(H(t.err)[0]) & 1
    orc = OS.SumTreeOracle(64)
    orc.update([3, 64, -1, 5], [1.0] * 4, 0.6)
    assert [int(x) for x in H(t.leaves)] == orc.q


def test_rebuild(rpl):
    g = rng(12)
    t = rpl.SumTree(20000, 32)
    t.update(T_(np.arange(20000, dtype=np.int64)), T_(td_abs(g, 20000)), 0.9)
    ref = H(t.storage).copy()
    for l in range(t.depth):
        t.level(l).zero_()
    t.rebuild()
    assert np.array_equal(H(t.storage), ref)


def test_sharded_equals_concatenated(rpl):
    import torch
    g = rng(21)
    G, n_local = 4, 3000
    shards, orcs = [], []
    for s in range(G):
        t = rpl.SumTree(n_local, 32)
        td = td_abs(g, n_local)
        t.update(T_(np.arange(n_local, dtype=np.int64)), T_(td), 0.9)
        o = OS.SumTreeOracle(n_local)
        o.update(list(range(n_local)), [float(x) for x in td], 0.9)
        shards.append(t)
        orcs.append(o)
    totals = torch.cat([t.total() for t in shards])
    n = 256
    draws = OP.draws_u64(9, 0, n)
    ref_idx, ref_q, ref_qmin = OS.sharded_sample(orcs, n, draws)
    got = np.full(n, -1, np.int64)
    qmins = []
    for rank, t in enumerate(shards):
        idx, q, qmin = t.sample_sharded(rank, G, totals, n, draws=T_(as_i64(draws)))
        idx = H(idx)
        own = idx >= 0
        assert np.all(got[own] == -1)
        got[own] = idx[own]
        qmins.append(int(H(qmin)[0]))
        # the owned draws are one contiguous run of strata
        pos = np.nonzero(own)[0]
        if pos.size:
            assert pos[-1] - pos[0] + 1 == pos.size
    assert list(got) == ref_idx
    assert min(qmins) == ref_qmin


def _oracle_q_parallel(td, alpha, eps_p, F, N):
    """oracle.priority.priority_q for every entry (mpmath, ~40 us each), spread over the
    host's cores; the oracle function itself, unchanged."""
    import functools
    import multiprocessing as mp
    fn = functools.partial(OPR.priority_q, alpha=alpha, eps_p=eps_p, frac_bits=F, n_leaves=N)
    vals = [float(x) for x in td]
    procs = max(1, min(32, os.cpu_count() or 1))
    with mp.get_context("spawn").Pool(procs) as pool:
        return pool.map(fn, vals, chunksize=max(1, len(vals) // (procs * 8)))


def test_dqn_full_size_tree(rpl):
    # BASELINE.json configs[2]: 1M transitions (2^20 leaves), alpha 0.6, beta 0.4, batch 512.
    # EVERY leaf of the full-size update is compared with the oracle's transform (no GPU value
    # ever enters the oracle), every internal node with the oracle's exact range sum, then
    # three sample / update rounds are compared index for index.
    g = rng(31)
    N = 1 << 20
    t = rpl.SumTree(N, 32)
    orc = OS.SumTreeOracle(N)
    td = td_abs(g, N)
    t.update(T_(np.arange(N, dtype=np.int64)), T_(td), 0.6)
    orc.q = _oracle_q_parallel(td, 0.6, 1e-3, 32, N)
    orc.max_seen = max(orc.max_seen, max(orc.q))
    check_tree_consistent(t, orc)
    for step in range(3):
        draws = OP.draws_u64(100 + step, 0, 512)
        idx, q, qmin, w = t.sample(512, draws=T_(as_i64(draws)), beta=0.4)
        oi, oq, oqmin = orc.sample(512, draws)
        assert list(H(idx)) == oi and [int(x) for x in H(q)] == oq and int(H(qmin)[0]) == oqmin
        check_rel(H(w), OS.is_weights(oq, orc.total(), N, 0.4), what="dqn w")
        new_td = td_abs(g, 512)
        t.update(idx, T_(new_td), 0.6)
        orc.update(oi, [float(x) for x in new_td], 0.6)
    check_tree_consistent(t, orc)
    assert int(H(t.total())[0]) == orc.total()
    assert int(H(t.err)[0]) == 0


@pytest.mark.parametrize("lo,nr,cap,B,n", [(0, 1, 1, 1, 5), (41, 17, 50, 4, 1000), (3, 65530, 65536, 16, 256),
                                           (10, 4089, 4096, 256, 777)])
def test_sample_uniform_vs_oracle(rpl, lo, nr, cap, B, n):
    import torch
    from oracle import uniform as OU
    out = rpl.sample_uniform(n, seed=77, lo_row=lo, n_rows=nr, cap_T=cap, B=B, offset=5)
    assert H(out).tolist() == OU.uniform_indices(n, 77, 5, lo, nr, cap, B)
    # device stream counter: two calls draw consecutive counters and advance it by n each
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    a = rpl.sample_uniform(n, seed=3, lo_row=lo, n_rows=nr, cap_T=cap, B=B, ctr=ctr)
    b = rpl.sample_uniform(n, seed=3, lo_row=lo, n_rows=nr, cap_T=cap, B=B, ctr=ctr)
    assert int(H(ctr)[0]) == 2 * n
    assert H(a).tolist() == OU.uniform_indices(n, 3, 0, lo, nr, cap, B)
    assert H(b).tolist() == OU.uniform_indices(n, 3, n, lo, nr, cap, B)


def test_sample_uniform_errors(rpl):
    lib = rpl._lib.lib
    assert lib.rpl_sample_uniform(0, 1, 0, None, 0, 1, 1, 1, 1, None) == -1
    assert lib.rpl_sample_uniform(1, 1, 0, None, 5, 1, 4, 1, 1, None) == -1   # lo_row >= cap
    assert lib.rpl_sample_uniform(1, 1, 0, None, 0, 5, 4, 1, 1, None) == -1   # n_rows > cap


def test_stream_without_reduction_matches(rpl):
    # sample_stream with no qmin / IS weights (no grid-wide reduction) draws the same
    # strata and advances the stream exactly like the reducing call
    a = rpl.SumTree(25600, 32)
    b = rpl.SumTree(25600, 32)
    g = rng(21)
    td = T_(td_abs(g, 25600))
    ii = T_(np.arange(25600, dtype=np.int64))
    a.update(ii, td, 0.9)
    b.update(ii, td, 0.9)
    for _ in range(3):
        ia, qa, ma, wa = a.sample_stream(200, 9, beta=0.6)
        ib, qb, mb, wb = b.sample_stream(200, 9, want_qmin=False)
        assert mb is None and wb is None
        assert np.array_equal(H(ia), H(ib)) and np.array_equal(H(qa), H(qb))
    assert np.array_equal(H(a.header), H(b.header))


@pytest.mark.parametrize("mode", ["draws", "stream"])
def test_sharded_compacted(rpl, mode):
    # out_count: the owned draws move to the front in stratum order, the rest are -1 / 0;
    # the union over ranks (in rank order) equals the concatenated oracle's sample
    import torch
    g = rng(33)
    G, n_local, n = 3, 2000, 200
    shards, orcs = [], []
    for s in range(G):
        t = rpl.SumTree(n_local, 32)
        td = td_abs(g, n_local)
        t.update(T_(np.arange(n_local, dtype=np.int64)), T_(td), 0.9)
        o = OS.SumTreeOracle(n_local)
        o.update(list(range(n_local)), [float(x) for x in td], 0.9)
        shards.append(t)
        orcs.append(o)
    shards[1].update(T_(np.arange(0, n_local, 2, dtype=np.int64)),
                     T_(np.zeros(n_local // 2, np.float32)), 0.9)   # an uneven shard
    orcs[1].update(list(range(0, n_local, 2)), [0.0] * (n_local // 2), 0.9)
    totals = torch.cat([t.total() for t in shards])
    for step in range(2):
        draws = OP.draws_u64(4, step * n, n)
        ref_idx, ref_q, _ = OS.sharded_sample(orcs, n, draws)
        collected, collected_q = [], []
        for rank, t in enumerate(shards):
            cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
            if mode == "draws":
                idx, q, _ = t.sample_sharded(rank, G, totals, n, draws=T_(as_i64(draws)), count=cnt)
                full, fq, _ = t.sample_sharded(rank, G, totals, n, draws=T_(as_i64(draws)))
            else:
                full, fq, _ = t.sample_sharded(rank, G, totals, n, seed=4, use_stream=True)
                t.header[2] -= n  # rewind the stream: the compacted call must draw the same strata
                idx, q, _ = t.sample_sharded(rank, G, totals, n, seed=4, use_stream=True, count=cnt)
            m = int(H(cnt)[0])
            idx, q, full, fq = H(idx), H(q), H(full), H(fq)
            own = full >= 0
            assert m == int(own.sum())
            if m:
                assert int(H(cnt)[1]) == int(np.nonzero(own)[0][0])  # k0: global position of entry 0
            # compacted entries are LOCAL leaves (global = rank * shard_leaves + local)
            assert np.array_equal(idx[:m] + rank * n_local, full[own]) and np.array_equal(q[:m], fq[own])
            assert np.all(idx[m:] == -1) and np.all(q[m:] == 0)
            collected += (idx[:m] + rank * n_local).tolist()
            collected_q += q[:m].tolist()
        assert collected == ref_idx and collected_q == ref_q


@pytest.mark.parametrize("T_p,n,eta", [(80, 64, 0.9), (1, 5, 0.9), (7, 300, 0.0), (80, 1200, 1.0), (33, 64, 0.37),
                                        (90, 100, 0.9), (91, 100, 0.9), (200, 70, 0.5)])
def test_update_seq_vs_oracle(rpl, T_p, n, eta, upd_multi):
    # NEXT-1: R2D2 eta-mix of per-step |delta| per sequence, then the update — tree bit-exact
    import torch
    g = rng(T_p * 1000 + n)
    N = 25600
    steps = np.abs(g.lognormal(0, 2, (T_p, n))).astype(np.float32)
    steps[:, :3] = 0.0                                   # an all-zero sequence -> eps_p floor
    idx = g.integers(0, N, n).astype(np.int64)
    idx[5 % n] = idx[0]                                  # duplicate: the later column wins
    t = rpl.SumTree(N, 32)
    t.update_seq(T_(idx), T_(steps), 0.9, eta=eta)
    orc = OS.SumTreeOracle(N)
    td = [OPR.sequence_td(steps[:, k], eta) for k in range(n)]
    orc.update([int(x) for x in idx], td, 0.9)
    check_tree_consistent(t, orc)
    # == rpl_sumtree_update on the oracle's fp32 mixes
    t2 = rpl.SumTree(N, 32)
    t2.update(T_(idx), T_(np.array(td, np.float32)), 0.9)
    assert np.array_equal(H(t.storage), H(t2.storage))


def test_buffer_min_and_buffer_normalised_weights(rpl):
    # NEXT-4: rpl_sumtree_min over non-zero leaves; the gather normalises IS weights by it
    import torch
    g = rng(44)
    N = 1 << 20
    t = rpl.SumTree(N, 32)
    idx = np.unique(g.integers(0, N, 50000)).astype(np.int64)
    td = td_abs(g, idx.size)
    t.update(T_(idx), T_(td), 0.6)
    orc = OS.SumTreeOracle(N)
    orc.update([int(x) for x in idx], [float(x) for x in td], 0.6)
    m = t.min_q()
    assert int(H(m)[0]) == OS.buffer_min(orc.q)
    w = rpl.is_weights(t.leaves[torch.from_numpy(idx[:100]).cuda()].contiguous(), m, 0.4)
    ref = [(OS.buffer_min(orc.q) / orc.q[int(i)]) ** 0.4 for i in idx[:100]]
    check_rel(H(w), np.array(ref), what="buffer-normalised w")
    e = rpl.SumTree(64, 32)
    assert int(H(e.min_q())[0]) == (1 << 63) - 1


@pytest.mark.parametrize("seq", [False, True])
def test_update_live_only(rpl, seq, upd_multi):
    # RPL_UPD_LIVE_ONLY (R30): entries on zero leaves are skipped (no revival, no max-seen)
    g = rng(71)
    N = 5000
    t = rpl.SumTree(N, 32)
    orc = OS.SumTreeOracle(N)
    live = np.arange(0, N, 3, dtype=np.int64)
    td0 = td_abs(g, live.size)
    t.update(T_(live), T_(td0), 0.9)
    orc.update([int(x) for x in live], [float(x) for x in td0], 0.9)
    idx = g.integers(0, N, 700).astype(np.int64)
    if seq:
        steps = np.abs(g.lognormal(0, 3, (12, idx.size))).astype(np.float32)
        t.update_seq(T_(idx), T_(steps), 0.9, eta=0.9, live_only=True)
        td = [OPR.sequence_td(steps[:, k], 0.9) for k in range(idx.size)]
    else:
        tdv = (td_abs(g, idx.size) * 50).astype(np.float32)
        t.update(T_(idx), T_(tdv), 0.9, live_only=True)
        td = [float(x) for x in tdv]
    orc.update([int(x) for x in idx], td, 0.9, live_only=True)
    check_tree_consistent(t, orc)


@pytest.mark.parametrize("N,n,zeros", [(25600, 64, 0.2), (100, 60, 0.5), (40, 40, 0.3)])
def test_sample_unique_vs_oracle(rpl, N, n, zeros):
    # NEXT-4 (R32): distinct successive proportional draws, tree restored bit-exactly
    g = rng(N + n)
    t = rpl.SumTree(N, 32)
    orc = OS.SumTreeOracle(N)
    live = np.array([i for i in range(N) if g.random() >= zeros], np.int64)
    td = td_abs(g, live.size)
    t.update(T_(live), T_(td), 0.6)
    orc.update([int(x) for x in live], [float(x) for x in td], 0.6)
    before = H(t.storage).copy()
    idx, q = t.sample_unique(n, seed=123, offset=7)
    ref_i, ref_q = OS.sample_unique(orc.q, n, OP.draws_u64(123, 7, n))
    assert H(idx).tolist() == ref_i and H(q).tolist() == ref_q
    assert np.array_equal(H(t.storage), before)               # tree restored exactly
    got = [i for i in H(idx).tolist() if i >= 0]
    assert len(got) == len(set(got))


def test_more_strata_than_mass(rpl):
    # Q < n: empty strata take lo_k (§8c #8); zero leaves still never drawn
    import torch
    t = rpl.SumTree(5, 32, frac_bits=0)
    q = np.array([0, 2, 0, 1, 2], np.int64)
    t.set_q(T_(np.arange(5, dtype=np.int64)), T_(q))
    orc = OS.SumTreeOracle(5, 0)
    orc.q = [int(x) for x in q]
    for n in (5, 16, 33):
        draws = OP.draws_u64(31, n, n)
        idx, qq, qmin, _ = t.sample(n, draws=T_(as_i64(draws)))
        oi, oq, oqm = orc.sample(n, draws)
        assert H(idx).tolist() == oi and H(qq).tolist() == oq and int(H(qmin)[0]) == oqm
        assert all(q[i] > 0 for i in oi)


def test_gpu_frequencies_chi2_upper_tail(rpl):
    # S:653 / S:991: 1e5 stratified draws on 64 leaves follow p^alpha / sum p^alpha; stratified
    # sampling is under-dispersed, so only the upper tail is tested (§4 of SURVEY)
    import torch
    g = rng(99)
    N = 64
    t = rpl.SumTree(N, 32)
    td = (g.random(N) * 3).astype(np.float32)
    t.update(T_(np.arange(N, dtype=np.int64)), T_(td), 1.0)
    q = H(t.leaves).astype(np.float64)
    counts = np.zeros(N)
    for rep in range(20):
        idx, _, _, _ = t.sample(5000, seed=rep, offset=0)
        counts += np.bincount(H(idx), minlength=N)
    exp = counts.sum() * q / q.sum()
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    assert chi2 < 63 + 4 * np.sqrt(2 * 63)                  # far below: stratified draws
    assert (counts[q == 0] == 0).all()


def test_determinism_two_runs(rpl):
    # identical inputs -> bit-identical tree, samples and gathered batches (no float atomics)
    import torch
    from synth import make_ring

    def run():
        ring = make_ring(7, cap=400, B=4, ep_len=25.0, period=40, rnn_h=8, reward_kind="r2d2")
        dr = rpl.GatherRing(obs=T_(ring.obs), act=T_(ring.act), rew=T_(ring.rew), done=T_(ring.done),
                            cursor=ring.cursor, size=ring.size, rnn=T_(ring.rnn))
        t = rpl.SumTree(40, 32)
        t.update(T_(np.arange(40, dtype=np.int64)), T_(td_abs(rng(1), 40)), 0.9)
        outs = []
        for i in range(3):
            idx, q, _, _ = t.sample_stream(16, 5, want_qmin=False)
            idx = torch.where(idx >= 0, idx, torch.zeros_like(idx))
            o = rpl.gather(dr, idx, kind="sequence", k=4, seq_len=45, period=40, q=q, beta=0.6)
            t.update_seq(idx, T_(np.abs(rng(i).normal(size=(45, 16))).astype(np.float32)), 0.9)
            outs.append((H(idx), H(q), {k: H(v) for k, v in o.items()}))
        return outs, H(t.storage)

    a, ta = run()
    b, tb = run()
    assert np.array_equal(ta, tb)
    for (ia, qa, oa), (ib, qb, ob) in zip(a, b):
        assert np.array_equal(ia, ib) and np.array_equal(qa, qb)
        for k in oa:
            assert np.array_equal(oa[k], ob[k]), k


def test_checkpoint_resume(rpl):
    # save leaves + header, restore into a fresh tree, rebuild: identical storage and
    # identical subsequent samples (stream position included)
    import io
    import torch
    g = rng(31)
    t = rpl.SumTree(25600, 32)
    t.update(T_(np.arange(0, 25600, 2, dtype=np.int64)), T_(td_abs(g, 12800)), 0.9)
    t.sample_stream(64, 3)
    buf = io.BytesIO()
    torch.save(t.state_dict(), buf)
    buf.seek(0)
    u = rpl.SumTree(25600, 32)
    u.load_state_dict(torch.load(buf))
    assert np.array_equal(H(t.storage), H(u.storage))
    a = t.sample_stream(64, 3)
    b = u.sample_stream(64, 3)
    assert np.array_equal(H(a[0]), H(b[0])) and np.array_equal(H(a[1]), H(b[1]))


@pytest.mark.parametrize("T_p,n_upd,n,live", [(80, 64, 64, False), (0, 300, 200, False), (12, 1500, 5000, True),
                                              (80, 0, 64, False), (33, 64, 7, True)])
def test_update_sample_fused(rpl, T_p, n_upd, n, live):
    # rpl_sumtree_update_sample == update(_seq) then sample_stream (no reduction), and both
    # == the oracle: tree bit-exact, draws from the stream position the pair would use
    g = rng(T_p * 7 + n_upd + n)
    N = 25600
    a, b = rpl.SumTree(N, 32), rpl.SumTree(N, 32)
    orc = OS.SumTreeOracle(N)
    base = np.arange(0, N, 2, dtype=np.int64)
    td0 = td_abs(g, base.size)
    for t in (a, b):
        t.update(T_(base), T_(td0), 0.9)
    orc.update([int(x) for x in base], [float(x) for x in td0], 0.9)
    pos = 0
    for step in range(3):
        idx = g.integers(0, N, max(n_upd, 1)).astype(np.int64)[:n_upd]
        if T_p:
            td = np.abs(g.lognormal(0, 2, (T_p, n_upd))).astype(np.float32)
            mix = [OPR.sequence_td(td[:, k], 0.9) for k in range(n_upd)]
        else:
            td = (td_abs(g, n_upd) * 3).astype(np.float32)
            mix = [float(x) for x in td]
        if n_upd:
            ia, qa = a.update_sample(n, 11, idx=T_(idx), td=T_(td), alpha=0.9, eta=0.9, live_only=live)
            if T_p:
                b.update_seq(T_(idx), T_(td), 0.9, eta=0.9, live_only=live)
            else:
                b.update(T_(idx), T_(td), 0.9, live_only=live)
            orc.update([int(x) for x in idx], mix, 0.9, live_only=live)
        else:
            ia, qa = a.update_sample(n, 11)
        ib, qb, _, _ = b.sample_stream(n, 11, want_qmin=False)
        ri, rq, _ = orc.sample(n, OP.draws_u64(11, pos, n))
        pos += n
        assert np.array_equal(H(ia), H(ib)) and np.array_equal(H(qa), H(qb))
        assert H(ia).tolist() == list(ri) and H(qa).tolist() == list(rq)
        check_tree_consistent(a, orc)
        ha, hb = H(a.header), H(b.header)
        assert np.array_equal(ha[:4], hb[:4]) and int(ha[2]) == pos and int(ha[3]) == 0  # barrier count reset
    assert np.array_equal(H(a.storage)[:a.layout.hdr_off], H(b.storage)[:b.layout.hdr_off])


def test_update_sample_graph_replay(rpl):
    # captured in a CUDA graph, every replay advances the stream and re-arms the grid barrier
    import torch
    N = 4096
    t, r = rpl.SumTree(N, 32), rpl.SumTree(N, 32)
    g = rng(3)
    td = T_(td_abs(g, N))
    ii = T_(np.arange(N, dtype=np.int64))
    t.update(ii, td, 0.6)
    r.update(ii, td, 0.6)
    uidx = T_(g.integers(0, N, 64).astype(np.int64))
    utd = T_(np.abs(g.normal(size=(20, 64))).astype(np.float32))
    oi = torch.empty(64, dtype=torch.int64, device="cuda")
    oq = torch.empty_like(oi)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        t.update_sample(64, 5, idx=uidx, td=utd, alpha=0.6, out=(oi, oq))  # warm-up (step 0)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        t.update_sample(64, 5, idx=uidx, td=utd, alpha=0.6, out=(oi, oq))
    for step in range(4):
        if step:
            gr.replay()
        torch.cuda.synchronize()
        r.update_seq(uidx, utd, 0.6, eta=0.9)
        ri, rq, _, _ = r.sample_stream(64, 5, want_qmin=False)
        assert np.array_equal(H(oi), H(ri)) and np.array_equal(H(oq), H(rq)), step


def test_update_seq_exact_sum_order_independent(rpl):
    # Reading R26: the sequence mean uses the EXACT sum rounded once (oracle.priority.sequence_sum),
    # so the GPU must match for any order of the rows.  alpha = 1, eps_p = 0, F = 20 make the
    # leaf q = td * 2^20 exactly (td >= 8), i.e. the leaves expose td bit for bit.  Columns:
    # the order-sensitive column of test_oracle_priority (bigs first / permuted), wide-exponent
    # columns (2^-60 .. 2^24 plus zeros and subnormals: the superaccumulator path) and narrow
    # ones (the any-order fp64 fast path) — fast and slow sequences share warps.
    import torch
    g = rng(1234)
    N, T_p, n = 25600, 64, 96
    base = np.array([2.0 ** 40] * 31 + [2.0 ** 20] + [2.0 ** -10] * 32, np.float32)
    base_small = (base.astype(np.float64) / 2.0 ** 20).astype(np.float32)  # same shape, fits F=20
    cols = []
    for k in range(n):
        kind = k % 4
        if kind == 0:
            cols.append(base_small)
        elif kind == 1:
            cols.append(g.permutation(base_small))
        elif kind == 2:
            c = (2.0 ** g.uniform(-60, 24, T_p)).astype(np.float32)
            c[g.random(T_p) < 0.1] = 0.0
            c[0] = np.float32(1e-44)                      # a subnormal
            cols.append(c)
        else:
            cols.append((np.abs(g.normal(0, 1, T_p)) * 64 + 8).astype(np.float32))
    steps = np.ascontiguousarray(np.stack(cols, axis=1))
    idx = g.choice(N, n, replace=False).astype(np.int64)
    t = rpl.SumTree(N, 32, 20)
    t.update_seq(T_(idx), T_(steps), 1.0, eta=0.0, eps_p=0.0)
    orc = OS.SumTreeOracle(N, 20)
    td = [OPR.sequence_td(steps[:, k], 0.0) for k in range(n)]
    orc.update([int(x) for x in idx], td, 1.0, 0.0)
    check_tree_consistent(t, orc)
    leaves = H(t.leaves)
    for k in range(n):
        assert int(leaves[idx[k]]) == orc.q[int(idx[k])], k
    # the order-sensitive columns take the exact-sum value (a lossy order rounds one ulp lower)
    assert orc.q[int(idx[0])] == int((31 * 2.0 ** 14 + 2.0 ** -5) * 2 ** 20)
    # eta = 0.9 on the same columns plus NaN / inf columns: saturation flags, tree consistent
    steps2 = steps.copy()
    steps2[3, 2] = np.inf
    steps2[5, 6] = np.nan
    t2 = rpl.SumTree(N, 32, 20)
    t2.update_seq(T_(idx), T_(steps2), 0.9, eta=0.9, eps_p=1e-3)
    orc2 = OS.SumTreeOracle(N, 20)
    orc2.update([int(x) for x in idx], [OPR.sequence_td(steps2[:, k], 0.9) for k in range(n)], 0.9, 1e-3)
    check_tree_consistent(t2, orc2)


def _oracle_min_levels(tree, q):
    """Every internal node of the min-tree by its definition: min over the positive leaves of
    the node's range (INT64_MAX when none), padding nodes included (R29)."""
    MAX = (1 << 63) - 1
    out = []
    W, D, N = tree.fanout, tree.depth, tree.n_leaves
    for l in range(D):
        span = W ** (D - l)
        ln = int(tree.layout.level_len[l])
        lvl = []
        for j in range(ln):
            lo, hi = j * span, min((j + 1) * span, N)
            lvl.append(OS.buffer_min(q[lo:hi]) if lo < N else MAX)
        out.append(lvl)
    return out


def _check_min_tree(t, orc):
    ref = _oracle_min_levels(t, orc.q)
    for l in range(t.depth):
        assert [int(x) for x in H(t.min_level(l))] == ref[l], l
    assert int(H(t.min_root)[0]) == OS.buffer_min(orc.q)


@pytest.mark.parametrize("N,W", [(25600, 32), (3000, 4), (1, 32), (100, 2)])
def test_min_tree_maintained_by_every_writer(rpl, N, W, upd_multi):
    # NEXT-4 / R29: the min-tree beside the sum tree stays exact through update, duplicate-heavy
    # update, update_seq, set_q (explicit zeros = invalidated leaves, max-seen), the fused
    # update+sample, replay validity and rebuild; the root is the buffer-wide normaliser
    import torch
    g = rng(N + W)
    t = rpl.SumTree(N, W)
    orc = OS.SumTreeOracle(N)
    t.attach_min_tree()
    _check_min_tree(t, orc)                              # empty tree: every node INT64_MAX
    idx = g.integers(0, N, 3 * N // 2 + 1).astype(np.int64)
    td = td_abs(g, idx.size)
    t.update(T_(idx), T_(td), 0.6)
    orc.update([int(x) for x in idx], [float(x) for x in td], 0.6)
    _check_min_tree(t, orc)
    for _ in range(3):
        n = int(g.integers(1, 700))
        idx = g.integers(0, N, n).astype(np.int64)
        idx[::3] = idx[0]                                # duplicates: the last one wins
        td = (td_abs(g, n) * 10.0 ** g.uniform(-3, 3, n)).astype(np.float32)
        t.update(T_(idx), T_(td), 0.6)
        orc.update([int(x) for x in idx], [float(x) for x in td], 0.6)
        _check_min_tree(t, orc)
        z = g.integers(0, N, max(1, N // 10)).astype(np.int64)   # invalidate: q := 0
        t.set_q(T_(z), T_(np.zeros(z.size, np.int64)))
        orc.set_q([int(x) for x in z], [0] * z.size)
        _check_min_tree(t, orc)
        t.set_q(T_(z[: z.size // 2]))                    # re-validate at max-seen
        orc.set_q([int(x) for x in z[: z.size // 2]])
        _check_min_tree(t, orc)
    steps = np.abs(g.normal(size=(16, 40))).astype(np.float32)
    sidx = g.integers(0, N, 40).astype(np.int64)
    t.update_seq(T_(sidx), T_(steps), 0.9, eta=0.9)
    orc.update([int(x) for x in sidx], [OPR.sequence_td(steps[:, k], 0.9) for k in range(40)], 0.9)
    _check_min_tree(t, orc)
    fi = g.integers(0, N, 32).astype(np.int64)
    ftd = td_abs(g, 32)
    t.update_sample(64, 9, idx=T_(fi), td=T_(ftd), alpha=0.6)
    orc.update([int(x) for x in fi], [float(x) for x in ftd], 0.6)
    torch.cuda.synchronize()
    _check_min_tree(t, orc)
    # a corrupted min-tree is restored by rebuild (resume path)
    t.mins.fill_(5)
    t.rebuild()
    _check_min_tree(t, orc)


def test_min_tree_validity_and_buffer_weights(rpl):
    # appends change leaf validity (rpl_replay_validity): the min-tree follows; IS weights
    # normalised by its root equal the PER buffer-wide formula (N P_i)^-beta / max_j
    import torch
    cap, B, k, n_step = 64, 16, 4, 3
    N = cap * B
    t = rpl.SumTree(N, 32)
    orc = OS.SumTreeOracle(N)
    t.attach_min_tree()
    g = rng(99)
    for c_old, s_old, c_new, s_new in [(0, 0, 20, 20), (20, 20, 50, 50), (50, 50, 10, 64), (10, 64, 40, 64)]:
        t.validity("transition", cap, B, k, c_old, s_old, c_new, s_new, n_step=n_step)
        for row in range(cap):
            v0 = OG.window_valid_transition(row, cap, c_old, s_old, k, n_step) if s_old else False
            v1 = OG.window_valid_transition(row, cap, c_new, s_new, k, n_step) if s_new else False
            if v0 != v1:
                leaves = [row * B + b for b in range(B)]
                if v1:
                    orc.set_q(leaves)
                else:
                    orc.set_q(leaves, [0] * B)
        _check_min_tree(t, orc)
        live = [i for i, x in enumerate(orc.q) if x > 0]
        if live:  # fresh priorities on the live leaves, then buffer-normalised weights
            pick = np.array(g.choice(live, min(200, len(live)), replace=False), np.int64)
            td = td_abs(g, pick.size)
            t.update(T_(pick), T_(td), 0.6)
            orc.update([int(x) for x in pick], [float(x) for x in td], 0.6)
            _check_min_tree(t, orc)
            qs = [orc.q[int(i)] for i in pick[:50]]
            w = rpl.is_weights(T_(np.array(qs, np.int64)), t.min_root, 0.4)
            Q, qmin = orc.total(), OS.buffer_min(orc.q)
            ref = [((N * qi / Q) ** -0.4) / ((N * qmin / Q) ** -0.4) for qi in qs]
            check_rel(H(w), ref, what="buffer-normalised w")


def test_min_tree_sharded_exchanges(rpl):
    # the buffer min travels with the K5 total: (a) peer boards (header word 6 of every rank's
    # tree), (b) the {total, min} all-gather record and rpl_sumtree_sample_sharded_pairs; the
    # global min equals the oracle's over all shards and the sample equals the concatenated one
    import torch
    from paper_1909_01500_b200.shard import PeerBoards
    G, n_local, n, seed = 3, 2000, 48, 11
    g = rng(123)
    trees, orcs = [], []
    for r in range(G):
        t = rpl.SumTree(n_local, 32)
        t.attach_min_tree()
        o = OS.SumTreeOracle(n_local)
        idx = g.integers(0, n_local, 1500).astype(np.int64)
        td = (td_abs(g, 1500) * (1 + 3 * r)).astype(np.float32)
        t.update(T_(idx), T_(td), 0.9)
        o.update([int(x) for x in idx], [float(x) for x in td], 0.9)
        trees.append(t)
        orcs.append(o)
    gmin = min(OS.buffer_min(o.q) for o in orcs)
    # (a) peer boards, all ranks' samplers concurrently on their own streams
    boards = [torch.zeros(6 * G, dtype=torch.int64, device="cuda") for _ in range(G)]
    ptrs = PeerBoards.local(boards)
    streams = [torch.cuda.Stream() for _ in range(G)]
    counts = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()
    for r in range(G):
        with torch.cuda.stream(streams[r]):
            trees[r].sample_sharded_p2p(r, G, ptrs, n, seed, counts[r])
    torch.cuda.synchronize()
    for r in range(G):
        assert int(H(trees[r].header)[6]) == gmin
        assert H(boards[r])[4 * G::2].tolist() == [OS.buffer_min(o.q) for o in orcs]
    # (b) the all-gathered {total, min} record (here: concatenated on one device)
    pairs = torch.cat([t.total_min() for t in trees]).view(G, 2)
    assert H(pairs).tolist() == [[o.total(), OS.buffer_min(o.q)] for o in orcs]
    ref_idx, ref_q, _ = OS.sharded_sample(orcs, n, OP.draws_u64(seed, n, n))  # stream position n after (a)
    got = []
    for r in range(G):
        cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
        idx, q, _, bm = trees[r].sample_sharded_pairs(r, G, pairs, n, seed, cnt)
        torch.cuda.synchronize()
        m = int(H(cnt)[0])
        got += (H(idx)[:m] + r * n_local).tolist()
        assert int(H(bm)[0]) == gmin and int(H(trees[r].header)[6]) == gmin
    assert got == ref_idx


@pytest.mark.parametrize("alpha", [0.6, 0.9, 0.5, 0.123, 0.75, 2.0, 3.5, 0.999])
def test_fast_power_path_equals_correctly_rounded(rpl, alpha):
    # R7: the fast exp(alpha ln p) evaluation (crpow.cuh fast_pow, Ziv margin (|t|+8) 2^-47) must
    # give the correctly rounded fp32 power on every input: 1.5M values spanning |delta| from
    # 1e-9 to 1e9 (and the eps_p floor, p near 1, exact powers of two) against the forced
    # double-double path, bit for bit
    g = rng(int(alpha * 1000) + 7)
    parts = [np.exp(g.uniform(np.log(1e-9), np.log(1e9), 1_000_000)),
             g.uniform(0.0, 4.0, 300_000),
             1.0 + g.normal(0, 1e-6, 100_000),
             np.ldexp(1.0, g.integers(-30, 30, 50_000)),
             np.zeros(50_000)]
    td = np.abs(np.concatenate(parts)).astype(np.float32)
    v_fast, _ = rpl.debug_priority_values(T_(td), alpha, 1e-3, force_slow=False)
    v_slow, _ = rpl.debug_priority_values(T_(td), alpha, 1e-3, force_slow=True)
    a, b = H(v_fast), H(v_slow)
    bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
    assert bad.size == 0, (alpha, td[bad[:5]], a[bad[:5]], b[bad[:5]])
