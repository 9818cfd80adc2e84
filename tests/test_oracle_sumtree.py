"""Pins for oracle.sumtree: SPEC worked example, brute force, exhaustive prefix
enumeration, last-write-wins, IS-weight closed forms and sampling statistics."""
import itertools
import math

import numpy as np
import pytest

from oracle import philox
from oracle import priority as P
from oracle import sumtree as S


def linear_find(q, prefix):
    """Brute-force linear scan, independent of the oracle's bisect."""
    run = 0
    for i, v in enumerate(q):
        if run <= prefix < run + v:
            return i
        run += v
    return None


def test_spec_tree_example():
    # S:607-609 with leaves scaled by 2 so the half-integer prefixes are integers:
    # leaves [3,1,4,2] -> total 10, find(4.5) -> 2, find(0) -> 0;
    # update leaf 1 -> 5: total 14, find(3.5) -> 1.
    t = S.SumTreeOracle(4, frac_bits=0)
    t.set_q([0, 1, 2, 3], [6, 2, 8, 4])
    assert t.total() == 20
    assert t.find(9) == 2
    assert t.find(0) == 0
    t.set_q([1], [10])
    assert t.total() == 28
    assert t.find(7) == 1


def test_find_matches_linear_scan():
    g = np.random.default_rng(0)
    for _ in range(200):
        n = int(g.integers(1, 65))
        q = [int(x) for x in g.integers(0, 50, n)]
        if sum(q) == 0:
            continue
        t = S.SumTreeOracle(n, 0)
        t.q = list(q)
        for prefix in g.integers(0, sum(q), 20):
            assert t.find(int(prefix)) == linear_find(q, int(prefix))


def test_exhaustive_prefix_counts_equal_q():
    g = np.random.default_rng(1)
    for _ in range(20):
        n = int(g.integers(1, 33))
        q = [int(x) for x in g.integers(0, 12, n)]
        if sum(q) == 0:
            continue
        t = S.SumTreeOracle(n, 0)
        t.q = list(q)
        counts = [0] * n
        for prefix in range(sum(q)):
            counts[t.find(prefix)] += 1
        assert counts == q                       # zero-q leaves never chosen


def test_update_last_write_wins_and_max_seen():
    g = np.random.default_rng(2)
    t = S.SumTreeOracle(16)
    idx = [int(x) for x in g.integers(0, 16, 64)]
    td = [float(x) for x in np.abs(g.normal(size=64)).astype(np.float32)]
    t.update(idx, td, 0.6)
    final = {}
    for i, d in zip(idx, td):
        final[i] = P.priority_q(d, 0.6, 1e-3, 32, 16)
    for i in range(16):
        assert t.q[i] == final.get(i, 0)
    assert t.max_seen == max([1 << 32] + [P.priority_q(d, 0.6, 1e-3, 32, 16) for d in td])


def test_update_floor_eps():
    # delta = 0 -> priority eps_p (never zero)
    t = S.SumTreeOracle(4)
    t.update([2], [0.0], 1.0, 1e-3)
    assert t.q[2] == P.quantise(*P.priority_value(0.0, 1.0, 1e-3), 32, t.cap)[0]
    assert t.q[2] > 0


def test_update_bad_index_skipped():
    t = S.SumTreeOracle(4)
    t.update([-1, 1], [1.0, 1.0], 1.0)
    assert not t.err_idx                      # negative = padding, skipped silently
    t.update([5, -1, 1], [1.0, 1.0, 1.0], 1.0)
    assert t.err_idx and t.q == [0, P.priority_q(1.0, 1.0, 1e-3, 32, 4), 0, 0]


def test_strata_identity_split_form():
    # The overflow-safe split form used on the GPU equals floor(k Q / n).
    g = np.random.default_rng(3)
    for _ in range(2000):
        Q = int(g.integers(1, 1 << 62)) * int(g.integers(1, 3))
        n = int(g.integers(1, 4097))
        k = int(g.integers(0, n + 1))
        split = k * (Q // n) + (k * (Q % n)) // n
        assert split == (k * Q) // n


def test_stratified_exact_mass_ratio():
    # p = [1, 3], alpha = 1 -> 1:3.  With integer strata and the full draw
    # range, the number of prefixes mapped to each leaf is exactly q.
    t = S.SumTreeOracle(2, 0)
    t.set_q([0, 1], [1, 3])
    idx, q, qmin = t.sample(4, [0, 0, 0, 0])
    assert sorted(idx) == [0, 1, 1, 1]


def test_alpha0_uniform_and_weights_one():
    # alpha = 0 -> all leaves equal -> uniform strata, weights all 1
    t = S.SumTreeOracle(64)
    g = np.random.default_rng(4)
    t.update(list(range(64)), [float(x) for x in g.lognormal(0, 2, 64).astype(np.float32)], 0.0)
    assert len(set(t.q)) == 1
    draws = philox.draws_u64(7, 0, 64)
    idx, q, qmin = t.sample(64, draws)
    assert sorted(idx) == list(range(64))       # one draw per equal-width stratum
    w = S.is_weights(q, t.total(), 64, 0.4)
    assert w == [1.0] * 64


def test_is_weights_closed_form():
    g = np.random.default_rng(5)
    q = [int(x) for x in g.integers(1, 1 << 40, 50)]
    Q = sum(q) + 12345
    for beta in [0.0, 0.4, 0.6, 1.0]:
        w = S.is_weights(q, Q, 1 << 20, beta)
        qmin = min(q)
        for wi, qi in zip(w, q):
            assert abs(wi - (qmin / qi) ** beta) <= 1e-13
        assert max(w) == 1.0
    assert S.is_weights(q, Q, 1 << 20, 0.0) == [1.0] * 50


def test_empty_tree_sample():
    t = S.SumTreeOracle(8)
    idx, q, qmin = t.sample(3, [1, 2, 3])
    assert idx == [-1, -1, -1]


def test_small_Q_empty_strata():
    # Q < n: empty strata take lo_k; every prefix is < Q
    t = S.SumTreeOracle(4, 0)
    t.set_q([1, 3], [1, 1])
    idx, q, _ = t.sample(5, [2 ** 64 - 1] * 5)
    assert all(i in (1, 3) for i in idx)


def test_chi2_upper_tail():
    # S:653 / S:991: frequencies match p^alpha / sum over 1e5 draws on 64 leaves
    # (upper tail only: stratified sampling is under-dispersed).
    g = np.random.default_rng(6)
    t = S.SumTreeOracle(64)
    t.update(list(range(64)), [float(x) for x in np.abs(g.normal(size=64)).astype(np.float32)], 0.6)
    Q = t.total()
    counts = np.zeros(64)
    n = 1000
    for rep in range(100):
        idx, _, _ = t.sample(n, philox.draws_u64(11, rep * n, n))
        np.add.at(counts, idx, 1)
    exp = np.array(t.q, np.float64) / Q * counts.sum()
    chi2 = float(((counts - exp) ** 2 / exp).sum())
    # 63 dof: the 0.99 quantile is ~92.0
    assert chi2 < 92.0


def test_sharded_equals_concatenated():
    g = np.random.default_rng(8)
    shards = []
    for s in range(4):
        t = S.SumTreeOracle(16)
        t.update(list(range(16)), [float(x) for x in np.abs(g.normal(size=16)).astype(np.float32)], 0.6)
        shards.append(t)
    draws = philox.draws_u64(3, 0, 32)
    idx, q, qmin = S.sharded_sample(shards, 32, draws)
    allq = list(itertools.chain.from_iterable(s.q for s in shards))
    Q = sum(allq)
    for k, i in enumerate(idx):
        lo, hi = (k * Q) // 32, ((k + 1) * Q) // 32
        prefix = lo + ((draws[k] * (hi - lo)) >> 64)
        assert linear_find(allq, prefix) == i


def test_buffer_min_is_the_per_normaliser():
    # NEXT-4 (R29): normalising by the buffer's largest weight, w_i = (N P_i)^-b / max_j (N P_j)^-b
    # over every stored leaf with P_j > 0, equals (q_min / q_i)^b with q_min = buffer_min
    import random
    rnd = random.Random(5)
    q = [rnd.randint(1, 1 << 40) if rnd.random() < 0.8 else 0 for _ in range(200)]
    Q = sum(q)
    N = len(q)
    beta = 0.4
    wmax = max((N * qi / Q) ** -beta for qi in q if qi > 0)
    qm = S.buffer_min(q)
    assert qm == min(x for x in q if x > 0)
    for qi in q:
        if qi > 0:
            assert abs((N * qi / Q) ** -beta / wmax - (qm / qi) ** beta) <= 1e-12
    assert S.buffer_min([0, 0]) == (1 << 63) - 1


def test_live_only_update_never_revives_and_keeps_max_seen():
    # R30: entries on zero leaves are skipped entirely (value and max-seen); live leaves update
    t = S.SumTreeOracle(8, 0)
    t.q = [5, 0, 7, 0, 0, 3, 0, 1]
    before_max = t.max_seen
    t.update([1, 3, 4], [100.0, 200.0, 300.0], 1.0, 0.0, live_only=True)
    assert t.q == [5, 0, 7, 0, 0, 3, 0, 1] and t.max_seen == before_max
    t.update([0, 1], [2.0, 9.0], 1.0, 0.0, live_only=True)
    assert t.q[0] == 2 and t.q[1] == 0                  # F = 0: q = RNE(p^1) = 2
    t.update([1], [9.0], 1.0, 0.0)                      # the plain update writes it
    assert t.q[1] == 9 and t.max_seen == 9


def test_sample_unique_pins():
    # R32: successive proportional draws without replacement
    import random
    rnd = random.Random(3)
    q = [0, 4, 0, 1, 7, 2, 0, 9]
    draws = [rnd.getrandbits(64) for _ in range(8)]
    idx, qq = S.sample_unique(q, 8, draws)
    nz = [i for i, v in enumerate(q) if v > 0]
    assert sorted(i for i in idx if i >= 0) == nz            # every non-zero leaf exactly once
    assert idx[len(nz):] == [-1] * (8 - len(nz)) and all(q[i] == v for i, v in zip(idx, qq) if i >= 0)
    t = S.SumTreeOracle(len(q), 0)
    t.q = list(q)
    assert idx[0] == t.find((draws[0] * sum(q)) >> 64)       # the first draw is the proportional one
    # two leaves, q = [1, 3]: first draw is leaf 1 with probability 3/4 exactly over u
    assert S.sample_unique([1, 3], 2, [0, 0])[0] == [0, 1]
    assert S.sample_unique([1, 3], 2, [2 ** 62, 0])[0] == [1, 0]   # u/2^64 = 1/4 -> prefix 1
    counts = [0, 0]
    for _ in range(4000):
        counts[S.sample_unique([1, 3], 1, [rnd.getrandbits(64)])[0][0]] += 1
    assert abs(counts[1] / 4000 - 0.75) < 0.03
