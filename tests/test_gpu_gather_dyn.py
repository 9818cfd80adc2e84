"""GPU parity: the dynamic-tail sequence gather (rpl_gather_desc.work, k_gather_seq_dyn) against
the oracle under every schedule shape — all rows dynamic (pct 0, 1- and 3-row units), the
default 80 % static share (and 78 %, the previous 88 %), a tiny look-ahead, 32-row units, all static (pct 100), and the
static kernel (pct -1) — with
stacked and unique output, both padding modes, skipped samples, fused rescaled targets and
batch-min IS weights; the unit counter is zero again after every call."""
import numpy as np
import pytest

from oracle import gather as OG
from oracle import returns as OR
from synth import make_ring, rng
from tests._tol import check_rel

pytestmark = pytest.mark.gpu

SCHEDULES = [(78, 16, 16), (80, 16, 16), (88, 16, 12), (88, 10, 10), (0, 1, 1), (0, 3, 4), (50, 7, 30), (100, 5, 8), (90, 32, 8), (60, 2, 64), (-1, 10, 10)]


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


@pytest.fixture(params=SCHEDULES, ids=[f"pct{a}_rows{b}_look{c}" for a, b, c in SCHEDULES])
def schedule(rpl, request):
    assert rpl._lib.lib.rpl_debug_set_gather_dyn(*request.param) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_gather_dyn(80, 16, 16)  # the defaults


def T_(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def H(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("L,k,n_s,out_mode,pad_mode", [(125, 4, 64, 0, 0), (125, 4, 64, 1, 0), (47, 2, 190, 0, 1),
                                                       (5, 4, 33, 0, 0), (1, 4, 7, 1, 1), (40, 1, 50, 0, 0),
                                                       (120, 8, 20, 0, 1), (2, 4, 300, 1, 0),
                                                       # beyond the dynamic kernel's capacity (static split):
                                                       (125, 4, 320, 0, 0), (1, 4, 20000, 0, 0),
                                                       # many pieces per CTA at the edge of the piece table:
                                                       (2, 4, 2400, 0, 1), (3, 4, 1900, 0, 0)])
def test_dynamic_tail_vs_oracle(rpl, schedule, L, k, n_s, out_mode, pad_mode):
    import torch
    period = 40
    cap, B = 400, 3
    ring = make_ring(90 + L + k + out_mode, cap=cap, B=B, ep_len=7.0, period=period, rnn_h=8, reward_kind="r2d2",
                     obs_shape=(16, 24))
    dr = rpl.GatherRing(obs=T_(ring.obs), act=T_(ring.act), rew=T_(ring.rew), done=T_(ring.done),
                        cursor=ring.cursor, size=ring.size, rnn=T_(ring.rnn))
    g = rng(L * 7 + k + n_s)
    idx = []
    while len(idx) < n_s:
        blk, b = int(g.integers(0, cap // period)), int(g.integers(0, B))
        if OG.window_valid_sequence(blk * period, cap, ring.cursor, ring.size, k, L):
            idx.append(blk * B + b)
    idx = np.array(idx, np.int64)
    idx[len(idx) // 2] = -1  # a skipped sample
    q = g.integers(1, 1 << 40, n_s).astype(np.int64)
    tg = None
    if L >= 10 and out_mode == 0:
        qv = g.normal(0, 10, (L, n_s)).astype(np.float32)
        tg = dict(lo=2, T=L - 8, n_step=5, gamma=0.997, rescale=True, eps=1e-3, q=T_(qv))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    plan = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, pad_mode=pad_mode,
                          out_mode=out_mode, with_weights=True, targets=tg)
    for rep in range(2):  # twice: the unit counter must have been re-zeroed by the first call
        out = plan.run(T_(idx), q=T_(q), beta=0.6, err=err)
        torch.cuda.synchronize()
        assert int(H(err)[0]) == 0
        assert H(plan._work).tolist() == [0, 0, 0, 0]
        ref = OG.gather_sequences(idx, B, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period, pad_mode,
                                  stacked=(out_mode == 0))
        ok = idx >= 0
        for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
            assert np.array_equal(H(out[name])[:, ok], ref[name][:, ok]), (rep, name)
        qm = int(q[ok].min())
        w_ref = np.where(ok, (qm / q.astype(np.float64)) ** 0.6, 0.0)
        check_rel(H(out["w"])[ok], w_ref[ok], what="w")
        if tg is not None:
            lo, Tt = tg["lo"], tg["T"]
            Tn = Tt + 4
            yr, dnr = OR.nstep_return(ref["rew"][lo:lo + Tn], ref["done"][lo:lo + Tn], 5, 0.997, q=qv[lo:lo + Tn],
                                      q_boot=qv[lo + Tn], rescale=True)
            check_rel(H(out["tgt"])[:, ok], yr[:, ok], (np.abs(yr) + 1e-3)[:, ok], what="targets")
            assert np.array_equal(H(out["tgt_done"])[:, ok], dnr[:, ok])


@pytest.fixture(params=[10, 0, 28], ids=["early10", "early0", "early28"])
def early(rpl, request):
    # first-frame loads a CTA issues right after its fused descent (10: the default)
    assert rpl._lib.lib.rpl_debug_set_gather_dyn(1000 + request.param, 1, 1) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_gather_dyn(1010, 1, 1)


@pytest.mark.parametrize("L,k,n_s,period", [(125, 4, 64, 40), (45, 4, 300, 40), (5, 4, 33, 8), (1, 1, 7, 4)])
def test_dynamic_tail_fused_sampling(rpl, schedule, early, L, k, n_s, period):
    # rpl_gather_sample with the dynamic tail: indices, q, weights, tree header and every output
    # equal rpl_sumtree_sample_stream + rpl_gather with the static split, over chained calls
    import torch
    cap, B = 400, 4
    ring = make_ring(170 + L, cap=cap, B=B, ep_len=12.0, period=period, rnn_h=8, reward_kind="r2d2",
                     obs_shape=(16, 24))
    dr = rpl.GatherRing(obs=T_(ring.obs), act=T_(ring.act), rew=T_(ring.rew), done=T_(ring.done),
                        cursor=ring.cursor, size=ring.size, rnn=T_(ring.rnn))
    nb = cap // period
    g = rng(L + n_s + 5)
    t1, t2 = rpl.SumTree(nb * B, 32), rpl.SumTree(nb * B, 32)
    valid = [b_ * B + c for b_ in range(nb) if OG.window_valid_sequence(b_ * period, cap, ring.cursor, ring.size, k, L)
             for c in range(B)]
    td = np.abs(g.normal(size=len(valid))).astype(np.float32)
    for t in (t1, t2):
        t.update(T_(np.array(valid, np.int64)), T_(td), 0.9)
    tg = dict(lo=0, T=max(1, L - 6), n_step=5, gamma=0.99, rescale=True,
              q=T_(g.normal(0, 5, (L, n_s)).astype(np.float32))) if L > 6 else None
    p1 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
    p2 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
    p1.desc.work = None  # the static split for the reference
    e1, e2 = (torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(2))
    for step in range(3):
        i1, q1 = (torch.empty(n_s, dtype=torch.int64, device="cuda") for _ in range(2))
        t1.sample_stream(n_s, 77, out=(i1, q1, None, None), err=e1, want_qmin=False)
        o1 = p1.run(i1, q=q1, beta=0.6, err=e1)
        i2, q2 = (torch.full((n_s,), -9, dtype=torch.int64, device="cuda") for _ in range(2))
        o2 = p2.run_sample(t2, 77, i2, q2, beta=0.6, err=e2)
        torch.cuda.synchronize()
        assert np.array_equal(H(i1), H(i2)) and np.array_equal(H(q1), H(q2)), step
        for name in o1:
            assert np.array_equal(H(o1[name]), H(o2[name])), (step, name)
        assert np.array_equal(H(t1.header), H(t2.header)), step
        assert int(H(e1)[0]) == int(H(e2)[0]) == 0
        assert H(p2._work).tolist() == [0, 0, 0, 0]
        ntd = np.abs(g.normal(size=n_s)).astype(np.float32)
        t1.update(i1, T_(ntd), 0.9)
        t2.update(i2, T_(ntd), 0.9)


@pytest.mark.parametrize("L,k,n_s,period,case", [(125, 4, 64, 40, "plain"), (125, 4, 64, 40, "dups"),
                                                 (45, 4, 120, 40, "live"), (5, 4, 33, 8, "mintree"),
                                                 (125, 4, 64, 40, "padding")])
def test_fused_update_sample_equals_two_launches(rpl, L, k, n_s, period, case):
    # rpl_gather_update_sample (update + sampling + gather in one launch) against
    # rpl_sumtree_update_seq followed by rpl_gather_sample, over chained calls: the whole tree
    # storage (leaves, nodes, header), an attached min-tree, indices, q, weights and every output
    import torch
    cap, B = 400, 4
    ring = make_ring(190 + L, cap=cap, B=B, ep_len=12.0, period=period, rnn_h=8, reward_kind="r2d2",
                     obs_shape=(16, 24))
    dr = rpl.GatherRing(obs=T_(ring.obs), act=T_(ring.act), rew=T_(ring.rew), done=T_(ring.done),
                        cursor=ring.cursor, size=ring.size, rnn=T_(ring.rnn))
    nb = cap // period
    g = rng(L * 3 + n_s)
    N = nb * B
    t1, t2 = rpl.SumTree(N, 32), rpl.SumTree(N, 32)
    valid = [b_ * B + c for b_ in range(nb) if OG.window_valid_sequence(b_ * period, cap, ring.cursor, ring.size, k, L)
             for c in range(B)]
    td = np.abs(g.normal(size=len(valid))).astype(np.float32)
    mins = []
    for t in (t1, t2):
        t.update(T_(np.array(valid, np.int64)), T_(td), 0.9)
        if case == "mintree":
            mins.append(t.attach_min_tree())
    tg = dict(lo=0, T=max(1, L - 6), n_step=5, gamma=0.99, rescale=True,
              q=T_(g.normal(0, 5, (L, n_s)).astype(np.float32))) if L > 6 else None
    p1 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
    p2 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
    e1, e2 = (torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(2))
    prev = torch.full((n_s,), -1, dtype=torch.int64, device="cuda")
    live = case == "live"
    for step in range(4):
        T_p = 80 if L == 125 else 7
        steps = np.abs(g.lognormal(0, 2, (T_p, n_s))).astype(np.float32)
        pidx = prev.clone()
        if case == "dups" and step > 0:
            pidx[5] = pidx[0]
            pidx[9] = pidx[0]
        if case == "padding":
            pidx[::7] = -1
        if case == "live" and step > 0:  # some of the batch's leaves were invalidated meanwhile
            z = pidx[pidx >= 0][:5]
            for t in (t1, t2):
                t.set_q(z, torch.zeros_like(z))
        std = T_(steps)
        i1, q1 = (torch.empty(n_s, dtype=torch.int64, device="cuda") for _ in range(2))
        if step > 0:
            t1.update_seq(pidx, std, 0.9, eta=0.9, live_only=live)
        o1 = p1.run_sample(t1, 77, i1, q1, beta=0.6, err=e1)
        i2, q2 = (torch.full((n_s,), -9, dtype=torch.int64, device="cuda") for _ in range(2))
        if step > 0:
            o2 = p2.run_update_sample(t2, pidx, std, 77, i2, q2, eta=0.9, alpha=0.9, beta=0.6, live_only=live, err=e2)
        else:
            o2 = p2.run_sample(t2, 77, i2, q2, beta=0.6, err=e2)
        torch.cuda.synchronize()
        s1, s2 = H(t1.storage).copy(), H(t2.storage).copy()
        hdr = int(t1.layout.hdr_off)
        s1[hdr + 5] = s2[hdr + 5] = 0  # header word 5: each tree's own min-tree address
        assert np.array_equal(s1, s2), (case, step, "tree")
        if mins:
            assert np.array_equal(H(mins[0]), H(mins[1])), (case, step, "min-tree")
        assert np.array_equal(H(i1), H(i2)) and np.array_equal(H(q1), H(q2)), (case, step)
        for name in o1:
            assert np.array_equal(H(o1[name]), H(o2[name])), (case, step, name)
        assert int(H(e1)[0]) == int(H(e2)[0]), (case, step)
        assert H(p2._work).tolist() == [0, 0, 0, 0]
        prev = i2.clone()
