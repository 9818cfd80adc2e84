"""GPU parity: rpl_gather (transition and sequence gathers) vs the naive
full-stack oracle — bytes bit-exact, n-step returns within 1e-5 relative."""
import numpy as np
import pytest

from oracle import gather as OG
from oracle import returns as OR
from oracle import sumtree as OS
from synth import make_ring, rng
from tests._tol import check_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def T_(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def H(t):
    return t.cpu().numpy()


def dev_ring(rpl, ring):
    return rpl.GatherRing(obs=T_(ring.obs), act=T_(ring.act), rew=T_(ring.rew), done=T_(ring.done),
                          cursor=ring.cursor, size=ring.size, rnn=None if ring.rnn is None else T_(ring.rnn))


def valid_transition_leaves(ring, k, n, count, g):
    cap, B = ring.obs.shape[:2]
    out = []
    while len(out) < count:
        row, b = int(g.integers(0, cap)), int(g.integers(0, B))
        if OG.window_valid_transition(row, cap, ring.cursor, ring.size, k, n):
            out.append(row * B + b)
    return np.array(out, np.int64)


@pytest.mark.parametrize("pad_mode", [0, 1])
@pytest.mark.parametrize("n_step", [1, 3, 5])
def test_transition_frames(rpl, pad_mode, n_step):
    import torch
    ring = make_ring(5 + n_step, cap=64, B=8, ep_len=6.0, reward_kind="heavy")
    dr = dev_ring(rpl, ring)
    g = rng(7)
    idx = valid_transition_leaves(ring, 4, n_step, 300, g)
    # also include ring-wrapping windows and a skipped entry
    idx[0] = (ring.cursor + 3) % 64 * 8 + 1
    idx[1] = -1
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=n_step, gamma=0.99, pad_mode=pad_mode, err=err)
    ref = OG.gather_transitions(idx, 8, ring.obs, ring.act, ring.rew, ring.done, 4, n_step, 0.99, pad_mode)
    ok = idx >= 0
    assert np.array_equal(H(out["obs"])[ok], ref["obs"][ok])
    assert np.array_equal(H(out["next_obs"])[ok], ref["next_obs"][ok])
    assert np.array_equal(H(out["act"])[ok], ref["act"][ok])
    assert np.array_equal(H(out["done_n"])[ok], ref["done_n"][ok])
    absR = OG.gather_transitions(idx, 8, ring.obs, ring.act, np.abs(ring.rew), ring.done, 4, n_step, 0.99)["ret"]
    check_rel(H(out["ret"])[ok], ref["ret"][ok], absR[ok], what="fused n-step")


def test_transition_invalid_window_flag(rpl):
    import torch
    ring = make_ring(3, cap=32, B=2, ep_len=100.0)
    dr = dev_ring(rpl, ring)
    bad_row = (ring.cursor - 1) % 32  # newest row: its n-step lookahead is not stored
    idx = np.array([bad_row * 2], np.int64)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=3, err=err)
    assert int(H(err)[0]) & 8


def test_transition_vector_obs(rpl):
    # Mujoco: obs f32 D=17 (68 B, LSU path) and D=376, actions f32 [A]
    for D, A in [(17, 6), (376, 17)]:
        ring = make_ring(11 + D, cap=128, B=16, obs_shape=(D,), obs_dtype=np.float32, act_dim=A, ep_len=50.0,
                         reward_kind="mujoco")
        dr = dev_ring(rpl, ring)
        idx = valid_transition_leaves(ring, 1, 3, 256, rng(D))
        out = rpl.gather(dr, T_(idx), kind="transition", k=1, n_step=3, gamma=0.99)
        ref = OG.gather_transitions(idx, 16, ring.obs, ring.act, ring.rew, ring.done, 1, 3, 0.99)
        assert np.array_equal(H(out["obs"]), ref["obs"])
        assert np.array_equal(H(out["next_obs"]), ref["next_obs"])
        assert np.array_equal(H(out["act"]), ref["act"])
        check_rel(H(out["ret"]), ref["ret"], np.abs(ref["ret"]) + 10.0, what="mujoco ret")


def test_transition_fused_is_weights(rpl):
    import torch
    ring = make_ring(21, cap=64, B=4, ep_len=20.0)
    dr = dev_ring(rpl, ring)
    idx = valid_transition_leaves(ring, 4, 3, 64, rng(1))
    g = rng(2)
    q = g.integers(1, 1 << 40, 64).astype(np.int64)
    qmin = np.array([q.min()], np.int64)
    out = rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=3, q=T_(q), qmin=T_(qmin), beta=0.4)
    ref = OS.is_weights([int(x) for x in q], int(q.sum()), 256, 0.4)
    check_rel(H(out["w"]), ref, what="fused w")


@pytest.fixture(params=[0, 1, 2, 3, 4, 5, 6], ids=["pipe", "chunk", "lsu", "tmapipe", "pipe14", "pipe8", "ldgbulk"])
def variant(rpl, request):
    assert rpl._lib.lib.rpl_debug_set_gather_variant(request.param) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_gather_variant(0)


@pytest.mark.parametrize("out_mode", [0, 1])
@pytest.mark.parametrize("pad_mode", [0, 1])
def test_sequences(rpl, out_mode, pad_mode, variant):
    import torch
    period, L, k = 40, 125, 4
    ring = make_ring(31 + out_mode, cap=400, B=4, ep_len=30.0, period=period, rnn_h=64, reward_kind="r2d2")
    dr = dev_ring(rpl, ring)
    g = rng(3)
    nblk = 400 // period
    idx = []
    while len(idx) < 24:
        blk, b = int(g.integers(0, nblk)), int(g.integers(0, 4))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 4 + b)
    idx = np.array(idx, np.int64)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, pad_mode=pad_mode,
                     out_mode=out_mode, err=err)
    ref = OG.gather_sequences(idx, 4, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period, pad_mode,
                              stacked=(out_mode == 0))
    for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
        assert np.array_equal(H(out[name]), ref[name]), name
    assert int(H(err)[0]) == 0


def test_sequence_then_nstep_target(rpl):
    # R2D2 step tail: gathered rows 40..123 of L=125 -> rescaled 5-step targets for the 80 train rows
    import torch
    period, L, k = 40, 125, 4
    ring = make_ring(41, cap=400, B=8, ep_len=200.0, period=period, rnn_h=32, reward_kind="r2d2")
    dr = dev_ring(rpl, ring)
    idx = []
    g = rng(4)
    while len(idx) < 16:
        blk, b = int(g.integers(0, 10)), int(g.integers(0, 8))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 8 + b)
    idx = np.array(idx, np.int64)
    out = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, want=["rew", "done"])
    qv = g.normal(0, 10, (L, 16)).astype(np.float32)
    r_tr = out["rew"][40:124].contiguous()
    d_tr = out["done"][40:124].contiguous()
    q_tr = T_(qv[40:124])
    y, dn = rpl.returns_nstep(r_tr, d_tr, 5, 0.997, q=q_tr, q_boot=T_(qv[124]), rescale=True)
    ref_seq = OG.gather_sequences(idx, 8, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period)
    yr, dnr = OR.nstep_return(ref_seq["rew"][40:124], ref_seq["done"][40:124], 5, 0.997, q=qv[40:124],
                              q_boot=qv[124], rescale=True)
    assert y.shape == (80, 16)
    check_rel(H(y), yr, np.abs(yr) + 1e-3, what="r2d2 targets")
    assert np.array_equal(H(dn), dnr)


@pytest.mark.parametrize("L,k,n_s", [(1, 4, 7), (2, 4, 300), (5, 4, 33), (40, 1, 50), (47, 2, 190), (125, 4, 64),
                                     (120, 8, 20)])
def test_sequence_shapes(rpl, L, k, n_s, variant):
    # degenerate and ragged lengths exercise the pipeline's piece logic (rows split
    # across CTAs, short pieces, ring-slot wrap) and every stack depth
    import torch
    period = 40
    ring = make_ring(50 + L + k, cap=400, B=3, ep_len=7.0, period=period, rnn_h=8, reward_kind="r2d2",
                     obs_shape=(16, 24))
    dr = dev_ring(rpl, ring)
    g = rng(L * 31 + k)
    nblk = 400 // period
    idx = []
    while len(idx) < n_s:
        blk, b = int(g.integers(0, nblk)), int(g.integers(0, 3))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 3 + b)
    idx = np.array(idx, np.int64)
    idx[len(idx) // 2] = -1  # a skipped sample in the middle
    out = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period)
    ref = OG.gather_sequences(idx, 3, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period)
    ok = idx >= 0
    assert np.array_equal(H(out["obs"])[:, ok], ref["obs"][:, ok])
    for name in ("act", "prev_act", "rew", "prev_rew", "done"):
        assert np.array_equal(H(out[name])[:, ok], ref[name][:, ok]), name
    assert np.array_equal(H(out["rnn"])[:, ok], ref["rnn"][:, ok])


def _column_ring(dr, b, with_rnn):
    """Host copy of ring column b (all rows) as a [cap_T, 1] ring for the oracle."""
    obs = H(dr.obs[:, b:b + 1])
    rnn = H(dr.rnn[:, b:b + 1]) if with_rnn else None
    return obs, H(dr.act[:, b:b + 1]), H(dr.rew[:, b:b + 1]), H(dr.done[:, b:b + 1]), rnn


def test_r2d2_full_size_sampled(rpl):
    # BASELINE configs[4] in bench.py's launch configuration: [4000, 256] ring (7.2 GB),
    # 64 sequences x 125 rows, k=4, stored (h, c) 512 — sampled sequences vs the oracle
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    dev = torch.device("cuda")
    cap, B, period, L, k = 4000, 256, 40, 125, 4
    dr = make_ring_device(2019, cap, B, dev, ep_len=2000.0, period=period, rnn_h=512, cursor=1234)
    blocks = R.valid_sequence_blocks(cap, period, dr.cursor, dr.size, k, L)
    g = rng(11)
    leaves = g.choice(R.leaves_of(blocks, B), 64).astype(np.int64)
    # the oldest and the newest valid blocks (ring wrap around the cursor)
    age = (dr.cursor - 1 - blocks * period) % cap
    leaves[5] = int(blocks[np.argmax(age)]) * B + 7
    leaves[6] = int(blocks[np.argmin(age)]) * B + 255
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    plan = rpl.GatherPlan(dr, 64, kind="sequence", k=k, seq_len=L, period=period)
    out = plan.run(T_(leaves), err=err)
    torch.cuda.synchronize()
    assert int(H(err)[0]) == 0
    for s in list(range(0, 64, 9)) + [5, 6, 63]:
        blk, b = divmod(int(leaves[s]), B)
        obs, act, rew, done, rnn = _column_ring(dr, b, True)
        ref = OG.gather_sequences(np.array([blk], np.int64), 1, obs, act, rew, done, rnn, k, L, period)
        assert np.array_equal(H(out["obs"][:, s]), ref["obs"][:, 0]), s
        for name in ("act", "prev_act", "rew", "prev_rew", "done"):
            assert np.array_equal(H(out[name][:, s]), ref[name][:, 0]), (name, s)
        assert np.array_equal(H(out["rnn"][:, s]), ref["rnn"][:, 0]), s
    del dr
    torch.cuda.empty_cache()


def _row_window(dr, row, b, lo, hi):
    """Host copy of ring rows row+lo .. row+hi-1 (mod cap_T) of column b as a one-column ring."""
    import torch
    cap = dr.obs.shape[0]
    rows = torch.from_numpy((row + np.arange(lo, hi)) % cap).cuda()
    return (H(dr.obs[rows, b:b + 1]), H(dr.act[rows, b:b + 1]), H(dr.rew[rows, b:b + 1]), H(dr.done[rows, b:b + 1]))


def test_dqn_full_size_sampled(rpl):
    # BASELINE configs[2]: [4096, 256] frame ring (2^20 transitions, 7.4 GB), batch 512,
    # k=4, n=3, gamma=0.99 with fused n-step and IS weights — EVERY transition of the batch vs
    # the oracle, on a ring with short episodes (mean 30 rows) so that episode starts inside
    # the frame stacks occur at full size
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    dev = torch.device("cuda")
    cap, B, k, n = 4096, 256, 4, 3
    dr = make_ring_device(7, cap, B, dev, ep_len=30.0, period=64, rnn_h=1, cursor=777)
    dr.rnn = None
    rows = R.valid_transition_rows(cap, dr.cursor, dr.size, k, n)
    g = rng(12)
    leaves = g.choice(R.leaves_of(rows, B), 512).astype(np.int64)
    q = g.integers(1 << 20, 1 << 34, 512).astype(np.int64)
    qmin = np.array([q.min()], np.int64)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    out = rpl.gather(dr, T_(leaves), kind="transition", k=k, n_step=n, gamma=0.99, q=T_(q), qmin=T_(qmin),
                     beta=0.4, err=err)
    torch.cuda.synchronize()
    assert int(H(err)[0]) == 0
    w_ref = OS.is_weights([int(x) for x in q], int(q.sum()), cap * B, 0.4)
    check_rel(H(out["w"]), w_ref, what="w")
    o_obs, o_next, o_act, o_dn, o_ret = (H(out[x]) for x in ("obs", "next_obs", "act", "done_n", "ret"))
    padded = 0
    for s in range(512):
        row, b = divmod(int(leaves[s]), B)
        obs, act, rew, done = _row_window(dr, row, b, -8, n + 2)   # the transition sits at window row 8
        ref = OG.gather_transitions(np.array([8], np.int64), 1, obs, act, rew, done, k, n, 0.99)
        assert np.array_equal(o_obs[s], ref["obs"][0]), s
        assert np.array_equal(o_next[s], ref["next_obs"][0]), s
        assert int(o_act[s]) == int(ref["act"][0]) and int(o_dn[s]) == int(ref["done_n"][0]), s
        check_rel(o_ret[s:s + 1], ref["ret"][:1], np.abs(ref["ret"][:1]) + 1.0, what="ret")
        padded += int(done[4:8, 0].any() or done[4 + n:8 + n, 0].any())
    assert padded > 0  # some stacks crossed an episode start
    del dr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", ["transition", "sequence"])
def test_gather_batch_min_weights(rpl, kind, variant):
    # qmin = NULL: the gather normalises the IS weights by the batch min over idx >= 0
    g = rng(8)
    if kind == "transition":
        ring = make_ring(71, cap=64, B=8, ep_len=9.0)
        idx = valid_transition_leaves(ring, 4, 3, 40, g)
        kw = dict(kind="transition", k=4, n_step=3)
    else:
        ring = make_ring(72, cap=400, B=4, ep_len=30.0, period=40, rnn_h=8, reward_kind="r2d2")
        idx = []
        while len(idx) < 40:
            blk, b = int(g.integers(0, 10)), int(g.integers(0, 4))
            if OG.window_valid_sequence(blk * 40, 400, ring.cursor, ring.size, 4, 45):
                idx.append(blk * 4 + b)
        idx = np.array(idx, np.int64)
        kw = dict(kind="sequence", k=4, seq_len=45, period=40)
    idx[3] = -1  # skipped entry: its (tiny) q must not enter the min
    q = g.integers(1 << 20, 1 << 40, idx.size).astype(np.int64)
    q[3] = 1
    dr = dev_ring(rpl, ring)
    out = rpl.gather(dr, T_(idx), q=T_(q), qmin=None, beta=0.6, want=["w", "obs"], **kw)
    qm = int(q[idx >= 0].min())
    ok = idx >= 0
    check_rel(H(out["w"])[ok], (qm / q[ok].astype(np.float64)) ** 0.6, what="batch-min w")


def test_sequence_n_active(rpl, variant):
    # rpl_gather_desc.n_active: only entries k < *n_active are gathered; the rest are
    # skipped exactly as idx < 0 (outputs left untouched) — every kernel variant
    import torch
    period, L, k = 40, 45, 4
    ring = make_ring(91, cap=400, B=4, ep_len=25.0, period=period, rnn_h=16, reward_kind="r2d2")
    dr = dev_ring(rpl, ring)
    g = rng(9)
    idx = []
    while len(idx) < 30:
        blk, b = int(g.integers(0, 10)), int(g.integers(0, 4))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 4 + b)
    idx = np.array(idx, np.int64)
    m = 17
    plan = rpl.GatherPlan(dr, idx.size, kind="sequence", k=k, seq_len=L, period=period)
    for t in plan.outputs.values():
        t.fill_(7) if t.dtype != torch.float32 else t.fill_(7.5)
    cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
    plan.desc.n_active = cnt.data_ptr()
    out = plan.run(T_(idx))
    ref = OG.gather_sequences(idx[:m], 4, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period)
    for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done"):
        o = H(out[name])
        assert np.array_equal(o[:, :m], ref[name]), name
        assert np.all(o[:, m:] == (7.5 if o.dtype == np.float32 else 7)), name
    assert np.array_equal(H(out["rnn"])[:, :m], ref["rnn"])


@pytest.mark.parametrize("nn,m", [(50, 23), (400, 333)])  # 400: the persistent pipeline path
def test_transition_n_active(rpl, nn, m):
    import torch
    ring = make_ring(92, cap=64, B=8, ep_len=9.0)
    dr = dev_ring(rpl, ring)
    idx = valid_transition_leaves(ring, 4, 3, nn, rng(10))
    plan = rpl.GatherPlan(dr, idx.size, kind="transition", k=4, n_step=3, gamma=0.99)
    for t in plan.outputs.values():
        t.zero_()
    cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
    plan.desc.n_active = cnt.data_ptr()
    out = plan.run(T_(idx))
    ref = OG.gather_transitions(idx[:m], 8, ring.obs, ring.act, ring.rew, ring.done, 4, 3, 0.99)
    assert np.array_equal(H(out["obs"])[:m], ref["obs"]) and np.all(H(out["obs"])[m:] == 0)
    assert np.array_equal(H(out["next_obs"])[:m], ref["next_obs"])


@pytest.mark.parametrize("kind", ["sequence", "transition", "sequence_unique"])
def test_col_offset(rpl, kind):
    # rpl_gather_desc.col_offset: entry k lands in output column *col_offset + k of arrays
    # with n columns; other columns untouched (Mode C writes into a central batch)
    import torch
    g = rng(13)
    if kind == "transition":
        ring = make_ring(93, cap=64, B=8, ep_len=9.0)
        idx = valid_transition_leaves(ring, 4, 3, 40, g)
        kw = dict(kind="transition", k=4, n_step=3, gamma=0.99)
    else:
        ring = make_ring(94, cap=400, B=4, ep_len=25.0, period=40, rnn_h=16, reward_kind="r2d2")
        idx = []
        while len(idx) < 40:
            blk, b = int(g.integers(0, 10)), int(g.integers(0, 4))
            if OG.window_valid_sequence(blk * 40, 400, ring.cursor, ring.size, 4, 45):
                idx.append(blk * 4 + b)
        idx = np.array(idx, np.int64)
        kw = dict(kind="sequence", k=4, seq_len=45, period=40, out_mode=1 if kind.endswith("unique") else 0)
    dr = dev_ring(rpl, ring)
    m, off = 11, 23
    sub = idx.copy()
    sub[m:] = -1
    plan = rpl.GatherPlan(dr, idx.size, **kw)
    for t in plan.outputs.values():
        t.zero_()
    cnt = torch.tensor([m, off], dtype=torch.int64, device="cuda")
    plan.desc.n_active = cnt.data_ptr()
    plan.desc.col_offset = cnt.data_ptr() + 8
    out = {kk: H(v) for kk, v in plan.run(T_(idx)).items()}
    ref = rpl.gather(dr, T_(idx[:m]), **kw)
    axis = 0 if kind == "transition" else 1
    for name, r in ref.items():
        r = H(r)
        o = out[name]
        got = np.take(o, np.arange(off, off + m), axis=axis)
        assert np.array_equal(got, r), name
        rest = np.delete(o, np.arange(off, off + m), axis=axis)
        assert not rest.any(), name


@pytest.mark.parametrize("pad_mode", [0, 1])
def test_unique_plus_start_stacks_equal_stacked(rpl, pad_mode):
    # Mode C shipping: RPL_OUT_UNIQUE rows + o_start offsets, re-stacked by rpl_stack_frames,
    # are bit-identical to the stacked gather (and to the oracle)
    import torch
    period, L, k = 40, 125, 4
    ring = make_ring(97, cap=400, B=4, ep_len=12.0, period=period, rnn_h=8, reward_kind="r2d2")
    dr = dev_ring(rpl, ring)
    g = rng(19)
    idx = []
    while len(idx) < 20:
        blk, b = int(g.integers(0, 10)), int(g.integers(0, 4))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 4 + b)
    idx = np.array(idx, np.int64)
    uq = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, pad_mode=pad_mode, out_mode=1,
                    want=["obs", "start"])
    st = rpl.stack_frames(uq["obs"], uq["start"], k, pad_mode=pad_mode)
    ref = OG.gather_sequences(idx, 4, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period, pad_mode)
    assert np.array_equal(H(st), ref["obs"])
    sg = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, pad_mode=pad_mode, want=["obs"])
    assert np.array_equal(H(st), H(sg["obs"]))


def test_random_gather_stress(rpl):
    # >= 1e4 random frame and sequence gathers (random geometry, ring wrap,
    # episode starts inside stacks, both paddings and output modes) bit-exact vs the oracle
    g = rng(2024)
    total_seq = total_tr = 0
    cfg = 0
    while total_seq < 6000 or total_tr < 6000:
        cfg += 1
        period = int(g.choice([4, 8, 20]))
        cap = period * int(g.integers(8, 20))
        B = int(g.integers(1, 6))
        k = int(g.integers(1, 6))
        pad = int(g.integers(0, 2))
        ring = make_ring(5000 + cfg, cap=cap, B=B, ep_len=float(g.uniform(3, 30)), period=period, rnn_h=4,
                         reward_kind="r2d2", obs_shape=(4, 8))
        dr = dev_ring(rpl, ring)
        if cfg % 2:
            L = int(g.integers(1, 3 * period))
            if not any(OG.window_valid_sequence(b * period, cap, ring.cursor, ring.size, k, L) for b in range(cap // period)):
                continue
            idx = []
            while len(idx) < 400:
                blk, b = int(g.integers(0, cap // period)), int(g.integers(0, B))
                if OG.window_valid_sequence(blk * period, cap, ring.cursor, ring.size, k, L):
                    idx.append(blk * B + b)
            idx = np.array(idx, np.int64)
            om = int(g.integers(0, 2))
            out = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, pad_mode=pad, out_mode=om)
            ref = OG.gather_sequences(idx, B, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period, pad,
                                      stacked=(om == 0))
            for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
                assert np.array_equal(H(out[name]), ref[name]), (cfg, name)
            total_seq += idx.size
        else:
            n = int(g.integers(1, 6))
            idx = valid_transition_leaves(ring, k, n, 400, g)
            out = rpl.gather(dr, T_(idx), kind="transition", k=k, n_step=n, gamma=0.97, pad_mode=pad)
            ref = OG.gather_transitions(idx, B, ring.obs, ring.act, ring.rew, ring.done, k, n, 0.97, pad)
            assert np.array_equal(H(out["obs"]), ref["obs"]) and np.array_equal(H(out["next_obs"]), ref["next_obs"])
            assert np.array_equal(H(out["act"]), ref["act"]) and np.array_equal(H(out["done_n"]), ref["done_n"])
            check_rel(H(out["ret"]), ref["ret"], np.abs(ref["ret"]) + 1.0, what="stress ret")
            total_tr += idx.size


@pytest.mark.parametrize("skip_pattern,n_step", [("isolated", 3), ("odd_runs", 3), ("isolated", 5), ("odd_runs", 6)])
def test_transition_pipeline_skipped_entries(rpl, skip_pattern, n_step):
    # n_step 5 / 6 give 9 / 10 frames per sample, i.e. 3 / 2 slot groups (an odd group count:
    # consumer warps then run ahead of the group's previous sample, the armed counter case)
    # Persistent transition pipeline with more samples per CTA than slot groups (n = 2048,
    # Atari frames: ~14 samples per CTA, 4 groups) and skipped entries (idx = -1) in between:
    # slot groups / mbarrier phases follow the loaded samples only (a skipped entry used to
    # leave a phase that never completed).  Bit-exact vs the oracle, no hang.
    import torch
    ring = make_ring(77, cap=256, B=8, ep_len=40.0)
    dr = dev_ring(rpl, ring)
    g = rng(8)
    idx = valid_transition_leaves(ring, 4, n_step, 2048, g)
    if skip_pattern == "isolated":
        idx[1::7] = -1
    else:  # runs of 1, 3 and 5 skipped entries
        for s0, ln in ((1, 1), (20, 3), (100, 5), (1500, 1), (2040, 3)):
            idx[s0:s0 + ln] = -1
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=n_step, gamma=0.99, err=err)
    torch.cuda.synchronize()
    assert int(H(err)[0]) == 0
    ref = OG.gather_transitions(idx, 8, ring.obs, ring.act, ring.rew, ring.done, 4, n_step, 0.99)
    ok = idx >= 0
    assert np.array_equal(H(out["obs"])[ok], ref["obs"][ok])
    assert np.array_equal(H(out["next_obs"])[ok], ref["next_obs"][ok])
    assert np.array_equal(H(out["act"])[ok], ref["act"][ok])
    assert np.array_equal(H(out["done_n"])[ok], ref["done_n"][ok])


def test_transition_pipeline_scalars_only(rpl):
    # want = ret / act only at a pipeline-sized batch: no frame output, so no frame loads
    import torch
    ring = make_ring(78, cap=128, B=8, ep_len=20.0, reward_kind="heavy")
    dr = dev_ring(rpl, ring)
    idx = valid_transition_leaves(ring, 4, 3, 600, rng(9))
    out = rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=3, gamma=0.99, want=["ret", "act", "done_n"])
    ref = OG.gather_transitions(idx, 8, ring.obs, ring.act, ring.rew, ring.done, 4, 3, 0.99)
    absR = OG.gather_transitions(idx, 8, ring.obs, ring.act, np.abs(ring.rew), ring.done, 4, 3, 0.99)["ret"]
    assert np.array_equal(H(out["act"]), ref["act"])
    assert np.array_equal(H(out["done_n"]), ref["done_n"])
    check_rel(H(out["ret"]), ref["ret"], absR, what="scalars-only ret")


def _with_timeouts(ring, g, frac=0.5):
    """Turn a fraction of the ring's episode ends into time-limit ends (done = 2) and give
    every row a terminal value (read only at those rows, R34)."""
    done = ring.done.copy()
    ends = np.argwhere(done == 1)
    pick = ends[g.random(len(ends)) < frac]
    done[pick[:, 0], pick[:, 1]] = 2
    v_term = g.normal(0, 10, done.shape).astype(np.float32)
    return done, v_term


@pytest.mark.parametrize("rescale,with_q,timeouts,lo,Tt", [(True, True, False, 40, 80), (False, True, True, 40, 80),
                                                            (True, True, True, 0, 120), (False, False, False, 3, 1),
                                                            (True, False, True, 7, 113)])
def test_sequence_fused_targets(rpl, rescale, with_q, timeouts, lo, Tt):
    # a2 + a4 fused into the sequence gather (rpl_gather_desc.o_tgt): rescaled 5-step targets of
    # the target rows vs the oracle's n-step over the oracle-gathered rows (and, without time
    # limits, bit-identical to rpl_returns_nstep over the gathered rows)
    import torch
    period, L, k, n_s, ns, gamma = 40, 125, 4, 64, 5, 0.997
    ring = make_ring(61, cap=400, B=4, ep_len=12.0, period=period, rnn_h=8, reward_kind="r2d2")
    g = rng(62)
    v_term = None
    if timeouts:
        ring.done, v_term = _with_timeouts(ring, g)
    dr = dev_ring(rpl, ring)
    if v_term is not None:
        dr.v_term = T_(v_term)
    idx = []
    while len(idx) < n_s:
        blk, b = int(g.integers(0, 10)), int(g.integers(0, 4))
        if OG.window_valid_sequence(blk * period, 400, ring.cursor, ring.size, k, L):
            idx.append(blk * 4 + b)
    idx = np.array(idx, np.int64)
    idx[9] = -1
    qv = g.normal(0, 10, (L, n_s)).astype(np.float32)
    tg = dict(lo=lo, T=Tt, n_step=ns, gamma=gamma, rescale=rescale, eps=1e-3, q=T_(qv) if with_q else None)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = rpl.gather(dr, T_(idx), kind="sequence", k=k, seq_len=L, period=period, targets=tg, err=err)
    torch.cuda.synchronize()
    assert int(H(err)[0]) == 0
    ref = OG.gather_sequences(idx, 4, ring.obs, ring.act, ring.rew, ring.done, ring.rnn, k, L, period)
    Tn = Tt + ns - 1
    vt_rows = None
    if v_term is not None:  # per gathered row: v_term of its ring row
        vt_rows = np.zeros((L, n_s), np.float32)
        for s_, leaf in enumerate(idx):
            if leaf >= 0:
                blk, b = divmod(int(leaf), 4)
                vt_rows[:, s_] = v_term[(blk * period + np.arange(L)) % 400, b]
        vt_rows = vt_rows[lo:lo + Tn]
    yr, dnr = OR.nstep_return(ref["rew"][lo:lo + Tn], ref["done"][lo:lo + Tn], ns, gamma,
                              q=qv[lo:lo + Tn] if with_q else None, q_boot=qv[lo + Tn] if with_q else None,
                              rescale=rescale, v_term=vt_rows)
    ok = idx >= 0
    assert out["tgt"].shape == (Tt, n_s)
    check_rel(H(out["tgt"])[:, ok], yr[:, ok], (np.abs(yr) + 1e-3)[:, ok], what="fused targets")
    assert np.array_equal(H(out["tgt_done"])[:, ok], dnr[:, ok])
    if v_term is None:  # the same arithmetic as the standalone kernel, bit for bit
        y2, dn2 = rpl.returns_nstep(out["rew"][lo:lo + Tn].contiguous(), out["done"][lo:lo + Tn].contiguous(), ns,
                                    gamma, q=T_(qv[lo:lo + Tn]) if with_q else None,
                                    q_boot=T_(qv[lo + Tn]) if with_q else None, rescale=rescale)
        assert np.array_equal(H(y2)[:, ok], H(out["tgt"])[:, ok])


def test_transition_time_limit_bootstrap(rpl):
    # R34 in the transition gather: n-step returns stopping at a time-limit row add gamma^(j+1) v_term
    import torch
    ring = make_ring(63, cap=128, B=8, ep_len=5.0, reward_kind="heavy")
    g = rng(64)
    ring.done, v_term = _with_timeouts(ring, g)
    dr = dev_ring(rpl, ring)
    dr.v_term = T_(v_term)
    for nn in (37, 700):  # one-CTA-per-sample kernel and the persistent pipeline
        idx = valid_transition_leaves(ring, 4, 3, nn, g)
        out = rpl.gather(dr, T_(idx), kind="transition", k=4, n_step=3, gamma=0.99)
        ref = OG.gather_transitions(idx, 8, ring.obs, ring.act, ring.rew, ring.done, 4, 3, 0.99, v_term=v_term)
        absR = OG.gather_transitions(idx, 8, ring.obs, ring.act, np.abs(ring.rew), ring.done, 4, 3, 0.99,
                                     v_term=np.abs(v_term))["ret"]
        check_rel(H(out["ret"]), ref["ret"], absR, what="time-limit ret")
        assert np.array_equal(H(out["done_n"]), ref["done_n"])
        assert np.array_equal(H(out["obs"]), ref["obs"]) and np.array_equal(H(out["next_obs"]), ref["next_obs"])


@pytest.mark.parametrize("L,k,n_s,period", [(125, 4, 64, 40), (45, 4, 300, 40), (5, 4, 33, 8), (1, 1, 7, 4)])
def test_gather_sample_equals_sample_then_gather(rpl, L, k, n_s, period):
    # a8 fused into the sequence gather (rpl_gather_sample): same indices, q, IS weights and
    # every output as rpl_sumtree_sample_stream followed by rpl_gather, over three chained
    # calls (the tree's stream position advances identically)
    import torch
    cap, B = 400, 4
    ring = make_ring(70 + L, cap=cap, B=B, ep_len=12.0, period=period, rnn_h=8, reward_kind="r2d2",
                     obs_shape=(16, 24))
    dr = dev_ring(rpl, ring)
    nb = cap // period
    g = rng(L + n_s)
    t1, t2 = rpl.SumTree(nb * B, 32), rpl.SumTree(nb * B, 32)
    valid = [b_ * B + c for b_ in range(nb) if OG.window_valid_sequence(b_ * period, cap, ring.cursor, ring.size, k, L)
             for c in range(B)]
    td = np.abs(g.normal(size=len(valid))).astype(np.float32)
    for t in (t1, t2):
        t.update(T_(np.array(valid, np.int64)), T_(td), 0.9)
    tg = dict(lo=0, T=max(1, L - 6), n_step=5, gamma=0.99, rescale=True, q=T_(g.normal(0, 5, (L, n_s)).astype(np.float32))) if L > 6 else None
    p1 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
    p2 = rpl.GatherPlan(dr, n_s, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, targets=tg)
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
        # the next step's priorities for the sampled leaves (same on both trees)
        ntd = np.abs(g.normal(size=n_s)).astype(np.float32)
        t1.update(i1, T_(ntd), 0.9)
        t2.update(i2, T_(ntd), 0.9)
