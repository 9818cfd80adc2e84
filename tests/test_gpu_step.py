"""The bench's R2D2 step, chained and graph-replayed, against the oracle chain (VERDICT r1
item 3; BASELINE north_star's full-step parity target, PAPER.md:38, P:123 fn).

Launch configuration of bench.py: [4000, 256] ring (7.2 GB, BASELINE configs[4]) with SHORT
episodes (mean 25 rows, so episode starts fall inside frame stacks), 25,600-leaf tree,
64 sequences x 125 rows, k = 4, n = 5, gamma 0.997, alpha 0.9, beta 0.6, eta 0.9, the
three-launch step (update_seq -> sample_stream -> gather with stacked frames, batch-min IS
weights and fused rescaled 5-step targets) and bench.py's default two-launch step
(update_seq -> rpl_gather_sample: the stratified draws inside the gather), PDL-chained and captured in one CUDA graph of P
steps, replayed twice.  Every step's tree, indices, q, weights, every output of all 64
sequences and every target are compared with the oracle doing the same chain from the same
seeded inputs (its own priority transform, sequence mix, Philox draws, stratified search,
naive full-stack gather and mpmath targets)."""
import numpy as np
import pytest

from oracle import gather as OG
from oracle import philox as OP
from oracle import priority as OPR
from oracle import returns as OR
from oracle import sumtree as OS
from tests._tol import check_rel

pytestmark = pytest.mark.gpu

CAP, B, PERIOD, BURN, TRAIN, TAIL, K, NS = 4000, 256, 40, 40, 80, 5, 4, 5
L = BURN + TRAIN + TAIL
GAMMA, ALPHA, BETA, ETA, EPS, EPS_P, SEED = 0.997, 0.9, 0.6, 0.9, 1e-3, 1e-3, 0x5EED
N = 64
P = 4


def _window(dr, leaf):
    """Host copy of the ring rows a sequence reads (row0-8 .. row0+L-1 of its column) as a
    one-column ring of L+8 rows, with the sequence at block 1 of period 8."""
    import torch
    blk, b = divmod(int(leaf), B)
    rows = (blk * PERIOD - 8 + np.arange(L + 8)) % CAP
    ri = torch.from_numpy(rows).cuda()
    obs = dr.obs[ri, b:b + 1].cpu().numpy()
    act = dr.act[ri, b:b + 1].cpu().numpy()
    rew = dr.rew[ri, b:b + 1].cpu().numpy()
    done = dr.done[ri, b:b + 1].cpu().numpy()
    rnn = np.zeros((2, 1) + tuple(dr.rnn.shape[2:]), np.float32)
    rnn[1, 0] = dr.rnn[blk, b].cpu().numpy()
    return obs, act, rew, done, rnn


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode", ["fused", "pair"])
def test_r2d2_step_chain_vs_oracle(cuda, mode):
    import torch
    import paper_1909_01500_b200 as rpl
    from synth.device import make_ring_device
    dev = torch.device("cuda")
    dr = make_ring_device(4242, CAP, B, dev, ep_len=25.0, period=PERIOD, rnn_h=512, cursor=1234)
    n_leaves = (CAP // PERIOD) * B
    # initial priorities of every valid sequence leaf (oracle window rule, §8c #16)
    valid = [blk * B + b for blk in range(CAP // PERIOD)
             if OG.window_valid_sequence(blk * PERIOD, CAP, dr.cursor, dr.size, K, L) for b in range(B)]
    g = np.random.default_rng(77)
    td0 = np.abs(g.normal(size=len(valid))).astype(np.float32)
    tree = rpl.SumTree(n_leaves, 32, 32, device=dev)
    tree.update(torch.tensor(valid, dtype=torch.int64, device=dev), torch.from_numpy(td0).to(dev), ALPHA, EPS_P)
    orc = OS.SumTreeOracle(n_leaves)
    orc.update(valid, [float(x) for x in td0], ALPHA, EPS_P)
    # per-step inputs: the learner's per-step |delta| of the previous batch and target-net Q
    steps_td = [np.abs(g.normal(size=(TRAIN, N))).astype(np.float32) for _ in range(2 * P)]
    steps_q = [g.normal(0, 10, (L, N)).astype(np.float32) for _ in range(2 * P)]
    td_dev = [torch.from_numpy(x).to(dev) for x in steps_td]
    q_dev = [torch.from_numpy(x).to(dev) for x in steps_q]
    idx_b = [torch.full((N,), -1, dtype=torch.int64, device=dev) for _ in range(P)]
    q_b = [torch.zeros(N, dtype=torch.int64, device=dev) for _ in range(P)]
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    tg = dict(lo=BURN, T=TRAIN, n_step=NS, gamma=GAMMA, rescale=True, eps=EPS, q=q_dev[0])
    plans = [rpl.GatherPlan(dr, N, kind="sequence", k=K, seq_len=L, period=PERIOD, with_weights=True, targets=tg)
             for _ in range(P)]
    lib, P_ = rpl._lib.lib, rpl.ops._ptr
    replay_no = [0]

    def step(j):  # graph step j of P; inputs of global step r*P + j are copied into slot j
        s = rpl.ops._stream(dev)
        cur, prev = idx_b[j], idx_b[(j - 1) % P]
        rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(prev), P_(td_slot[j]), TRAIN, N,
                                                  ETA, ALPHA, EPS_P, 0, None, s), "update_seq")
        if mode == "fused":
            plans[j].run_sample(tree, SEED, cur, q_b[j], beta=BETA, err=err, stream=s, q_tgt=q_slot[j])
            return
        rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), N, SEED, BETA, P_(cur),
                                                     P_(q_b[j]), None, None, P_(err), s), "sample")
        plans[j].run(cur, q=q_b[j], qmin=None, beta=BETA, err=err, stream=s, q_tgt=q_slot[j])

    td_slot = [torch.empty_like(td_dev[0]) for _ in range(P)]
    q_slot = [torch.empty_like(q_dev[0]) for _ in range(P)]
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for j in range(P):
            step(j)
    torch.cuda.synchronize()

    prev_o = []
    ctr = 0
    for rep in range(2):
        for j in range(P):
            td_slot[j].copy_(td_dev[rep * P + j])
            q_slot[j].copy_(q_dev[rep * P + j])
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        assert int(err.cpu()[0]) & ~1 == 0  # RPL_DERR_IDX only from the first step's -1 padding
        for j in range(P):
            i = rep * P + j
            # ---- oracle chain: update (eta-mixed sequence priorities) -> sample -> gather -> targets
            if prev_o:
                orc.update(prev_o, [OPR.sequence_td(steps_td[i][:, c], ETA) for c in range(N)], ALPHA, EPS_P)
            draws = OP.draws_u64(SEED, ctr, N)
            ctr += N
            oi, oq, oqmin = orc.sample(N, draws)
            idx = [int(x) for x in idx_b[j].cpu().tolist()]
            assert idx == oi, (i, "indices")
            assert [int(x) for x in q_b[j].cpu().tolist()] == oq, (i, "q")
            out = {k_: v.cpu().numpy() for k_, v in plans[j].outputs.items()}
            check_rel(out["w"], OS.is_weights(oq, orc.total(), n_leaves, BETA), what=f"w step {i}")
            for c, leaf in enumerate(oi):
                obs, act, rew, done, rnn = _window(dr, leaf)
                ref = OG.gather_sequences(np.array([1], np.int64), 1, obs, act, rew, done, rnn, K, L, 8)
                for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
                    assert np.array_equal(out[name][:, c], ref[name][:, 0]), (i, c, name)
                Tn = TRAIN + NS - 1
                yr, dnr = OR.nstep_return(ref["rew"][BURN:BURN + Tn], ref["done"][BURN:BURN + Tn], NS, GAMMA,
                                          q=steps_q[i][BURN:BURN + Tn, c:c + 1],
                                          q_boot=steps_q[i][BURN + Tn, c:c + 1], rescale=True, eps=EPS)
                check_rel(out["tgt"][:, c], yr[:, 0], np.abs(yr[:, 0]) + 1e-3, what=f"targets step {i} seq {c}")
                assert np.array_equal(out["tgt_done"][:, c], dnr[:, 0]), (i, c)
            prev_o = oi
        # the tree after the replay: leaves bit-equal, root = exact sum
        assert [int(x) for x in tree.leaves.cpu().tolist()] == orc.q
        assert int(tree.total().cpu()[0]) == orc.total()
    # episode starts inside stacks did occur (short episodes), so the padding path was compared
    starts = sum(int((plans[j].outputs["done"][:-1].cpu().numpy() != 0).sum()) for j in range(P))
    assert starts > 0
    del dr
    torch.cuda.empty_cache()
