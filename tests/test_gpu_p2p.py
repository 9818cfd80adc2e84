"""GPU tests of the peer-board exchanges (rpl.h RPL_BOARD_WORDS; SURVEY.md §8e K5 / K7
without NCCL): G 'ranks' in one process on one GPU, each with its own tree, ring and board,
their kernels launched on separate streams so they run concurrently and spin on each
other's slots.  The fused sampler must equal the oracle's sample of the concatenated trees
(bit-exact), and the fused gather must equal a plain gather given the global batch min."""
import numpy as np
import pytest

from oracle import philox as OP
from oracle import sumtree as OS
from synth import rng, td_abs

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


def _shards(rpl, G, n_local, seed, empty=()):
    g = rng(seed)
    trees, orcs = [], []
    for s in range(G):
        t = rpl.SumTree(n_local, 32)
        o = OS.SumTreeOracle(n_local)
        if s not in empty:
            td = td_abs(g, n_local) * (1 + s)
            t.update(T_(np.arange(n_local, dtype=np.int64)), T_(td), 0.9)
            o.update(list(range(n_local)), [float(x) for x in td], 0.9)
        trees.append(t)
        orcs.append(o)
    return trees, orcs


@pytest.mark.parametrize("G,empty", [(2, ()), (3, ()), (2, (1,)), (4, (0, 2))])
def test_p2p_sampler_equals_oracle(rpl, G, empty):
    import torch
    from paper_1909_01500_b200.shard import PeerBoards
    n_local, n, seed = 3000, 96, 7
    trees, orcs = _shards(rpl, G, n_local, 40 + G, empty)
    boards = [torch.zeros(6 * G, dtype=torch.int64, device="cuda") for _ in range(G)]
    ptrs = PeerBoards.local(boards)
    streams = [torch.cuda.Stream() for _ in range(G)]
    errs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(G)]
    counts = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()
    for step in range(3):
        outs = []
        for r in range(G):  # all launched before any completes: they wait on each other
            with torch.cuda.stream(streams[r]):
                outs.append(trees[r].sample_sharded_p2p(r, G, ptrs, n, seed, counts[r], err=errs[r]))
        torch.cuda.synchronize()
        ref_idx, ref_q, _ = OS.sharded_sample(orcs, n, OP.draws_u64(seed, step * n, n))
        got_i, got_q = [], []
        for r in range(G):
            m = int(H(counts[r])[0])
            i, q = H(outs[r][0]), H(outs[r][1])
            assert np.all(i[m:] == -1) and np.all(q[m:] == 0)
            got_i += (i[:m] + r * n_local).tolist()
            got_q += q[:m].tolist()
            assert int(H(errs[r])[0]) == 0
        assert got_i == ref_idx and got_q == ref_q
        for r in range(G):  # every board holds every rank's total under this step's tag
            b = H(boards[r])
            assert b[1:2 * G:2].tolist() == [(step + 1) * n] * G
            assert b[0:2 * G:2].tolist() == [o.total() for o in orcs]


@pytest.mark.parametrize("empty", [(), (1,)])
def test_p2p_gather_weights(rpl, empty):
    # K7 fused into the sequence gather: the IS weights use the min over every rank's owned q;
    # every output equals a plain gather given that global min (bit-exact).  A rank that owns
    # nothing still publishes (INT64_MAX) so its peers do not wait.
    import torch
    from paper_1909_01500_b200 import replay as R
    from paper_1909_01500_b200.shard import PeerBoards
    from synth.device import make_ring_device
    G, cap, B, period, L, k, n = 2, 400, 4, 40, 45, 4, 8
    dev = torch.device("cuda")
    rings, trees = [], []
    for r in range(G):
        ring = make_ring_device(300 + r, cap, B, dev, ep_len=30.0, period=period, rnn_h=8, cursor=123,
                                frame_shape=(8, 16))
        t = rpl.SumTree((cap // period) * B, 32)
        if r not in empty:
            valid = R.leaves_of(R.valid_sequence_blocks(cap, period, ring.cursor, ring.size, k, L), B)
            t.update(T_(valid), T_(td_abs(rng(r), valid.size)), 0.9)
        rings.append(ring)
        trees.append(t)
    boards = [torch.zeros(6 * G, dtype=torch.int64, device=dev) for _ in range(G)]
    ptrs = PeerBoards.local(boards)
    streams = [torch.cuda.Stream() for _ in range(G)]
    errs = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(G)]
    counts = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(G)]
    plans, refs = [], []
    for r in range(G):
        p = rpl.GatherPlan(rings[r], n * G, kind="sequence", k=k, seq_len=L, period=period, with_weights=True)
        p.desc.n_active = counts[r].data_ptr()
        p.set_peers(ptrs, G, r)
        plans.append(p)
        q_ = rpl.GatherPlan(rings[r], n * G, kind="sequence", k=k, seq_len=L, period=period, with_weights=True)
        q_.desc.n_active = counts[r].data_ptr()
        refs.append(q_)
    torch.cuda.synchronize()
    for step in range(3):
        res = []
        for r in range(G):
            with torch.cuda.stream(streams[r]):
                idx, q = trees[r].sample_sharded_p2p(r, G, ptrs, n * G, 5, counts[r], err=errs[r])
                plans[r].run(idx, q=q, beta=0.6, err=errs[r])
                res.append((idx, q))
        torch.cuda.synchronize()
        mins = []
        for r in range(G):
            m = int(H(counts[r])[0])
            qq = H(res[r][1])[:m]
            mins.append(int(qq.min()) if m else (1 << 63) - 1)
        gmin = torch.tensor([min(mins)], dtype=torch.int64, device=dev)
        for r in range(G):
            assert int(H(errs[r])[0]) == 0, (step, r)
            out_ref = refs[r].run(res[r][0], q=res[r][1], qmin=gmin, beta=0.6)
            torch.cuda.synchronize()
            m = int(H(counts[r])[0])
            for name in out_ref:  # the m active columns (the rest are untouched by both)
                a, b_ = H(plans[r].outputs[name]), H(out_ref[name])
                if name == "w":
                    a, b_ = a[:m], b_[:m]
                else:
                    a, b_ = a[:, :m], b_[:, :m]
                assert np.array_equal(a, b_), (step, r, name)
            b = H(boards[r])
            assert b[2 * G:4 * G:2].tolist() == mins


def test_p2p_timeout_fails_loudly(cuda):
    # a peer that never publishes: after ~2 s the sampler sets RPL_DERR_PEER and traps, so the
    # step fails at the next synchronisation (run in a child process: the trap ends its context)
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = """
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1909_01500_b200 as rpl
t = rpl.SumTree(100, 32)
t.update(torch.arange(100, device="cuda"), torch.ones(100, device="cuda"), 0.9)
boards = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(2)]
ptrs = torch.tensor([b.data_ptr() for b in boards], dtype=torch.int64, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
t.sample_sharded_p2p(0, 2, ptrs, 16, 1, cnt, err=err)
try:
    torch.cuda.synchronize()
except RuntimeError as e:
    print("FAILED-LOUDLY", str(e).splitlines()[0])
    sys.exit(3)
print("CONTINUED", int(err.cpu()[0]))
""" % root
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert res.returncode == 3 and "FAILED-LOUDLY" in res.stdout, (res.returncode, res.stdout, res.stderr[-500:])


def test_p2p_prefilled_peer(rpl):
    # one rank's kernels alone, the peer's slots pre-written by the host with the step's tag
    # (no concurrent kernel needed: also the sanitizer-friendly form of the protocol)
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    G, cap, B, period, L, k, n = 2, 400, 4, 40, 45, 4, 8
    dev = torch.device("cuda")
    ring = make_ring_device(301, cap, B, dev, ep_len=30.0, period=period, rnn_h=8, cursor=123, frame_shape=(8, 16))
    t = rpl.SumTree((cap // period) * B, 32)
    valid = R.leaves_of(R.valid_sequence_blocks(cap, period, ring.cursor, ring.size, k, L), B)
    td = td_abs(rng(3), valid.size)
    t.update(T_(valid), T_(td), 0.9)
    o = OS.SumTreeOracle(t.n_leaves)
    o.update([int(x) for x in valid], [float(x) for x in td], 0.9)
    peer = OS.SumTreeOracle(t.n_leaves)  # rank 1: a copy of rank 0's shard
    peer.q = list(o.q)
    tag = n * G                           # stream position after the first step
    board = torch.zeros(6 * G, dtype=torch.int64, device=dev)
    board[2 * 1], board[2 * 1 + 1] = peer.total(), tag           # rank 1's K5 slot
    ptrs = torch.tensor([board.data_ptr(), board.data_ptr()], dtype=torch.int64, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    idx, q = t.sample_sharded_p2p(0, G, ptrs, n * G, 5, cnt, err=err)
    torch.cuda.synchronize()
    ref_idx, ref_q, _ = OS.sharded_sample([o, peer], n * G, OP.draws_u64(5, 0, n * G))
    m = int(H(cnt)[0])
    own = [(i, qq) for i, qq in zip(ref_idx, ref_q) if i < t.n_leaves]
    assert m == len(own) and H(idx)[:m].tolist() == [i for i, _ in own] and H(q)[:m].tolist() == [qq for _, qq in own]
    peer_min = min(qq for i, qq in zip(ref_idx, ref_q) if i >= t.n_leaves)
    board[2 * G + 2], board[2 * G + 3] = peer_min, tag          # rank 1's K7 slot
    plan = rpl.GatherPlan(ring, n * G, kind="sequence", k=k, seq_len=L, period=period, with_weights=True)
    plan.desc.n_active = cnt.data_ptr()
    plan.set_peers(ptrs, G, 0)
    out = plan.run(idx, q=q, beta=0.6, err=err)
    torch.cuda.synchronize()
    assert int(H(err)[0]) == 0
    gmin = min(min(qq for _, qq in own), peer_min)
    w = H(out["w"])[:m]
    ref_w = [(gmin / qq) ** 0.6 for _, qq in own]
    assert np.allclose(w, ref_w, rtol=1e-6, atol=0)
    assert int(H(board)[2 * G]) == min(qq for _, qq in own) and int(H(board)[2 * G + 1]) == tag
