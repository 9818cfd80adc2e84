"""GPU tests of the asynchronous replay pipeline (NEXT-2, paper_1909_01500_b200/pipeline.py):
(1) with flush() before each learner step the schedule is deterministic and every sampled
batch equals the oracle's (tree maintained by appends + eta-mixed updates, Philox stream
draws, naive full-stack gather); (2) without flushes, copies overlap learner steps and every
gathered sequence still equals the ring content the host submitted (no torn or overwritten
rows), with the replay ratio under its cap."""
import numpy as np
import pytest

from oracle import gather as OG
from oracle import philox as OP
from oracle import priority as OPR
from oracle import sumtree as OS
from synth import rng

pytestmark = pytest.mark.gpu

CAP, B, K, PERIOD, L, TB, N = 240, 3, 4, 20, 45, 40, 6


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def H(t):
    return t.cpu().numpy()


def _setup(rpl, cap_ratio):
    import torch
    from paper_1909_01500_b200.pipeline import ReplayPipeline
    dev = torch.device("cuda")
    ring = rpl.GatherRing(obs=torch.zeros((CAP, B, 8, 16), dtype=torch.uint8, device=dev),
                          act=torch.zeros((CAP, B), dtype=torch.int64, device=dev),
                          rew=torch.zeros((CAP, B), dtype=torch.float32, device=dev),
                          done=torch.zeros((CAP, B), dtype=torch.uint8, device=dev), cursor=0, size=0,
                          rnn=torch.zeros((CAP // PERIOD, B, 2, 4), dtype=torch.float32, device=dev))
    tree = rpl.SumTree((CAP // PERIOD) * B, 32)
    pipe = ReplayPipeline(ring, tree, "sequence", TB, k=K, seq_len=L, period=PERIOD, train_steps=L, cap=cap_ratio)
    plan = rpl.GatherPlan(ring, N, kind="sequence", k=K, seq_len=L, period=PERIOD, with_weights=True)
    return ring, tree, pipe, plan


def _fill(pipe, g, host):
    hb = pipe.host_batch()
    t = hb.tensors
    c0 = pipe.ring.cursor
    obs = g.integers(0, 256, t["obs"].shape, dtype=np.uint8)
    act = g.integers(0, 18, t["act"].shape).astype(np.int64)
    rew = g.normal(size=t["rew"].shape).astype(np.float32)
    done = (g.random(t["done"].shape) < 0.05).astype(np.uint8)
    rows = pipe.rnn_rows()
    rnn = g.normal(size=(len(rows), B, 2, 4)).astype(np.float32)
    t["obs"].numpy()[...] = obs
    t["act"].numpy()[...] = act
    t["rew"].numpy()[...] = rew
    t["done"].numpy()[...] = done
    if rows:
        t["rnn"].numpy()[:len(rows)] = rnn
    rr = [(c0 + i) % CAP for i in range(TB)]
    host["obs"][rr], host["act"][rr], host["rew"][rr], host["done"][rr] = obs, act, rew, done
    for j, i in enumerate(rows):
        host["rnn"][((c0 + i) % CAP) // PERIOD] = rnn[j]
    pipe.submit(hb)


def _host():
    return {"obs": np.zeros((CAP, B, 8, 16), np.uint8), "act": np.zeros((CAP, B), np.int64),
            "rew": np.zeros((CAP, B), np.float32), "done": np.zeros((CAP, B), np.uint8),
            "rnn": np.zeros((CAP // PERIOD, B, 2, 4), np.float32)}


def test_pipeline_deterministic_vs_oracle(rpl):
    import torch
    ring, tree, pipe, plan = _setup(rpl, cap_ratio=10.0)
    host = _host()
    g = rng(61)
    nl = (CAP // PERIOD) * B
    orc = OS.SumTreeOracle(nl)
    cursor, size, ctr = 0, 0, 0
    idx = [torch.full((N,), -1, dtype=torch.int64, device="cuda") for _ in range(2)]
    q = torch.zeros(N, dtype=torch.int64, device="cuda")
    prev_td = None
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for it in range(10):
        _fill(pipe, g, host)
        c1, s1 = (cursor + TB) % CAP, min(CAP, size + TB)
        for leaf in range(nl):  # oracle validity maintenance (§8c #16)
            blk = leaf // B
            v0 = size > 0 and OG.window_valid_sequence(blk * PERIOD, CAP, cursor, size, K, L)
            v1 = OG.window_valid_sequence(blk * PERIOD, CAP, c1, s1, K, L)
            if v0 != v1:
                orc.q[leaf] = orc.max_seen if v1 else 0
        cursor, size = c1, s1
        pipe.flush()
        if orc.total() == 0:
            continue
        cur, prev = idx[it % 2], idx[(it + 1) % 2]
        has_prev = prev_td is not None
        out = pipe.step(N, prev if has_prev else None, torch.from_numpy(prev_td).cuda() if has_prev else None, plan,
                        cur, q, seed=9, alpha=0.9, beta=0.6, err=err)
        if has_prev:
            pv = [int(x) for x in H(prev)]
            orc.update(pv, [OPR.sequence_td(prev_td[:, j], 0.9) for j in range(N)], 0.9, live_only=True)
        oi, oq, _ = orc.sample(N, OP.draws_u64(9, ctr, N))
        ctr += N
        torch.cuda.synchronize()
        assert H(cur).tolist() == oi and H(q).tolist() == oq
        ref = OG.gather_sequences(np.array(oi), B, host["obs"], host["act"], host["rew"], host["done"], host["rnn"],
                                  K, L, PERIOD)
        for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
            assert np.array_equal(H(out[name]), ref[name]), (it, name)
        prev_td = np.abs(g.normal(size=(L, N))).astype(np.float32)
        e = int(H(err)[0])
        if e:
            ages = [((cursor - 1 - (i // B) * PERIOD) % CAP, size) for i in oi]
            raise AssertionError(f"it {it}: err {e}, cursor {cursor} size {size} desc {plan.desc.cursor} "
                                 f"{plan.desc.size} ages {ages}")
    assert int(H(err)[0]) == 0


def test_pipeline_overlapped_integrity(rpl):
    import torch
    ring, tree, pipe, plan = _setup(rpl, cap_ratio=1.0)
    host = _host()
    g = rng(62)
    idx = [torch.full((N,), -1, dtype=torch.int64, device="cuda") for _ in range(2)]
    q = torch.zeros(N, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    checks = 0
    for it in range(40):
        _fill(pipe, g, host)                  # no flush: copies run while the learner steps
        snap = {k: v.copy() for k, v in host.items()}
        for j in range(3):
            if not pipe.can_step(N):
                break
            if it < 3:
                pipe.flush()
            cur = idx[(it * 3 + j) % 2]
            out = pipe.step(N, None, None, plan, cur, q, seed=5, alpha=0.9, beta=0.6, err=err)
            pipe.learn_stream.synchronize()
            ii = H(cur)
            if (ii < 0).any():
                continue
            ref = OG.gather_sequences(ii, B, snap["obs"], snap["act"], snap["rew"], snap["done"], snap["rnn"], K, L,
                                      PERIOD)
            for name in ("obs", "rew", "done", "rnn"):
                assert np.array_equal(H(out[name]), ref[name]), (it, j, name)
            checks += 1
        assert pipe.throttle.consumed <= pipe.throttle.cap * pipe.throttle.generated
    torch.cuda.synchronize()
    assert checks > 10 and int(H(err)[0]) == 0


@pytest.mark.parametrize("kind", ["sequence", "transition"])
def test_pipeline_initial_priorities(rpl, kind):
    # NEXT-1 (R33): with init_priority, every valid leaf holds the priority of its n-step TD
    # errors over the rows the ring holds (leaves cannot change rows while valid); invalid
    # leaves hold 0.  Checked after every append against the oracle.
    import torch
    from oracle import targets as OT
    from paper_1909_01500_b200.pipeline import ReplayPipeline
    dev = torch.device("cuda")
    ring = rpl.GatherRing(obs=torch.zeros((CAP, B, 8, 16), dtype=torch.uint8, device=dev),
                          act=torch.zeros((CAP, B), dtype=torch.int64, device=dev),
                          rew=torch.zeros((CAP, B), dtype=torch.float32, device=dev),
                          done=torch.zeros((CAP, B), dtype=torch.uint8, device=dev), cursor=0, size=0,
                          rnn=torch.zeros((CAP // PERIOD, B, 2, 4), dtype=torch.float32, device=dev))
    ip = dict(n=5 if kind == "sequence" else 3, gamma=0.997, rescale=kind == "sequence", alpha=0.9, eta=0.9,
              burn_in=10)
    if kind == "sequence":
        nl = (CAP // PERIOD) * B
        pipe = ReplayPipeline(ring, rpl.SumTree(nl, 32), "sequence", TB, k=K, seq_len=L, period=PERIOD,
                              train_steps=30, init_priority=ip)
    else:
        nl = CAP * B
        pipe = ReplayPipeline(ring, rpl.SumTree(nl, 32), "transition", TB, k=K, n_step=3, init_priority=ip)
    host = _host()
    hq = {"q_taken": np.zeros((CAP, B), np.float32), "q_boot": np.zeros((CAP, B), np.float32)}
    g = rng(64)
    for it in range(9):
        hb_next = pipe._bufs[pipe._next]
        hb_next.ready.synchronize()  # its previous copy has finished
        c0 = ring.cursor
        for name in ("q_taken", "q_boot"):  # the actor's values for the rows of this batch
            v = g.normal(0, 3, (TB, B)).astype(np.float32)
            hb_next.tensors[name].numpy()[...] = v
            hq[name][[(c0 + i) % CAP for i in range(TB)]] = v
        if kind == "sequence":
            _fill(pipe, g, host)
        else:
            hb = pipe.host_batch()
            t = hb.tensors
            t["obs"].numpy()[...] = g.integers(0, 256, t["obs"].shape, dtype=np.uint8)
            rew = g.normal(size=(TB, B)).astype(np.float32)
            done = (g.random((TB, B)) < 0.05).astype(np.uint8)
            t["rew"].numpy()[...] = rew
            t["done"].numpy()[...] = done
            rr = [(c0 + i) % CAP for i in range(TB)]
            host["rew"][rr], host["done"][rr] = rew, done
            pipe.submit(hb)
        pipe.flush()
        pipe.learn_stream.synchronize()
        leaves = H(pipe.tree.leaves)
        cur, size = ring.cursor, ring.size
        if kind == "sequence":
            from paper_1909_01500_b200 import replay as RP
            valid = RP.valid_sequence_blocks(CAP, PERIOD, cur, size, K, L)
            orc = OS.SumTreeOracle(nl)
            for blk in valid:
                p = OT.initial_sequence_priorities(host["rew"], host["done"], hq["q_taken"], hq["q_boot"], int(blk),
                                                   PERIOD, 10, 30, 5, 0.997, 0.9, rescale=True)
                orc.update([int(blk) * B + b for b in range(B)], p, 0.9)
            units = set(int(x) * B + b for x in valid for b in range(B))
        else:
            from paper_1909_01500_b200 import replay as RP
            valid = RP.valid_transition_rows(CAP, cur, size, K, 3)
            orc = OS.SumTreeOracle(nl)
            for r in valid:
                td = OT.ring_td_abs(host["rew"], host["done"], hq["q_taken"], hq["q_boot"], int(r), 1, 3,
                                    0.997).astype(np.float32)
                orc.update([int(r) * B + b for b in range(B)], [float(x) for x in td[0]], 0.9)
            units = set(int(x) * B + b for x in valid for b in range(B))
        ref = np.array(orc.q, np.int64)
        for leaf in range(nl):
            if leaf in units:
                assert abs(int(leaves[leaf]) - int(ref[leaf])) <= 1e-6 * ref[leaf] + 2, (it, leaf)
            else:
                assert leaves[leaf] == 0, (it, leaf)
        tot = int(H(pipe.tree.total())[0])
        assert tot == int(leaves.sum())
    assert len(units) > 0
