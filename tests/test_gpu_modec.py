"""Mode C end to end on one GPU: two ranks (gloo, both on cuda:0) each own half of the
ring columns and one sum tree; the compacted sharded sampler + rpl_gather (unique rows +
episode-start offsets) with n_active / col_offset write every owned sequence straight into
rank 0's batch buffers (mapped through CUDA IPC, CentralBatch); rank 0 re-stacks the frames
(rpl_stack_frames) and checks the whole central batch against the oracle gather of the
global sample (sharded == concatenated, §8c #17)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PERIOD, L, K, CAP, B_TOT, N_PER = 40, 45, 4, 400, 4, 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rings():
    from synth import make_ring
    return [make_ring(300 + r, cap=CAP, B=B_TOT // 2, ep_len=20.0, period=PERIOD, rnn_h=16, reward_kind="r2d2")
            for r in range(2)]


def _worker(rank, world, port, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1909_01500_b200 as rpl
    from paper_1909_01500_b200.replay import leaves_of, valid_sequence_blocks
    from paper_1909_01500_b200.shard import CentralBatch, ShardedSampler
    dev = torch.device("cuda", 0)
    host = _rings()[rank]
    ring = rpl.GatherRing(obs=torch.from_numpy(host.obs).to(dev), act=torch.from_numpy(host.act).to(dev),
                          rew=torch.from_numpy(host.rew).to(dev), done=torch.from_numpy(host.done).to(dev),
                          cursor=host.cursor, size=host.size, rnn=torch.from_numpy(host.rnn).to(dev))
    Bl = B_TOT // 2
    n_leaves = (CAP // PERIOD) * Bl
    tree = rpl.SumTree(n_leaves, 32, device=dev)
    valid = leaves_of(valid_sequence_blocks(CAP, PERIOD, host.cursor, host.size, K, L), Bl)
    g = np.random.default_rng(5 + rank)
    tree.update(torch.from_numpy(valid).to(dev), torch.from_numpy(np.abs(g.normal(size=valid.size)).astype(np.float32)).to(dev), 0.9)
    smp = ShardedSampler(tree, N_PER, seed=17, compact=True)
    n_glob = N_PER * world
    want = ["obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn", "start"]
    root_plan = rpl.GatherPlan(ring, n_glob, kind="sequence", k=K, seq_len=L, period=PERIOD, with_weights=True,
                               out_mode=1, want=want) if rank == 0 else None
    cb = CentralBatch(root_plan.outputs if rank == 0 else None)
    plan = root_plan if rank == 0 else rpl.GatherPlan(ring, n_glob, kind="sequence", k=K, seq_len=L, period=PERIOD,
                                                      with_weights=True, out_mode=1, want=want, outputs=cb.outputs)
    plan.desc.n_active = smp.count.data_ptr()
    plan.desc.col_offset = smp.count.data_ptr() + 8
    cb.attach(plan)  # completion flag (K8) instead of a collective
    if rank == 0:
        for t in cb.outputs.values():
            t.zero_()
    dist.barrier()
    idx, q, w = smp.sample(0.6)  # compacted: this rank's LOCAL leaves first
    plan.run(idx, q=q, qmin=smp.qmin, beta=0.6)
    if rank == 0:
        cb.wait()  # spins until both ranks' gathers signalled (st.release.sys flags)
    torch.cuda.synchronize()
    # every rank reports its global sample (compacted) so rank 0 can rebuild the global order
    m = int(smp.count[0].item())
    mine = [rank * n_leaves + int(x) for x in idx[:m].cpu()]
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        res = {name: t.cpu().numpy() for name, t in cb.outputs.items()}
        # learner side: k-stacks rebuilt from the shipped unique rows + episode-start offsets
        res["obs"] = rpl.stack_frames(cb.outputs["obs"], cb.outputs["start"], K).cpu().numpy()
        queue.put((parts, res, n_leaves))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_mode_c_central_batch(cuda):
    import torch.multiprocessing as mp
    from oracle import gather as OG
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    parts, res, n_leaves = qu.get(timeout=280)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glob = parts[0] + parts[1]           # stratum order: rank 0's run precedes rank 1's
    assert len(glob) == 2 * N_PER
    rings = _rings()
    for col, gl in enumerate(glob):
        r, leaf = divmod(gl, n_leaves)
        h = rings[r]
        ref = OG.gather_sequences(np.array([leaf], np.int64), B_TOT // 2, h.obs, h.act, h.rew, h.done, h.rnn, K, L,
                                  PERIOD)
        for name in ("obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn"):
            assert np.array_equal(res[name][:, col], ref[name][:, 0]), (name, col)
    # IS weights and the sample itself vs the oracle: sharded sampling == sampling the
    # shard-major concatenation (§8c #17) with the same Philox stream; weights normalised by
    # the global batch max (§8c #10)
    from oracle import philox as OP
    from oracle import sumtree as OS
    from tests._tol import check_rel
    shards = []
    for r, h in enumerate(rings):
        Bl = B_TOT // 2
        o = OS.SumTreeOracle((CAP // PERIOD) * Bl)
        valid = [blk * Bl + b for blk in range(CAP // PERIOD)
                 if OG.window_valid_sequence(blk * PERIOD, CAP, h.cursor, h.size, K, L) for b in range(Bl)]
        g = np.random.default_rng(5 + r)
        td = np.abs(g.normal(size=len(valid))).astype(np.float32)
        o.update(valid, [float(x) for x in td], 0.9)
        shards.append(o)
    n_glob = 2 * N_PER
    oi, oq, _ = OS.sharded_sample(shards, n_glob, OP.draws_u64(17, 0, n_glob))
    assert glob == oi
    Q = sum(sh.total() for sh in shards)
    check_rel(res["w"], OS.is_weights(oq, Q, 2 * n_leaves, 0.6), what="mode C w")
