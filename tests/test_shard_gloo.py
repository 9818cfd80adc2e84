"""World-size-2 gloo test of the Mode-L sharded sampling protocol
(paper_1909_01500_b200/shard.py) on CPU.  The per-rank tree is an oracle-backed
stand-in with the rpl SumTree interface (the kernels themselves are covered by
tests/test_gpu_sumtree.py::test_sharded_equals_concatenated); what is tested
here is the exchange: all-gather of totals, shared strata, ownership split and
the global batch-min for the IS weights."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import philox as OP
from oracle import sumtree as OS

N_LOCAL, N_PER_RANK, SEED, STEPS, BETA = 40, 8, 99, 3, 0.6


class OracleShardTree:
    """CPU stand-in with the SumTree methods ShardedSampler calls."""

    def __init__(self, q):
        self.o = OS.SumTreeOracle(len(q), 0)
        self.o.q = list(q)
        self.n_leaves = len(q)
        self.device = torch.device("cpu")
        self.pos = 0  # Philox stream position (tree header word 2)

    def total(self, out):
        out[0] = self.o.total()
        return out

    def sample_sharded(self, rank, n_shards, shard_totals, n, seed=0, out=None, use_stream=False, count=None):
        idx, q, qmin = out
        totals = [int(x) for x in shard_totals]
        Q = sum(totals)
        lo_own = sum(totals[:rank])
        draws = OP.draws_u64(seed, self.pos, n)
        self.pos += n
        m = None
        for k in range(n):
            lo, hi = (k * Q) // n, ((k + 1) * Q) // n
            prefix = lo + ((draws[k] * (hi - lo)) >> 64)
            if lo_own <= prefix < lo_own + totals[rank]:
                i = self.o.find(prefix - lo_own)
                idx[k] = rank * self.n_leaves + i
                q[k] = self.o.q[i]
                m = q[k].item() if m is None else min(m, q[k].item())
            else:
                idx[k] = -1
                q[k] = 0
        qmin[0] = m if m is not None else (1 << 63) - 1
        if count is not None:  # compacted output (rpl_sumtree_sample_sharded with out_count)
            own = idx >= 0
            c = int(own.sum())
            idx[:c], q[:c] = idx[own].clone() - rank * self.n_leaves, q[own].clone()  # local leaves
            idx[c:], q[c:] = -1, 0
            count[0] = c
            count[1] = int(np.nonzero(own.numpy())[0][0]) if c else 0


    # buffer-wide normaliser (R29): {total, min} records, compacted pairs sampler
    def total_min(self, out):
        out[0] = self.o.total()
        out[1] = OS.buffer_min(self.o.q)
        return out

    def sample_sharded_pairs(self, rank, n_shards, pairs, n, seed, count, out=None, bufmin=None):
        idx, q, qmin = out
        self.sample_sharded(rank, n_shards, pairs[:, 0].contiguous(), n, seed=seed, out=out, use_stream=True,
                            count=count)
        bufmin[0] = min(int(x) for x in pairs[:, 1])
        return idx, q, qmin, bufmin


def cpu_is_weights(q, qmin, beta, out):
    m = float(qmin[0])
    for k in range(q.numel()):
        out[k] = (m / float(q[k])) ** beta if q[k] > 0 else 0.0


def leaves_of(rank):
    g = np.random.default_rng(1000 + rank)
    return [int(x) for x in g.integers(1, 1 << 20, N_LOCAL)]


def worker(rank, world, port, queue, compact=False, buffer_norm=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_01500_b200.shard import ShardedSampler
    tree = OracleShardTree(leaves_of(rank))
    smp = ShardedSampler(tree, N_PER_RANK, SEED, is_weights=cpu_is_weights, compact=compact, buffer_norm=buffer_norm)
    res = []
    for _ in range(STEPS):
        idx, q, w = smp.sample(BETA)
        res.append((idx.clone().numpy(), q.clone().numpy(), w.clone().numpy(), smp.totals.clone().numpy(),
                    int(smp.count[0])))
    queue.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_mode_l_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = []
    for r in range(world):
        t = OS.SumTreeOracle(N_LOCAL, 0)
        t.q = leaves_of(r)
        shards.append(t)
    n_glob = N_PER_RANK * world
    for step in range(STEPS):
        draws = OP.draws_u64(SEED, step * n_glob, n_glob)
        ref_idx, ref_q, ref_qmin = OS.sharded_sample(shards, n_glob, draws)
        merged = np.full(n_glob, -1, np.int64)
        w_merged = np.zeros(n_glob)
        for r in range(world):
            idx, qq, w, totals, _ = out[r][step]
            assert list(totals) == [sum(s.q) for s in shards]          # K5 all-gather
            own = idx >= 0
            assert not (merged[own] >= 0).any()                          # disjoint ownership
            merged[own] = idx[own]
            w_merged[own] = w[own]
            pos = np.nonzero(own)[0]
            if pos.size:
                assert pos[-1] - pos[0] + 1 == pos.size                  # one contiguous run of strata
        assert list(merged) == ref_idx                                   # == concatenated oracle
        ref_w = OS.is_weights(ref_q, sum(sum(s.q) for s in shards), world * N_LOCAL, BETA)
        np.testing.assert_allclose(w_merged, ref_w, rtol=1e-6)           # K7 global batch min (f32)


@pytest.mark.timeout(120)
def test_mode_l_two_ranks_gloo_compacted():
    # compacted protocol: each rank's owned draws first; concatenating the ranks' first
    # `count` entries in rank order reproduces the global sample in stratum order
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = []
    for r in range(world):
        t = OS.SumTreeOracle(N_LOCAL, 0)
        t.q = leaves_of(r)
        shards.append(t)
    n_glob = N_PER_RANK * world
    for step in range(STEPS):
        draws = OP.draws_u64(SEED, step * n_glob, n_glob)
        ref_idx, ref_q, _ = OS.sharded_sample(shards, n_glob, draws)
        merged, merged_w = [], []
        for r in range(world):
            idx, qq, w, totals, cnt = out[r][step]
            assert (idx[:cnt] >= 0).all() and (idx[cnt:] == -1).all()
            merged += (idx[:cnt] + r * N_LOCAL).tolist()   # compacted entries are local leaves
            merged_w += w[:cnt].tolist()
        assert merged == ref_idx
        ref_w = OS.is_weights(ref_q, sum(sum(s.q) for s in shards), world * N_LOCAL, BETA)
        np.testing.assert_allclose(merged_w, ref_w, rtol=1e-6)


@pytest.mark.timeout(120)
def test_mode_l_two_ranks_gloo_buffer_normaliser():
    # R29 sharded: one all-gather of {total, min} records; the weights use the global buffer
    # min (PER's (N P_i)^-beta / max over the whole buffer) and there is no K7 all-reduce
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, True, True)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = []
    for r in range(world):
        t = OS.SumTreeOracle(N_LOCAL, 0)
        t.q = leaves_of(r)
        shards.append(t)
    n_glob = N_PER_RANK * world
    N = world * N_LOCAL
    Q = sum(sum(s.q) for s in shards)
    qmin = min(OS.buffer_min(s.q) for s in shards)
    for step in range(STEPS):
        draws = OP.draws_u64(SEED, step * n_glob, n_glob)
        ref_idx, ref_q, _ = OS.sharded_sample(shards, n_glob, draws)
        merged, merged_w = [], []
        for r in range(world):
            idx, qq, w, totals, cnt = out[r][step]
            merged += (idx[:cnt] + r * N_LOCAL).tolist()
            merged_w += w[:cnt].tolist()
        assert merged == ref_idx
        ref_w = [((N * qi / Q) ** -BETA) / ((N * qmin / Q) ** -BETA) for qi in ref_q]
        np.testing.assert_allclose(merged_w, ref_w, rtol=1e-6)
