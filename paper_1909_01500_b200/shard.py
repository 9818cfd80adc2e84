"""Multi-GPU prioritized sampling, Mode L.

One process per GPU (P:64's data-parallel layout).  Each rank holds the ring
columns it samples into and ONE sum tree over its own leaves.  A global
proportional sample over the union of the shards needs one exchange per step:

  K5  all-gather of the G per-shard totals (8 B per rank, NCCL over NVLink);
      every rank then evaluates the SAME global strata (shared counter-based
      Philox stream) and descends only the strata whose prefix falls in its own
      shard (rpl_sumtree_sample_sharded) -- no index scatter is needed;
  K7  all-reduce MIN of the owned batch-min q, so the IS weights are normalised
      by the global batch max weight (§8c #10).

Frames never cross NVLink: each rank gathers its owned samples locally and feeds
its own learner.  With compact=True the owned draws come first as LOCAL leaf indices
(count = [m, k0] on the device), so the rank's update and gather take them directly and
the gather schedules only them (rpl_gather_desc.n_active).  The result equals rpl_sumtree_sample on the shard-major
concatenation of the trees (§8c #17; tests/test_gpu_sumtree.py).

The tree object is duck-typed (total(), sample_sharded(), .device) so the
protocol can be exercised with world-size-2 gloo on CPU (tests/test_shard_gloo.py).

PeerBoards replaces both NCCL exchanges with stores into the peers' memory, fused into
the kernels that need them: the sampler publishes its total and reads everyone's
(rpl_sumtree_sample_sharded_p2p, K5), the gather publishes the batch-min q and reads
everyone's while its frame copy runs (rpl_gather_desc.peer_boards, K7).  The step then has
no collective launch at all: update -> sample -> gather -> n-step, as on one GPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class ShardedSampler:
    def __init__(self, tree, n_per_rank: int, seed: int, group=None, is_weights=None, compact=False,
                 buffer_norm=False):
        """buffer_norm: IS weights normalised over the whole (sharded) buffer (R29): the
        tree carries an attached min-tree and the K5 all-gather exchanges {total, min}
        records — the K7 all-reduce disappears.  Requires compact."""
        self.tree = tree
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n_glob = int(n_per_rank) * self.world
        self.seed = int(seed)
        dev = tree.device
        self.totals = torch.zeros(self.world, dtype=torch.int64, device=dev)
        self.my_total = torch.zeros(1, dtype=torch.int64, device=dev)
        self.idx = torch.full((self.n_glob,), -1, dtype=torch.int64, device=dev)
        self.q = torch.zeros(self.n_glob, dtype=torch.int64, device=dev)
        self.qmin = torch.zeros(1, dtype=torch.int64, device=dev)
        self.w = torch.zeros(self.n_glob, dtype=torch.float32, device=dev)
        self._is_weights = is_weights
        self.compact = bool(compact)
        self.count = torch.zeros(2, dtype=torch.int64, device=dev)  # [owned m, first stratum k0]
        self.buffer_norm = bool(buffer_norm)
        if self.buffer_norm and not self.compact:
            raise ValueError("buffer_norm needs the compacted sampler")
        self.my_pair = torch.zeros(2, dtype=torch.int64, device=dev)
        self.pairs = torch.zeros((self.world, 2), dtype=torch.int64, device=dev)
        self.local_qmin = torch.zeros(1, dtype=torch.int64, device=dev)

    def sample(self, beta: float):
        """One global stratified sample of n_glob draws.  Returns (idx, q, w): idx[k] is
        the GLOBAL leaf (rank * shard_leaves + local) for the draws this rank owns and
        -1 elsewhere; w is normalised by the global batch min q."""
        if self.buffer_norm:  # K5 carries {total, buffer min}; the global min is the normaliser
            self.tree.total_min(out=self.my_pair)
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(self.pairs.view(-1), self.my_pair, group=self.group)
            else:
                dist.all_gather(list(self.pairs.unbind(0)), self.my_pair, group=self.group)
            self.totals.copy_(self.pairs[:, 0])  # (diagnostics only; the sampler reads the pairs)
            self.tree.sample_sharded_pairs(self.rank, self.world, self.pairs, self.n_glob, self.seed, self.count,
                                           out=(self.idx, self.q, self.local_qmin), bufmin=self.qmin)
            wfn = self._is_weights
            if wfn is None:
                from .ops import is_weights as wfn
            wfn(self.q, self.qmin, beta, out=self.w)
            return self.idx, self.q, self.w
        self.tree.total(out=self.my_total)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.totals, self.my_total, group=self.group)      # K5
        else:  # gloo (CPU tests, functional checks): list form
            dist.all_gather(list(self.totals.chunk(self.world)), self.my_total, group=self.group)
        kw = {"count": self.count} if self.compact else {}
        self.tree.sample_sharded(self.rank, self.world, self.totals, self.n_glob, seed=self.seed,
                                 out=(self.idx, self.q, self.qmin), use_stream=True, **kw)
        dist.all_reduce(self.qmin, op=dist.ReduceOp.MIN, group=self.group)                 # K7
        if self._is_weights is None:
            from .ops import is_weights
            is_weights(self.q, self.qmin, beta, out=self.w)
        else:
            self._is_weights(self.q, self.qmin, beta, out=self.w)
        return self.idx, self.q, self.w

    def owned(self):
        """Boolean mask of the draws this rank owns (host sync; diagnostics)."""
        return self.idx >= 0


class CentralBatch:
    """Mode C (BASELINE north_star "gathers the batch back to the learner
    GPU"): the learner rank owns the batch buffers; every other rank maps them through
    CUDA IPC (peer memory over NVLink) so that its gather kernel writes its owned samples
    straight into the learner's batch at their global positions — the transfer is fused
    into the gather, no staging copy and no NCCL send of frames.  Used with a compacted
    ShardedSampler: count = [m, k0] feeds rpl_gather_desc.n_active / col_offset.

    Completion (K8) needs no collective either: the learner also owns a flag word per rank
    (int64 [world], mapped like the outputs).  `attach(plan)` makes a rank's gather signal
    its flag when its last CTA finishes (rpl_gather_desc.done_flag: every store made visible
    at system scope, then st.release.sys of the rank's call counter); on the learner
    `wait()` enqueues rpl_wait_flags, which spins until every rank's flag has reached the
    learner's own call count (fails loudly after ~2 s), so work enqueued after it reads the
    complete batch.  A mapped buffer in another GPU's memory gets peer access from this
    rank's device (rpl_peer_access); all ranks agree on the outcome before raising."""

    def __init__(self, outputs_on_root, group=None, root: int = 0):
        from torch.multiprocessing.reductions import reduce_tensor
        self.group = group
        self.root = root
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        local = torch.device("cuda", torch.cuda.current_device())
        names = sorted(outputs_on_root) if outputs_on_root is not None else None
        if self.rank == root:
            dev = next(iter(outputs_on_root.values())).device
            self.flags = torch.zeros(self.world, dtype=torch.int64, device=dev)
            torch.cuda.synchronize(dev)
            payload = [[(n, reduce_tensor(outputs_on_root[n])) for n in names] +
                       [("__flags__", reduce_tensor(self.flags))]]
        else:
            payload = [None]
        dist.broadcast_object_list(payload, src=root, group=group)
        failure = None
        if self.rank == root:
            self.outputs = dict(outputs_on_root)
        else:
            mapped = {n: fn(*args) for n, (fn, args) in payload[0]}
            self.flags = mapped.pop("__flags__")
            self.outputs = mapped
            failure = self._peer_access(list(mapped.values()) + [self.flags], local)
        ok = torch.tensor([0 if failure else 1], dtype=torch.int32, device=local)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            raise RuntimeError(f"central batch unreachable from some rank ({failure or 'a peer failed'})")
        self.seq = torch.zeros(2, dtype=torch.int64, device=local)  # rpl_gather_desc.done_seq
        self.err = torch.zeros(1, dtype=torch.int32, device=local)

    @staticmethod
    def _peer_access(tensors, local):
        from . import _lib
        for dev_index in sorted({t.device.index for t in tensors if t.device != local}):
            with torch.cuda.device(local):
                rc = _lib.lib.rpl_peer_access(dev_index)
            if rc != 0:
                return f"rpl_peer_access({dev_index}) from {local}: {_lib.lib.rpl_strerror(rc).decode()}"
        return None

    def attach(self, plan):
        """Make this rank's gather (a GatherPlan writing into self.outputs) signal completion."""
        plan.desc.done_flag = self.flags[self.rank].data_ptr()
        plan.desc.done_seq = self.seq.data_ptr()

    def wait(self, stream=None):
        """Learner only: enqueue the wait for every rank's completion flag (K8)."""
        from . import _lib
        from .ops import _stream
        s = _stream(self.flags.device) if stream is None else stream
        _lib.check(_lib.lib.rpl_wait_flags(self.flags.data_ptr(), self.world, self.seq.data_ptr(),
                                           self.err.data_ptr(), s), "rpl_wait_flags")


class PeerBoards:
    """The exchange boards of rpl.h (RPL_BOARD_WORDS = 6 * world int64 words per rank):
    this rank's board is allocated here, zeroed, exported through CUDA IPC and mapped by
    every peer (all_gather_object of the IPC handles; NVLink P2P between GPUs, plain device
    memory on a shared GPU).  `ptrs` is the device int64 [world] array of board addresses
    the kernels take.  Construct on every rank at the same point (collective)."""

    def __init__(self, group=None, device=None):
        from torch.multiprocessing.reductions import reduce_tensor
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.board = torch.zeros(6 * self.world, dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)
        handles = [None] * self.world
        dist.all_gather_object(handles, reduce_tensor(self.board), group=group)
        self._mapped = []
        addrs = []
        failure = None
        try:
            self._map(handles, dev, addrs)
        except RuntimeError as e:  # agree on the outcome before raising (no rank left in a collective)
            failure = e
        ok = torch.tensor([0 if failure else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            raise RuntimeError(f"peer boards unavailable on some rank ({failure or 'a peer failed'})")
        self.ptrs = torch.tensor(addrs, dtype=torch.int64, device=dev)

    def _map(self, handles, dev, addrs):
        for g, (fn, args) in enumerate(handles):
            if g == self.rank:
                addrs.append(self.board.data_ptr())
            else:
                t = fn(*args)  # opens the peer's IPC handle in this process
                if t.device != self.board.device:
                    # the mapping lives in the peer GPU's memory: this device's kernels need
                    # peer access to it (NVLink P2P); fail loudly when there is no path
                    from . import _lib
                    with torch.cuda.device(self.board.device):
                        rc = _lib.lib.rpl_peer_access(t.device.index)
                    if rc != 0:
                        raise RuntimeError(f"rpl_peer_access({t.device.index}) from {self.board.device}: "
                                           f"{_lib.lib.rpl_strerror(rc).decode()}")
                self._mapped.append(t)
                addrs.append(t.data_ptr())

    @staticmethod
    def local(boards):
        """In-process boards for G 'ranks' sharing one process (tests): boards is a list of
        device int64 tensors of 6*G words; returns the shared pointer array."""
        return torch.tensor([b.data_ptr() for b in boards], dtype=torch.int64, device=boards[0].device)
