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
its own learner.  With compact=True the owned draws come first (count on the device),
so the rank's gather schedules only them (rpl_gather_desc.n_active).  The result equals rpl_sumtree_sample on the shard-major
concatenation of the trees (§8c #17; tests/test_gpu_sumtree.py).

The tree object is duck-typed (total(), sample_sharded(), .device) so the
protocol can be exercised with world-size-2 gloo on CPU (tests/test_shard_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class ShardedSampler:
    def __init__(self, tree, n_per_rank: int, seed: int, group=None, is_weights=None, compact=False):
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
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)

    def sample(self, beta: float):
        """One global stratified sample of n_glob draws.  Returns (idx, q, w): idx[k] is
        the GLOBAL leaf (rank * shard_leaves + local) for the draws this rank owns and
        -1 elsewhere; w is normalised by the global batch min q."""
        self.tree.total(out=self.my_total)
        dist.all_gather_into_tensor(self.totals, self.my_total, group=self.group)          # K5
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
