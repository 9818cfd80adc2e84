"""Oracle: prioritized replay over a list of integer leaves — no tree at all.

Paper: "prioritized replay (sum tree)" [EXT: PER].  SPEC: sum-tree
total/find/update, stratified proportional sampling and importance
weights, priority updates with last-write-wins,
max-priority-seen initial priority.

The plain definitions:

  total        Q = sum_i q_i                                   (Python int, exact)
  find(x)      the unique i with C_i <= x < C_{i+1}, C = exclusive prefix sums of q
               (half-open intervals: zero-q leaves are never returned, §8c #8)
  update       apply (idx, |delta|) pairs sequentially in batch order, so the last
               write to a leaf wins (§8c #9); max_seen tracks every q written
  strata       lo_k = floor(k Q / n), hi_k = lo_{k+1}; prefix_k = lo_k +
               floor(u_k (hi_k - lo_k) / 2**64), u_k a uint64 draw (§8c #8)
  IS weights   w_i = (N P_i)^-beta / max_j (N P_j)^-beta over the sampled batch,
               P_i = q_i / Q (§8c #10), float64

The sum tree the GPU keeps only accelerates `find`; its internal nodes are
checked against `range_sum` here, so this module never mirrors the GPU layout.
"""
from __future__ import annotations

import bisect
import itertools

from . import priority as _pr


class SumTreeOracle:
    def __init__(self, n_leaves: int, frac_bits: int = _pr.F_DEFAULT):
        self.n_leaves = int(n_leaves)
        self.frac_bits = int(frac_bits)
        self.cap = _pr.q_cap(self.n_leaves)
        self.q = [0] * self.n_leaves
        self.max_seen = 1 << self.frac_bits          # Q(1.0^alpha) before any write (§8c #12)
        self.err_idx = False
        self.err_saturated = False

    # ---- S:601-609 -------------------------------------------------------
    def total(self) -> int:
        return sum(self.q)

    def range_sum(self, lo: int, hi: int) -> int:
        return sum(self.q[max(0, lo):min(hi, self.n_leaves)])

    def find(self, prefix: int) -> int:
        incl = list(itertools.accumulate(self.q))    # incl[i] = C_{i+1}
        i = bisect.bisect_right(incl, prefix)        # first i with C_{i+1} > prefix
        return i

    # ---- S:621-629, S:660 -----------------------------------------------
    def update(self, idx, td_abs, alpha: float, eps_p: float = 1e-3, live_only: bool = False):
        """live_only (reading R30): a leaf whose q is 0 when its entry is applied (invalid
        since it was sampled, or never written) is skipped."""
        for i, d in zip(idx, td_abs):
            i = int(i)
            if i < 0:                                 # padding entry (rpl.h): skipped silently
                continue
            if i >= self.n_leaves:
                self.err_idx = True
                continue
            if live_only and self.q[i] == 0:
                continue
            M, E = _pr.priority_value(float(d), alpha, eps_p)
            qv, sat = _pr.quantise(M, E, self.frac_bits, self.cap)
            if sat:
                self.err_saturated = True
            self.q[i] = qv
            self.max_seen = max(self.max_seen, qv)

    def set_q(self, idx, q=None):
        """Direct leaf write (append / validity maintenance, §8a row a12);
        q=None writes max_seen."""
        for k, i in enumerate(idx):
            i = int(i)
            v = self.max_seen if q is None else int(q[k])
            if i < 0:
                continue
            if i >= self.n_leaves or v < 0:
                self.err_idx = True
                continue
            if v > self.cap:
                v = self.cap
                self.err_saturated = True
            self.q[i] = v
            if q is not None:
                self.max_seen = max(self.max_seen, v)

    # ---- S:611-619 --------------------------------------------------------
    def sample(self, n: int, draws):
        """Stratified proportional sampling. Returns (idx, q, qmin); idx = -1
        everywhere when Q == 0 (S:615 'empty buffer')."""
        Q = self.total()
        if Q == 0:
            return [-1] * n, [0] * n, 0
        idx, qs = [], []
        incl = list(itertools.accumulate(self.q))
        for k in range(n):
            lo = (k * Q) // n
            hi = ((k + 1) * Q) // n
            u = int(draws[k]) & ((1 << 64) - 1)
            prefix = lo + ((u * (hi - lo)) >> 64)
            i = bisect.bisect_right(incl, prefix)
            idx.append(i)
            qs.append(self.q[i])
        return idx, qs, min(qs)


def strata(Q: int, n: int):
    return [((k * Q) // n, ((k + 1) * Q) // n) for k in range(n)]


def is_weights(q_sampled, Q: int, N: int, beta: float):
    """w_i = (N P_i)^-beta normalised by the batch max (§8c #10), float64."""
    raw = [(N * (qi / Q)) ** (-beta) for qi in q_sampled]
    m = max(raw)
    return [x / m for x in raw]


def sharded_sample(shards, n: int, draws):
    """Sharded sampling = sampling on the shard-major concatenation (§8c #17).
    Returns global idx (shard g, local i -> g*len(shard_0) + i) and q."""
    cat = SumTreeOracle(sum(s.n_leaves for s in shards), shards[0].frac_bits)
    cat.q = list(itertools.chain.from_iterable(s.q for s in shards))
    return cat.sample(n, draws)


def buffer_min(q_leaves) -> int:
    """Buffer-wide IS normaliser (§8f NEXT-4, R29): min over the leaves with q > 0
    (2**63 - 1 when there are none); w_i = (q_min / q_i)^beta then normalises by the
    largest weight any stored transition could receive (PER), not the batch's."""
    pos = [int(x) for x in q_leaves if int(x) > 0]
    return min(pos) if pos else (1 << 63) - 1


def sample_unique(q_leaves, n, draws):
    """Sampling WITHOUT replacement (§8f NEXT-4, R32): successive proportional draws; draw k
    takes prefix = floor(u_k Q_k / 2**64) over the leaves not drawn yet (Q_k their total) and
    the unique leaf whose half-open interval holds it.  Returns (idx, q) lists; -1 / 0 once
    no mass is left."""
    q = [int(x) for x in q_leaves]
    out_i, out_q = [], []
    for k in range(n):
        Q = sum(q)
        if Q == 0:
            out_i.append(-1)
            out_q.append(0)
            continue
        prefix = (int(draws[k]) * Q) >> 64
        acc = 0
        for i, v in enumerate(q):
            if acc <= prefix < acc + v:
                break
            acc += v
        out_i.append(i)
        out_q.append(q[i])
        q[i] = 0
    return out_i, out_q
