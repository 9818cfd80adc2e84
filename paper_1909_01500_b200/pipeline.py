"""Asynchronous replay pipeline on one GPU (Fig. 3).

rlpyt's asynchronous mode runs the sampler and the optimiser in separate
processes tied together by a shared-memory replay buffer: the sampler writes into a
double buffer, a copier process moves finished batches into the main buffer under a
read-write lock, and the optimiser is throttled so that its replay ratio (consumption
rate / generation rate) does not exceed a cap.

The B200 version keeps the roles and replaces the mechanisms:

  * double buffer   two pinned host batch buffers; the host sampler fills one while the
                    copy engine moves the other (rpl_ring_append on a copy stream);
  * read-write lock stream ordering with CUDA events, so copies overlap learner steps:
                    (1) on the learner stream, the leaves whose windows touch the rows
                    about to be overwritten are invalidated (no later sample can pick
                    them) and an event is recorded; (2) the copy stream waits for that
                    event — every gather that could still read those rows precedes it —
                    and runs rpl_ring_append; (3) once that copy has completed, the next
                    learner step first validates the leaves the new rows complete.  All
                    tree writes stay on the learner stream;
  * throttle        an exact budget counter (SPEC's design decision): every appended
                    step credits `cap` units, every consumed sample debits its counted
                    steps; `can_step()` is false while a step would overdraw the budget.
  * initial         (optional, NEXT-1, P:123 fn "5-step TD initial priorities", S:660,
    priorities      reading R33) the sampler also hands over the actor's q_taken / q_boot
                    per row; they are appended to two ring arrays, and a leaf that an append
                    makes valid gets, instead of max-seen, the priority of its n-step TD
                    errors (rpl_ring_td_abs -> rpl_sumtree_update_seq / _update_ex).

Host logic only (argument marshalling and event bookkeeping); every data movement and
tree update runs in librpl.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import ops
from . import replay as _rp


@dataclass
class ReplayRatio:
    """Budget counter for the replay-ratio cap (SPEC "optimizer blocks on a budget
    counter credited by the copier (generated x cap), debited per consumed sample").
    Warm-up steps count as generated (P:123 fn: "replay ratio of 1, including the warmup
    samples")."""
    cap: float
    generated: int = 0
    consumed: int = 0

    def credit(self, steps: int):
        self.generated += int(steps)

    def can_consume(self, steps: int) -> bool:
        return self.consumed + int(steps) <= self.cap * self.generated

    def debit(self, steps: int):
        self.consumed += int(steps)

    @property
    def ratio(self) -> float:
        return self.consumed / self.generated if self.generated else 0.0


@dataclass
class _HostBatch:
    tensors: dict
    ready: torch.cuda.Event = field(default_factory=torch.cuda.Event)  # copy finished: reusable


class ReplayPipeline:
    """Sequence (R2D2) or transition replay with asynchronous appends.

    ring: an ops.GatherRing (device); tree: ops.SumTree over its leaves; the batch
    shape [T_b, B, ...] is fixed.  Typical loop:

        h = pipe.host_batch()          # a free pinned buffer (waits if both are in flight)
        <sampler writes h.tensors>
        pipe.submit(h)                 # copy stream: append + validity
        if pipe.can_step(): pipe.step(...)   # learner stream: update + sample + gather
    """

    def __init__(self, ring: ops.GatherRing, tree: ops.SumTree, kind: str, T_b: int, k: int = 4, n_step: int = 1,
                 seq_len: int = 1, period: int = 1, train_steps: int = 1, cap: float = 1.0, rnn_parts: int = 2,
                 rnn_h: int = 512, init_priority: dict | None = None):
        self.ring, self.tree = ring, tree
        self.kind, self.T_b, self.k, self.n_step = kind, int(T_b), int(k), int(n_step)
        self.seq_len, self.period, self.train_steps = int(seq_len), int(period), int(train_steps)
        dev = ring.obs.device
        self.device = dev
        # init_priority: dict(n, gamma, rescale, eps, alpha, eps_p[, eta, burn_in] for sequences)
        self.init = dict(init_priority) if init_priority is not None else None
        if self.init is not None:
            ip = self.init
            ip.setdefault("rescale", False)
            ip.setdefault("eps", 1e-3)
            ip.setdefault("eps_p", 1e-3)
            ip.setdefault("eta", 0.9)
            ip.setdefault("burn_in", 0)
            if kind == "sequence" and ip["burn_in"] + train_steps + ip["n"] > seq_len:
                raise ValueError("burn_in + train_steps + n must fit in the sequence window")
            shape = (ring.cap_T, ring.B)
            self.q_taken = torch.zeros(shape, dtype=torch.float32, device=dev)
            self.q_boot = torch.zeros(shape, dtype=torch.float32, device=dev)
            self._leaf_ids = torch.arange(tree.n_leaves, dtype=torch.int64, device=dev)
            t_out = train_steps if kind == "sequence" else ring.cap_T
            self._td = torch.empty((t_out, ring.B), dtype=torch.float32, device=dev)
        self.copy_stream = torch.cuda.Stream(dev)
        self.learn_stream = torch.cuda.Stream(dev)
        self.throttle = ReplayRatio(cap)
        B = ring.B
        shp = (self.T_b, B)

        def pinned(shape, dtype):
            return torch.empty(shape, dtype=dtype).pin_memory()

        self._bufs = []
        for _ in range(2):  # double buffer (Fig. 3)
            t = {"obs": pinned(shp + ring.item_shape, ring.obs.dtype),
                 "act": pinned(shp + ring.act_shape, ring.act.dtype),
                 "rew": pinned(shp, torch.float32), "done": pinned(shp, torch.uint8)}
            if kind == "sequence" and ring.rnn is not None:
                nblk = (self.T_b + self.period - 1) // self.period + 1
                t["rnn"] = pinned((nblk,) + tuple(ring.rnn.shape[1:]), ring.rnn.dtype)
            if self.init is not None:  # the actor's Q(s_t, a_t) and bootstrap value of s_t
                t["q_taken"] = pinned(shp, torch.float32)
                t["q_boot"] = pinned(shp, torch.float32)
            hb = _HostBatch(t)
            hb.ready.record(torch.cuda.current_stream(dev))
            self._bufs.append(hb)
        self._next = 0
        self._pending = []

    # ---- sampler side -------------------------------------------------------------
    def host_batch(self) -> _HostBatch:
        """The next pinned batch buffer, once its previous copy has finished."""
        hb = self._bufs[self._next]
        hb.ready.synchronize()
        self._next ^= 1
        return hb

    def rnn_rows(self) -> list[int]:
        """Batch rows (relative to the next append) whose stored RNN state the sampler must
        provide, in order (rows landing on a storage-block start)."""
        c = self.ring.cursor
        return [t for t in range(self.T_b) if (c + t) % self.period == 0]

    def submit(self, hb: _HostBatch):
        """(1) invalidate the leaves that touch the rows about to be overwritten (learner
        stream), (2) copy the batch into the ring on the copy stream after every earlier
        learner op, (3) queue the validation of the newly complete leaves for the first
        learner step after the copy has finished (`_apply_ready`)."""
        L, C = self.learn_stream, self.copy_stream
        cap = self.ring.cap_T
        c0, s0 = self.ring.cursor, self.ring.size
        drop = max(0, s0 + self.T_b - cap)  # oldest rows the append overwrites
        with torch.cuda.stream(L):
            if drop:
                self.tree.validity(self.kind, cap, self.ring.B, self.k, c0, s0, c0, s0 - drop, n_step=self.n_step,
                                   seq_len=self.seq_len, period=self.period)
            inv = torch.cuda.Event()
            inv.record(L)
        C.wait_event(inv)
        with torch.cuda.stream(C):
            t = hb.tensors
            rows = self.rnn_rows()
            rnn = t["rnn"][:len(rows)] if ("rnn" in t and rows) else None
            if self.init is not None:  # at the cursor, before ring_append advances it
                ops.ring_append_rows(self.q_taken, t["q_taken"], c0)
                ops.ring_append_rows(self.q_boot, t["q_boot"], c0)
            ops.ring_append(self.ring, obs=t["obs"], act=t["act"], rew=t["rew"], done=t["done"], rnn=rnn,
                            period=self.period)
            copied = torch.cuda.Event()
            copied.record(C)
            hb.ready.record(C)
        self._pending.append((copied, (c0, s0 - drop), (self.ring.cursor, self.ring.size)))
        self.throttle.credit(self.T_b * self.ring.B)

    def _apply_ready(self, wait=False):
        """Learner stream: validate the leaves completed by every append whose copy is done
        (in submission order; `wait` = also the ones still copying)."""
        L = self.learn_stream
        while self._pending and (wait or self._pending[0][0].query()):
            copied, (c0, s0), (c1, s1) = self._pending.pop(0)
            L.wait_event(copied)
            with torch.cuda.stream(L):
                self.tree.validity(self.kind, self.ring.cap_T, self.ring.B, self.k, c0, s0, c1, s1,
                                   n_step=self.n_step, seq_len=self.seq_len, period=self.period)
                if self.init is not None:
                    self._initial_priorities(c0, s0, c1, s1)

    def newly_valid(self, c0, s0, c1, s1):
        """Host bookkeeping: the rows (transitions) or blocks (sequences) an append made valid."""
        cap = self.ring.cap_T
        if self.kind == "sequence":
            before = _rp.valid_sequence_blocks(cap, self.period, c0, s0, self.k, self.seq_len)
            after = _rp.valid_sequence_blocks(cap, self.period, c1, s1, self.k, self.seq_len)
        else:
            before = _rp.valid_transition_rows(cap, c0, s0, self.k, self.n_step)
            after = _rp.valid_transition_rows(cap, c1, s1, self.k, self.n_step)
        return sorted(set(after.tolist()) - set(before.tolist()))

    def _initial_priorities(self, c0, s0, c1, s1):
        """Learner stream, right after validity: n-step TD initial priorities (R33) for every
        leaf the append made valid (replacing the max-seen validity gave them)."""
        ip, ring, B = self.init, self.ring, self.ring.B
        units = self.newly_valid(c0, s0, c1, s1)
        if self.kind == "sequence":
            for blk in units:
                td = ops.ring_td_abs(ring.rew, ring.done, self.q_taken, self.q_boot, blk * self.period + ip["burn_in"],
                                     self.train_steps, ip["n"], ip["gamma"], ip["rescale"], ip["eps"], out=self._td)
                self.tree.update_seq(self._leaf_ids[blk * B:(blk + 1) * B], td, ip["alpha"], eta=ip["eta"],
                                     eps_p=ip["eps_p"])
            return
        runs, start = [], None  # runs of consecutive rows (leaf ranges never wrap)
        for i, r in enumerate(units):
            if start is None:
                start = r
            if i + 1 == len(units) or units[i + 1] != r + 1:
                runs.append((start, r + 1))
                start = None
        for r0, r1 in runs:
            td = ops.ring_td_abs(ring.rew, ring.done, self.q_taken, self.q_boot, r0, r1 - r0, ip["n"], ip["gamma"],
                                 ip["rescale"], ip["eps"], out=self._td[:r1 - r0])
            self.tree.update(self._leaf_ids[r0 * B:r1 * B], td.view(-1), ip["alpha"], eps_p=ip["eps_p"])

    def flush(self):
        """Make every submitted batch sampleable before the next step (deterministic order)."""
        self._apply_ready(wait=True)

    # ---- learner side -------------------------------------------------------------
    def can_step(self, n: int) -> bool:
        return self.throttle.can_consume(n * self.train_steps)

    def step(self, n, prev_idx, prev_td, plan, out_idx, out_q, seed, alpha, beta, eta=0.9, err=None):
        """Learner stream: validity of finished appends -> (sequence) priorities of the
        previous batch -> sample -> gather.  prev_td: [train_steps, n] per-step |delta|
        (sequences) or [n] (transitions); prev_idx may be None on the first step."""
        self._apply_ready()
        s = self.learn_stream
        plan.set_cursor(self.ring.cursor, self.ring.size)
        with torch.cuda.stream(s):
            if prev_idx is not None:
                # live-only (R30): a leaf invalidated by an append since it was sampled
                # must not be revived by the late priority
                if self.kind == "sequence":
                    self.tree.update_seq(prev_idx, prev_td, alpha, eta=eta, err=err, live_only=True)
                else:
                    self.tree.update(prev_idx, prev_td, alpha, err=err, live_only=True)
            self.tree.sample_stream(n, seed, out=(out_idx, out_q, None, None), want_qmin=False, err=err)
            plan.run(out_idx, q=out_q, qmin=None, beta=beta, err=err)
        self.throttle.debit(n * self.train_steps)
        return plan.outputs
