#!/usr/bin/env python
"""bench.py — B200 replay + return-estimation hot path of rlpyt (arXiv 1909.01500).

Metric (BASELINE.json): "prioritized samples/sec (update+sample+gather) and return
elems/sec, 1/2/4/8 B200".  One STEP = one learner update's replay work on the
R2D2 config (BASELINE.json configs[4]):

    rpl_sumtree_update   64 sequence priorities of the previous batch  (a5-a7)
    rpl_sumtree_sample   64 stratified draws                            (a8)
    rpl_gather           64 sequences x 125 rows, frame stacks, prev fields,
                         stored LSTM state, IS weights (a9) and the
                         rescaled 5-step targets of the 80 train rows   (a11, a2, a4)

`value` = sequences/s over all ranks (weak scaling: 64 sequences per rank per
step, Mode L of SURVEY.md §8e).  A secondary line-item times GAE + discounted
returns on the PPO config [128, 4096] (configs[1]; a1, a3) in elements/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl rpl|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, NCCL)

--impl reference times the CPU oracle (oracle/) on the same workload: the
reference arm of this tier (no upstream code exists).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

FRAME = 84 * 84

# R2D2: 1M-step ring [4000, 256] (configs[4]), sharded by env columns in Mode L.
R2D2 = dict(cap_T=4000, B=256, period=40, burn_in=40, train=80, tail=5, k=4, n_step=5, gamma=0.997,
            alpha=0.9, beta=0.6, batch=64, rnn_h=512, rnn_parts=2, eps=1e-3, eps_p=1e-3, fanout=32, eta=0.9)
R2D2["L"] = R2D2["burn_in"] + R2D2["train"] + R2D2["tail"]
PPO = dict(T=128, B=4096, gamma=0.99, lam=0.95)
SPEC_HBM_GBS = 8000.0
# north_star's "1M-sequence R2D2 buffer": 2^20 sequence leaves over 8 GPUs; one shard per GPU
R2D2_1MSEQ_SHARD = dict(cap_T=40960, B=128)
# DQN/Rainbow Atari (configs[2]) and SAC/TD3 Mujoco (configs[3]) secondary line items
DQN = dict(cap_T=4096, B=256, k=4, n_step=3, gamma=0.99, alpha=0.6, beta=0.4, eps_p=1e-3, fanout=32,
           batches=(32, 128, 512))
MUJOCO = dict(cap_T=65536, B=16, n_step=3, gamma=0.99, batch=256, dims=((17, 6), (376, 17)))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="rpl", choices=["rpl", "reference"])
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--graph-steps", type=int, default=8, help="steps per captured CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle sample budget (cpu_baseline)")
    ap.add_argument("--cpu-baseline-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/baseline/e2e)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "collective"],
                    help="N>1: K5/K7 over peer-memory boards fused into the sampler and gather (p2p) or "
                         "torch.distributed collectives (collective); auto = p2p with nccl, else collective")
    ap.add_argument("--tree-fused", type=int, default=0, choices=[0, 1],
                    help="1 GPU: priority update + sampling as one launch (rpl_sumtree_update_sample; "
                         "measured 1.7 us/step slower than the PDL-chained pair)")
    ap.add_argument("--seq-variant", type=int, default=None, help="diagnostics: sequence-gather kernel variant")
    ap.add_argument("--gather-dyn", default=None,
                    help="measurement: the dynamic-tail schedule pct,rows,lookahead (rpl_debug_set_gather_dyn)")
    ap.add_argument("--fused-sample", type=int, default=1, choices=[0, 1],
                    help="1 GPU: stratified sampling inside the sequence gather (rpl_gather_sample), so the step "
                         "is update_seq -> gather (default: same-box A/B 68.1 vs 69.45 us per step with the "
                         "top levels staged in shared memory, profiles/r2/ab_fused_sample_staged.txt); 0: a "
                         "separate rpl_sumtree_sample_stream launch")
    ap.add_argument("--fused-update", type=int, default=0, choices=[0, 1],
                    help="1 GPU with --fused-sample 1: the priority update runs inside the gather too "
                         "(rpl_gather_update_sample: ONE launch per step; in-process A/B 64.8 vs 62.9 us, "
                         "profiles/r2/ab_one_launch.txt); 0 (default): the 8-CTA update_seq, then the gather")
    ap.add_argument("--mode", default="L", choices=["L", "C"],
                    help="N > 1 replay mode (SURVEY §8e): L = owner computes, each rank feeds its own learner; "
                         "C = every owner's gather writes into the rank-0 learner's batch over NVLink (CUDA IPC)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional checks only)")
    ap.add_argument("--same-device", action="store_true",
                    help="functional check: every rank on cuda:0 (with --backend gloo on a 1-GPU box)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def r2d2_config(c, world, mode="L"):
    """The workload description both arms print (BASELINE configs[4])."""
    Bl = c["B"] // max(1, world)
    return {"workload": "r2d2_1mstep", "ring": [c["cap_T"], c["B"]], "ring_per_gpu": [c["cap_T"], Bl],
            "leaves_per_gpu": (c["cap_T"] // c["period"]) * Bl, "batch_per_gpu": c["batch"], "seq_len": c["L"],
            "burn_in": c["burn_in"], "train": c["train"], "tail": c["tail"], "frame_stack": c["k"],
            "n_step": c["n_step"], "gamma": c["gamma"], "alpha": c["alpha"], "beta": c["beta"], "eta": c["eta"],
            "out": "stacked", "parallelism": (f"mode-{mode} x{world}" if world > 1 else "single"),
            "l2": "inputs larger than L2 (7.2 GB ring, random sequences every step)"}


def gather_traffic():
    """DRAM bytes (read + write) per launch of the sequence gather from the committed
    ncu --set full capture (profiles/gather_traffic.json, written by
    scripts/ncu_summary.py from the same launch configuration)."""
    p = os.path.join(ROOT, "profiles", "gather_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"bytes": d["dram_bytes_read"] + d["dram_bytes_write"], "source": d["source"]}
    except (OSError, KeyError, ValueError):
        return {}


def r2d2_targets(c, q):
    """Fused rescaled n-step targets of the train rows (rpl_gather_desc.o_tgt): rows
    burn_in .. burn_in+train-1, bootstrap q [L, n] at row tau + n_step (R5, R24)."""
    return dict(lo=c["burn_in"], T=c["train"], n_step=c["n_step"], gamma=c["gamma"], rescale=True, eps=c["eps"], q=q)


def seq_bytes_per_sample(c, act_bytes=8):
    """Algorithmic HBM bytes one sequence of rpl_gather moves:
    reads the L+k-1 unique frames, the per-row scalars and the stored state;
    writes L k-stacks and the per-row fields."""
    L, k = c["L"], c["k"]
    rd = (L + k - 1) * FRAME                      # unique frames
    rd += (L + 1) * (act_bytes + 4 + 1)           # act, rew, done of rows row0-1 .. row0+L-1
    rd += c["rnn_parts"] * c["rnn_h"] * 4         # stored (h, c)
    wr = L * k * FRAME                            # stacked observations
    wr += L * (2 * act_bytes + 4 + 4 + 1)         # act, prev_act, rew, prev_rew, done
    wr += c["rnn_parts"] * c["rnn_h"] * 4
    rd += c["train"] * 4                          # fused targets: bootstrap q of each train row
    wr += c["train"] * (4 + 1)                    # target y and done^n
    return rd + wr


# ----------------------------------------------------------------------------- GPU arm
def run_rpl(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if args.gpus > 1 and world == 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    local = 0 if args.same_device else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    import paper_1909_01500_b200 as rpl
    from paper_1909_01500_b200 import replay as R
    from synth import make_ring, rng
    FUSED_SAMPLE[0] = bool(args.fused_sample) and not args.tree_fused
    if args.gather_dyn is not None:
        rpl._lib.check(rpl._lib.lib.rpl_debug_set_gather_dyn(*(int(x) for x in args.gather_dyn.split(","))),
                       "gather_dyn")
    if args.seq_variant is not None:
        rpl._lib.check(rpl._lib.lib.rpl_debug_set_gather_variant(int(args.seq_variant)), "variant")

    c = dict(R2D2)
    b0, b1 = R.shard_columns(c["B"], world, rank)
    Bl = b1 - b0
    n = c["batch"]
    L, k, period = c["L"], c["k"], c["period"]

    # ---- inputs (seeded synthetic, resident in HBM before timing) ----
    t_setup = time.time()
    if world == 1:
        host = make_ring(2019, c["cap_T"], Bl, ep_len=2000.0, reward_kind="r2d2", period=period,
                         rnn_parts=c["rnn_parts"], rnn_h=c["rnn_h"], cursor=1234 % c["cap_T"])
        ring = rpl.GatherRing(obs=torch.from_numpy(host.obs).to(dev), act=torch.from_numpy(host.act).to(dev),
                              rew=torch.from_numpy(host.rew).to(dev), done=torch.from_numpy(host.done).to(dev),
                              cursor=host.cursor, size=host.size, rnn=torch.from_numpy(host.rnn).to(dev))
    else:
        from synth.device import make_ring_device
        host = None
        ring = make_ring_device(2019 + 7919 * rank, c["cap_T"], Bl, dev, ep_len=2000.0, period=period,
                                rnn_parts=c["rnn_parts"], rnn_h=c["rnn_h"], cursor=1234 % c["cap_T"])
    n_leaves = (c["cap_T"] // period) * Bl
    tree = rpl.SumTree(n_leaves, c["fanout"], 32, device=dev)
    blocks = R.valid_sequence_blocks(c["cap_T"], period, ring.cursor, ring.size, k, L)
    valid = torch.from_numpy(R.leaves_of(blocks, Bl)).to(dev)
    g = rng(77 + rank)
    td0 = np.abs(g.normal(size=valid.numel())).astype(np.float32)
    tree.update(valid, torch.from_numpy(td0).to(dev), c["alpha"], c["eps_p"])
    P = max(2, args.graph_steps + (args.graph_steps % 2))  # steps per CUDA graph (even: idx buffers alternate)
    if args.steps % P:
        # exactly K steps without a short remainder graph (its replay carries the graph launch
        # over fewer steps): the even divisor of K in [4, 16] closest to the requested size
        divs = [d for d in range(4, 17, 2) if args.steps % d == 0]
        if divs:
            P = min(divs, key=lambda d: (abs(d - P), -d))
    # per-step |delta| of the previous batch's train rows, [P][train, n_glob] (R2D2 learner output)
    td_pool = torch.from_numpy(np.abs(g.normal(size=(P, c["train"], n * max(1, world)))).astype(np.float32)).to(dev)
    n_glob = n * world
    q_pool = torch.from_numpy(g.normal(0, 10, (P, L, n_glob)).astype(np.float32)).to(dev)
    seed = 0x5EED

    mode_c = world > 1 and args.mode == "C"
    learner = (not mode_c) or rank == 0  # ranks that consume a batch (and compute its targets)
    central = None
    stacked = None
    if mode_c:
        # Mode C: rank 0's batch buffers, mapped into every rank (CUDA IPC over NVLink).  The owners
        # ship UNIQUE frame rows + episode-start offsets (116 MB per 64 sequences instead of 284 MB
        # of stacks); the learner rebuilds the k-stacks locally (rpl_stack_frames).
        from paper_1909_01500_b200 import _lib as _L
        from paper_1909_01500_b200.shard import CentralBatch
        want = ["obs", "act", "prev_act", "rew", "prev_rew", "done", "rnn", "start"]
        root_plan = (rpl.GatherPlan(ring, n_glob, kind="sequence", k=k, seq_len=L, period=period, with_weights=True,
                                    out_mode=_L.OUT_UNIQUE, want=want) if rank == 0 else None)
        central = CentralBatch(root_plan.outputs if rank == 0 else None)
        plan = root_plan if rank == 0 else rpl.GatherPlan(ring, n_glob, kind="sequence", k=k, seq_len=L,
                                                          period=period, with_weights=True, out_mode=_L.OUT_UNIQUE,
                                                          want=want, outputs=central.outputs)
        central.attach(plan)  # the gather signals the learner's flag when its last CTA is done
        if rank == 0:
            stacked = torch.empty((L, n_glob, k) + tuple(ring.item_shape), dtype=torch.uint8, device=dev)
    else:
        plan = rpl.GatherPlan(ring, n_glob, kind="sequence", k=k, seq_len=L, period=period, with_weights=True,
                              targets=r2d2_targets(c, q_pool[0]))
    out = plan.outputs
    fused_tgt = not mode_c  # Mode C: the learner computes targets after the central batch lands
    idx_buf = [torch.full((n_glob,), -1, dtype=torch.int64, device=dev) for _ in range(2)]
    q_buf = torch.zeros(n_glob, dtype=torch.int64, device=dev)
    qmin = torch.zeros(1, dtype=torch.int64, device=dev)
    w = plan.outputs["w"]  # IS weights: written by the gather (1 GPU) or rpl_is_weights (Mode L)
    if fused_tgt:
        y, dn = out["tgt"], out["tgt_done"]
    else:
        y = torch.empty((c["train"], n_glob), dtype=torch.float32, device=dev)
        dn = torch.empty((c["train"], n_glob), dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    totals = torch.zeros(world, dtype=torch.int64, device=dev)
    my_total = torch.zeros(1, dtype=torch.int64, device=dev)
    n_owned = torch.zeros(2, dtype=torch.int64, device=dev)  # [owned m, first owned stratum k0]
    p2p = world > 1 and (args.exchange == "p2p" or (args.exchange == "auto" and args.backend == "nccl"))
    boards = None
    if world > 1:
        # compacted sharded sample: this rank's owned draws first, the gather schedules only those
        plan.desc.n_active = n_owned.data_ptr()
        if mode_c:  # ... and writes them at their global batch positions in the learner's buffers
            plan.desc.col_offset = n_owned.data_ptr() + 8
        if p2p:  # K5 / K7 through peer-memory boards, fused into the sampler and the gather
            from paper_1909_01500_b200.shard import PeerBoards
            try:
                boards = PeerBoards(device=dev)
                ok = torch.tensor([1], dtype=torch.int32, device=dev)
            except RuntimeError as e:  # no peer path to some rank: every rank falls back together
                print(f"[bench] rank {rank}: peer boards unavailable ({e}); using NCCL collectives", file=sys.stderr)
                ok = torch.tensor([0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 1:
                plan.set_peers(boards.ptrs, world, rank)
            else:
                p2p, boards = False, None

    def all_gather_totals():
        if args.backend == "nccl":
            dist.all_gather_into_tensor(totals, my_total)
        else:
            dist.all_gather(list(totals.chunk(world)), my_total)
    r_tr = out["rew"][c["burn_in"]:c["burn_in"] + c["train"] + c["n_step"] - 1]
    d_tr = out["done"][c["burn_in"]:c["burn_in"] + c["train"] + c["n_step"] - 1]
    Tn = c["train"] + c["n_step"] - 1
    lib, P_ = rpl._lib.lib, rpl.ops._ptr

    def step(i, gather_events=None, y_out=None, w_out=None, io=None, skip_gather=False):
        # y_out / w_out: per-step output buffers; io = (td, q, cur_idx, prev_idx) per-step
        # inputs / index buffers (the e2e schedule gives every step of a graph its own)
        s = rpl.ops._stream(dev)
        cur, prev = idx_buf[i % 2], idx_buf[(i + 1) % 2]
        td_i, q_i = td_pool[i % P], q_pool[i % P]
        if io is not None:
            td_i, q_i, cur, prev = io
        # (a5-a7) new priorities for the previous batch (entries < 0 — not owned — are skipped, R22)
        # (NEXT-1 fused) sequence priority = eta max + (1 - eta) mean of the 80 per-step |delta| (R26)
        one_launch = world == 1 and args.fused_sample and args.fused_update and not args.tree_fused
        if one_launch and not skip_gather:
            # (a5-a8 + a9 + a11 + a2/a4) the whole step in one launch: every gather CTA applies
            # the update to its staged copy of the tree and samples it; CTA 0 writes the update
            if gather_events is not None:  # the one kernel is the step: events around it
                gather_events[0].record()
            if w_out is not None:
                plan.desc.o_w = w_out.data_ptr()
            if y_out is not None:
                plan.desc.o_tgt = y_out.data_ptr()
            plan.run_update_sample(tree, prev, td_i, seed, cur, q_buf, eta=c["eta"], alpha=c["alpha"],
                                   eps_p=c["eps_p"], beta=c["beta"], err=err, stream=s, q_tgt=q_i)
            if w_out is not None:
                plan.desc.o_w = w.data_ptr()
            if y_out is not None:
                plan.desc.o_tgt = y.data_ptr()
            if gather_events is not None:
                gather_events[1].record()
            return
        if world == 1 and args.tree_fused:
            # (a5-a8) update + stratified draws in one launch (grid barrier between them);
            # the batch-min normaliser and IS weights (a9) are fused into the gather
            rpl._lib.check(lib.rpl_sumtree_update_sample(tree._lp, P_(tree.storage), P_(prev), P_(td_i),
                                                         c["train"], n_glob, c["eta"], c["alpha"], c["eps_p"], 0, n,
                                                         seed, P_(cur), P_(q_buf), P_(err), s), "update_sample")
        else:
            rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(prev), P_(td_i),
                                                      c["train"], n_glob, c["eta"], c["alpha"], c["eps_p"], 0, None,
                                                      s), "update_seq")
        if world == 1 and not args.tree_fused and not args.fused_sample:
            # (a8) draws only; the batch-min normaliser and IS weights (a9) are fused into the gather
            rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, seed, c["beta"], P_(cur),
                                                         P_(q_buf), None, None, P_(err), s), "sample")
        elif p2p:
            # (a8, K5 fused) every rank publishes its total into the peers' boards and reads all of
            # them inside the sampler; no collective launch
            rpl._lib.check(lib.rpl_sumtree_sample_sharded_p2p(tree._lp, P_(tree.storage), rank, world, n_leaves,
                                                              P_(boards.ptrs), n_glob, seed, P_(cur), P_(q_buf),
                                                              P_(n_owned), P_(err), s), "sample_sharded_p2p")
        elif world > 1:
            rpl._lib.check(lib.rpl_sumtree_total(tree._lp, P_(tree.storage), P_(my_total), s), "total")
            all_gather_totals()                                                  # K5: 8 B per rank
            rpl._lib.check(lib.rpl_sumtree_sample_sharded(tree._lp, P_(tree.storage), rank, world, n_leaves,
                                                          P_(totals), n_glob, None, seed, 0, 1, P_(cur), P_(q_buf),
                                                          P_(qmin), P_(n_owned), P_(err), s), "sample_sharded")
            dist.all_reduce(qmin, op=dist.ReduceOp.MIN)                          # K7: global batch min
        if skip_gather:  # marginal-cost measurement: the same step without the gather launch
            return
        if gather_events is not None:
            # the start event sits on a side branch that depends on the update's completion,
            # so the update -> gather programmatic (PDL) edge stays intact; the gather itself
            # waits for the same completion in its griddepcontrol.wait
            side = gather_events[2]
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                gather_events[0].record()
        # IS weights fused into the gather: batch min (1 GPU) or the all-reduced global min (Mode L)
        if w_out is not None:
            plan.desc.o_w = w_out.data_ptr()
        if fused_tgt and y_out is not None:
            plan.desc.o_tgt = y_out.data_ptr()
        # (K7 fused with p2p: the gather publishes / reads the batch mins over the boards;
        #  a2 + a4 fused: the rescaled 5-step targets of the train rows, bootstrap q_i)
        if world == 1 and args.fused_sample and not args.tree_fused:
            # (a8 + a9 + a11 + a2/a4) the gather draws its own strata from the updated tree
            plan.run_sample(tree, seed, cur, q_buf, beta=c["beta"], err=err, stream=s, q_tgt=q_i)
        else:
            plan.run(cur, q=q_buf, qmin=None if (world == 1 or p2p) else qmin, beta=c["beta"], err=err, stream=s,
                     q_tgt=q_i if fused_tgt else None)
        if w_out is not None:
            plan.desc.o_w = w.data_ptr()
        if fused_tgt and y_out is not None:
            plan.desc.o_tgt = y.data_ptr()
        if gather_events is not None:
            gather_events[1].record()
            torch.cuda.current_stream(dev).wait_stream(gather_events[2])  # rejoin the side branch
        if mode_c:
            if rank == 0:  # learner: wait for every owner's completion flag (K8, no collective),
                central.wait(stream=s)  # then the k-stacks from the shipped unique rows (local HBM)
                rpl._lib.check(lib.rpl_stack_frames(P_(out["obs"]), P_(out["start"]), L, n_glob, k, ring.obs_bytes,
                                                    0, P_(stacked), None, s), "stack")
        if learner and not fused_tgt:
            rpl._lib.check(lib.rpl_returns_nstep(P_(r_tr), P_(d_tr), Tn, n_glob, c["n_step"], c["gamma"],
                                                 P_(q_i[c["burn_in"]:c["burn_in"] + Tn]),
                                                 P_(q_i[c["burn_in"] + Tn]), 1, c["eps"],
                                                 P_(y if y_out is None else y_out), P_(dn), s), "nstep")

    # idx < 0 entries (first step / not-owned) make the update kernel flag RPL_DERR_IDX; allow that bit.
    # warm-up (also primes lazy module loading and cudaFuncSetAttribute outside capture)
    for i in range(max(args.warmup, 2)):
        step(i)
    torch.cuda.synchronize()
    rpl.check_err(err)

    # CUDA graphs: one of P steps, replayed K // P times, and one of the K % P remaining steps,
    # so exactly K steps are timed.  With N > 1 the NCCL collectives are captured too (gloo: eager).
    K = args.steps
    reps, rem = divmod(K, P)
    use_graph = (not args.no_graph) and (world == 1 or args.backend == "nccl")
    graph = graph_rem = None
    per_graph = per_rem = 0
    if use_graph:
        try:
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            c0 = rpl.launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for i in range(P):
                    step(i)
            per_graph = rpl.launch_count() - c0
            if rem:
                c0 = rpl.launch_count()
                graph_rem = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph_rem, stream=s):
                    for i in range(rem):  # P is even: step 0 here continues after step P-1
                        step(i)
                per_rem = rpl.launch_count() - c0
            torch.cuda.synchronize()
            # warm the captured graphs (first replays upload / instantiate lazily)
            for _ in range(3):
                graph.replay()
            if graph_rem is not None:
                graph_rem.replay()
            torch.cuda.synchronize()
        except Exception as e:  # capture unsupported here: fall back to eager launches
            print(f"[bench] graph capture failed ({type(e).__name__}: {e}); timing eager steps", file=sys.stderr)
            graph = graph_rem = None
            use_graph = False
            torch.cuda.synchronize()
    K_eff = K

    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    # keep the GPU busy up to the timed region (after the sampler's start-up idle): ~30 ms of
    # replays of the same warm graph, so the first timed replay does not start from idle
    if use_graph:
        for _ in range(max(1, int(30e-3 / (P * 70e-6)))):
            graph.replay()
    # timed region: exactly K steps; an event before each replay gives per-replay durations
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 2)] if use_graph else []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = rpl.launch_count()
    # a ~100 us device spin BEFORE the start event (outside the timed region): the host enqueues
    # the start event and all K steps' graph replays while it runs, so the region times K steps
    # of device work back to back rather than the first graph launch's host submission latency
    # (with K = 20 that gap alone read as +1.8 us per step: 65.07 vs 63.09 us per replay)
    torch.cuda._sleep(int(2e5))
    e0.record()
    if use_graph:
        for j in range(reps):
            evs[j].record()
            graph.replay()
        evs[reps].record()
        if graph_rem is not None:
            graph_rem.replay()
    else:
        for i in range(K_eff):
            step(i)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ((rpl.launch_count() - launches0) if not use_graph else per_graph * reps + per_rem)
    clk = clocks.stop() if not args.profile else {}
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = K_eff * n * world / (ms / 1e3)
    timed_stats = None
    if use_graph and reps >= 1:
        per = [evs[j].elapsed_time(evs[j + 1]) / P * 1e3 for j in range(reps)]
        timed_stats = _stats(per)
    # SURVEY §8d protocol on the same warm graph: >= 200 replays, per-replay durations
    replay_stats = None
    if use_graph and not args.profile:
        nr = 200
        ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(nr + 1)]
        torch.cuda.synchronize()
        for j in range(nr):
            ev2[j].record()
            graph.replay()
        ev2[nr].record()
        torch.cuda.synchronize()
        replay_stats = dict(_stats([ev2[j].elapsed_time(ev2[j + 1]) / P * 1e3 for j in range(nr)]), replays=nr)

    pipelined = None
    if world == 1 and not args.no_secondary and not args.profile:
        try:
            pipelined = pipelined_step(dev, rpl, tree, plan, idx_buf, td_pool, q_pool, err, c, n, P, seed)
        except Exception as e:  # pragma: no cover
            pipelined = {"error": f"{type(e).__name__}: {e}"[:300]}

    # dominant kernel (sequence gather): average launch duration with CUDA events on
    # the launching stream, over K eager steps of the same workload
    Kg = min(K_eff, 200)
    side = torch.cuda.Stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), side) for _ in range(Kg)]
    torch.cuda.synchronize()
    for i in range(Kg):
        step(i, evs[i])
    torch.cuda.synchronize()
    g_ms_eager = float(np.mean([a.elapsed_time(b) for a, b, _ in evs]))
    # the same launch inside the timed configuration: a graph of P steps whose gathers are
    # bracketed by event-record nodes (cudaEventRecordExternal), so no host enqueue gap
    # falls inside the interval.  The start node sits on a side branch that waits for the
    # update kernel's completion, so the update -> gather PDL edge stays intact (the gather's
    # launch overlaps the update, and the interval starts where the gather's dependency wait
    # ends); the end node follows the gather on the launching stream.
    g_ms_graph = None
    if use_graph and world == 1:
        try:
            g_ms_graph = gather_ms_in_graph(dev, step, P)
        except Exception as e:  # pragma: no cover - keep the eager figure
            print(f"[bench] in-graph gather timing failed ({type(e).__name__}: {e})", file=sys.stderr)
    g_ms = g_ms_graph if g_ms_graph is not None else g_ms_eager
    # the gather's marginal cost in the timed configuration: graphs of P steps with and
    # without the gather launch (no event node inside the graph, so the PDL edges stay intact)
    g_ms_marginal = None
    if use_graph and world == 1:
        try:
            full_ms = _graph_time(dev, step, P=P, reps=50)
            nog_ms = _graph_time(dev, lambda i: step(i, skip_gather=True), P=P, reps=50)
            g_ms_marginal = full_ms - nog_ms
        except Exception as e:  # pragma: no cover
            print(f"[bench] marginal gather timing failed ({type(e).__name__}: {e})", file=sys.stderr)
    owned = n  # per rank, on average
    alg_bytes = owned * seq_bytes_per_sample(c)
    if mode_c:  # Mode C gathers unique rows (the learner re-stacks them)
        alg_bytes = owned * (seq_bytes_per_sample(c) - L * k * FRAME + (L + k - 1) * FRAME)
    peak, peak_kind = measured_peaks()
    achieved = alg_bytes / (g_ms / 1e3) / 1e9

    rpl.check_err(err)
    traffic = gather_traffic()

    result = {
        "metric": "prioritized samples/sec (update+sample+gather)",
        "value": value,
        "unit": "sequences/s",
        "n_gpus": world,
        "steps": K_eff,
        "warmup": max(args.warmup, 2),
        "ms_per_step": ms / K_eff,
        "step_us_stats": {"timed": timed_stats, "replays_200": replay_stats,
                          "note": ("per-step us over the timed region's graph replays (timed) and over 200 further "
                                   "replays of the same warm graph (SURVEY §8d protocol); value = K / timed total")},
        "knobs": dict(rpl._lib.config(), env={k_: v_ for k_, v_ in os.environ.items() if k_.startswith("RPL_")}),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 frames + f32 (fp64 accum) + int64 tree",
        "data": "synthetic (seeded; uniform-random 84x84 u8 frames, R2D2 reward/episode recipe, DESIGN.md)",
        "config": dict(r2d2_config(c, world, args.mode),
                       timing=(f"cuda graph of {P} steps replayed {reps}x" + (f" + a graph of {rem} steps" if rem else "")
                               + (" (both warmed" if rem else " (warmed") + " by 3 replays first); exactly K steps timed" if use_graph
                               else "eager launches"),
                       tree=("update+sample fused (rpl_sumtree_update_sample)" if world == 1 and args.tree_fused
                             else "update_seq, then sampling inside the gather (rpl_gather_sample)"
                             if world == 1 and args.fused_sample else "update_seq, then sample"),
                       exchange=(None if world == 1 else "p2p boards (K5 in the sampler, K7 in the gather)" if p2p
                                 else f"{args.backend} collectives")),
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_gather_seq_pipe_lsu", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic.get("bytes"), "traffic_source": traffic.get("source"),
                     "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": g_ms,
                     "avg_launch_ms_eager": g_ms_eager,
                     "marginal_ms": g_ms_marginal,
                     "frac_marginal": (alg_bytes / (g_ms_marginal / 1e3) / 1e9 / peak) if g_ms_marginal else None,
                     "marginal_note": ("step graph minus the same graph without the gather launch: the gather's "
                                       "in-step cost with the PDL edges intact (frac uses the event-bracketed "
                                       "avg_launch_ms)"),
                     "launch_timing": ("event-record nodes around each gather in the CUDA graph of the timed "
                                       "steps (the start node on a side branch after the update, so the PDL edge "
                                       "into the gather stays intact; mean of P launches x 25 replays)"
                                       if g_ms_graph is not None
                                       else "events around the gather in eager steps (start event on a side branch)"),
                     "step_share": g_ms / (ms / K_eff),
                     "frac_of_spec": achieved / SPEC_HBM_GBS, "spec_peak": SPEC_HBM_GBS,
                     "spec_note": "north_star's ~8 TB/s nominal (DGX B200 figure) as the second denominator"},
    }
    if not args.profile:
        result["clocks"] = clk
    if mode_c:
        # the central learner's NVLink ingress bounds Mode C — the other ranks' unique
        # rows + fields cross into rank 0 every step (spec 900 GB/s per direction; not measured here)
        per_seq = seq_bytes_per_sample(c) - L * k * FRAME + (L + k - 1) * FRAME
        ingress = (world - 1) / world * n_glob * per_seq
        result["mode_c_ceiling"] = {"bytes_into_learner_per_step": ingress, "nvlink_ingress_GBps_spec": 900.0,
                                    "us_per_step_floor": ingress / 900e9 * 1e6,
                                    "sequences_per_s_ceiling": n_glob / (ingress / 900e9) if ingress else None,
                                    "note": "the learner then re-stacks the k-frame stacks locally (rpl_stack_frames)"}
    result["e2e"] = e2e_rpl(args, dev, step, idx_buf, y, w, td_pool, q_pool, n, P, K_eff, world)
    # a1-a4 at every N: each rank scans its own [128, 4096] columns, no collective
    try:
        result["returns"] = returns_line(dev, rpl, world, dist if world > 1 else None)
    except Exception as e:  # pragma: no cover
        result["returns"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if world == 1 and not args.no_secondary and not args.profile:
        # each secondary is isolated: a failure is reported in its slot, never loses the line
        jobs = [("r2d2_seeds", lambda: seed_sweep(dev, rpl, c, ms / K_eff * 1e3)),
                ("r2d2_pipelined", lambda: pipelined),
                ("r2d2_1mseq", lambda: bench_r2d2_1mseq(dev, rpl, c)),
                ("r2d2_unique_output", lambda: unique_output_step(dev, rpl, tree, ring, idx_buf, td_pool, q_pool, err,
                                                                  c, n, P, seed)),
                ("tree_latency", lambda: tree_latency(dev, rpl)),
                ("dqn_replay", lambda: bench_dqn(dev, rpl)),
                ("mujoco_replay", lambda: bench_mujoco(dev, rpl))]
        result["secondary"] = {}
        for name, fn in jobs:
            try:
                result["secondary"][name] = fn()
            except Exception as e:  # pragma: no cover
                result["secondary"][name] = {"error": f"{type(e).__name__}: {e}"[:300]}
                try:
                    torch.cuda.synchronize()
                    torch.cuda.empty_cache()
                except Exception:  # pragma: no cover  (sticky CUDA error: skip the rest)
                    break
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        try:
            del host  # the leg rebuilds the same seeded ring in its own process
            result["cpu_baseline"] = cpu_baseline_subprocess(args.cpu_seconds)
        except Exception as e:  # pragma: no cover
            result["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"[:300], "kind": "oracle"}
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


def e2e_rpl(args, dev, step, idx_buf, y, w, td_pool, q_pool, n, P, K, world):
    """Same metric through the public API with HOST buffers: every step copies its
    inputs (the previous batch's |delta| and the target-net Q rows) from pinned host
    memory and reads the step's result (targets, IS weights, indices) back."""
    import torch
    K = min(K, 320)
    # graphs of PE steps: the one join per graph (the last step's D2H read-back) is paid
    # once per PE steps; every step still copies its own inputs and results
    PE = 32 if world == 1 and not args.no_graph else P
    rep = [j % P for j in range(PE)]
    td0, q0 = td_pool, q_pool  # the buffers step(i) reads in the eager path
    td_pool = td_pool[rep].contiguous()
    q_pool = q_pool[rep].contiguous()
    h_td = torch.empty(td_pool.shape, dtype=torch.float32).pin_memory()
    h_q = torch.empty(q_pool.shape, dtype=torch.float32).pin_memory()
    h_td.copy_(td_pool.cpu())
    h_q.copy_(q_pool.cpu())
    h_y = torch.empty(y.shape, dtype=torch.float32).pin_memory()
    h_w = torch.empty(w.shape, dtype=torch.float32).pin_memory()
    h_i = torch.empty(idx_buf[0].shape, dtype=torch.int64).pin_memory()
    torch.cuda.synchronize()

    def e2e_step(i):
        td0[i % P].copy_(h_td[i % P], non_blocking=True)
        q0[i % P].copy_(h_q[i % P], non_blocking=True)
        step(i)
        h_y.copy_(y, non_blocking=True)
        h_w.copy_(w, non_blocking=True)
        h_i.copy_(idx_buf[i % 2], non_blocking=True)

    # 1 GPU: the same calls in CUDA graphs of P steps.  Every step of a graph has its own
    # input slots, index and output buffers, so no step waits on a copy: the copy stream
    # brings up the NEXT graph's P input sets (two slot sets, alternating graphs A / B) and
    # takes each step's results down right after that step (fork only; one join at the graph
    # end).  Every copy is inside the timed region; multi-rank: eager, serial.
    cs = torch.cuda.Stream(dev)
    td_set = [td_pool, torch.empty_like(td_pool)]
    q_set = [q_pool, torch.empty_like(q_pool)]
    idx_all = [torch.full_like(idx_buf[0], -1) for _ in range(PE)]
    y_all = [torch.empty_like(y) for _ in range(PE)]
    w_all = [torch.empty_like(w) for _ in range(PE)]
    h_y_all = [torch.empty(y.shape, dtype=torch.float32).pin_memory() for _ in range(PE)]
    h_w_all = [torch.empty(w.shape, dtype=torch.float32).pin_memory() for _ in range(PE)]
    h_i_all = [torch.empty(idx_buf[0].shape, dtype=torch.int64).pin_memory() for _ in range(PE)]

    def prefetched(par):
        main = torch.cuda.current_stream(dev)
        cs.wait_stream(main)
        with torch.cuda.stream(cs):  # the next graph's inputs (set 1 - par)
            for j in range(PE):
                td_set[1 - par][j].copy_(h_td[j], non_blocking=True)
                q_set[1 - par][j].copy_(h_q[j], non_blocking=True)
        for j in range(PE):
            step(j, y_out=y_all[j], w_out=w_all[j], io=(td_set[par][j], q_set[par][j], idx_all[j], idx_all[j - 1]))
            ev = torch.cuda.Event()
            ev.record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(ev)
                h_y_all[j].copy_(y_all[j], non_blocking=True)
                h_w_all[j].copy_(w_all[j], non_blocking=True)
                h_i_all[j].copy_(idx_all[j], non_blocking=True)
        main.wait_stream(cs)

    graphs = None
    if world == 1 and not args.no_graph:
        try:
            for par in (0, 1):
                prefetched(par)
            torch.cuda.synchronize()
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            graphs = []
            for par in (0, 1):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=s):
                    prefetched(par)
                graphs.append(gr)
            torch.cuda.synchronize()
            graphs[0].replay()  # fills set 1 for the first timed replay (graph B)
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover
            print(f"[bench] e2e graph capture failed ({e}); eager", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize()
    reps = max(2, K // PE)
    K = reps * PE if graphs is not None else K
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graphs is not None:
        for r_ in range(reps):
            graphs[(r_ + 1) % 2].replay()
    else:
        for i in range(K):
            e2e_step(i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    hb = td_pool[0].numel() * 4 + q_pool[0].numel() * 4
    db = y.numel() * 4 + w.numel() * 4 + idx_buf[0].numel() * 8
    return {"value": K * n * world / (ms / 1e3), "unit": "sequences/s", "h2d_bytes_per_step": hb,
            "d2h_bytes_per_step": db, "steps": K,
            "timing": (f"cuda graphs of {PE} steps; per step one pinned-host H2D input set (prefetched one graph "
                       "ahead into alternating slots) and the D2H of its results right after it, on a copy "
                       "stream overlapping compute") if graphs is not None
            else "eager launches incl. pinned-host H2D/D2H copies"}


def returns_line(dev, rpl, world, dist):
    """Return estimation (a1-a4) at N GPUs, weak scaling: every rank runs GAE, the discounted
    return and the rescaled 5-step target on its own PPO-shaped [128, 4096] buffers (columns
    are independent: no collective on the data path).  Per-call device time is the max over
    ranks; aggregate elems/s = N x 128 x 4096 / that time."""
    import torch
    r = bench_ppo(dev, rpl)
    keys = ("gae_us_per_call", "disc_us_per_call", "nstep_us_per_call")
    t = torch.tensor([r[k] for k in keys], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    T, B = PPO["T"], PPO["B"]
    out = {"workload": f"ppo_[{T},{B}] per rank", "unit": "elems/s", "n_gpus": world, "scaling": "weak",
           "exchange": "none (columns independent)", "timing": r["timing"], "l2": r["l2"]}
    peak, _ = measured_peaks()
    for k, nb in zip(keys, (17, 9, 14)):  # bytes per element: GAE, discounted, n-step with bootstrap q
        us = float(t[keys.index(k)].item())
        name = k.split("_")[0]
        out[f"{name}_us_per_call_max_over_ranks"] = us
        out[f"{name}_elems_per_s_aggregate"] = world * T * B / (us * 1e-6)
        out[f"{name}_frac_per_gpu"] = T * B * nb / (us * 1e-6) / 1e9 / peak
    return out


def bench_ppo(dev, rpl):
    """GAE + discounted returns on [128, 4096] (configs[1]); inputs rotate over a
    pool larger than L2 so every call reads HBM."""
    import torch
    from synth import returns_inputs
    T, B = PPO["T"], PPO["B"]
    r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    per = T * B * 17
    pool = max(4, int(math.ceil(4 * l2 / per)))
    R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
    V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
    D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
    BT = torch.from_numpy(boot).to(dev)
    A = torch.empty_like(R)
    RT = torch.empty_like(R)
    def capture(fn):
        for i in range(pool):  # warm (outside capture)
            fn(i)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream(dev)
        st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.graph(gr, stream=st):
            for i in range(pool):
                fn(i)
        torch.cuda.synchronize()
        return gr

    def timeit(gr, reps=10):
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (reps * pool)

    g_gae = capture(lambda i: rpl.gae(R[i], V[i], D[i], BT, PPO["gamma"], PPO["lam"], adv=A[i], ret=RT[i]))
    g_disc = capture(lambda i: rpl.returns_discounted(R[i], D[i], BT, PPO["gamma"], out=RT[i]))
    QB = torch.zeros_like(BT)
    DN = torch.empty((T - 4, B), dtype=torch.uint8, device=dev)
    g_nstep = capture(lambda i: rpl.returns_nstep(R[i], D[i], 5, PPO["gamma"], q=V[i], q_boot=QB, rescale=True,
                                                  out=A[i][:T - 4], done_out=DN))
    ms_gae = timeit(g_gae)
    ms_disc = timeit(g_disc)
    ms_nstep = timeit(g_nstep)
    peak, kind = measured_peaks()
    gae_gbs = T * B * 17 / (ms_gae / 1e3) / 1e9
    disc_gbs = (T * B * 9 + B * 4) / (ms_disc / 1e3) / 1e9
    return {"workload": "ppo_[128,4096]", "unit": "elems/s",
            "gae_elems_per_s": T * B / (ms_gae / 1e3), "gae_us_per_call": ms_gae * 1e3, "gae_GBps": gae_gbs,
            "gae_frac": gae_gbs / peak, "disc_elems_per_s": T * B / (ms_disc / 1e3),
            "disc_us_per_call": ms_disc * 1e3, "disc_GBps": disc_gbs, "disc_frac": disc_gbs / peak,
            "nstep_us_per_call": ms_nstep * 1e3, "nstep_note": "rescaled 5-step target, bootstrap q = V rows",
            "l2": f"input pool {pool} x {per/1e6:.1f} MB > 4 x L2",
            "timing": "CUDA graph of one call per pool entry, replayed; per-call average"}


def pipelined_step(dev, rpl, tree, plan, idx_buf, td_pool, q_pool, err, c, n, P, seed):
    """SURVEY §8d's secondary step variant: the same four calls, but update(i+1) +
    sample(i+1) run on a second stream while gather(i) + n-step(i) run (the paper's
    asynchronous sampler/optimiser overlap, Fig. 3).  Dependencies: gather(i) waits for
    sample(i); sample(i) waits for gather(i-2) (it overwrites that batch's idx / q)."""
    import torch
    lib, P_ = rpl._lib.lib, rpl.ops._ptr
    qb = [torch.zeros(n, dtype=torch.int64, device=dev) for _ in range(2)]
    sA, sB = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_s = [torch.cuda.Event() for _ in range(P)]
    ev_g = [torch.cuda.Event() for _ in range(P)]

    def run(P_steps):
        for i in range(P_steps):
            cur, prev = idx_buf[i % 2], idx_buf[(i + 1) % 2]
            with torch.cuda.stream(sA):
                if i >= 2:
                    sA.wait_event(ev_g[(i - 2) % P])
                a = rpl.ops._stream(dev)
                rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(prev), P_(td_pool[i % P]),
                                                          c["train"], n, c["eta"], c["alpha"], c["eps_p"], 0, None, a),
                               "update_seq")
                rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, seed, c["beta"],
                                                             P_(cur), P_(qb[i % 2]), None, None, P_(err), a),
                               "sample")
                ev_s[i % P].record(sA)
            with torch.cuda.stream(sB):
                sB.wait_event(ev_s[i % P])
                b = rpl.ops._stream(dev)
                plan.run(cur, q=qb[i % 2], qmin=None, beta=c["beta"], err=err, stream=b, q_tgt=q_pool[i % P])
                ev_g[i % P].record(sB)

    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    for s_ in (sA, sB):
        s_.wait_stream(cap)
    run(P)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        sA.wait_stream(cap)
        sB.wait_stream(cap)
        run(P)
        cap.wait_stream(sA)
        cap.wait_stream(sB)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    rpl.check_err(err)
    ms = e0.elapsed_time(e1) / (reps * P)
    return {"us_per_step": ms * 1e3, "sequences_per_s": n / (ms / 1e3),
            "timing": "CUDA graph of 8 steps on two streams (update+sample || gather with fused targets), replayed"}


def bench_r2d2_1mseq(dev, rpl, c):
    """The north_star's 1M-sequence buffer at N=1: ONE of its 8 shards, a [40960, 128] ring
    (37 GB of frames, 131,072 sequence leaves, D=4 tree), same 4-call step as the headline
    (graph of 8 steps).  The frames span ~145x the TLB reach."""
    return time_r2d2_step(dev, rpl, c, R2D2_1MSEQ_SHARD["cap_T"], R2D2_1MSEQ_SHARD["B"], 31337, 777,
                          "r2d2_1mseq_one_shard")


FUSED_SAMPLE = [True]  # set from --fused-sample (the secondaries time the headline's step shape)


def seed_sweep(dev, rpl, c, main_us):
    """seeds 0-4, median reported — seed 0 is the headline measurement; seeds 1-4
    rebuild the [4000, 256] ring (device generator), tree and graph and re-time the step."""
    us = [main_us] + [time_r2d2_step(dev, rpl, c, c["cap_T"], c["B"], 2019 + 101 * s, 1234 % c["cap_T"],
                                     "r2d2_1mstep")["us_per_step"] for s in range(1, 5)]
    med = sorted(us)[len(us) // 2]
    return {"us_per_step_by_seed": us, "median_us_per_step": med, "median_sequences_per_s": c["batch"] / (med / 1e6)}


def time_r2d2_step(dev, rpl, c, cap, B, seed, cursor, workload):
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    L, k, period, n = c["L"], c["k"], c["period"], c["batch"]
    ring = make_ring_device(seed, cap, B, dev, ep_len=2000.0, period=period, rnn_parts=c["rnn_parts"],
                            rnn_h=c["rnn_h"], cursor=cursor)
    n_leaves = (cap // period) * B
    tree = rpl.SumTree(n_leaves, c["fanout"], 32, device=dev)
    valid = torch.from_numpy(R.leaves_of(R.valid_sequence_blocks(cap, period, ring.cursor, ring.size, k, L), B)).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    tree.update(valid, torch.randn(valid.numel(), generator=g, device=dev).abs(), c["alpha"], c["eps_p"])
    qv = None
    plan = None
    idx = [torch.full((n,), -1, dtype=torch.int64, device=dev) for _ in range(2)]
    q = torch.zeros(n, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    td = torch.randn((8, c["train"], n), generator=g, device=dev).abs()
    qv = torch.randn((8, L, n), generator=g, device=dev) * 10
    plan = rpl.GatherPlan(ring, n, kind="sequence", k=k, seq_len=L, period=period, with_weights=True,
                          targets=r2d2_targets(c, qv[0]))
    out = plan.outputs
    lib, P_ = rpl._lib.lib, rpl.ops._ptr

    def step(i):
        s = rpl.ops._stream(dev)
        rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(idx[(i + 1) % 2]), P_(td[i % 8]),
                                                  c["train"], n, c["eta"], c["alpha"], c["eps_p"], 0, None, s), "upd")
        if FUSED_SAMPLE[0]:
            plan.run_sample(tree, 0xBEEF, idx[i % 2], q, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])
            return
        rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, 0xBEEF, c["beta"], P_(idx[i % 2]),
                                                     P_(q), None, None, P_(err), s), "sample")
        plan.run(idx[i % 2], q=q, qmin=None, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])

    ms = _graph_time(dev, step, P=8, reps=50)
    rpl.check_err(err)
    res = {"workload": workload, "seed": seed, "ring_per_gpu": [cap, B], "ring_gb": ring.obs.numel() / 1e9,
           "leaves_per_gpu": n_leaves, "tree_depth": tree.depth, "us_per_step": ms * 1e3,
           "sequences_per_s": n / (ms / 1e3), "timing": "CUDA graph of 8 steps, replayed"}
    del ring, tree, plan, out
    torch.cuda.empty_cache()
    return res


def unique_output_step(dev, rpl, tree, ring, idx_buf, td_pool, q_pool, err, c, n, P, seed):
    """The headline step with RPL_OUT_UNIQUE output: the gather writes each sequence's 128
    unique frames once ([L+k-1, n, 84, 84]) instead of 125 k-stacks (the learner's first
    layer stacks on the fly) — SURVEY §8d's 'unique' byte count: 116 MB per 64 sequences."""
    import torch
    from paper_1909_01500_b200 import _lib
    lib, P_ = rpl._lib.lib, rpl.ops._ptr
    L, k, period = c["L"], c["k"], c["period"]
    plan = rpl.GatherPlan(ring, n, kind="sequence", k=k, seq_len=L, period=period, with_weights=True,
                          out_mode=_lib.OUT_UNIQUE, targets=r2d2_targets(c, q_pool[0]))
    q = torch.zeros(n, dtype=torch.int64, device=dev)

    def step(i):
        s = rpl.ops._stream(dev)
        cur, prev = idx_buf[i % 2], idx_buf[(i + 1) % 2]
        rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(prev), P_(td_pool[i % P]),
                                                  c["train"], n, c["eta"], c["alpha"], c["eps_p"], 0, None, s), "upd")
        if FUSED_SAMPLE[0]:
            plan.run_sample(tree, seed, cur, q, beta=c["beta"], err=err, stream=s, q_tgt=q_pool[i % P])
            return
        rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, seed, c["beta"], P_(cur), P_(q),
                                                     None, None, P_(err), s), "sample")
        plan.run(cur, q=q, qmin=None, beta=c["beta"], err=err, stream=s, q_tgt=q_pool[i % P])

    ms = _graph_time(dev, step, P=8, reps=50)
    rpl.check_err(err)
    ub = seq_bytes_per_sample(c) - c["L"] * k * FRAME + (c["L"] + k - 1) * FRAME
    return {"out": "unique", "us_per_step": ms * 1e3, "sequences_per_s": n / (ms / 1e3),
            "alg_bytes_per_sequence": ub, "timing": "CUDA graph of 8 steps, replayed"}


def tree_latency(dev, rpl):
    """Sampled-lookup latency: events over a graph of 16 sample-only
    (and update-only) launches on the R2D2 (25,600 leaves, n=64) and DQN (2^20, n=512) trees."""
    import torch
    res = {}
    for N, n in ((25600, 64), (1 << 20, 512)):
        t = rpl.SumTree(N, 32, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(N)
        t.update(torch.arange(N, device=dev), torch.rand(N, generator=g, device=dev) + 1e-3, 0.9)
        idx = torch.randint(0, N, (n,), generator=g, device=dev)
        td = torch.rand(n, generator=g, device=dev)
        outs = (torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int64, device=dev), None,
                None)
        us_s = _graph_time(dev, lambda i: t.sample_stream(n, 3, out=outs, want_qmin=False), P=16, reps=20) * 1e3
        us_u = _graph_time(dev, lambda i: t.update(idx, td, 0.9), P=16, reps=20) * 1e3
        res[f"N{N}_n{n}"] = {"sample_us": us_s, "update_us": us_u, "depth": t.depth}
        del t
    return {"unit": "us per launch (graph-replayed, back to back)", **res}


class _ExtEvent:
    """A timing event recorded with cudaEventRecordExternal, so that inside stream capture
    it becomes an event-record node of the graph (torch's Event.record there only marks a
    capture dependency)."""
    _rt = None

    def __init__(self):
        import torch
        self.ev = torch.cuda.Event(enable_timing=True)
        self.ev.record()  # create the CUDA event
        if _ExtEvent._rt is None:
            import ctypes
            import glob
            import os as _os
            import nvidia.cuda_runtime as _cr
            libs = sorted(glob.glob(_os.path.join(list(_cr.__path__)[0], "lib", "libcudart.so*")))
            rt = ctypes.CDLL(libs[0])
            rt.cudaEventRecordWithFlags.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
            rt.cudaEventRecordWithFlags.restype = ctypes.c_int
            _ExtEvent._rt = rt

    def record(self):
        import torch
        st = torch.cuda.current_stream().cuda_stream
        rc = _ExtEvent._rt.cudaEventRecordWithFlags(self.ev.cuda_event, st, 1)  # cudaEventRecordExternal
        if rc != 0:
            raise RuntimeError(f"cudaEventRecordWithFlags failed ({rc})")


def gather_ms_in_graph(dev, step, P, reps=25):
    """Mean gather launch duration (ms) over the P gathers of a graph of P steps, each
    bracketed by event-record nodes; averaged over `reps` replays."""
    import torch
    side = torch.cuda.Stream(dev)
    evs = [(_ExtEvent(), _ExtEvent(), side) for _ in range(P)]
    torch.cuda.synchronize()
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for i in range(P):
            step(i, evs[i])
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        gr.replay()
        torch.cuda.synchronize()
        tot += sum(a.ev.elapsed_time(b.ev) for a, b, _ in evs) / P
    return tot / reps


def _stats(us):
    a = np.asarray(us, np.float64)
    return {"n": int(a.size), "median_us": float(np.median(a)), "p10_us": float(np.percentile(a, 10)),
            "p90_us": float(np.percentile(a, 90)), "mean_us": float(a.mean())}


def _graph_time(dev, step, P=8, reps=25):
    """Capture P consecutive steps in one CUDA graph (after warm-up) and return the
    mean device time per step over `reps` replays (CUDA events on the replay stream)."""
    import torch
    for i in range(2 * P):
        step(i)
    torch.cuda.synchronize()
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for i in range(P):
            step(i)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * P)


def transition_bytes(k, n, obs_bytes, act_bytes, stacked_frames=True):
    """Algorithmic bytes of one gathered transition: unique obs rows
    t-k+1..t+n read once, two k-stacks written, n rewards + n dones + action in,
    action + return + done_n + IS weight out."""
    rd = (k + n) * obs_bytes + n * 5 + act_bytes
    wr = 2 * k * obs_bytes + act_bytes + 4 + 1 + 4
    return rd + wr


def bench_dqn(dev, rpl):
    """configs[2]: 2^20-transition frame ring [4096, 256], tree of 2^20 leaves; one step
    = update(previous batch) -> sample_stream(bs) + IS weights -> transition gather
    (k=4 stacks at t and t+3, fused 3-step return)."""
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    c = DQN
    ring = make_ring_device(404, c["cap_T"], c["B"], dev, ep_len=2000.0, cursor=1111, with_rnn=False)
    N = c["cap_T"] * c["B"]
    tree = rpl.SumTree(N, c["fanout"], 32, device=dev)
    rows = R.valid_transition_rows(c["cap_T"], ring.cursor, ring.size, c["k"], c["n_step"])
    valid = torch.from_numpy(R.leaves_of(rows, c["B"])).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    tree.update(valid, torch.randn(valid.numel(), generator=g, device=dev).abs(), c["alpha"], c["eps_p"])
    out = {}
    lib, P_ = rpl._lib.lib, rpl.ops._ptr
    for bs in c["batches"]:
        plan = rpl.GatherPlan(ring, bs, kind="transition", k=c["k"], n_step=c["n_step"], gamma=c["gamma"],
                              with_weights=True)
        idx = [torch.full((bs,), -1, dtype=torch.int64, device=dev) for _ in range(2)]
        q = torch.zeros(bs, dtype=torch.int64, device=dev)
        td = torch.randn((8, bs), generator=g, device=dev).abs()
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        def step(i):
            s = rpl.ops._stream(dev)
            cur, prev = idx[i % 2], idx[(i + 1) % 2]
            rpl._lib.check(lib.rpl_sumtree_update(tree._lp, P_(tree.storage), P_(prev), P_(td[i % 8]), bs,
                                                  c["alpha"], c["eps_p"], None, s), "update")
            rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), bs, 0xD00, c["beta"], P_(cur),
                                                         P_(q), None, None, P_(err), s), "sample")
            plan.run(cur, q=q, qmin=None, beta=c["beta"], err=err, stream=s)  # IS weights fused

        ms = _graph_time(dev, step)
        rpl.check_err(err)
        nb = bs * transition_bytes(c["k"], c["n_step"], 7056, 8)
        out[f"bs{bs}"] = {"us_per_step": ms * 1e3, "samples_per_s": bs / (ms / 1e3),
                          "step_GBps": nb / (ms / 1e3) / 1e9}
    del ring, tree
    torch.cuda.empty_cache()
    return {"workload": "dqn_atari_1M_transitions", "unit": "transitions/s", "ring": [c["cap_T"], c["B"]],
            "leaves": N, "k": c["k"], "n_step": c["n_step"], "alpha": c["alpha"], "beta": c["beta"],
            "timing": "CUDA graph of 8 steps (update+sample+gather), replayed", **out}


def bench_mujoco(dev, rpl):
    """configs[3]: uniform + n-step replay over a [65536, 16] f32 vector ring (2^20
    transitions); one step = rpl_sample_uniform(256) -> transition gather (obs at t
    and t+3, action, fused 3-step return)."""
    import torch
    from paper_1909_01500_b200 import replay as R
    from synth.device import make_ring_device
    c = MUJOCO
    res = {}
    for D, A in c["dims"]:
        ring = make_ring_device(505 + D, c["cap_T"], c["B"], dev, ep_len=1000.0, cursor=2222, vec_dim=D, act_dim=A,
                                with_rnn=False)
        rows = R.valid_transition_rows(c["cap_T"], ring.cursor, ring.size, 1, c["n_step"])
        # valid rows form one ring interval: oldest valid row and count
        age = (ring.cursor - 1 - rows) % c["cap_T"]
        lo_row = int(rows[np.argmax(age)])
        n_rows = int(rows.size)
        bs = c["batch"]
        plan = rpl.GatherPlan(ring, bs, kind="transition", k=1, n_step=c["n_step"], gamma=c["gamma"])
        idx = torch.zeros(bs, dtype=torch.int64, device=dev)
        ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)

        def step(i):
            s = rpl.ops._stream(dev)
            rpl._lib.check(rpl._lib.lib.rpl_sample_uniform(bs, 0xA11, 0, rpl.ops._ptr(ctr), lo_row, n_rows,
                                                           c["cap_T"], c["B"], rpl.ops._ptr(idx), s), "uniform")
            plan.run(idx, err=err, stream=s)

        ms = _graph_time(dev, step)
        rpl.check_err(err)
        nb = bs * transition_bytes(1, c["n_step"], 4 * D, 4 * A)
        res[f"D{D}_A{A}"] = {"us_per_step": ms * 1e3, "samples_per_s": bs / (ms / 1e3),
                             "step_GBps": nb / (ms / 1e3) / 1e9}
        del ring
        torch.cuda.empty_cache()
    return {"workload": "mujoco_uniform_1M_transitions", "unit": "transitions/s", "ring": [c["cap_T"], c["B"]],
            "batch": c["batch"], "n_step": c["n_step"],
            "timing": "CUDA graph of 8 steps (uniform sample+gather), replayed", **res}


# ----------------------------------------------------------------------------- oracle arm
class OracleStep:
    """The CPU oracle doing the same R2D2 step (update + sample + gather + rescaled
    n-step targets) on host copies of the same inputs."""

    def __init__(self, c, host, seed=77):
        # oracle + synth only: this arm never imports the product package (no librpl.so)
        from oracle import gather as OG
        from oracle import sumtree as OS
        self.c, self.h = c, host
        B = host.obs.shape[1]
        self.B = B
        n_blocks = c["cap_T"] // c["period"]
        self.tree = OS.SumTreeOracle(n_blocks * B)
        # every leaf (block * B + b) whose sequence window is stored (§8c #16)
        valid = [blk * B + b for blk in range(n_blocks)
                 if OG.window_valid_sequence(blk * c["period"], c["cap_T"], host.cursor, host.size, c["k"], c["L"])
                 for b in range(B)]
        g = np.random.Generator(np.random.PCG64(seed))
        td0 = np.abs(g.normal(size=len(valid))).astype(np.float32)
        self.tree.update(valid, [float(x) for x in td0], c["alpha"], c["eps_p"])
        self.g = g
        self.prev = []
        self.ctr = 0

    def step(self, nseq):
        from oracle import gather as OG
        from oracle import philox as OP
        from oracle import returns as OR
        from oracle import sumtree as OS
        c, h = self.c, self.h
        from oracle import priority as OPR
        steps = np.abs(self.g.normal(size=(c["train"], len(self.prev)))).astype(np.float32)
        td = [OPR.sequence_td(steps[:, j], c["eta"]) for j in range(len(self.prev))]
        self.tree.update(self.prev, td, c["alpha"], c["eps_p"])
        draws = OP.draws_u64(0x5EED, self.ctr, nseq)
        self.ctr += nseq
        idx, q, qmin = self.tree.sample(nseq, draws)
        OS.is_weights(q, self.tree.total(), self.tree.n_leaves, c["beta"])
        out = OG.gather_sequences(idx, self.B, h.obs, h.act, h.rew, h.done, h.rnn, c["k"], c["L"], c["period"])
        lo = c["burn_in"]
        Tn = c["train"] + c["n_step"] - 1
        qv = self.g.normal(0, 10, (c["L"], nseq))
        OR.nstep_return(out["rew"][lo:lo + Tn], out["done"][lo:lo + Tn], c["n_step"], c["gamma"],
                        q=qv[lo:lo + Tn], q_boot=qv[lo + Tn], rescale=True, eps=c["eps"])
        self.prev = idx
        return nseq


def _cores():
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return aff, model


def cpu_baseline_subprocess(seconds):
    """The cpu_baseline leg in a fresh interpreter (oracle + synth only), so the oracle never
    runs in a process that has the product library mapped."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--cpu-baseline-leg",
           "--cpu-seconds", str(seconds)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    if res.returncode != 0 or not lines:
        raise RuntimeError(f"cpu_baseline leg failed (rc={res.returncode}): {res.stderr[-300:]}")
    return json.loads(lines[-1])


def cpu_baseline(c, host, seconds):
    for v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[v] = "1"
    o = OracleStep(c, host)
    o.step(4)  # warm
    t0 = time.time()
    done = 0
    nsteps = 0
    while time.time() - t0 < seconds:
        done += o.step(c["batch"])
        nsteps += 1
    dt = time.time() - t0
    aff, model = _cores()
    return {"value": done / dt, "unit": "sequences/s", "cores": 1, "kind": "oracle",
            "sample": f"{nsteps} full R2D2 steps ({c['batch']} sequences each: eta-mixed update + sample over "
                      f"{o.tree.n_leaves} leaves + stacked gather + rescaled 5-step targets), {dt:.1f} s",
            "host_cpus": os.cpu_count(), "affinity": aff, "cpu_model": model}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return  # N > 1: rank 0 alone runs the oracle
    for v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[v] = "1"
    from synth import make_ring
    c = dict(R2D2)
    host = make_ring(2019, c["cap_T"], c["B"], ep_len=2000.0, reward_kind="r2d2", period=c["period"],
                     rnn_parts=c["rnn_parts"], rnn_h=c["rnn_h"], cursor=1234 % c["cap_T"])
    if args.cpu_baseline_leg:  # the product arm's cpu_baseline, run in this separate process
        print(json.dumps(cpu_baseline(c, host, args.cpu_seconds)))
        return
    o = OracleStep(c, host)
    t0 = time.time()
    o.step(2)
    per_seq = max(1e-3, (time.time() - t0) / 2)
    K, W = args.steps, args.warmup
    budget = 150.0
    nseq = int(max(1, min(c["batch"], budget / max(1, K + min(W, 3)) / per_seq)))
    for _ in range(min(W, 3)):
        o.step(nseq)
    t0 = time.time()
    done = 0
    for _ in range(K):
        done += o.step(nseq)
    dt = time.time() - t0
    aff, model = _cores()
    val = done / dt
    res = {"impl": "reference", "metric": "prioritized samples/sec (update+sample+gather)", "value": val,
           "unit": "sequences/s", "n_gpus": world, "steps": K, "warmup": min(W, 3), "ms_per_step": dt / K * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 / python int",
           "data": "synthetic (seeded, same recipe)",
           "config": dict(r2d2_config(c, 1), timing="host wall clock, single thread",
                          oracle_batch_per_step=nseq),
           "cpu_baseline": {"value": val, "unit": "sequences/s", "cores": 1, "kind": "oracle",
                            "sample": f"{K} steps of {nseq} sequences (bounded sample of the 64-sequence step)",
                            "host_cpus": os.cpu_count(), "affinity": aff, "cpu_model": model},
           "e2e": {"value": val, "unit": "sequences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    res["native_so_loaded"] = _repo_so_mapped()  # evidence: the oracle arm maps no product library
    print(json.dumps(res))


def _repo_so_mapped():
    """Shared objects under this repository mapped into this process (/proc/self/maps)."""
    root = os.path.dirname(os.path.abspath(__file__))
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so") or ".so." in ln}
    except OSError:
        return None
    return sorted(p for p in paths if p.startswith(root))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_rpl(args)


if __name__ == "__main__":
    main()
