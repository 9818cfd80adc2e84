"""In-process A/B of a runtime knob on bench.py's R2D2 step (fused sampling): one ring, tree and
plan; graph A captured with the knob at its A value, graph B at its B value; the two graphs
replayed alternately (10 replays of 8 steps each, 20 rounds), so memory placement, clocks and
box are shared.  KNOB=upd_trigger A=-1 B=3 (rpl_debug_set_upd_trigger)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402
from paper_1909_01500_b200 import replay as R  # noqa: E402
from synth.device import make_ring_device  # noqa: E402

KNOB = os.environ.get("KNOB", "upd_trigger")
VA, VB = int(os.environ.get("A", "-1")), int(os.environ.get("B", "3"))
DYN_ROWS, DYN_LOOK = int(os.environ.get("DYN_ROWS", "5")), int(os.environ.get("DYN_LOOK", "8"))


def _set_dyn(v):  # KNOB=dyn_pct: the static share of the dynamic-tail gather (0 = all dynamic? no: 0 = off)
    return rpl._lib.lib.rpl_debug_set_gather_dyn(v, DYN_ROWS, DYN_LOOK)


setter = {"upd_trigger": rpl._lib.lib.rpl_debug_set_upd_trigger,
          "dyn_pct": _set_dyn,
          "gather_trigger": rpl._lib.lib.rpl_debug_set_gather_trigger,
          "upd_multi": rpl._lib.lib.rpl_debug_set_upd_multi,
          "gather_variant": rpl._lib.lib.rpl_debug_set_gather_variant,
          "scan_variant": rpl._lib.lib.rpl_debug_set_scan_variant}[KNOB]
dev = torch.device("cuda:0")
c = dict(bench.R2D2)
L, k, period, n = c["L"], c["k"], c["period"], c["batch"]
cap, B = c["cap_T"], c["B"]
ring = make_ring_device(2019, cap, B, dev, ep_len=2000.0, period=period, rnn_parts=c["rnn_parts"], rnn_h=c["rnn_h"],
                        cursor=1234 % cap)
tree = rpl.SumTree((cap // period) * B, c["fanout"], 32, device=dev)
valid = torch.from_numpy(R.leaves_of(R.valid_sequence_blocks(cap, period, ring.cursor, ring.size, k, L), B)).to(dev)
g = torch.Generator(device=dev)
g.manual_seed(5)
tree.update(valid, torch.randn(valid.numel(), generator=g, device=dev).abs(), c["alpha"], c["eps_p"])
idx = [torch.full((n,), -1, dtype=torch.int64, device=dev) for _ in range(2)]
q = torch.zeros(n, dtype=torch.int64, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
td = torch.randn((8, c["train"], n), generator=g, device=dev).abs()
qv = torch.randn((8, L, n), generator=g, device=dev) * 10
plan = rpl.GatherPlan(ring, n, kind="sequence", k=k, seq_len=L, period=period, with_weights=True,
                      targets=bench.r2d2_targets(c, qv[0]))
lib, P_ = rpl._lib.lib, rpl.ops._ptr
FUSED = os.environ.get("STEP", "fused") in ("fused", "one")


def step(i):
    s = rpl.ops._stream(dev)
    if os.environ.get("STEP") == "one":  # update + sampling + gather in one launch
        plan.run_update_sample(tree, idx[(i + 1) % 2], td[i % 8], 0xBEEF, idx[i % 2], q, eta=c["eta"], alpha=c["alpha"],
                               eps_p=c["eps_p"], beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])
        return
    rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(idx[(i + 1) % 2]), P_(td[i % 8]),
                                              c["train"], n, c["eta"], c["alpha"], c["eps_p"], 0, None, s), "upd")
    if FUSED:
        plan.run_sample(tree, 0xBEEF, idx[i % 2], q, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])
        return
    rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, 0xBEEF, c["beta"], P_(idx[i % 2]),
                                                 P_(q), None, None, P_(err), s), "sample")
    plan.run(idx[i % 2], q=q, qmin=None, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])


BASE = {k_: int(v_) for k_, v_ in (kv.split("=") for kv in os.environ.get("BASE", "").split(",") if kv)}
for k_, v_ in BASE.items():  # other knobs held fixed for both graphs, e.g. BASE=upd_trigger=2
    assert {"upd_trigger": rpl._lib.lib.rpl_debug_set_upd_trigger,
            "upd_multi": rpl._lib.lib.rpl_debug_set_upd_multi,
            "gather_trigger": rpl._lib.lib.rpl_debug_set_gather_trigger}[k_](v_) == 0


def capture(v):
    if v is not None:
        assert setter(v) == 0
    for i in range(16):
        step(i)
    torch.cuda.synchronize()
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for i in range(8):
            step(i)
    torch.cuda.synchronize()
    return gr


def compare(graphs, rounds=20, reps=10):
    """Median us per step of each graph, replayed round-robin (order rotated every round)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {name: [] for name in graphs}
    names = list(graphs)
    for r in range(rounds):
        for name in names[r % len(names):] + names[:r % len(names)]:
            gr = graphs[name]
            gr.replay()
            e0.record()
            for _ in range(reps):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) * 1e3 / (8 * reps))
    return {kk: sorted(v)[len(v) // 2] for kk, v in res.items()}


if __name__ == "__main__":
    med = compare({"A": capture(VA), "B": capture(VB)})
    print(json.dumps({"knob": KNOB, "A": VA, "B": VB, "step": "fused" if FUSED else "pair",
                      "median_us_per_step": med, "delta_B_minus_A_us": med["B"] - med["A"]}))
