"""R2D2 step timeline (needs a -DRPL_TRACE build): globaltimer stamps of the update, sampler and
sequence-gather kernels of the LAST step of a replayed 8-step graph (bench.py's step shape:
update_seq -> sample_stream -> gather with fused targets), ns relative to the update kernel's
entry.  Median over 30 replays."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402
from paper_1909_01500_b200 import replay as R  # noqa: E402
from synth.device import make_ring_device  # noqa: E402

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
if os.environ.get("UPD_TRIG"):  # rpl_debug_set_upd_trigger
    assert lib.rpl_debug_set_upd_trigger(int(os.environ["UPD_TRIG"])) == 0
if os.environ.get("DYN"):  # DYN=pct,rows,lookahead (rpl_debug_set_gather_dyn)
    assert lib.rpl_debug_set_gather_dyn(*(int(x) for x in os.environ["DYN"].split(","))) == 0
MODE = os.environ.get("STEP", "pair")  # pair: update -> sample -> gather; fused: update -> gather_sample


DOUBLE = os.environ.get("DOUBLE_UPD", "0") == "1"  # run the update twice (the trace shows the second)


def step(i):
    s = rpl.ops._stream(dev)
    if MODE == "one":  # update + sampling + gather in one launch
        plan.run_update_sample(tree, idx[(i + 1) % 2], td[i % 8], 0xBEEF, idx[i % 2], q, eta=c["eta"], alpha=c["alpha"],
                               eps_p=c["eps_p"], beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])
        return
    for _ in range(2 if DOUBLE else 1):
        rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(idx[(i + 1) % 2]), P_(td[i % 8]),
                                                  c["train"], n, c["eta"], c["alpha"], c["eps_p"], 0, None, s),
                       "upd")
    if MODE == "fused":
        plan.run_sample(tree, 0xBEEF, idx[i % 2], q, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])
        return
    rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, 0xBEEF, c["beta"], P_(idx[i % 2]),
                                                 P_(q), None, None, P_(err), s), "sample")
    plan.run(idx[i % 2], q=q, qmin=None, beta=c["beta"], err=err, stream=s, q_tgt=qv[i % 8])


for i in range(16):
    step(i)
torch.cuda.synchronize()
st = torch.cuda.Stream(dev)
st.wait_stream(torch.cuda.current_stream(dev))
gr = torch.cuda.CUDAGraph()
PSTEPS = int(os.environ.get("P_STEPS", "8"))
with torch.cuda.graph(gr, stream=st):
    for i in range(PSTEPS):
        step(i)
for _ in range(5):
    gr.replay()
torch.cuda.synchronize()
names_u = {7: "update_entry", 0: "update_past_wait", 2: "update_mixed", 3: "update_hash_reset",
           4: "update_dedupe", 5: "update_leaves", 6: "update_end", 8: "sample_past_wait", 9: "sample_end"}
DYN = os.environ.get("STEP", "pair") != "static"
names_g = {0: "gather_entry", 1: "gather_past_wait", 2: "gather_first_frames (dyn: staged)", 3: "gather_end",
           4: "gather_smp_staged (dyn: earliest CTA entry)", 5: "gather_smp_sampled (dyn: earliest past wait)",
           6: "gather_first_tma_issue (dyn: latest past wait)", 7: "gather_pieces_done (dyn: descents done)",
           8: "gather_first_cta_end"}
runs = []
bu, bg = (ctypes.c_int64 * 16)(), (ctypes.c_int64 * 9)()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
STEADY = os.environ.get("STEADY", "0") == "1"  # 1: 10 back-to-back replays per sample (steady state)
for _ in range(30):
    if not STEADY:
        lib.rpl_debug_trace_reset()
    e0.record()
    for _ in range(10 if STEADY else 1):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    if lib.rpl_debug_trace(bu, 16) != 0 or lib.rpl_debug_gather_trace(bg, 9) != 0:  # not a trace build
        runs.append({"graph_us_per_step": e0.elapsed_time(e1) * 1e3 / ((10 if STEADY else 1) * PSTEPS)})
        continue
    t0 = bu[7]
    r = {v: bu[kk] - t0 for kk, v in names_u.items() if kk != 8 or MODE != "fused"}
    r.update({v: bg[kk] - t0 for kk, v in names_g.items() if bg[kk] != 0})
    r["graph_us_per_step"] = e0.elapsed_time(e1) * 1e3 / ((10 if STEADY else 1) * PSTEPS)
    runs.append(r)
med = {kk: sorted(r[kk] for r in runs if kk in r)[len([r for r in runs if kk in r]) // 2] for kk in runs[0]}
ends = (ctypes.c_int64 * (3 * 146))()
if lib.rpl_debug_gather_cta_ends(ends, 146) == 0:  # the last launch's per-CTA ends, relative to its update
    import numpy as np
    allv = np.array(list(ends), np.int64)
    e = (allv[:146] - t0) / 1e3
    st_ = (allv[146:292] - t0) / 1e3
    un = allv[292:]
    if un.sum() > 0:
        order = np.argsort(e)
        med["dyn_units_total"] = int(un.sum())
        med["dyn_slowest8_end_static_units"] = [[int(i), round(float(e[i]), 2), round(float(st_[i]), 2), int(un[i])]
                                                for i in order[-8:]]
        med["dyn_fastest4_end_static_units"] = [[int(i), round(float(e[i]), 2), round(float(st_[i]), 2), int(un[i])]
                                                for i in order[:4]]
        gb = (ctypes.c_int64 * (16 * 146))()
        if lib.rpl_debug_gather_grabs(gb, 146) == 0:
            ga = np.array(list(gb), np.int64).reshape(146, 8, 2)
            med["dyn_slowest4_grabs_t_rows_queued"] = [
                [int(i), [[round((int(ga[i, j, 0]) - t0) / 1e3, 2), int(ga[i, j, 1]) >> 32, int(ga[i, j, 1]) & 0xffffffff]
                          for j in range(min(8, int(un[i])))]] for i in order[-4:]]
        med["dyn_static_done_p0_p50_p100"] = [round(float(np.percentile(st_[:145], p_)), 2) for p_ in (0, 50, 100)]
    med["cta_end_us_percentiles_p0_p10_p50_p90_p100_last"] = [round(float(np.percentile(e[:145], p_)), 2)
                                                            for p_ in (0, 10, 50, 90, 100)] + [round(float(e[145]), 2)]
    med["cta_end_us_slowest_ctas"] = [int(x) for x in np.argsort(e)[-8:]]
print(json.dumps({"mode": MODE, "steady": STEADY, "ns_from_update_entry_median": dict(sorted(med.items(), key=lambda kv: kv[1] if not isinstance(kv[1], list)
                                                                     else 1e18)),
                  "note": "last step of a replayed 8-step graph; -DRPL_TRACE build"}, indent=1))
