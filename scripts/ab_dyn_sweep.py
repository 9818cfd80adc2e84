"""In-process sweep of the dynamic-tail gather's schedule (rpl_debug_set_gather_dyn) on bench.py's
R2D2 step: one ring/tree/plan, one 8-step graph per setting, replayed round-robin; median us
per step per setting.  SETTINGS="100,5,8 80,8,8 ..." (pct,rows,lookahead; lookahead may be
look:end_look:threshold — the queue drops to end_look once fewer than threshold rows are
left in the pool); STEP=pair|fused."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("STEP", "pair")
import ab_inproc as A  # noqa: E402

graphs = {}
for st in os.environ.get("SETTINGS", "100,5,8 80,5,8 80,8,8").split():
    pct, rows, lk = st.split(",")
    pct, rows = int(pct), int(rows)
    lp = [int(x) for x in lk.split(":")]  # look[:end_look:end_threshold_rows]
    look = lp[0] | ((lp[1] if len(lp) > 1 else 0) << 8) | ((lp[2] if len(lp) > 2 else 0) << 16)
    assert A.rpl._lib.lib.rpl_debug_set_gather_dyn(pct, rows, look) == 0
    graphs[st] = A.capture(None)
print(json.dumps({"step": os.environ["STEP"], "median_us_per_step": A.compare(graphs, rounds=15)}))
