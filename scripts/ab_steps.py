"""In-process A/B of the R2D2 step SHAPES on one ring / tree / plan: 'one' (rpl_gather_update_sample,
one launch), 'fused' (update_seq -> rpl_gather_sample), 'pair' (update_seq -> sample_stream ->
gather), optionally with a gather PDL trigger (name:gt=T): one 8-step graph each, replayed round-robin; median us per step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ab_inproc as A  # noqa: E402

graphs = {}
for name in os.environ.get("SHAPES", "one fused pair").split():
    shape, _, gt = name.partition(":gt=")  # e.g. one:gt=0 captures with rpl_debug_set_gather_trigger(0)
    os.environ["STEP"] = shape
    A.FUSED = shape in ("fused", "one")
    if gt:
        assert A.lib.rpl_debug_set_gather_trigger(int(gt)) == 0
    graphs[name] = A.capture(None)
    if gt:
        assert A.lib.rpl_debug_set_gather_trigger(-1) == 0
print(json.dumps({"median_us_per_step": A.compare(graphs, rounds=15)}))
