"""In-process A/B of the R2D2 step SHAPES on one ring / tree / plan: 'one' (rpl_gather_update_sample,
one launch), 'fused' (update_seq -> rpl_gather_sample), 'pair' (update_seq -> sample_stream ->
gather): one 8-step graph each, replayed round-robin; median us per step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ab_inproc as A  # noqa: E402

graphs = {}
for shape in os.environ.get("SHAPES", "one fused pair").split():
    os.environ["STEP"] = shape
    A.FUSED = shape in ("fused", "one")
    graphs[shape] = A.capture(None)
print(json.dumps({"median_us_per_step": A.compare(graphs, rounds=15)}))
