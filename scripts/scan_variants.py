"""PPO [128, 4096] GAE / discounted timing per scan kernel variant (rpl_debug_set_scan_variant):
bench.py's ppo_returns measurement (graph of one call per pool entry, pool > 4x L2)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for var in [int(x) for x in os.environ.get("VARIANTS", "6,0,4,5,3,0").split(",")]:
    assert rpl._lib.lib.rpl_debug_set_scan_variant(var) == 0
    d = bench.bench_ppo(dev, rpl)
    res[f"v{var}" if f"v{var}" not in res else f"v{var}_again"] = {"gae_us": round(d["gae_us_per_call"], 3),
                                                                  "disc_us": round(d["disc_us_per_call"], 3)}
rpl._lib.lib.rpl_debug_set_scan_variant(0)
print(json.dumps(res, indent=1))
