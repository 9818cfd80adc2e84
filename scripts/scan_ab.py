"""Interleaved A/B of scan kernel variants at PPO [128, 4096] (bench.py's ppo_returns measurement,
rpl_debug_set_scan_variant): ROUNDS rounds, the variant order rotated every round, median GAE /
discounted us per call per variant — so a drift over the run hits every variant alike."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
variants = [int(x) for x in os.environ.get("VARIANTS", "0,19").split(",")]
rounds = int(os.environ.get("ROUNDS", "8"))
res = {v: {"gae": [], "disc": []} for v in variants}
for r in range(rounds):
    for v in variants[r % len(variants):] + variants[:r % len(variants)]:
        assert rpl._lib.lib.rpl_debug_set_scan_variant(v) == 0
        d = bench.bench_ppo(dev, rpl)
        res[v]["gae"].append(d["gae_us_per_call"])
        res[v]["disc"].append(d["disc_us_per_call"])
rpl._lib.lib.rpl_debug_set_scan_variant(0)
med = lambda x: sorted(x)[len(x) // 2]  # noqa: E731
print(json.dumps({f"v{v}": {"gae_us": round(med(x["gae"]), 3), "disc_us": round(med(x["disc"]), 3),
                            "gae_all": [round(y, 2) for y in x["gae"]]} for v, x in res.items()}))
