"""bench.py's PPO secondary (GAE + discounted, [128,4096], CUDA graph over a rotating
pool > 4x L2) on its own, for A/B of return-kernel configurations (RPL_SCAN_VARIANT)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402

r = bench.bench_ppo(torch.device("cuda:0"), rpl)
print(json.dumps({"variant": os.environ.get("RPL_SCAN_VARIANT", "0"), "gae_us": r["gae_us_per_call"],
                  "disc_us": r["disc_us_per_call"], "gae_frac": r["gae_frac"]}))
