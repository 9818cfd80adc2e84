"""DQN transition-gather probe: rpl_gather (k=4, n=3, IS weights) alone on the [4096, 256]
frame ring for batch 32 / 128 / 512, graph of 16 launches over rotating index sets,
us per launch and algorithmic GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402
from paper_1909_01500_b200 import replay as R  # noqa: E402
from synth.device import make_ring_device  # noqa: E402

dev = torch.device("cuda:0")
ring = make_ring_device(404, 4096, 256, dev, cursor=1111, with_rnn=False)
leaves = R.leaves_of(R.valid_transition_rows(4096, ring.cursor, ring.size, 4, 3), 256)
g = np.random.default_rng(0)
res = {}
for bs in (32, 128, 512):
    plan = rpl.GatherPlan(ring, bs, kind="transition", k=4, n_step=3, gamma=0.99, with_weights=True)
    idxs = [torch.from_numpy(g.choice(leaves, bs)).to(dev) for _ in range(16)]
    q = torch.randint(1 << 20, 1 << 30, (bs,), device=dev)
    ms = bench._graph_time(dev, lambda i: plan.run(idxs[i % 16], q=q, qmin=None, beta=0.4), P=16, reps=20)
    nb = bs * bench.transition_bytes(4, 3, 7056, 8)
    res[f"bs{bs}"] = {"us": round(ms * 1e3, 2), "GBps": round(nb / (ms / 1e3) / 1e9, 1)}
print(json.dumps(res))
