"""Sequence-gather probe: kernel time vs ring size (TLB reach / DRAM locality) and
variant, R2D2 shape (64 x 125 rows, k=4, 7056-B frames), CUDA events, mean of 50."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from paper_1909_01500_b200 import replay as R  # noqa: E402
from synth.device import make_ring_device  # noqa: E402

dev = torch.device("cuda:0")
res = {}
FR = 7056
for cap, B in [(4000, 256), (1024000, 1)]:
    ring = make_ring_device(1, cap, B, dev, period=40, rnn_h=512, cursor=17)
    blocks = R.valid_sequence_blocks(cap, 40, ring.cursor, ring.size, 4, 125)
    leaves = R.leaves_of(blocks, B)
    g = np.random.default_rng(0)
    for variant in [int(v) for v in os.environ.get("VARIANTS", "0,1,4,5").split(",")]:
        rpl._lib.lib.rpl_debug_set_gather_variant(variant)
        for mode in ("stacked", "unique"):
            if mode == "unique" and variant not in (0, 1):
                continue
            plan = rpl.GatherPlan(ring, 64, kind="sequence", k=4, seq_len=125, period=40,
                                  out_mode=0 if mode == "stacked" else 1)
            idxs = [torch.from_numpy(g.choice(leaves, 64)).to(dev) for _ in range(50)]
            for i in range(5):
                plan.run(idxs[i])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(50):
                plan.run(idxs[i])
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1e3
            nb = 64 * ((128 * FR) + (125 * 4 * FR if mode == "stacked" else 128 * FR))
            res[f"ring{cap}x{B}_v{variant}_{mode}"] = {"us": round(us, 2), "GBps": round(nb / us / 1e3, 1)}
    del ring
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
