"""Sequence-gather limiter probe: the default kernel with stores and/or loads
switched off, streaming stores, evict-first loads (rpl_debug_set_gather_diag);
R2D2 shape (64 x 125 rows, k=4), CUDA events, mean of 50 launches."""
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
variants = [int(v) for v in os.environ.get("VARIANTS", "0").split(",")]
diags = [int(v) for v in os.environ.get("DIAGS", "0,1,2,3,4,8,12").split(",")]
res = {}
cap, B = 4000, 256
ring = make_ring_device(1, cap, B, dev, period=40, rnn_h=512, cursor=17)
blocks = R.valid_sequence_blocks(cap, 40, ring.cursor, ring.size, 4, 125)
leaves = R.leaves_of(blocks, B)
g = np.random.default_rng(0)
idxs = [torch.from_numpy(g.choice(leaves, 64)).to(dev) for _ in range(50)]
plan = rpl.GatherPlan(ring, 64, kind="sequence", k=4, seq_len=125, period=40)
for variant in variants:
    rpl._lib.lib.rpl_debug_set_gather_variant(variant)
    for diag in diags:
        assert rpl._lib.lib.rpl_debug_set_gather_diag(diag) == 0
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
        rd = 64 * 128 * 7056 if not diag & 2 else 0
        wr = 64 * 125 * 4 * 7056 if not diag & 1 else 0
        res[f"v{variant}_diag{diag}"] = {"us": round(us, 2), "GBps_frames": round((rd + wr) / us / 1e3, 1)}
rpl._lib.lib.rpl_debug_set_gather_diag(0)
rpl._lib.lib.rpl_debug_set_gather_variant(0)
print(json.dumps(res, indent=1))
