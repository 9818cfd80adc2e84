"""rpl_stack_frames (Mode C learner side) on the R2D2 batch: unique [128, 64, 84, 84] +
start offsets -> stacked [125, 64, 4, 84, 84]; graph of 16 launches, us per launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
L, n, k = 125, 64, 4
uq = torch.randint(0, 255, (L + k - 1, n, 84, 84), dtype=torch.uint8, device=dev)
st = torch.randint(0, 2, (L, n), dtype=torch.int8, device=dev)
out = torch.empty((L, n, k, 84, 84), dtype=torch.uint8, device=dev)
ms = bench._graph_time(dev, lambda i: rpl.stack_frames(uq, st, k, out=out), P=16, reps=20)
nb = uq.numel() + st.numel() + out.numel()
print(json.dumps({"stack_us": ms * 1e3, "GBps_rw": nb / (ms / 1e3) / 1e9, "note": "reads are 1/4 unique (L2 reuse)"}))
