"""PPO GAE call timing: (a) rotating input pool > 4x L2 (TLB-cold, L2-cold); (b) one input
set re-used with a 256 MB L2 flush before every call (TLB-warm, L2-cold); per-call CUDA
events, eager, flush keeps the GPU busy while the call is enqueued."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

dev = torch.device("cuda:0")
r, v, d, boot = returns_inputs(5, 128, 4096, p_done=1e-3)
res = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for pool in (60, 1):
    R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
    V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
    D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
    BT = torch.from_numpy(boot).to(dev)
    A, RT = torch.empty_like(R), torch.empty_like(R)
    for kind in ("gae", "disc"):
        ts = []
        for it in range(60):
            i = it % pool
            flush.fill_(it & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "gae":
                rpl.gae(R[i], V[i], D[i], BT, 0.99, 0.95, adv=A[i], ret=RT[i])
            else:
                rpl.returns_discounted(R[i], D[i], BT, 0.99, out=RT[i])
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[10:])
        res[f"{kind}_pool{pool}"] = {"median_us": us[len(us) // 2], "min_us": us[0]}
    del R, V, D, A, RT
print(json.dumps(res, indent=1))
