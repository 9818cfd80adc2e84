"""Per-call time of rpl_returns_nstep at PPO size ([128, 4096], n = 5; rescaled with q and
plain), timed like bench.py's returns line (CUDA graph over a pool > 4x L2)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

dev = torch.device("cuda:0")
T, B = 128, 4096
r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
pool = max(4, int(math.ceil(4 * torch.cuda.get_device_properties(dev).L2_cache_size / (T * B * 14))))
R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
QB = torch.zeros(B, device=dev)
Y = torch.empty((pool, T - 4, B), device=dev)
DN = torch.empty((T - 4, B), dtype=torch.uint8, device=dev)


def per_call(fn, reps=10):
    for i in range(pool):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.graph(g, stream=s):
        for i in range(pool):
            fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * pool) * 1e3


res = {"rescaled_q_us": per_call(lambda i: rpl.returns_nstep(R[i], D[i], 5, 0.99, q=V[i], q_boot=QB, rescale=True,
                                                             out=Y[i], done_out=DN)),
       "plain_us": per_call(lambda i: rpl.returns_nstep(R[i], D[i], 5, 0.99, out=Y[i], done_out=DN))}
print(json.dumps(res))
