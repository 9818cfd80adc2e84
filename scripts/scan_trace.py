"""PPO [128, 4096] scan timeline (needs -DRPL_TRACE): a graph of back-to-back calls (bench.py's
ppo measurement); the last call's stamps, ns relative to CTA 0's entry; median of 20 replays."""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

dev = torch.device("cuda:0")
T, B = int(os.environ.get("T", "128")), int(os.environ.get("B", "4096"))
r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
pool = max(4, int(math.ceil(4 * l2 / (T * B * 17))))
R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
BT = torch.from_numpy(boot).to(dev)
A, RT = torch.empty_like(R), torch.empty_like(R)
GAE = os.environ.get("KIND", "gae") == "gae"


def call(i):
    if GAE:
        rpl.gae(R[i], V[i], D[i], BT, 0.99, 0.95, adv=A[i], ret=RT[i])
    else:
        rpl.returns_discounted(R[i], D[i], BT, 0.99, out=RT[i])


for i in range(pool):
    call(i)
torch.cuda.synchronize()
st = torch.cuda.Stream(dev)
st.wait_stream(torch.cuda.current_stream(dev))
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    for i in range(pool):
        call(i)
names = ["entry", "past_wait", "tiles", "bar1", "bar2", "bar3", "store_issued", "exit", "last_cta_exit",
         "first_cta_exit"]
buf = (ctypes.c_int64 * 10)()
runs = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(20):
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    assert rpl._lib.lib.rpl_debug_scan_trace(buf, 10) == 0
    t0 = buf[0]
    row = {n: buf[k] - t0 for k, n in enumerate(names)}
    row["us_per_call"] = e0.elapsed_time(e1) * 1e3 / pool
    runs.append(row)
med = {k: sorted(x[k] for x in runs)[len(runs) // 2] for k in runs[0]}
print(json.dumps({"T": T, "B": B, "kind": "gae" if GAE else "disc", "ns_from_cta0_entry": med}))
