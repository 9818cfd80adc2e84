"""Small driver for ncu captures of the return kernels and the tree kernels
(PPO [128,4096] GAE/discounted; DQN 2^20-leaf tree update/sample of 512)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs, rng, td_abs  # noqa: E402

dev = torch.device("cuda:0")
r, v, d, boot = returns_inputs(5, 128, 4096, p_done=1e-3)
R, V, D, BT = (torch.from_numpy(x).to(dev) for x in (r, v, d, boot))
for _ in range(3):
    rpl.gae(R, V, D, BT, 0.99, 0.95)
    rpl.returns_discounted(R, D, BT, 0.99)
    rpl.returns_nstep(R, D, 3, 0.99)
g = rng(1)
N = 1 << 20
t = rpl.SumTree(N, 32, device=dev)
t.update(torch.arange(N, device=dev), torch.from_numpy(td_abs(g, N)).to(dev), 0.6)
for i in range(3):
    idx, q, qmin, w = t.sample_stream(512, 7, beta=0.4)
    t.update(idx, torch.from_numpy(td_abs(g, 512)).to(dev), 0.6)
torch.cuda.synchronize()
print("ok")
