"""One rescaled 5-step target call at PPO size (for ncu captures of k_nstep)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

r, v, d, boot = returns_inputs(5, 128, 4096, reward_kind="clipped", p_done=1e-3)
dev = torch.device("cuda:0")
R, V, D, BT = (torch.from_numpy(x).to(dev) for x in (r, v, d, boot))
for _ in range(3):
    rpl.returns_nstep(R, D, 5, 0.99, q=V, q_boot=BT, rescale=True)
torch.cuda.synchronize()
