"""One GAE + one discounted call at a given size (for ncu captures of the scan kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

T, B = int(sys.argv[1]), int(sys.argv[2])
r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
dev = torch.device("cuda:0")
R, V, D, BT = (torch.from_numpy(x).to(dev) for x in (r, v, d, boot))
A, RT = torch.empty_like(R), torch.empty_like(R)
for _ in range(3):
    rpl.gae(R, V, D, BT, 0.99, 0.95, adv=A, ret=RT)
    rpl.returns_discounted(R, D, BT, 0.99, out=RT)
torch.cuda.synchronize()
