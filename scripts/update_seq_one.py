"""update_seq on the R2D2 tree, repeated (for ncu captures of k_tree_update in MODE_SEQ)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
N, n = 25600, 64
t = rpl.SumTree(N, 32)
g = torch.Generator(device=dev)
g.manual_seed(1)
t.update(torch.arange(N, device=dev), torch.rand(N, generator=g, device=dev) + 1e-3, 0.9)
idx = torch.randint(0, N, (n,), generator=g, device=dev)
td_seq = torch.rand((80, n), generator=g, device=dev)
for _ in range(6):
    t.update_seq(idx, td_seq, 0.9, eta=0.9)
torch.cuda.synchronize()
