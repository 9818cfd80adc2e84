"""Update-kernel latency, single-CTA vs multi-CTA (rpl_debug_set_upd_multi), MODE_TD and
MODE_SEQ, several batch sizes: a graph of 16 back-to-back updates, us per launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for N in (25600, 1 << 20):
    t = rpl.SumTree(N, 32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(N)
    t.update(torch.arange(N, device=dev), torch.rand(N, generator=g, device=dev) + 1e-3, 0.9)
    for n in (32, 64, 128, 256, 512, 1024):
        idx = torch.randint(0, N, (n,), generator=g, device=dev)
        td = torch.rand(n, generator=g, device=dev)
        steps = torch.rand((80, n), generator=g, device=dev)
        for multi in (0, 1):
            assert rpl._lib.lib.rpl_debug_set_upd_multi(multi) == 0
            us = bench._graph_time(dev, lambda i: t.update(idx, td, 0.9), P=16, reps=20) * 1e3
            us_s = bench._graph_time(dev, lambda i: t.update_seq(idx, steps, 0.9, eta=0.9), P=16, reps=20) * 1e3
            res[f"N{N}_n{n}_multi{multi}"] = {"td_us": round(us, 2), "seq_us": round(us_s, 2)}
    del t
rpl._lib.lib.rpl_debug_set_upd_multi(1)
print(json.dumps(res, indent=0))
