"""update_seq back-to-back cost vs T_p (rows of per-step |delta|), R2D2 tree, 64 sequences."""
import json
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


def graph_us(step, P=16, reps=50):
    for i in range(P):
        step(i)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.graph(gr, stream=s):
        for i in range(P):
            step(i)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * P) * 1e3


res = {}
td1 = torch.rand(n, generator=g, device=dev)
res["plain"] = graph_us(lambda i: t.update(idx, td1, 0.9))
res["plain_alpha1"] = graph_us(lambda i: t.update(idx, td1, 1.0))
for tp in (1, 8, 40, 80, 160):
    td = torch.rand((tp, n), generator=g, device=dev)
    res[f"seq_T{tp}"] = graph_us(lambda i: t.update_seq(idx, td, 0.9, eta=0.9))
    res[f"seq_T{tp}_alpha1"] = graph_us(lambda i: t.update_seq(idx, td, 1.0, eta=0.9))
print(json.dumps(res))
