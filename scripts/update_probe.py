"""Tree-step probe on the R2D2 tree (25,600 leaves, 64 draws): graphs of 8 x (update + sample)
with the sequence update (80 x 64 per-step |delta|) or the plain update (64 |delta|), to
isolate the cost of the eta-mixed sequence priority."""
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
idx = [torch.randint(0, N, (n,), generator=g, device=dev) for _ in range(2)]
q = torch.empty(n, dtype=torch.int64, device=dev)
td_seq = torch.rand((80, n), generator=g, device=dev)
td = torch.rand(n, generator=g, device=dev)
lib, P_ = rpl._lib.lib, rpl.ops._ptr


def graph_us(step, P=8, reps=50):
    for i in range(2 * P):
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


def seq(i):
    t.update_seq(idx[(i + 1) % 2], td_seq, 0.9, eta=0.9)
    t.sample_stream(n, 3, out=(idx[i % 2], q, None, None), want_qmin=False)


def plain(i):
    t.update(idx[(i + 1) % 2], td, 0.9)
    t.sample_stream(n, 3, out=(idx[i % 2], q, None, None), want_qmin=False)


def upd_only(i):
    t.update_seq(idx[i % 2], td_seq, 0.9, eta=0.9)


print(json.dumps({"update_seq_plus_sample_us": graph_us(seq), "update_plus_sample_us": graph_us(plain),
                  "update_seq_only_us": graph_us(upd_only)}))
