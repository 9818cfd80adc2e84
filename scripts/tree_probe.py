"""Sum-tree step probe: update(n)+sample_stream(n) as two launches vs the fused
rpl_sumtree_update_sample, R2D2 (25,600 leaves) and DQN (2^20 leaves) trees; CUDA
graph of 16 steps, replayed; us per step.  Also each kernel alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402

dev = torch.device("cuda:0")
res = {}


def gtime(fn, P=16, reps=20):
    for i in range(P):
        fn(i)
    torch.cuda.synchronize()
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(P):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / (reps * P) * 1e3, 2)


for N, ns in [(25600, (64,)), (1 << 20, (32, 128, 512))]:
    t = rpl.SumTree(N, 32, device=dev)
    t.update(torch.arange(N, device=dev), torch.rand(N, device=dev) + 0.01, 0.9)
    for n in ns:
        idx = [torch.randint(0, N, (n,), device=dev) for _ in range(2)]
        q = torch.empty(n, dtype=torch.int64, device=dev)
        qm = torch.empty(1, dtype=torch.int64, device=dev)
        w = torch.empty(n, dtype=torch.float32, device=dev)
        td = torch.rand(n, device=dev)
        out = (None, q, qm, w)

        def pair(i):
            t.update(idx[(i + 1) % 2], td, 0.9)
            t.sample_stream(n, 5, beta=0.6, out=(idx[i % 2], q, qm, w))

        def upd(i):
            t.update(idx[(i + 1) % 2], td, 0.9)

        def smp(i):
            t.sample_stream(n, 5, beta=0.6, out=(idx[0], q, qm, w))

        big_a = torch.empty(300 << 20, dtype=torch.uint8, device=dev)
        big_b = torch.empty_like(big_a)

        def pair_evict(i):  # a 300 MB copy between steps evicts the tree from L2, as the gather does
            big_b.copy_(big_a)
            pair(i)

        def copy_only(i):
            big_b.copy_(big_a)

        res[f"N{N}_n{n}"] = {"pair": gtime(pair), "update": gtime(upd), "sample": gtime(smp),
                             "pair_after_300MB_copy_minus_copy": round(gtime(pair_evict) - gtime(copy_only), 2)}
        del big_a, big_b
print(json.dumps(res, indent=1))
