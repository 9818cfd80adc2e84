"""Marginal cost of each call in the R2D2 step: graphs of 8 steps with the calls added one
at a time (update_seq; + sample; + gather; + n-step), stacked and unique output."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01500_b200 as rpl  # noqa: E402
from paper_1909_01500_b200 import replay as R  # noqa: E402
from synth.device import make_ring_device  # noqa: E402

dev = torch.device("cuda:0")
c = dict(bench.R2D2)
cap, B, L, k, period, n = c["cap_T"], c["B"], c["L"], c["k"], c["period"], c["batch"]
ring = make_ring_device(11, cap, B, dev, period=period, rnn_h=512, cursor=1234)
tree = rpl.SumTree((cap // period) * B, 32, device=dev)
valid = torch.from_numpy(R.leaves_of(R.valid_sequence_blocks(cap, period, ring.cursor, ring.size, k, L), B)).to(dev)
tree.update(valid, torch.rand(valid.numel(), device=dev) + 0.01, 0.9)
lib, P_ = rpl._lib.lib, rpl.ops._ptr
idx = [torch.full((n,), -1, dtype=torch.int64, device=dev) for _ in range(2)]
q = torch.zeros(n, dtype=torch.int64, device=dev)
td = torch.rand((8, 80, n), device=dev)
qv = torch.randn((8, L, n), device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
Tn = 84
res = {}
for fused in (0, 1):
    for mode in ((0, 1) if not fused else (0,)):
        plan = rpl.GatherPlan(ring, n, kind="sequence", k=k, seq_len=L, period=period, with_weights=True, out_mode=mode)
        out = plan.outputs
        y = torch.empty((80, n), device=dev)
        dn = torch.empty((80, n), dtype=torch.uint8, device=dev)
        for upto in range(2 if fused else 1, 5):
            def step(i):
                s = rpl.ops._stream(dev)
                if fused:  # rpl_sumtree_update_sample: update + sample in one launch
                    rpl._lib.check(lib.rpl_sumtree_update_sample(tree._lp, P_(tree.storage), P_(idx[(i + 1) % 2]),
                                                                 P_(td[i % 8]), 80, n, 0.9, 0.9, 1e-3, 0, n, 5,
                                                                 P_(idx[i % 2]), P_(q), P_(err), s), "us")
                else:
                    rpl._lib.check(lib.rpl_sumtree_update_seq(tree._lp, P_(tree.storage), P_(idx[(i + 1) % 2]),
                                                              P_(td[i % 8]), 80, n, 0.9, 0.9, 1e-3, 0, None, s), "u")
                if upto >= 2 and not fused:
                    rpl._lib.check(lib.rpl_sumtree_sample_stream(tree._lp, P_(tree.storage), n, 5, 0.6, P_(idx[i % 2]),
                                                                 P_(q), None, None, P_(err), s), "s")
                if upto >= 3:
                    plan.run(idx[i % 2], q=q, beta=0.6, err=err, stream=s)
                if upto >= 4:
                    rpl._lib.check(lib.rpl_returns_nstep(P_(out["rew"][40:124]), P_(out["done"][40:124]), Tn, n, 5, 0.997,
                                                         P_(qv[i % 8][40:124]), P_(qv[i % 8][124]), 1, 1e-3, P_(y),
                                                         P_(dn), s), "n")
            res[f"{'fused_' if fused else ''}{'stacked' if mode == 0 else 'unique'}_upto{upto}"] = round(bench._graph_time(dev, step, P=8, reps=50) * 1e3, 2)
print(json.dumps(res, indent=1))
