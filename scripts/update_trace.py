"""Timeline of one update launch (needs a -DRPL_TRACE build): ns from kernel start to each
stage, for the plain update and update_seq at T_p = 1 and 80 (R2D2 tree, 64 entries)."""
import ctypes
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
buf = (ctypes.c_int64 * 16)()
names = ["start", "staged", "mixed", "hash_reset", "dedupe", "leaves", "end"]
res = {}
for name, fn in [("plain", lambda: t.update(idx, torch.rand(n, generator=g, device=dev), 0.9)),
                 ("seq_T1", lambda: t.update_seq(idx, torch.rand((1, n), generator=g, device=dev), 0.9)),
                 ("seq_T80", lambda: t.update_seq(idx, torch.rand((80, n), generator=g, device=dev), 0.9))]:
    runs = []
    for _ in range(20):
        for k in range(16):
            buf[k] = 0
        fn()
        torch.cuda.synchronize()
        assert rpl._lib.lib.rpl_debug_trace(buf, 7) == 0
        t0 = buf[0]
        runs.append([(buf[k] - t0) if buf[k] >= t0 else None for k in range(7)])
    med = []
    for k in range(7):
        v = sorted(r[k] for r in runs if r[k] is not None)
        med.append(v[len(v) // 2] if v else None)
    res[name] = dict(zip(names, med))
print(json.dumps(res))
