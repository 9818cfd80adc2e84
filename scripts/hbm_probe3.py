"""Write-pattern probe: 28224-B stack tiles written time-major ([L, n], rows nsamp*tile
apart, as the sequence gather does) vs contiguous, TMA bulk vs LSU."""
import ctypes
import json
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "libprobe.so"))
lib.probe_rows.argtypes = [ctypes.c_int, ctypes.c_void_p] + [ctypes.c_int] * 5
dev = torch.device("cuda:0")
tile, rows = 28224, 125
res = {}
for nsamp, ctas in [(64, 64), (64, 128), (64, 256), (0, 148), (0, 296)]:
    buf = torch.empty(ctas * rows * tile, dtype=torch.uint8, device=dev)
    for which, G in [(0, 4), (0, 16), (1, 0)]:
        if which == 1 and G:
            continue
        lib.probe_rows(which, buf.data_ptr(), ctas, rows, tile, nsamp, G)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.probe_rows(which, buf.data_ptr(), ctas, rows, tile, nsamp, G)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[f"{'bulk' if which == 0 else 'lsu'}{G if which == 0 else ''}_nsamp{nsamp}_ctas{ctas}"] = round(
            buf.numel() / (best / 1e3) / 1e9, 1)
    del buf
print(json.dumps(res, indent=1))
