"""Custom-kernel HBM probes (scripts/probe/hbm_probe.cu): read-only, write-only,
copy, 1R:4W broadcast, TMA bulk-store-only.  GB/s = bytes moved / time, best of 10."""
import ctypes
import json
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "libprobe.so"))
lib.probe_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_int]
dev = torch.device("cuda:0")
N = 1 << 30
a = torch.empty(N, dtype=torch.uint8, device=dev).random_(0, 255)
b = torch.empty(4 * N, dtype=torch.uint8, device=dev)
sm = torch.cuda.get_device_properties(dev).multi_processor_count


def t(which, bytes_, moved, R=1, grid=None, block=256, tile=0, dst=None):
    g = grid or sm * 8
    x, y = (b, a) if which == 4 else (a, b)
    lib.probe_run(which, x.data_ptr(), y.data_ptr(), bytes_, R, g, block, tile)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.probe_run(which, x.data_ptr(), y.data_ptr(), bytes_, R, g, block, tile)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return round(moved / (best / 1e3) / 1e9, 1)


res = {
    "read": t(0, N, N),
    "write": t(1, N, N),
    "copy": t(2, N, 2 * N),
    "bcast_1R2W": t(3, N, 3 * N, R=2),
    "bcast_1R4W": t(3, N, 5 * N, R=4),
    "bulk_store_28KB_1cta": t(4, 4 * N, 4 * N, grid=sm, tile=28224 * 7),
    "bulk_store_28KB_2cta": t(4, 4 * N, 4 * N, grid=2 * sm, tile=28224 * 3),
}
print(json.dumps(res))
