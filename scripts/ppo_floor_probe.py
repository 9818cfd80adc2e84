"""PPO [128,4096] per-call floors, timed like bench.py's ppo_returns (CUDA graph of one
call per pool entry, pool > 4x L2): empty kernel, GAE-shaped streaming pass (same bytes,
no scan) at a few grid sizes, and rpl.gae / rpl.returns_discounted."""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_01500_b200 as rpl  # noqa: E402
from synth import returns_inputs  # noqa: E402

_so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "libppo_floor.so")
if not os.path.exists(_so):
    import subprocess
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", _so, _so.replace("libppo_floor.so", "ppo_floor.cu")])
lib = ctypes.CDLL(_so)
lib.ppo_floor.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                                   ctypes.c_void_p]
dev = torch.device("cuda:0")
T, B = 128, 4096
r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
pool = max(4, int(math.ceil(4 * l2 / (T * B * 17))))
R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
BT = torch.from_numpy(boot).to(dev)
A, RT = torch.empty_like(R), torch.empty_like(R)


def per_call_us(fn, reps=10):
    for i in range(pool):
        fn(i)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.graph(gr, stream=st):
        for i in range(pool):
            fn(i)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / (reps * pool) * 1e3, 3)


def floor(which, grid=0, block=256):
    def f(i):
        s = torch.cuda.current_stream(dev).cuda_stream
        lib.ppo_floor(which, R[i].data_ptr(), V[i].data_ptr(), D[i].data_ptr(), A[i].data_ptr(), RT[i].data_ptr(),
                      T * B, grid, block, s)
    return f


res = {"pool": pool, "empty_kernel_us": per_call_us(floor(0))}
for grid, block in [(128, 512), (148, 512), (296, 256), (512, 256), (1024, 128)]:
    res[f"stream_g{grid}_b{block}_us"] = per_call_us(floor(1, grid, block))
res["gae_us"] = per_call_us(lambda i: rpl.gae(R[i], V[i], D[i], BT, 0.99, 0.95, adv=A[i], ret=RT[i]))
res["disc_us"] = per_call_us(lambda i: rpl.returns_discounted(R[i], D[i], BT, 0.99, out=RT[i]))
res["env"] = {k: os.environ.get(k, "") for k in ("RPL_SCAN_VARIANT", "RPL_SCAN_TRIGGER", "RPL_PDL")}
print(json.dumps(res))
