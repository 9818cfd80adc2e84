"""Return-scan size sweep: GAE and discounted return per call at PPO
and larger sizes, timed like bench.py's ppo_returns (CUDA graph of one call per pool entry,
input pool >= 4x L2 so every call reads HBM), with the achieved GB/s of the algorithmic
bytes (GAE 17 B/elem, discounted 9 B/elem + 4 B/column) and a same-bytes streaming floor."""
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
flib = ctypes.CDLL(_so)
flib.ppo_floor.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                                    ctypes.c_void_p]
dev = torch.device("cuda:0")
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
l2 = torch.cuda.get_device_properties(dev).L2_cache_size


def per_call_us(fn, pool, reps=10):
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
    return e0.elapsed_time(e1) / (reps * pool) * 1e3


def sweep(shapes):
    out = []
    for T, B in shapes:
        r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
        per = T * B * 17
        pool = max(2, int(math.ceil(4 * l2 / per)))
        R = torch.from_numpy(r).to(dev).repeat(pool, 1, 1).contiguous()
        V = torch.from_numpy(v).to(dev).repeat(pool, 1, 1).contiguous()
        D = torch.from_numpy(d).to(dev).repeat(pool, 1, 1).contiguous()
        BT = torch.from_numpy(boot).to(dev)
        A, RT = torch.empty_like(R), torch.empty_like(R)
        gae = per_call_us(lambda i: rpl.gae(R[i], V[i], D[i], BT, 0.99, 0.95, adv=A[i], ret=RT[i]), pool)
        disc = per_call_us(lambda i: rpl.returns_discounted(R[i], D[i], BT, 0.99, out=RT[i]), pool)

        def fl(i):
            s = torch.cuda.current_stream(dev).cuda_stream
            flib.ppo_floor(1, R[i].data_ptr(), V[i].data_ptr(), D[i].data_ptr(), A[i].data_ptr(), RT[i].data_ptr(),
                           T * B, 0, 512, s)
        floor = per_call_us(fl, pool)
        gb_gae = T * B * 17 / (gae * 1e-6) / 1e9
        gb_disc = (T * B * 9 + 4 * B) / (disc * 1e-6) / 1e9
        out.append({"T": T, "B": B, "mb_gae": per / 1e6, "pool": pool, "gae_us": gae, "gae_GBps": gb_gae,
                    "gae_frac": gb_gae / PEAK, "disc_us": disc, "disc_GBps": gb_disc, "disc_frac": gb_disc / PEAK,
                    "floor_stream_us": floor, "floor_frac": per / (floor * 1e-6) / 1e9 / PEAK})
        del R, V, D, A, RT
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    shapes = [(128, 4096), (256, 4096), (512, 4096), (1024, 4096), (2048, 4096), (128, 16384), (128, 65536),
              (1024, 16384)]
    if os.environ.get("SHAPES"):  # e.g. SHAPES="2048x4736,1024x18944"
        shapes = [tuple(int(x) for x in sh.split("x")) for sh in os.environ["SHAPES"].split(",")]
    print(json.dumps({"peak_gbs": PEAK, "sweep": sweep(shapes)}))
