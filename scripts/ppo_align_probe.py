import sys, os, math, json
sys.path.insert(0, os.getcwd())
import torch, bench, paper_1909_01500_b200 as rpl
from synth import returns_inputs
dev = torch.device("cuda:0")
T, B = 128, 4096
r, v, d, boot = returns_inputs(5, T, B, reward_kind="clipped", p_done=1e-3)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
pool = max(4, int(math.ceil(4 * l2 / (T * B * 17))))
def run(shift_bytes):
    # flat buffers with an explicit byte offset from a 2 MB-aligned base
    def mk(x, dtype):
        per = x.nbytes
        raw = torch.empty(pool * per + (4 << 20), dtype=torch.uint8, device=dev)
        base = raw.data_ptr()
        off = ((-base) % (2 << 20)) + shift_bytes
        t = raw[off:off + pool * per].view(dtype).view(pool, *x.shape)
        t.copy_(torch.from_numpy(x).to(dev).expand(pool, *x.shape))
        return raw, t
    rR, R = mk(r, torch.float32); rV, V = mk(v, torch.float32); rD, D = mk(d, torch.uint8)
    BT = torch.from_numpy(boot).to(dev)
    A, RT = torch.empty_like(R), torch.empty_like(R)
    def cap(fn):
        for i in range(pool): fn(i)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph(); st = torch.cuda.Stream(dev); st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.graph(gr, stream=st):
            for i in range(pool): fn(i)
        torch.cuda.synchronize(); return gr
    def tm(gr, reps=10):
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): gr.replay()
        e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / (reps * pool) * 1e3
    g1 = cap(lambda i: rpl.gae(R[i], V[i], D[i], BT, 0.99, 0.95, adv=A[i], ret=RT[i]))
    g2 = cap(lambda i: rpl.returns_discounted(R[i], D[i], BT, 0.99, out=RT[i]))
    return round(tm(g1), 3), round(tm(g2), 3), A.data_ptr() % (2 << 20), RT.data_ptr() % (2 << 20)
res = {}
for sh in (0, 0, 4096, 65536, 512 * 1024, 1 << 20, 0):
    res.setdefault(str(sh), []).append(run(sh))
print(json.dumps(res))
d2 = bench.bench_ppo(dev, rpl); d3 = bench.bench_ppo(dev, rpl)
print(round(d2["gae_us_per_call"], 3), round(d3["gae_us_per_call"], 3))
