"""HBM probes for context on the write-heavy gather: copy (1R:1W), fill (0R:1W),
broadcast (1R:4W, the shape of the k=4 frame-stack gather), all with torch on
>= 1 GiB tensors, CUDA events, best of 10."""
import json
import torch

dev = torch.device("cuda:0")
N = 1 << 30
src = torch.empty(N, dtype=torch.uint8, device=dev).random_(0, 255)
dst = torch.empty(N, dtype=torch.uint8, device=dev)
big = torch.empty(4 * (N // 4), dtype=torch.uint8, device=dev)
q = src[: N // 4]


def best(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    ms = min(out)
    return nbytes / (ms / 1e3) / 1e9


res = {
    "copy_1R1W_GBps": best(lambda: dst.copy_(src), 2 * N),
    "fill_0R1W_GBps": best(lambda: dst.zero_(), N),
    "bcast_1R4W_GBps": best(lambda: big.view(4, -1).copy_(q.view(1, -1).expand(4, -1)), N // 4 + N),
}
print(json.dumps(res))
