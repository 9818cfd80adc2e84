import sys, torch
sys.path.insert(0, '.')
import paper_1909_01500_b200 as rpl
t = rpl.SumTree(25600, 32)
m = t.attach_min_tree()
torch.cuda.synchronize()
print("hdr", t.header.cpu().tolist(), "mins ptr", m.data_ptr(), "err", torch.cuda.synchronize())
for l in range(t.depth):
    x = t.min_level(l).cpu()
    print(l, x[:4].tolist(), int(x.min()), int(x.max()), x.numel())
print(rpl._lib.config())
