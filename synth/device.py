"""Seeded synthetic replay rings generated directly in HBM (torch RNG on the GPU).

Same recipe as synth.workloads.make_ring for buffers too
large to build on the host (one 7.2-37 GB shard per rank).  Input plumbing only:
no hot-path arithmetic.
"""
from __future__ import annotations

import torch


def make_ring_device(seed, cap, B, device, ep_len=2000.0, period=40, rnn_parts=2, rnn_h=512, cursor=0,
                     frame_shape=(84, 84), vec_dim=None, act_dim=None, with_rnn=True):
    """Atari rings: u8 frames, int64 actions.  vec_dim=D: Mujoco rings with f32 N(0,1)
    observations [cap, B, D] and (act_dim=A) f32 actions [cap, B, A]."""
    from paper_1909_01500_b200.ops import GatherRing
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    if vec_dim is None:
        obs = torch.empty((cap, B) + tuple(frame_shape), dtype=torch.uint8, device=device)
        flat = obs.view(-1)
        chunk = 1 << 30
        for s in range(0, flat.numel(), chunk):
            e = min(flat.numel(), s + chunk)
            flat[s:e].random_(0, 256, generator=g)
    else:
        obs = torch.randn((cap, B, int(vec_dim)), generator=g, device=device, dtype=torch.float32)
    if act_dim is None:
        act = torch.randint(0, 18, (cap, B), generator=g, device=device, dtype=torch.int64)
    else:
        act = torch.rand((cap, B, int(act_dim)), generator=g, device=device, dtype=torch.float32) * 2 - 1
    nz = torch.rand((cap, B), generator=g, device=device) < 0.05
    mag = torch.exp(torch.rand((cap, B), generator=g, device=device) * torch.log(torch.tensor(1000.0)))
    sign = torch.where(torch.rand((cap, B), generator=g, device=device) < 0.5, -1.0, 1.0)
    rew = (nz * sign * mag).to(torch.float32).contiguous()
    done = (torch.rand((cap, B), generator=g, device=device) < 1.0 / ep_len).to(torch.uint8)
    rnn = (torch.randn((cap // period, B, rnn_parts, rnn_h), generator=g, device=device, dtype=torch.float32)
           if with_rnn else None)
    return GatherRing(obs=obs, act=act, rew=rew, done=done, cursor=int(cursor), size=cap, rnn=rnn)
