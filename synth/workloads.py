"""Seeded synthetic workloads (numpy, host).  DESIGN.md "Input recipe".

Shapes follow BASELINE.json configs; value distributions follow SURVEY.md §8(d):
  * rewards: clipped Atari rewards r in {-1, 0, 1} with P(r != 0) = 0.05, or a
    "heavy" set of signed log-normal(0, 2) rewards that stresses cancellation,
    or R2D2's unclipped rewards (P(r != 0) = 0.05, |r| log-uniform in [1, 1000]);
  * values V ~ N(0, 5^2); dones ~ Bernoulli(p_done);
  * |delta| ~ |N(0, 1)| or log-normal(0, 2) (heavy tail);
  * frames: uniform random bytes with bytes 0..15 overwritten by (row, b, tag)
    so that a mis-gathered frame is caught immediately;
  * episodes: geometric lengths (mean `ep_len`) via Bernoulli(1/ep_len) dones.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "rng", "rewards", "values", "dones", "td_abs", "returns_inputs", "Ring", "make_ring",
    "FRAME_H", "FRAME_W", "FRAME_BYTES", "TOY",
]

FRAME_H = 84
FRAME_W = 84
FRAME_BYTES = FRAME_H * FRAME_W  # 7056 = 441 * 16


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def rewards(g, shape, kind="clipped"):
    if kind == "clipped":
        nz = g.random(shape) < 0.05
        sign = np.where(g.random(shape) < 0.5, -1.0, 1.0)
        return (nz * sign).astype(np.float32)
    if kind == "heavy":
        sign = np.where(g.random(shape) < 0.5, -1.0, 1.0)
        return (sign * g.lognormal(0.0, 2.0, shape)).astype(np.float32)
    if kind == "r2d2":
        nz = g.random(shape) < 0.05
        mag = np.exp(g.uniform(0.0, np.log(1000.0), shape))
        sign = np.where(g.random(shape) < 0.5, -1.0, 1.0)
        return (nz * sign * mag).astype(np.float32)
    if kind == "mujoco":
        return g.normal(1.0, 1.0, shape).astype(np.float32)
    if kind == "small":  # toy: values from a small exact set
        return g.choice(np.array([-1.0, 0.0, 0.5, 1.0, 2.0], np.float32), size=shape)
    raise ValueError(kind)


def values(g, shape, scale=5.0):
    return (g.normal(0.0, scale, shape)).astype(np.float32)


def dones(g, shape, p):
    return (g.random(shape) < p).astype(np.uint8)


def td_abs(g, n, kind="normal"):
    if kind == "normal":
        return np.abs(g.normal(0.0, 1.0, n)).astype(np.float32)
    if kind == "heavy":
        return g.lognormal(0.0, 2.0, n).astype(np.float32)
    raise ValueError(kind)


def returns_inputs(seed, T, B, reward_kind="clipped", p_done=0.05):
    """(r, v, d, bootstrap_v) for a [T, B] return-estimation call."""
    g = rng(seed)
    r = rewards(g, (T, B), reward_kind)
    v = values(g, (T, B))
    d = dones(g, (T, B), p_done)
    boot = values(g, (B,))
    return r, v, d, boot


@dataclass
class Ring:
    """Host copy of a replay ring: rows are ring slots, [cap_T, B, ...]."""
    obs: np.ndarray       # [cap, B, item...] u8 frames or f32 vectors
    act: np.ndarray       # [cap, B] int64 or [cap, B, A] f32
    rew: np.ndarray       # [cap, B] f32
    done: np.ndarray      # [cap, B] u8
    rnn: np.ndarray | None  # [cap/period, B, parts, H] f32 (sequence replay)
    cursor: int           # ring row of the next append
    size: int             # number of valid rows


def _stamp_frames(obs, cap, B, tag):
    # bytes 0..3 row, 4..7 column, 8..11 tag, 12..15 row ^ column  (misgather detector)
    rows = np.arange(cap, dtype=np.uint32)[:, None]
    cols = np.arange(B, dtype=np.uint32)[None, :]
    flat = obs.reshape(cap, B, -1)
    stamp = np.stack(np.broadcast_arrays(rows, cols, np.uint32(tag) + 0 * rows, rows ^ cols), -1)
    flat[:, :, :16] = stamp.astype("<u4").view(np.uint8).reshape(cap, B, 16)


def make_ring(seed, cap, B, obs_shape=(FRAME_H, FRAME_W), obs_dtype=np.uint8, act_dim=None,
              ep_len=2000.0, reward_kind="clipped", period=None, rnn_parts=2, rnn_h=512,
              cursor=None, size=None):
    """A filled ring with geometric episodes (Bernoulli(1/ep_len) dones)."""
    g = rng(seed)
    if obs_dtype == np.uint8:
        obs = g.integers(0, 256, size=(cap, B) + tuple(obs_shape), dtype=np.uint8)
        if int(np.prod(obs_shape)) >= 16:
            _stamp_frames(obs, cap, B, seed & 0xFFFF)
    else:
        obs = g.normal(0.0, 1.0, (cap, B) + tuple(obs_shape)).astype(np.float32)
    if act_dim is None:
        act = g.integers(0, 18, size=(cap, B), dtype=np.int64)
    else:
        act = g.uniform(-1.0, 1.0, (cap, B, act_dim)).astype(np.float32)
    rew = rewards(g, (cap, B), reward_kind)
    done = dones(g, (cap, B), 1.0 / ep_len)
    rnn = None
    if period is not None:
        rnn = g.normal(0.0, 1.0, (cap // period, B, rnn_parts, rnn_h)).astype(np.float32)
    if cursor is None:
        cursor = int(g.integers(0, cap))
    if size is None:
        size = cap
    return Ring(obs=obs, act=act, rew=rew, done=done, rnn=rnn, cursor=cursor, size=size)


# The toy config of BASELINE.json configs[0]: sum tree 16 leaves, [T=8, B=2] buffer,
# n_step=3, gamma=0.99, GAE lambda=0.95, batch 4.
TOY = dict(T=8, B=2, n_step=3, gamma=0.99, lam=0.95, n_leaves=16, batch=4, alpha=0.6, beta=0.4,
           eps_p=1e-3, frac_bits=32)
