"""Oracle: Philox4x32-10 counter-based RNG in Python ints [EXT: Salmon et al. 2011,
"Parallel random numbers: as easy as 1, 2, 3" (Random123)].

Used only to define the sampler's draws when the caller passes draws = NULL:
    u_k = x0 | (x1 << 32),  (x0, x1, x2, x3) = philox4x32_10(ctr, key)
    ctr = (lo32(offset + k), hi32(offset + k), 0, 0),  key = (lo32(seed), hi32(seed))
(DESIGN.md "Readings" R-philox.)  Pinned by the Random123 known-answer vectors
in tests/test_oracle_philox.py.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85


def _mulhilo(a: int, b: int) -> tuple[int, int]:
    p = (a & M32) * (b & M32)
    return (p >> 32) & M32, p & M32


def _round(c, k):
    hi0, lo0 = _mulhilo(PHILOX_M0, c[0])
    hi1, lo1 = _mulhilo(PHILOX_M1, c[2])
    return [(hi1 ^ c[1] ^ k[0]) & M32, lo1, (hi0 ^ c[3] ^ k[1]) & M32, lo0]


def philox4x32(ctr, key, rounds: int = 10):
    c = [x & M32 for x in ctr]
    k = [x & M32 for x in key]
    for r in range(rounds):
        if r > 0:
            k = [(k[0] + PHILOX_W0) & M32, (k[1] + PHILOX_W1) & M32]
        c = _round(c, k)
    return c


def draw_u64(seed: int, offset: int, k: int) -> int:
    """The k-th uint64 draw of stream (seed, offset)."""
    ctr_v = (offset + k) & ((1 << 64) - 1)
    x = philox4x32([ctr_v & M32, ctr_v >> 32, 0, 0], [seed & M32, (seed >> 32) & M32])
    return x[0] | (x[1] << 32)


def draws_u64(seed: int, offset: int, n: int) -> list[int]:
    return [draw_u64(seed, offset, k) for k in range(n)]
