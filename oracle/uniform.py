"""Oracle: uniform replay indices (SAC/TD3 Mujoco config, BASELINE configs[3]).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs; never by the product package.

SPEC: uniform replay samples transitions "uniformly with replacement" from the
stored ones; a transition is valid when its k-frame history and
n-step lookahead are stored (§8c #2, #14).  The plain definition, with the
draws passed in as uint64 Philox values (R23):

    M = n_rows * B;  m_k = floor(u_k * M / 2**64)        (Python ints, exact)
    leaf_k = ((lo_row + m_k // B) mod cap) * B + m_k mod B

Every value of m in [0, M) receives floor or ceil of 2**64 / M of the 2**64
possible u (pinned in tests/test_oracle_uniform.py).
"""
from __future__ import annotations

from . import philox as _ph


def uniform_leaf(u: int, lo_row: int, n_rows: int, cap: int, B: int) -> int:
    M = n_rows * B
    m = (u * M) >> 64
    row = (lo_row + m // B) % cap
    return row * B + m % B


def uniform_indices(n, seed, offset, lo_row, n_rows, cap, B):
    return [uniform_leaf(u, lo_row, n_rows, cap, B) for u in _ph.draws_u64(seed, offset, n)]
