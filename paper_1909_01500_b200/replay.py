"""Host-side replay logic around the kernels: ring validity windows, leaf
numbering and the multi-GPU shard protocol.  No hot-path math:
index bookkeeping that decides WHICH leaves/shards a kernel touches.

Conventions (rpl.h): ring rows are slots 0..cap_T-1, `cursor` is the row the
next append writes, `size` rows are valid; transition leaf = row*B + b,
sequence leaf = block*B + b with row0 = block*period (P:38, P:123 fn).
"""
from __future__ import annotations

import numpy as np


def row_age(row, cap_T, cursor):
    """0 for the newest row (cursor-1), cap_T-1 for the oldest."""
    return (np.asarray(cursor) - 1 - np.asarray(row)) % cap_T


def valid_transition_rows(cap_T, cursor, size, k, n_step):
    """Rows whose frame history (k-1 rows back) and n-step lookahead are stored."""
    rows = np.arange(cap_T)
    age = row_age(rows, cap_T, cursor)
    return rows[(age >= n_step) & (age <= size - k)]


def valid_sequence_blocks(cap_T, period, cursor, size, k, seq_len):
    """Blocks whose sequence rows row0-max(k-1,1) .. row0+L-1 are all stored."""
    blocks = np.arange(cap_T // period)
    age = row_age(blocks * period, cap_T, cursor)
    hist = max(k - 1, 1)
    return blocks[(age >= seq_len - 1) & (age + hist <= size - 1)]


def leaves_of(rows_or_blocks, B):
    r = np.asarray(rows_or_blocks, np.int64)[:, None]
    return (r * B + np.arange(B, dtype=np.int64)[None, :]).reshape(-1)


def shard_columns(B_total, world, rank):
    """Mode L partitioning: rank owns env columns [rank*B/G, (rank+1)*B/G) (P:64 data-parallel)."""
    if B_total % world:
        raise ValueError("B must divide evenly over the ranks")
    w = B_total // world
    return rank * w, (rank + 1) * w


def owner_of_prefix(prefix, totals):
    """Shard owning a global prefix under shard-major order, and the local prefix."""
    acc = 0
    for g, t in enumerate(totals):
        if acc <= prefix < acc + t:
            return g, prefix - acc
        acc += t
    raise ValueError("prefix outside [0, sum(totals))")
