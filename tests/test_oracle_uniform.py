"""Pins for oracle/uniform.py (uniform replay indices): extreme draws, the exact
share of the 2^64 draws each index receives, window membership with ring wrap,
and a chi-square upper tail on Philox draws."""
import numpy as np
import pytest

from oracle import philox as OP
from oracle import uniform as OU


def test_extreme_draws_hit_window_ends():
    # u = 0 -> first row, column 0; u = 2^64 - 1 -> last row, last column (wrapping the ring)
    assert OU.uniform_leaf(0, 90, 20, 100, 8) == 90 * 8
    assert OU.uniform_leaf(2**64 - 1, 90, 20, 100, 8) == ((90 + 19) % 100) * 8 + 7


@pytest.mark.parametrize("M", [1, 3, 7, 10, 12])
def test_every_index_gets_floor_or_ceil_share(M):
    # count, for each m, the draws u with floor(u M / 2^64) == m: the first u reaching m is
    # ceil(m 2^64 / M), so the share is ceil((m+1) 2^64/M) - ceil(m 2^64/M) in {floor, ceil}(2^64/M)
    def first_u(m):
        return -((-m * 2**64) // M)
    shares = [first_u(m + 1) - first_u(m) for m in range(M)]
    assert sum(shares) == 2**64
    assert set(shares) <= {2**64 // M, -(-2**64 // M)}
    for m in range(M):  # the boundary draws land on m and m-1
        u = first_u(m)
        B = 1
        assert OU.uniform_leaf(u, 0, M, M, B) == m
        if m > 0:
            assert OU.uniform_leaf(u - 1, 0, M, M, B) == m - 1


def test_window_membership_and_chi2():
    cap, B, lo, nr = 50, 4, 41, 17  # window wraps the ring end
    idx = OU.uniform_indices(20000, seed=9, offset=3, lo_row=lo, n_rows=nr, cap=cap, B=B)
    rows = {(lo + i) % cap for i in range(nr)}
    assert all((i // B) in rows for i in idx)
    cnt = np.bincount([((i // B - lo) % cap) * B + i % B for i in idx], minlength=nr * B)
    assert len(cnt) == nr * B
    exp = len(idx) / (nr * B)
    chi2 = float(((cnt - exp) ** 2 / exp).sum())
    assert chi2 < 67 + 5 * np.sqrt(2 * 67)  # 67 dof upper tail


def test_uses_the_philox_stream():
    u = OP.draws_u64(5, 100, 3)
    assert OU.uniform_indices(3, 5, 100, 0, 10, 10, 2) == [OU.uniform_leaf(x, 0, 10, 10, 2) for x in u]
