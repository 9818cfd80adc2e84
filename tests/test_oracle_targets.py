"""Pins for oracle/targets.py (NEXT-3): argmax conventions, reductions of double-Q to the
plain max / single-action cases, and the C51 projection's closed forms (identity, mass
conservation, mean preservation without clipping, point masses, clipping)."""
import math

import numpy as np

from oracle import returns as OR
from oracle import targets as OT


def test_argmax_first_ties_and_nan():
    assert OT.argmax_first([1.0, 3.0, 3.0, 2.0]) == 1
    assert OT.argmax_first([float("nan"), -1.0, -2.0]) == 1
    assert OT.argmax_first([float("nan")] * 3) == 0


def test_double_q_with_equal_nets_is_max():
    g = np.random.default_rng(0)
    q = g.normal(size=(4, 3, 6))
    a, v = OT.double_q_bootstrap(q, q)
    assert np.array_equal(v, q.max(-1)) and np.array_equal(a, q.argmax(-1))


def test_nstep_double_q_single_action_reduces_to_nstep():
    g = np.random.default_rng(1)
    T, B, n = 9, 4, 3
    r = g.normal(size=(T, B))
    d = (g.random((T, B)) < 0.2).astype(np.uint8)
    qt = g.normal(size=(T + 1, B, 1))
    y, dn, a = OT.nstep_double_q(r, d, n, 0.99, g.normal(size=(T + 1, B, 1)), qt)
    y2, dn2 = OR.nstep_return(r, d, n, 0.99, q=qt[:T, :, 0], q_boot=qt[T, :, 0])
    assert np.array_equal(y, y2) and np.array_equal(dn, dn2) and not a.any()


def test_c51_identity_conservation_and_mean():
    g = np.random.default_rng(2)
    N, vmin, vmax = 51, -10.0, 10.0
    p = g.random(N)
    p /= p.sum()
    m = OT.c51_project(p, 0.0, 1.0, vmin, vmax)              # R = 0, g = 1: identity
    assert np.allclose(m, p, atol=1e-15)
    z = np.linspace(vmin, vmax, N)
    p2 = np.zeros(N)
    p2[20:31] = g.random(11)
    p2 /= p2.sum()                                            # support well inside: no clipping
    R, gg = 0.37, 0.9
    m2 = np.array(OT.c51_project(p2, R, gg, vmin, vmax))
    assert math.isclose(m2.sum(), 1.0, rel_tol=1e-14)         # mass conservation
    assert math.isclose((m2 * z).sum(), R + gg * (p2 * z).sum(), rel_tol=1e-12)  # mean preserved


def test_c51_point_masses_and_clipping():
    N, vmin, vmax = 11, -5.0, 5.0                             # dz = 1
    p = np.full(N, 1.0 / N)
    m = OT.c51_project(p, 2.0, 0.0, vmin, vmax)               # terminal, R on atom 7
    assert math.isclose(m[7], 1.0, rel_tol=1e-15) and sum(m) == m[7]   # all mass on atom 7
    m = OT.c51_project(p, 2.25, 0.0, vmin, vmax)              # between atoms 7 and 8
    assert math.isclose(m[7], 0.75) and math.isclose(m[8], 0.25)
    m = OT.c51_project(p, 40.0, 0.5, vmin, vmax)              # everything clipped to v_max
    assert math.isclose(m[-1], 1.0) and sum(m[:-1]) == 0.0
