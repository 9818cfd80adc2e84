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


# ---- initial priorities (NEXT-1, R33) ---------------------------------------------------------

def test_ring_td_constant_closed_form():
    # r = 1.5, no dones, q_boot = 4, q_taken = 2: y = r (1 - g^n) / (1 - g) + g^n 4 on every row
    cap, B, n, g = 20, 3, 5, 0.9
    rew = np.full((cap, B), 1.5, np.float32)
    done = np.zeros((cap, B), np.uint8)
    qb = np.full((cap, B), 4.0, np.float32)
    qt = np.full((cap, B), 2.0, np.float32)
    td = OT.ring_td_abs(rew, done, qt, qb, 17, 10, n, g)       # wraps the ring end
    y = 1.5 * (1 - g ** n) / (1 - g) + g ** n * 4.0
    assert td.shape == (10, B) and np.allclose(td, abs(y - 2.0), rtol=0, atol=1e-12)


def test_ring_td_worked_example_with_done():
    # rewards 1, 2, 3 (rows 0-2), done at row 1, n = 2, gamma = 0.5, q_boot = 10 everywhere:
    #   row 0: 1 + 0.5 * 2 = 2 (the episode ends at row 1: no bootstrap)
    #   row 1: 2 (done at once)
    #   row 2: 3 + 0.5 * r_3 + 0.25 * q_boot_4 = 3 + 0.5 * 4 + 2.5 = 7.5
    rew = np.array([[1.0], [2.0], [3.0], [4.0], [0.0], [0.0]], np.float32)
    done = np.array([[0], [1], [0], [0], [0], [0]], np.uint8)
    qb = np.full((6, 1), 10.0, np.float32)
    qt = np.array([[0.5], [2.5], [7.0], [0.0], [0.0], [0.0]], np.float32)
    td = OT.ring_td_abs(rew, done, qt, qb, 0, 3, 2, 0.5)
    assert td[:, 0].tolist() == [1.5, 0.5, 0.5]


def test_ring_td_one_step_and_rescaled_closed_forms():
    g = np.random.default_rng(3)
    cap, B = 12, 4
    rew = g.normal(size=(cap, B)).astype(np.float32)
    done = (g.random((cap, B)) < 0.3).astype(np.uint8)
    qb = g.normal(size=(cap, B)).astype(np.float32)
    qt = g.normal(size=(cap, B)).astype(np.float32)
    td = OT.ring_td_abs(rew, done, qt, qb, 5, 6, 1, 0.99)        # n = 1: the 1-step TD error
    for t in range(6):
        r0, r1 = (5 + t) % cap, (6 + t) % cap
        ref = np.abs(rew[r0].astype(np.float64) + 0.99 * (1 - done[r0]) * qb[r1] - qt[r0])
        assert np.allclose(td[t], ref, rtol=1e-12, atol=1e-12)
    # rescaled, terminal: y = h(3) = sqrt(4) - 1 + 3 eps = 1 + 3 eps exactly
    e = 1e-3
    td = OT.ring_td_abs(np.array([[3.0]]), np.array([[1]]), np.array([[0.5]]), np.array([[0.0]]), 0, 1, 1, 0.9,
                        rescale=True, eps=e)
    assert abs(td[0, 0] - (0.5 + 3 * e)) < 1e-15


def test_ring_td_rotation_invariance():
    # rotating the ring by s rows and shifting row0 by s changes nothing
    g = np.random.default_rng(4)
    cap, B = 16, 3
    arrs = [g.normal(size=(cap, B)).astype(np.float32), (g.random((cap, B)) < 0.2).astype(np.uint8),
            g.normal(size=(cap, B)).astype(np.float32), g.normal(size=(cap, B)).astype(np.float32)]
    a = OT.ring_td_abs(*arrs, 11, 9, 3, 0.97, rescale=True)
    rolled = [np.roll(x, 6, axis=0) for x in arrs]
    b = OT.ring_td_abs(*rolled, (11 + 6) % cap, 9, 3, 0.97, rescale=True)
    assert np.array_equal(a, b)


def test_initial_sequence_priority_constant_td_is_td():
    # a constant per-step |delta| mixes to itself (max = mean), for any eta
    cap, B, period = 80, 2, 10
    rew = np.full((cap, B), 1.0, np.float32)
    done = np.zeros((cap, B), np.uint8)
    qb = np.zeros((cap, B), np.float32)
    qt = np.zeros((cap, B), np.float32)
    p = OT.initial_sequence_priorities(rew, done, qt, qb, 3, period, 4, 16, 1, 0.9, 0.9, rescale=False)
    assert p == [1.0, 1.0]
