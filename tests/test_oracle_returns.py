"""Pins for oracle.returns against SPEC worked examples, closed forms and
independent exact-rational (sum-form) evaluations."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import returns as R
from synth import returns_inputs, rng


# ---- SPEC worked examples -------------------------------------------------
def test_nstep_spec_example_5_23():
    # r=[1,2,3], gamma=0.9, n=3, no done -> 5.23, done_n false
    r = np.array([[1.0], [2.0], [3.0]])
    d = np.zeros((3, 1), np.uint8)
    Rn, dn = R.nstep_return(r, d, 3, 0.9)
    assert Rn.shape == (1, 1)
    assert abs(Rn[0, 0] - 5.23) < 1e-12 and dn[0, 0] == 0


def test_nstep_spec_truncation():
    # done after the first reward -> return 1.0, done_n true
    r = np.array([[1.0], [2.0], [3.0]])
    d = np.array([[1], [0], [0]], np.uint8)
    Rn, dn = R.nstep_return(r, d, 3, 0.9)
    assert Rn[0, 0] == 1.0 and dn[0, 0] == 1


def test_nstep_n1_degenerate():
    # n=1 reduces to the single reward
    g = rng(1)
    r = g.normal(size=(7, 3))
    d = (g.random((7, 3)) < 0.3).astype(np.uint8)
    Rn, dn = R.nstep_return(r, d, 1, 0.97)
    assert np.array_equal(Rn, r) and np.array_equal(dn, d)


def test_discounted_spec_2_62():
    # rewards [1,0,2], discount 0.9 -> 2.62
    r = np.array([[1.0], [0.0], [2.0]])
    out = R.discounted_return(r, np.zeros((3, 1)), None, 0.9)
    assert abs(out[0, 0] - 2.62) < 1e-12


def test_gae_spec_0_5():
    # r=1, gamma=1, V=2.5, V'=2, lambda=0 -> adv 0.5
    adv, ret = R.gae(np.array([[1.0]]), np.array([[2.5]]), np.zeros((1, 1)), np.array([2.0]), 1.0, 0.0)
    assert adv[0, 0] == 0.5 and ret[0, 0] == 3.0


# ---- closed forms ---------------------------------------------------------
@pytest.mark.parametrize("gamma", [0.9, 0.99, 0.997])
def test_discounted_geometric(gamma):
    T, B, c = 50, 3, 0.7
    boot = np.array([1.5, -2.0, 0.0])
    out = R.discounted_return(np.full((T, B), c), np.zeros((T, B)), boot, gamma)
    for t in range(T):
        m = T - t
        ref = c * (1 - gamma ** m) / (1 - gamma) + gamma ** m * boot
        np.testing.assert_allclose(out[t], ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_nstep_geometric(n):
    T, c, gamma = 20, -1.25, 0.99
    Rn, dn = R.nstep_return(np.full((T, 2), c), np.zeros((T, 2), np.uint8), n, gamma)
    np.testing.assert_allclose(Rn, c * (1 - gamma ** n) / (1 - gamma), rtol=1e-13)
    assert not dn.any()


def test_gae_lambda0_is_td_residual():
    # S:754
    r, v, d, boot = returns_inputs(3, 16, 5, p_done=0.2)
    adv, _ = R.gae(r, v, d, boot, 0.99, 0.0)
    vn = np.concatenate([v[1:].astype(np.float64), boot[None].astype(np.float64)])
    delta = r.astype(np.float64) + 0.99 * (1 - d) * vn - v
    np.testing.assert_allclose(adv, delta, rtol=1e-14, atol=1e-14)


def test_gae_lambda1_is_return_minus_value():
    # S:755 (telescoping): lambda=1 -> adv = discounted return (with bootstrap) - V,
    # and this holds with dones too because both mask the same terms.
    r, v, d, boot = returns_inputs(4, 40, 6, p_done=0.1)
    adv, ret = R.gae(r, v, d, boot, 0.99, 1.0)
    disc = R.discounted_return(r, d, boot, 0.99)
    np.testing.assert_allclose(adv, disc - v, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(ret, disc, rtol=1e-10, atol=1e-10)


def test_nstep_target_full_window_equals_discounted():
    # n = T with bootstrap q_T: the single target row is the bootstrapped discounted return.
    r, v, d, boot = returns_inputs(5, 6, 4, p_done=0.2)
    y, dn = R.nstep_return(r, d, 6, 0.95, q=v, q_boot=boot)
    disc = R.discounted_return(r, d, boot, 0.95)
    np.testing.assert_allclose(y[0], disc[0], rtol=1e-13, atol=1e-13)


def test_nstep_target_done_no_bootstrap():
    # done_n true -> y = return_n exactly
    r = np.array([[1.0], [2.0], [3.0], [4.0]])
    d = np.array([[0], [1], [0], [0]], np.uint8)
    q = np.full((4, 1), 100.0)
    y, dn = R.nstep_return(r, d, 3, 0.9, q=q, q_boot=np.array([100.0]))
    assert dn[0, 0] == 1 and y[0, 0] == 1.0 + 0.9 * 2.0
    assert dn[1, 0] == 1 and y[1, 0] == 2.0


# ---- exact rational sum-form evaluation (independent formulation) -----------
def _frac(x):
    return Fraction(float(x))


def _sum_form_discounted(r, d, boot, gamma):
    T, B = r.shape
    g = _frac(gamma)
    out = [[None] * B for _ in range(T)]
    for b in range(B):
        for t in range(T):
            tot, disc, alive = Fraction(0), Fraction(1), True
            for i in range(t, T):
                tot += disc * _frac(r[i, b])
                if d[i, b]:
                    alive = False
                    break
                disc *= g
            if alive:
                tot += disc * _frac(boot[b])
            out[t][b] = tot
    return out


def _sum_form_gae(r, v, d, boot, gamma, lam):
    T, B = r.shape
    g, l = _frac(gamma), _frac(lam)
    adv = [[None] * B for _ in range(T)]
    for b in range(B):
        delta = []
        for t in range(T):
            vn = _frac(boot[b]) if t == T - 1 else _frac(v[t + 1, b])
            delta.append(_frac(r[t, b]) + g * (1 - int(d[t, b])) * vn - _frac(v[t, b]))
        for t in range(T):
            tot, w = Fraction(0), Fraction(1)
            for i in range(t, T):
                tot += w * delta[i]
                if d[i, b]:
                    break
                w *= g * l
            adv[t][b] = tot
    return adv


def test_discounted_vs_exact_sum_form():
    r, v, d, boot = returns_inputs(11, 8, 2, reward_kind="small", p_done=0.25)
    out = R.discounted_return(r, d, boot, 0.99)
    ex = _sum_form_discounted(r, d, boot, 0.99)
    for t in range(8):
        for b in range(2):
            assert abs(out[t, b] - float(ex[t][b])) <= 1e-14 * max(1.0, abs(float(ex[t][b])))


def test_gae_vs_exact_sum_form():
    r, v, d, boot = returns_inputs(12, 8, 2, reward_kind="small", p_done=0.25)
    adv, ret = R.gae(r, v, d, boot, 0.99, 0.95)
    ex = _sum_form_gae(r, v, d, boot, 0.99, 0.95)
    for t in range(8):
        for b in range(2):
            e = float(ex[t][b])
            assert abs(adv[t, b] - e) <= 1e-13 * max(1.0, abs(e))
            assert abs(ret[t, b] - (e + float(v[t, b]))) <= 1e-13 * max(1.0, abs(e) + abs(float(v[t, b])))


def test_nstep_random_vs_direct_loops():
    # n-step vs direct summation on random buffers (scalar loop, Fractions)
    g = rng(13)
    for trial in range(30):
        T = int(g.integers(3, 12))
        n = int(g.integers(1, T + 1))
        gamma = float(g.uniform(0.5, 1.0))
        r = g.normal(size=(T, 2))
        d = (g.random((T, 2)) < g.uniform(0, 0.5)).astype(np.uint8)
        Rn, dn = R.nstep_return(r, d, n, gamma)
        for t in range(T - n + 1):
            for b in range(2):
                tot, disc, done = Fraction(0), Fraction(1), 0
                for i in range(n):
                    tot += disc * _frac(r[t + i, b])
                    if d[t + i, b]:
                        done = 1
                        break
                    disc *= _frac(gamma)
                assert abs(Rn[t, b] - float(tot)) <= 1e-13 * max(1, abs(float(tot)))
                assert dn[t, b] == done


# ---- time-limit bootstrap (reading R34; P:95 fn) ----
def _truncated_pair(seed, T=40, B=6, k=17):
    """A long episode (no dones, bootstrap b) and the same rows cut by a time limit after
    row k, whose v_term is the untruncated return / value of row k+1; the rows after k are
    replaced by an unrelated new episode."""
    g = np.random.default_rng(seed)
    r = g.normal(0, 1, (T, B))
    v = g.normal(0, 3, (T, B))
    boot = g.normal(0, 3, B)
    d0 = np.zeros((T, B), np.uint8)
    r2, v2 = r.copy(), v.copy()
    r2[k + 1:] = g.normal(0, 5, (T - k - 1, B))
    v2[k + 1:] = g.normal(0, 5, (T - k - 1, B))
    d2 = np.zeros((T, B), np.uint8)
    d2[k] = 2
    return r, v, boot, d0, r2, v2, d2, k


def test_timeout_with_exact_bootstrap_equals_untruncated():
    gamma = 0.97
    r, v, boot, d0, r2, v2, d2, k = _truncated_pair(1)
    full = R.discounted_return(r, d0, boot, gamma)
    vt = np.zeros_like(r)
    vt[k] = full[k + 1]                                   # the value the cut removed
    cut = R.discounted_return(r2, d2, np.zeros(r.shape[1]), gamma, v_term=vt)
    np.testing.assert_allclose(cut[:k + 1], full[:k + 1], rtol=1e-12, atol=1e-12)
    # n-step: a window containing row k equals the untruncated full return (its v_term is
    # exactly what the cut removed); a window before the cut equals the plain n-step sum
    n = 5
    Rn_plain, _ = R.nstep_return(r, d0, n, gamma)
    Rn_cut, dn = R.nstep_return(r2, d2, n, gamma, v_term=vt)
    for t in range(k - n + 1, k + 1):
        np.testing.assert_allclose(Rn_cut[t], full[t], rtol=1e-12, atol=1e-12)
        assert dn[t].all()
    np.testing.assert_allclose(Rn_cut[:k - n + 1], Rn_plain[:k - n + 1], rtol=1e-12, atol=1e-12)
    assert not dn[:k - n + 1].any()
    # identity check of the plain sum itself: R^n_t = R_t - gamma^n R_{t+n} without dones
    np.testing.assert_allclose(Rn_plain[:k], full[:k] - gamma ** n * full[n:k + n], rtol=1e-9, atol=1e-9)


def test_timeout_gae_lambda_limits():
    gamma = 0.99
    r, v, boot, d0, r2, v2, d2, k = _truncated_pair(2)
    vt = np.zeros_like(r)
    vt[k] = v[k + 1]                                      # V of the final observation
    # lambda = 0: A_t = delta_t, identical to the untruncated delta for t <= k
    a0, _ = R.gae(r, v, d0, boot, gamma, 0.0)
    a0c, _ = R.gae(r2, v, d2, boot, gamma, 0.0, v_term=vt)
    np.testing.assert_allclose(a0c[:k + 1], a0[:k + 1], rtol=1e-12, atol=1e-12)
    # lambda = 1: ret = the discounted return with the same time-limit bootstrap
    _, ret1 = R.gae(r2, v2, d2, boot, gamma, 1.0, v_term=vt)
    np.testing.assert_allclose(ret1, R.discounted_return(r2, d2, boot, gamma, v_term=vt), rtol=1e-10, atol=1e-10)


def test_timeout_closed_form_and_plain_terminal_without_values():
    gamma, c, rc, k = 0.9, 7.0, 1.5, 6
    T = 12
    r = np.full((T, 1), rc)
    d = np.zeros((T, 1), np.uint8)
    d[k] = 2
    vt = np.zeros((T, 1))
    vt[k] = c
    Rt = R.discounted_return(r, d, np.array([100.0]), gamma, v_term=vt)
    assert abs(Rt[0, 0] - (rc * (1 - gamma ** (k + 1)) / (1 - gamma) + gamma ** (k + 1) * c)) < 1e-12
    # without v_term a time-limit row is a plain terminal: same as done = 1
    d1 = np.where(d == 2, 1, 0).astype(np.uint8)
    np.testing.assert_array_equal(R.discounted_return(r, d, None, gamma), R.discounted_return(r, d1, None, gamma))
    y2, dn2 = R.nstep_return(r, d, 3, gamma)
    y1, dn1 = R.nstep_return(r, d1, 3, gamma)
    np.testing.assert_array_equal(y2, y1)
    np.testing.assert_array_equal(dn2, dn1)
