"""Property-based pins of the return oracle (hypothesis): identities that hold for every
input, so a dropped term, a wrong sign or an index slip in oracle/returns.py fails here even
where no worked example reaches (SURVEY.md §8c pins; readings R1, R24, R34)."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import returns as OR

shapes = st.tuples(st.integers(1, 40), st.integers(1, 6))


def _inputs(seed, T, B, p_done, p_timeout=0.0):
    g = np.random.default_rng(seed)
    r = g.normal(0, 3, (T, B))
    v = g.normal(0, 5, (T, B))
    boot = g.normal(0, 5, B)
    d = (g.random((T, B)) < p_done).astype(np.uint8)
    d[(d == 1) & (g.random((T, B)) < p_timeout)] = 2
    vt = g.normal(0, 5, (T, B))
    return r, v, d, boot, vt


@settings(max_examples=60, deadline=None)
@given(shapes, st.integers(0, 10**6), st.floats(0.5, 0.999), st.floats(0.0, 0.3))
def test_gae_lambda_one_is_discounted_minus_value(shape, seed, gamma, p_done):
    # GAE with lambda = 1 gives A_t = R_t - V_t (the discounted return bootstrapped from
    # V_T), with or without time limits (R34)
    T, B = shape
    r, v, d, boot, vt = _inputs(seed, T, B, p_done, 0.5)
    for vterm in (None, vt):
        adv, ret = OR.gae(r, v, d, boot, gamma, 1.0, v_term=vterm)
        np.testing.assert_allclose(ret, OR.discounted_return(r, d, boot, gamma, v_term=vterm), rtol=1e-9, atol=1e-9)


@settings(max_examples=60, deadline=None)
@given(shapes, st.integers(0, 10**6), st.floats(0.5, 0.999))
def test_gae_lambda_zero_is_td_error(shape, seed, gamma):
    # lambda = 0 gives the one-step TD error delta_t
    T, B = shape
    r, v, d, boot, _ = _inputs(seed, T, B, 0.2)
    adv, _ = OR.gae(r, v, d, boot, gamma, 0.0)
    v_next = np.concatenate([v[1:], boot[None]], 0)
    np.testing.assert_allclose(adv, r + gamma * (1 - d) * v_next - v, rtol=1e-12, atol=1e-12)


@settings(max_examples=60, deadline=None)
@given(shapes, st.integers(0, 10**6), st.floats(0.5, 0.999), st.integers(1, 6))
def test_nstep_telescopes_into_the_discounted_return(shape, seed, gamma, n):
    # without dones: R_t = R^n_t + gamma^n R_{t+n} (the n-step return is the discounted return
    # truncated after n rewards); with q = R and q_boot the target reproduces R_t exactly
    T, B = shape
    if n > T:
        n = T
    r, _, _, boot, _ = _inputs(seed, T, B, 0.0)
    d = np.zeros((T, B), np.uint8)
    R = OR.discounted_return(r, d, boot, gamma)
    Rn, dn = OR.nstep_return(r, d, n, gamma)
    assert not dn.any()
    Rfull = np.concatenate([R, boot[None]], 0)
    np.testing.assert_allclose(Rn, R[:T - n + 1] - gamma ** n * Rfull[n:], rtol=1e-9, atol=1e-9)
    y, _ = OR.nstep_return(r, d, n, gamma, q=Rfull[:T], q_boot=boot)
    np.testing.assert_allclose(y, R[:T - n + 1], rtol=1e-9, atol=1e-9)


@settings(max_examples=60, deadline=None)
@given(shapes, st.integers(0, 10**6), st.floats(0.5, 0.999), st.integers(1, 6))
def test_nstep_equals_discounted_return_of_the_window(shape, seed, gamma, n):
    # with dones: R^n_t equals the discounted return of rows t..t+n-1 alone (bootstrap 0), and
    # done^n_t is the OR of those done flags — the definition computed a second way (R1, R24)
    T, B = shape
    n = min(n, T)
    r, _, d, _, _ = _inputs(seed, T, B, 0.3)
    Rn, dn = OR.nstep_return(r, d, n, gamma)
    for t in range(T - n + 1):
        w = OR.discounted_return(r[t:t + n], d[t:t + n], None, gamma)[0]
        np.testing.assert_allclose(Rn[t], w, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(dn[t], (d[t:t + n] != 0).any(0).astype(np.uint8))


@settings(max_examples=40, deadline=None)
@given(st.integers(2, 40), st.integers(0, 10**6), st.floats(0.5, 0.999), st.data())
def test_time_limit_cut_with_exact_value_changes_nothing(T, seed, gamma, data):
    # R34: cutting an episode at row k by a time limit whose v_term is the removed continuation
    # leaves every return up to row k unchanged, for any k and any later rows
    k = data.draw(st.integers(0, T - 2))
    g = np.random.default_rng(seed)
    r = g.normal(0, 2, (T, 1))
    boot = g.normal(0, 2, 1)
    d0 = np.zeros((T, 1), np.uint8)
    full = OR.discounted_return(r, d0, boot, gamma)
    r2 = r.copy()
    r2[k + 1:] = g.normal(0, 9, (T - k - 1, 1))
    d2 = d0.copy()
    d2[k] = 2
    vt = np.zeros((T, 1))
    vt[k] = full[k + 1]
    cut = OR.discounted_return(r2, d2, g.normal(0, 9, 1), gamma, v_term=vt)
    np.testing.assert_allclose(cut[:k + 1], full[:k + 1], rtol=1e-10, atol=1e-10)
