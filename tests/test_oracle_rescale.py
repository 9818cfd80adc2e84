"""Pins for oracle.rescale: special values, symmetry, derivative and inverse."""
import math

import mpmath
import numpy as np

from oracle import rescale as H


def test_h_special_values():
    eps = 1e-3
    assert H.h(0.0, eps) == 0.0
    # sqrt(4) - 1 + 3 eps, sqrt(9) - 1 + 8 eps: perfect squares give exact closed forms
    assert abs(H.h(3.0, eps) - (1.0 + 3e-3)) < 1e-15
    assert abs(H.h(8.0, eps) - (2.0 + 8e-3)) < 1e-15
    assert abs(H.h(-8.0, eps) + (2.0 + 8e-3)) < 1e-15
    assert abs(H.h_inv(1.0 + 3e-3, eps) - 3.0) < 1e-12


def test_h_odd_and_inverse():
    g = np.random.default_rng(0)
    xs = np.concatenate([g.normal(0, 1, 50), g.normal(0, 1000, 50), 10.0 ** g.uniform(-20, 6, 50)])
    for x in xs:
        assert H.h(-x) == -H.h(x)
        y = H.h_inv_mp(H.h_mp(float(x), 1e-3), 1e-3)
        assert abs(float(y) - x) <= 1e-14 * max(abs(x), 1e-300)
        z = H.h_mp(H.h_inv_mp(float(x), 1e-3), 1e-3)
        assert abs(float(z) - x) <= 1e-14 * max(abs(x), 1e-300)


def test_h_derivative_at_zero():
    # h'(0) = 1/2 + eps
    with mpmath.workdps(60):
        dx = mpmath.mpf("1e-30")
        der = (H.h_mp(dx, 1e-3) - H.h_mp(-dx, 1e-3)) / (2 * dx)
    assert abs(float(der) - (0.5 + 1e-3)) < 1e-15


def test_h_tiny_is_linear():
    # for |x| << 1: h(x) = x (1/2 + eps) - x^2/8 + ... ; relative error of the
    # linear term is O(x), so at 1e-14 the textbook float64 form (which loses it)
    # would fail while the mpmath oracle holds.
    x = 1e-14
    assert abs(H.h(x) / (x * (0.5 + 1e-3)) - 1) < 1e-12


def test_rescaled_target_done_is_h_of_return():
    from oracle import returns as R
    r = np.array([[1.0], [2.0], [3.0]])
    d = np.array([[1], [0], [0]], np.uint8)
    y, dn = R.nstep_return(r, d, 3, 0.997, q=np.full((3, 1), 50.0), q_boot=np.array([50.0]), rescale=True)
    assert y[0, 0] == H.h(1.0)


def test_rescaled_target_identity():
    # R^n = 0 and gamma^n (1-done) = 1 (gamma = 1, no done) -> y = h(h^-1(q)) = q
    r = np.zeros((4, 1))
    d = np.zeros((4, 1), np.uint8)
    q = np.array([[3.7], [-12.5], [0.01], [1e4]])
    y, _ = R_nstep(r, d, q)
    np.testing.assert_allclose(y[:, 0], [-12.5, 0.01, 1e4, 77.0][: y.shape[0]], rtol=1e-14)


def R_nstep(r, d, q):
    from oracle import returns as R
    return R.nstep_return(r, d, 1, 1.0, q=q, q_boot=np.array([77.0]), rescale=True)
