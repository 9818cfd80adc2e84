"""Oracle: R2D2 value rescaling h and its inverse (mpmath, 60 significant digits).

The paper names R2D1 value rescaling only through its R2D2 reproduction (P:34,
P:122-132); the formula is S:810:

    h(x)      = sign(x) (sqrt(|x| + 1) - 1) + eps x
    h^-1(y)   = sign(y) ( ((sqrt(1 + 4 eps (|y| + 1 + eps)) - 1) / (2 eps))^2 - 1 )

(the inverse is the closed-form root of h(x) = y, [EXT: Pohlen et al. 2018 /
R2D2]; eps = 1e-3 by default, §8c #4).  Both are evaluated in the textbook form
at 60 digits, where cancellation costs nothing, and rounded once to float64.
"""
from __future__ import annotations

import mpmath
import numpy as np

_DPS = 60


def _ctx():
    ctx = mpmath.MPContext()
    ctx.dps = _DPS
    return ctx


_C = _ctx()


def h_mp(x, eps):
    x = _C.mpf(x)
    e = _C.mpf(eps)
    s = _C.sign(x)
    return s * (_C.sqrt(abs(x) + 1) - 1) + e * x


def h_inv_mp(y, eps):
    y = _C.mpf(y)
    e = _C.mpf(eps)
    s = _C.sign(y)
    u = (_C.sqrt(1 + 4 * e * (abs(y) + 1 + e)) - 1) / (2 * e)
    return s * (u * u - 1)


def h(x, eps=1e-3):
    return float(h_mp(float(x), float(eps)))


def h_inv(y, eps=1e-3):
    return float(h_inv_mp(float(y), float(eps)))


def h_array(x, eps=1e-3):
    x = np.asarray(x, np.float64)
    out = np.empty_like(x)
    flat = x.reshape(-1)
    o = out.reshape(-1)
    for i in range(flat.size):
        o[i] = float(h_mp(float(flat[i]), float(eps)))
    return out


def h_inv_array(y, eps=1e-3):
    y = np.asarray(y, np.float64)
    out = np.empty_like(y)
    flat = y.reshape(-1)
    o = out.reshape(-1)
    for i in range(flat.size):
        o[i] = float(h_inv_mp(float(flat[i]), float(eps)))
    return out


def h_of_target(Rn, gamma_n, done_n, q_boot, eps=1e-3):
    """y = h(R^n + gamma^n (1 - done^n) h^-1(q_{t+n})) at 60 digits (§8c #5)."""
    inner = _C.mpf(float(Rn)) + _C.mpf(float(gamma_n)) * (1 - int(done_n)) * h_inv_mp(float(q_boot), eps)
    return float(h_mp(inner, eps))
