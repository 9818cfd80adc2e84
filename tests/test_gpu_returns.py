"""GPU parity: return kernels (rpl_returns_discounted / _nstep / rpl_gae /
rpl_value_rescale) vs the float64 oracle, through the C ABI."""
import json
import os

import numpy as np
import pytest

from oracle import rescale as ORS
from oracle import returns as OR
from synth import returns_inputs, rng
from tests._tol import check_rel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def T_(x, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def H(t):
    return t.cpu().numpy()


def test_toy_golden(rpl):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "toy.json")))
    I = g["inputs"]
    c = g["config"]
    r = T_(np.array(I["r"], np.float32))
    d = T_(np.array(I["d"], np.uint8))
    v = T_(np.array(I["v"], np.float32))
    boot = T_(np.array(I["bootstrap"], np.float32))
    qt = T_(np.array(I["q_target"], np.float32))
    qb = T_(np.array(I["q_boot"], np.float32))
    check_rel(H(rpl.returns_discounted(r, d, boot, c["gamma"])), g["discounted"], what="discounted")
    Rn, dn = rpl.returns_nstep(r, d, c["n_step"], c["gamma"])
    check_rel(H(Rn), g["nstep"], what="nstep")
    assert np.array_equal(H(dn), np.array(g["done_n"], np.uint8))
    y, _ = rpl.returns_nstep(r, d, c["n_step"], c["gamma"], q=qt, q_boot=qb)
    check_rel(H(y), g["nstep_target"], what="target")
    yr, _ = rpl.returns_nstep(r, d, c["n_step"], c["gamma"], q=qt, q_boot=qb, rescale=True, eps=c["rescale_eps"])
    check_rel(H(yr), g["nstep_target_rescaled"], what="target rescaled")
    adv, ret = rpl.gae(r, v, d, boot, c["gamma"], c["lam"])
    check_rel(H(adv), g["gae_adv"], what="adv")
    check_rel(H(ret), g["gae_ret"], what="ret")


# B % 16 == 0 takes a TMA kernel — whole-column tiles (multi-chunk T, partial 32-column
# blocks) or, under scan variants 4 / 5, the cluster split when T <= 128 (ragged last CTA,
# CTAs past T) — other B the LDG kernel
SHAPES = [(1, 1), (1, 7), (5, 3), (16, 32), (127, 33), (128, 64), (129, 31), (300, 100), (1000, 5), (300, 48),
          (129, 16), (1000, 80), (257, 4096), (20, 64), (65, 16), (97, 48), (33, 4096)]


@pytest.fixture(params=[0, 9, 6, 4, 5, 3, 7, 16])
def scan_variant(rpl, request):
    assert rpl._lib.lib.rpl_debug_set_scan_variant(request.param) == 0
    yield request.param
    rpl._lib.lib.rpl_debug_set_scan_variant(0)


@pytest.mark.parametrize("T,B", SHAPES)
@pytest.mark.parametrize("kind", ["clipped", "heavy"])
def test_discounted_and_gae_random(rpl, T, B, kind, scan_variant):
    seed = 1000 + T * 7 + B
    r, v, d, boot = returns_inputs(seed, T, B, reward_kind=kind, p_done=0.05)
    for gamma, lam in [(0.99, 0.95), (0.997, 1.0), (0.9, 0.0)]:
        ref = OR.discounted_return(r, d, boot, gamma)
        S = OR.abs_scale_discounted(r, d, boot, gamma)
        check_rel(H(rpl.returns_discounted(T_(r), T_(d), T_(boot), gamma)), ref, S, what="disc")
        check_rel(H(rpl.returns_discounted(T_(r), T_(d), None, gamma)), OR.discounted_return(r, d, None, gamma),
                  OR.abs_scale_discounted(r, d, None, gamma), what="disc no boot")
        adv_ref, ret_ref = OR.gae(r, v, d, boot, gamma, lam)
        Sg = OR.abs_scale_gae(r, v, d, boot, gamma, lam)
        adv, ret = rpl.gae(T_(r), T_(v), T_(d), T_(boot), gamma, lam)
        check_rel(H(adv), adv_ref, Sg, what="adv")
        check_rel(H(ret), ret_ref, Sg, what="ret")


def test_ppo_full_size(rpl, scan_variant):
    # BASELINE.json configs[1]: [T=128, B=4096], gamma 0.99, lambda 0.95; every element
    T, B = 128, 4096
    for kind, pd in [("clipped", 0.05), ("heavy", 0.001)]:
        r, v, d, boot = returns_inputs(77, T, B, reward_kind=kind, p_done=pd)
        adv, ret = rpl.gae(T_(r), T_(v), T_(d), T_(boot), 0.99, 0.95)
        a_ref, r_ref = OR.gae(r, v, d, boot, 0.99, 0.95)
        Sg = OR.abs_scale_gae(r, v, d, boot, 0.99, 0.95)
        check_rel(H(adv), a_ref, Sg, what="ppo adv")
        check_rel(H(ret), r_ref, Sg, what="ppo ret")
        disc = rpl.returns_discounted(T_(r), T_(d), T_(boot), 0.99)
        check_rel(H(disc), OR.discounted_return(r, d, boot, 0.99), OR.abs_scale_discounted(r, d, boot, 0.99),
                  what="ppo disc")


@pytest.mark.parametrize("T,B,n", [(8, 2, 3), (3, 1, 3), (50, 37, 1), (50, 37, 5), (128, 256, 3), (7, 5, 7)])
def test_nstep_random(rpl, T, B, n):
    r, v, d, boot = returns_inputs(2000 + T + B + n, T, B, reward_kind="heavy", p_done=0.2)
    gamma = 0.99
    R, dn = OR.nstep_return(r, d, n, gamma)
    absR, _ = OR.nstep_return(np.abs(r), d, n, gamma)
    g_R, g_dn = rpl.returns_nstep(T_(r), T_(d), n, gamma)
    check_rel(H(g_R), R, absR, what="nstep")
    assert np.array_equal(H(g_dn), dn)
    y, _ = OR.nstep_return(r, d, n, gamma, q=v, q_boot=boot)
    g_y, _ = rpl.returns_nstep(T_(r), T_(d), n, gamma, q=T_(v), q_boot=T_(boot))
    qabs = np.concatenate([np.abs(v), np.abs(boot)[None]], 0)
    scale = absR + gamma ** n * qabs[n:n + R.shape[0]]
    check_rel(H(g_y), y, scale, what="nstep target")


def test_nstep_rescaled_r2d2_shape(rpl):
    # R2D2: n=5, gamma=0.997, rescaling on, train rows [80, 64] from an 84-row slice
    g = rng(5)
    T, B, n = 84, 64, 5
    r = (g.normal(size=(T, B)) * (g.random((T, B)) < 0.05) * 100).astype(np.float32)
    d = (g.random((T, B)) < 0.01).astype(np.uint8)
    q = g.normal(0, 10, (T, B)).astype(np.float32)
    qb = g.normal(0, 10, B).astype(np.float32)
    y, dn = OR.nstep_return(r, d, n, 0.997, q=q, q_boot=qb, rescale=True, eps=1e-3)
    g_y, g_dn = rpl.returns_nstep(T_(r), T_(d), n, 0.997, q=T_(q), q_boot=T_(qb), rescale=True, eps=1e-3)
    assert g_y.shape == (80, 64)
    check_rel(H(g_y), y, np.abs(y) + 1e-3, what="rescaled target")
    assert np.array_equal(H(g_dn), dn)


def test_value_rescale(rpl):
    g = rng(9)
    x = np.concatenate([g.normal(0, 1, 2000), g.normal(0, 1000, 2000), 10.0 ** g.uniform(-30, 8, 2000),
                        -(10.0 ** g.uniform(-30, 8, 2000)), [0.0, -0.0, 1.0, -1.0, 3.0, 8.0]]).astype(np.float32)
    for inverse in (False, True):
        out = H(rpl.value_rescale(T_(x), 1e-3, inverse=inverse))
        ref = ORS.h_inv_array(x.astype(np.float64)) if inverse else ORS.h_array(x.astype(np.float64))
        check_rel(out, ref, what=f"rescale inverse={inverse}")
    # odd-length tail / misaligned view path
    xs = T_(x)[1:1000]
    out = H(rpl.value_rescale(xs.contiguous()[0:999], 1e-3))
    check_rel(out, ORS.h_array(x[1:1000].astype(np.float64)), what="rescale tail")


def test_errors(rpl):
    import torch
    r = torch.zeros(4, 3, device="cuda")
    d = torch.zeros(4, 3, dtype=torch.uint8, device="cuda")
    with pytest.raises(rpl._lib.RplError):
        rpl.returns_nstep(r, d, 5, 0.9)
    with pytest.raises(ValueError):
        rpl.returns_discounted(r.cpu(), d, None, 0.9)
    with pytest.raises(rpl._lib.RplError):
        rpl.returns_nstep(r, d, 2, 0.9, rescale=True, eps=0.0)


@pytest.mark.parametrize("T,B", [(1, 1), (16, 32), (129, 31), (300, 48), (1000, 16), (33, 256)])
def test_time_limit_bootstrap_tl_entries(rpl, T, B, scan_variant):
    _time_limit_case(rpl, T, B)


@pytest.mark.parametrize("T,B", [(128, 4096), (1000, 80)])
def test_time_limit_bootstrap_ppo_size(rpl, T, B):
    _time_limit_case(rpl, T, B)


def _time_limit_case(rpl, T, B):
    # R34: half of the episode ends are time limits (d = 2) with terminal values v_term;
    # discounted / GAE / n-step through the rpl_*_tl entries vs the oracle, every element
    g = rng(T * 13 + B)
    r, v, d, boot = returns_inputs(2000 + T + B, T, B, reward_kind="heavy", p_done=0.08)
    d = d.copy()
    d[(d == 1) & (g.random(d.shape) < 0.5)] = 2
    vt = g.normal(0, 5, (T, B)).astype(np.float32)
    for gamma, lam in [(0.99, 0.95), (0.997, 1.0)]:
        ref = OR.discounted_return(r, d, boot, gamma, v_term=vt)
        S = OR.abs_scale_discounted(r, d, boot, gamma, v_term=vt)
        check_rel(H(rpl.returns_discounted(T_(r), T_(d), T_(boot), gamma, v_term=T_(vt))), ref, S, what="disc tl")
        adv_ref, ret_ref = OR.gae(r, v, d, boot, gamma, lam, v_term=vt)
        Sg = OR.abs_scale_gae(r, v, d, boot, gamma, lam, v_term=vt)
        adv, ret = rpl.gae(T_(r), T_(v), T_(d), T_(boot), gamma, lam, v_term=T_(vt))
        check_rel(H(adv), adv_ref, Sg, what="adv tl")
        check_rel(H(ret), ret_ref, Sg, what="ret tl")
        # without v_term a time-limit row is a plain terminal (== d = 1)
        d1 = np.where(d != 0, 1, 0).astype(np.uint8)
        assert np.array_equal(H(rpl.returns_discounted(T_(r), T_(d), T_(boot), gamma)),
                              H(rpl.returns_discounted(T_(r), T_(d1), T_(boot), gamma)))
    for n in (1, 3, 5):
        if n > T:
            continue
        q = g.normal(0, 10, (T, B)).astype(np.float32)
        qb = g.normal(0, 10, B).astype(np.float32)
        # the rescaled oracle is mpmath per element: only on the small shapes
        for rescale in ((False, True) if T * B <= 20000 else (False,)):
            y, dn = rpl.returns_nstep(T_(r), T_(d), n, 0.99, q=T_(q), q_boot=T_(qb), rescale=rescale, v_term=T_(vt))
            yr, dnr = OR.nstep_return(r, d, n, 0.99, q=q, q_boot=qb, rescale=rescale, v_term=vt)
            sc, _ = OR.nstep_return(np.abs(r), d, n, 0.99, q=np.abs(q), q_boot=np.abs(qb), v_term=np.abs(vt))
            check_rel(H(y), yr, sc + np.abs(yr) + 1e-3, what=f"nstep tl n={n} rescale={rescale}")
            assert np.array_equal(H(dn), dnr)
