"""GPU parity for NEXT-3 targets: rpl_returns_nstep_dq (double-Q selection + n-step +
rescaling) and rpl_c51_project vs oracle/targets.py."""
import numpy as np
import pytest

from oracle import targets as OT
from synth import rng
from tests._tol import check_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rpl(cuda):
    import paper_1909_01500_b200 as rpl
    return rpl


def T_(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def H(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("T,B,A,n,rescale", [(84, 64, 18, 5, True), (9, 7, 4, 3, False), (5, 3, 1, 5, True),
                                             (40, 33, 18, 1, False)])
def test_nstep_double_q(rpl, T, B, A, n, rescale):
    g = rng(T * 7 + A)
    r = (g.normal(size=(T, B)) * (g.random((T, B)) < 0.3) * 50).astype(np.float32)
    d = (g.random((T, B)) < 0.05).astype(np.uint8)
    qo = g.normal(0, 10, (T + 1, B, A)).astype(np.float32)
    qo[1, 0, :] = qo[1, 0, 0]                                 # ties: first maximum wins
    qo[2, 1 % B, 0] = np.nan                                  # NaN never wins
    qt = g.normal(0, 10, (T + 1, B, A)).astype(np.float32)
    y, dn, a = rpl.returns_nstep_dq(T_(r), T_(d), n, 0.997, T_(qo), T_(qt), rescale=rescale)
    yr, dnr, ar = OT.nstep_double_q(r, d, n, 0.997, qo, qt, rescale=rescale)
    assert np.array_equal(H(a), ar) and np.array_equal(H(dn), dnr)
    check_rel(H(y), yr, np.abs(yr) + 1e-3, what="double-q target")


@pytest.mark.parametrize("n,A,N", [(512, 18, 51), (7, 1, 51), (33, 6, 11)])
def test_c51_projection(rpl, n, A, N):
    g = rng(n + A + N)
    logits = g.normal(size=(n, A, N))
    p = np.exp(logits)
    p /= p.sum(-1, keepdims=True)
    p = p.astype(np.float32)
    qo = g.normal(size=(n, A)).astype(np.float32) if A > 1 else None
    R = (g.normal(size=n) * 3).astype(np.float32)
    R[0], R[1 % n] = 25.0, -25.0                              # clipped both ways
    dn = (g.random(n) < 0.1).astype(np.uint8)
    m, a = rpl.c51_project(T_(p), None if qo is None else T_(qo), T_(R), T_(dn), -10.0, 10.0, 0.99 ** 3)
    ref = OT.c51_targets(p, qo, R, dn, 0.99 ** 3, -10.0, 10.0)
    mm = H(m)
    # R21's rule with the distribution's total mass (1) as the scale: 1e-5 relative per atom,
    # and for atoms below 1e-6 of the mass (pure rounding territory) 1e-11 absolute
    check_rel(mm, ref, np.ones_like(ref), what="c51 projection")
    assert np.allclose(mm.sum(-1), p.sum(-1)[np.arange(n), H(a)], atol=1e-5)
    if qo is not None:
        assert np.array_equal(H(a), [OT.argmax_first(qo[s]) for s in range(n)])


@pytest.mark.parametrize("cap,B,row0,T_out,n,rescale", [(200, 64, 40, 80, 5, True), (200, 64, 150, 80, 5, True),
                                                        (37, 5, 30, 20, 1, False), (12, 3, 0, 7, 5, False),
                                                        (4096, 256, 4000, 96, 3, False)])
def test_ring_td_abs_vs_oracle(rpl, cap, B, row0, T_out, n, rescale):
    # NEXT-1 initial priorities (R33): per-step |n-step TD| from ring arrays, rows mod cap
    g = rng(cap + row0 + n)
    rew = (g.normal(size=(cap, B)) * (g.random((cap, B)) < 0.4) * 20).astype(np.float32)
    done = (g.random((cap, B)) < 0.05).astype(np.uint8)
    qt = g.normal(0, 5, (cap, B)).astype(np.float32)
    qb = g.normal(0, 5, (cap, B)).astype(np.float32)
    qt[row0, 0] = 0.0
    out = rpl.ring_td_abs(T_(rew), T_(done), T_(qt), T_(qb), row0, T_out, n, 0.997, rescale=rescale)
    ref = OT.ring_td_abs(rew, done, qt, qb, row0, T_out, n, 0.997, rescale=rescale)
    rows = [(row0 + t) % cap for t in range(T_out)]
    scale = np.abs(ref) + np.abs(qt[rows].astype(np.float64)) + 1.0
    check_rel(H(out), ref, scale=scale, what="ring td")


def test_ring_td_abs_errors(rpl):
    import torch
    z = torch.zeros((10, 2), device="cuda")
    d = torch.zeros((10, 2), dtype=torch.uint8, device="cuda")
    with pytest.raises(RuntimeError):
        rpl.ring_td_abs(z, d, z, z, 0, 6, 5, 0.9)          # T_out + n > cap
    with pytest.raises(RuntimeError):
        rpl.ring_td_abs(z, d, z, z, 10, 1, 1, 0.9)         # row0 outside the ring


def test_ring_append_rows(rpl):
    import torch
    ring = torch.zeros((10, 3), device="cuda")
    src = torch.arange(12, dtype=torch.float32).reshape(4, 3).pin_memory()
    rpl.ring_append_rows(ring, src, 8)                   # wraps: rows 8, 9, 0, 1
    torch.cuda.synchronize()
    h = H(ring)
    assert h[[8, 9, 0, 1]].tolist() == src.numpy().tolist() and not h[2:8].any()
