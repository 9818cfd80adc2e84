"""CPU test of the async pipeline's replay-ratio budget (SPEC: measured ratio never
exceeds the cap beyond one optimiser batch of slack)."""
from paper_1909_01500_b200.pipeline import ReplayRatio


def test_budget_counter_caps_the_ratio():
    rr = ReplayRatio(cap=1.0)
    assert not rr.can_consume(1)                    # nothing generated yet
    rr.credit(40 * 4)                               # one sampler batch: 40 steps x 4 envs
    steps = 0
    while rr.can_consume(64):
        rr.debit(64)
        steps += 1
    assert steps == 2 and rr.consumed == 128 and rr.ratio <= 1.0
    for _ in range(100):                            # generation and consumption interleaved
        rr.credit(160)
        while rr.can_consume(64):
            rr.debit(64)
        assert rr.consumed <= rr.cap * rr.generated
        assert rr.generated * rr.cap - rr.consumed < 64   # at most one batch of slack unused


def test_fractional_cap():
    rr = ReplayRatio(cap=0.67)
    rr.credit(1000)
    n = 0
    while rr.can_consume(10):
        rr.debit(10)
        n += 1
    assert n == 67 and abs(rr.ratio - 0.67) < 1e-12
