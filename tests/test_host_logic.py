"""Host-side index logic of the product package checked against the oracle's
definitions, and the bench's oracle arm checked for independence from the product
(CPU only)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import gather as OG

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _geometries(count, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    for _ in range(count):
        period = int(g.choice([1, 4, 8, 40]))
        cap = period * int(g.integers(2, 40))
        cursor = int(g.integers(0, cap))
        size = int(g.integers(0, cap + 1))
        k = int(g.integers(1, 6))
        yield g, period, cap, cursor, size, k


def test_valid_transition_rows_equal_oracle_windows():
    # replay.valid_transition_rows picks the initial leaves in bench and pipeline: every row
    # it returns (and no other) must satisfy the oracle's window rule (§8c #2, #14)
    from paper_1909_01500_b200 import replay as R
    for g, _, cap, cursor, size, k in _geometries(400, 1):
        n = int(g.integers(1, 8))
        got = set(int(r) for r in R.valid_transition_rows(cap, cursor, size, k, n))
        ref = {r for r in range(cap) if OG.window_valid_transition(r, cap, cursor, size, k, n)}
        assert got == ref, (cap, cursor, size, k, n)


def test_valid_sequence_blocks_equal_oracle_windows():
    from paper_1909_01500_b200 import replay as R
    for g, period, cap, cursor, size, k in _geometries(400, 2):
        L = int(g.integers(1, 3 * period + 2))
        got = set(int(b) for b in R.valid_sequence_blocks(cap, period, cursor, size, k, L))
        ref = {b for b in range(cap // period)
               if OG.window_valid_sequence(b * period, cap, cursor, size, k, L)}
        assert got == ref, (cap, period, cursor, size, k, L)
        leaves = R.leaves_of(sorted(got), 3)
        assert leaves.tolist() == [b * 3 + j for b in sorted(got) for j in range(3)]


def test_bench_oracle_arm_never_imports_the_product():
    # the --impl reference / cpu_baseline arm runs oracle + synth only: no librpl.so mapped
    code = r"""
import json, sys
sys.path.insert(0, %r)
import bench
from synth import make_ring
c = dict(bench.R2D2)
c.update(cap_T=400, B=4)
h = make_ring(5, 400, 4, ep_len=50.0, reward_kind="r2d2", period=40, rnn_parts=2, rnn_h=8, cursor=123)
o = bench.OracleStep(c, h)
o.step(3); o.step(3)
maps = open("/proc/self/maps").read()
print(json.dumps({"mods": sorted(m for m in sys.modules if m.startswith("paper_1909_01500_b200")),
                  "so": "librpl" in maps}))
""" % ROOT
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out == {"mods": [], "so": False}
