"""The toy golden file (BASELINE.json configs[0]) is reproducible from the oracle
and agrees with values computed by hand from its definitions."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "toy.json")


def load():
    with open(GOLD) as f:
        return json.load(f)


def test_golden_regenerates(tmp_path):
    before = open(GOLD).read()
    subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "make_golden.py")],
                          stdout=subprocess.DEVNULL)
    assert open(GOLD).read() == before


def test_golden_hand_values():
    g = load()
    # n-step row 0, column 0: r = 1, 0, 2 with the episode ending after row 2:
    # 1 + 0.99*0 + 0.99^2 * 2 = 2.9602, done_n = 1
    assert abs(g["nstep"][0][0] - 2.9602) < 1e-12 and g["done_n"][0][0] == 1
    # column 1, rows 0..2: 0 - 0.99 + 0.99^2*0.5 = -0.49995, no done
    assert abs(g["nstep"][0][1] - (-0.49995)) < 1e-12 and g["done_n"][0][1] == 0
    # discounted, last row col 0: done at T-1 -> R = r = 1.0 (no bootstrap)
    assert g["discounted"][7][0] == 1.0
    # discounted, last row col 1: -1 + 0.99 * (-1.5)
    assert abs(g["discounted"][7][1] - (-1.0 + 0.99 * -1.5)) < 1e-15
    # GAE, last row col 1: delta = -1 + 0.99*(-1.5) - 0 ; adv = delta
    assert abs(g["gae_adv"][7][1] - (-1.0 + 0.99 * -1.5)) < 1e-15
    # the tree root is the sum of the leaves; the duplicate update's last write wins
    assert int(g["tree_total"]) == sum(int(x) for x in g["tree_q"])
    assert len(g["sample_idx"]) == 4 and max(g["is_weights"]) == 1.0
