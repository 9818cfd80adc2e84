"""bench.py's JSON-line contract on a short run (the driver parses these keys): the headline,
`roofline`, `clocks`, `e2e` (host<->device copies declared), the a1-a4 `returns` line and
`gpu_launches` must all be present at N = 1.  Guards against a key silently dropping out of
the line (round 2: `e2e` and `returns` were once indented under the Mode C branch)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_line_carries_every_contract_key(cuda):
    out = subprocess.run([sys.executable, "bench.py", "--steps", "8", "--warmup", "3", "--no-secondary",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e",
                "returns"):
        assert key in d, key
    assert d["steps"] == 8 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["gpu_launches"] >= 2 * 8  # update + gather (sampling fused) per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    ret = d["returns"]
    assert "error" not in ret, ret
    for name in ("gae", "disc", "nstep"):
        assert ret[f"{name}_us_per_call_max_over_ranks"] > 0
