"""Summarise ncu output for profiles/: key counters of a --set full capture and the
per-kernel shares of a gpu__time_duration launch list.

    python scripts/ncu_summary.py full gpurun_out/prof.ncu-rep        -> JSON per kernel
    python scripts/ncu_summary.py launches gpurun_out/launches.csv    -> JSON per kernel name
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u.get(k, '')}".strip()
        out.append(ent)
    return out


def launches(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    t = defaultdict(list)
    for r in rows:
        t[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in t.values())
    return {k: {"launches": len(v), "avg_ns": sum(v) / len(v), "share": sum(v) / tot} for k, v in t.items()}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(full(path) if mode == "full" else launches(path), indent=1))
