"""Brief of an ncu report (--set full): duration, DRAM throughput and bytes, issue and pipe
utilisation, top stall reasons — per kernel.  Usage: python scripts/ncu_brief.py file.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d.get("Kernel Name", "")[:90])
    for k in want:
        if k in d:
            print(f"  {k} = {d[k]} {units[hdr.index(k)]}")
    stalls = [(float(d[h] or 0), h) for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled")
              or (h.startswith("smsp__warp_issue_stalled") and h.endswith("per_warp_active.pct"))]
    for v, h in sorted(stalls, reverse=True)[:6]:
        print(f"  stall {h.split('stalled_')[-1]} = {v:.1f}")
