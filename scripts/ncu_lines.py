"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
    python scripts/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
rows, cur, hdr = [], None, None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] in ("File Path", "File Name"):
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            smp = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            smp = 0
        stalls = {k: float(d[k] or 0) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
                  and (d[k] or "0").replace(".", "").isdigit()}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        rows.append((smp, cur.split("/")[-1], int(r[0]), r[1].strip()[:80], top))
tot = sum(x[0] for x in rows) or 1
for x in sorted(rows, key=lambda x: -x[0])[:N]:
    print(f"{x[0]:6d} {x[0]/tot:5.3f} {x[1]}:{x[2]} {x[3]}  {[(k[6:], int(v)) for k, v in x[4]]}")
