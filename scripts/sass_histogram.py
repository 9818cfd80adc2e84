"""Per-kernel SASS opcode histogram of the built objects (cuobjdump -sass), for the evidence
that the hot kernels use the Blackwell paths: UTMALDG / UTMASTG (TMA tensor copies), UBLKCP
(bulk copies), SYNCS (mbarriers), STG.E.EF (evict-first streaming stores), DFMA (fp64 scans).
Usage: python scripts/sass_histogram.py [out.json]  (CPU only; reads paper_1909_01500_b200/build/*.o)."""
import collections
import glob
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1909_01500_b200", "build")
KEY = ("UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "STG.E.EF", "LDG.E.EF", "DFMA", "DADD", "DMUL", "F2F", "SHFL",
       "ATOMG", "REDG", "RED", "BAR", "LDS", "STS", "STG", "LDG", "UTMAPF", "ELECT", "BSSY")


def demangle(names):
    res = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return res.stdout.splitlines() if res.returncode == 0 else names


out = {}
for obj in sorted(glob.glob(os.path.join(BUILD, "*.o"))):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, counts = None, {}
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            op = m.group(1)
            counts[cur][op] += 1
    names = list(counts)
    for raw, nice in zip(names, demangle(names)):
        c = counts[raw]
        if not any(k.startswith("k_") for k in re.findall(r"k_\w+", nice)):
            continue
        short = nice.replace("(anonymous namespace)::", "").replace("rpl::", "")
        short = re.sub(r"^void ", "", short)
        short = re.sub(r"\((?!.*<).*$", "", short)  # drop the parameter list
        agg = {k: sum(v for op, v in c.items() if op == k or op.startswith(k + ".")) for k in KEY}
        out[f"{os.path.basename(obj)}:{short}"] = {"instructions": sum(c.values()),
                                                    "key_ops": {k: v for k, v in agg.items() if v},
                                                    "top": dict(c.most_common(12))}
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2", "sass_histogram.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1, sort_keys=True)
for k, v in sorted(out.items()):
    print(f"{k[:90]:90s} n={v['instructions']:5d} " + " ".join(f"{a}={b}" for a, b in v["key_ops"].items()))
