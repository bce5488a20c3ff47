"""Aggregate an ncu source-page capture (SASS view) by opcode: samples, stall reasons,
executed instructions.  python tools/ncu_sass_stalls.py prof.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(lambda: defaultdict(float))
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split(" ")[0].split(".")[0]
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    a = agg[op]
    a["samples"] += s
    a["exec"] += float(r[ix["Instructions Executed"]] or 0)
    for k in keys:
        a[k] += float(r[ix[k]] or 0)
print(f"total samples {tot:.0f}")
cols = ["stall_wait", "stall_math", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_long_sb",
        "stall_barrier", "stall_mio", "stall_lg", "stall_branch_resolving", "stall_dispatch", "stall_no_inst"]
cols = [c for c in cols if c in keys]
print(f"{'op':10} {'samp%':>6} {'exec':>12} " + " ".join(f"{c[6:14]:>8}" for c in cols))
for op, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:30]:
    print(f"{op:10} {a['samples'] / tot * 100:6.1f} {a['exec']:12.0f} " + " ".join(f"{a[c] / tot * 100:8.1f}" for c in cols))
