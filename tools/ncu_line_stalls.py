"""Aggregate an ncu capture's stall samples by CUDA source line (cuda,sass view; needs -lineinfo).
   python tools/ncu_line_stalls.py prof.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
text = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(text)))
cur_file, hdr, ix = None, None, None
agg = defaultdict(lambda: defaultdict(float))
per_file = defaultdict(float)
tot = 0.0
last_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        last_line = (cur_file, int(r[0]), r[1].strip()[:70])
    if not r[2].startswith("0x"):
        continue
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    a = agg[last_line]
    a["samples"] += s
    a["exec"] += float(r[ix["Instructions Executed"]] or 0)
    for k in ("stall_wait", "stall_math", "stall_short_sb", "stall_barrier", "stall_not_selected", "stall_selected",
              "stall_branch_resolving", "stall_mio", "stall_long_sb"):
        if k in ix:
            a[k] += float(r[ix[k]] or 0)
    per_file[cur_file] += s
    tot += s
print(f"total samples {tot:.0f}")
for f, s in sorted(per_file.items(), key=lambda kv: -kv[1]):
    print(f"  {f:24} {s / tot * 100:5.1f}%")
print(f"{'file:line':28} {'samp%':>6} {'wait':>5} {'math':>5} {'ssb':>5} {'bar':>5} {'nsel':>5} {'sel':>5} {'br':>5}  source")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    f, ln, src = key
    g = lambda k: a.get(k, 0) / tot * 100  # noqa: E731
    print(f"{f + ':' + str(ln):28} {a['samples'] / tot * 100:6.2f} {g('stall_wait'):5.1f} {g('stall_math'):5.1f} "
          f"{g('stall_short_sb'):5.1f} {g('stall_barrier'):5.1f} {g('stall_not_selected'):5.1f} {g('stall_selected'):5.1f} "
          f"{g('stall_branch_resolving'):5.1f}  {src}")
