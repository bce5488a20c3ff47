"""FMA-pipe cycles of the largest loop body of each kernel in a binary's SASS (2 per packed
FP32x2 op, 1 per scalar FP32 op).  python tools/sass_loop_count.py <binary>"""
import re
import subprocess
import sys

txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    rows = [(int(m.group(1), 16), m.group(2).strip()) for m in
            (re.match(r"^\s+/\*([0-9a-f]{4,})\*/\s+(.*?);?\s*(?:/\*.*)?$", ln) for ln in f.split("\n")) if m]
    addrs = [a for a, _ in rows]
    best = None
    for i, (a, ins) in enumerate(rows):
        m = re.search(r"BRA (?:.*?)0x([0-9a-f]+)", ins)
        if m:
            t = int(m.group(1), 16)
            if t < a and t in addrs:
                j = addrs.index(t)
                if best is None or i - j > best[1] - best[0]:
                    best = (j, i)
    body = rows[best[0]:best[1] + 1] if best else rows
    cyc, ops = 0, {}
    for _, ins in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", ins).split(" ")[0].split(".")[0]
        ops[op] = ops.get(op, 0) + 1
        cyc += 2 if op in ("FFMA2", "FADD2", "FMUL2") else 1 if op in ("FFMA", "FADD", "FMUL") else 0
    top = dict(sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print(f"{name[:50]} loop {len(body)} instrs, {cyc} FMA-pipe cycles {top}")
