"""SASS opcode histogram of the hot kernels of libgacq.so (whole function and, for K2, the
round loop between the mbarrier wait's enclosing back-edge): evidence that the packed FP32x2
pipe, UBLKCP/SYNCS (bulk copy + mbarrier) and no local-memory spills are what runs.
    python tools/sass_histogram.py [lib] > profiles/<tag>_sass_histogram.md"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_1309_0052_b200" / "libgacq.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
WANT = ("gacq_corr_pfa_kernelILb1", "gacq_fwd_pfa_kernelILi4ELi4", "gacq_gen_corr_kernelILi2", "gacq_gen_fwd_kernelILi2")
KEYS = ("FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL",
        "UBLKCP", "SYNCS", "LDGSTS", "BAR", "UCGABAR_ARV", "UCGABAR_WAIT", "FMNMX", "IMAD", "IADD3", "ISETP")


def ops(lines):
    c = Counter()
    for ln in lines:
        m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", ln)
        if m:
            c[m.group(2)] += 1
    return c


print("# SASS opcode histograms (cuobjdump -sass of the shipped libgacq.so, sm_100a)\n")
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0].strip()
    if not any(w in name for w in WANT):
        continue
    lines = [ln for ln in f.split("\n") if re.match(r"^\s+/\*[0-9a-f]{4,}\*/", ln)]
    whole = ops(lines)
    print(f"## `{name}`\n")
    print(f"{len(lines)} instructions. Selected opcodes (whole function):\n")
    print("| " + " | ".join(KEYS) + " |")
    print("|" + "---|" * len(KEYS))
    print("| " + " | ".join(str(whole.get(k, 0)) for k in KEYS) + " |\n")
    if "corr_pfa" in name:
        # the round loop: from the mbarrier try-wait back to the loop's backward branch
        addr = [int(re.match(r"^\s+/\*([0-9a-f]+)\*/", ln).group(1), 16) for ln in lines]
        wait = next(i for i, ln in enumerate(lines) if "SYNCS.PHASECHK" in ln)
        back = None
        for i, ln in enumerate(lines):
            m = re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", ln)
            if m and i > wait and int(m.group(1), 16) <= addr[wait] and (back is None or i < back):
                back = i
        tgt = int(re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", lines[back]).group(1), 16)
        start = addr.index(tgt) if tgt in addr else wait
        loop = ops(lines[start:back + 1])
        fma = 2 * (loop["FFMA2"] + loop["FADD2"] + loop["FMUL2"]) + loop["FFMA"] + loop["FADD"] + loop["FMUL"]
        print(f"Round loop (one 1023-point inverse transform per iteration): {back + 1 - start} instructions, "
              f"{fma} FMA-pipe cycles (2 per packed op):\n")
        print("| " + " | ".join(KEYS) + " |")
        print("|" + "---|" * len(KEYS))
        print("| " + " | ".join(str(loop.get(k, 0)) for k in KEYS) + " |\n")
