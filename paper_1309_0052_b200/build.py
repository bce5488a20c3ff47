"""Build libgacq.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

    python -m paper_1309_0052_b200.build [-v]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "libgacq.so"
SOURCES = [PKG / "csrc" / "gacq.cu"]
DEPS = SOURCES + [PKG / "csrc" / h for h in ("gacq_kernels.cuh", "gacq_pfa.cuh", "pfa.cuh", "pfa_tables.cuh",
                                             "codelets.cuh", "gtrk_kernels.cuh", "gacq_tables.cuh", "gacq_generic.cuh", "rader31.cuh", "gtrk_close.h")] + [ROOT / "include" / "gacq.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def flags(verbose: bool = False) -> list[str]:
    f = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "--shared", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off,-fopenmp", "-I", str(ROOT / "include"), "-lpthread", "-lgomp"]
    if verbose:
        f += ["-Xptxas", "-v"]
    return f


def up_to_date() -> bool:
    return LIB.exists() and all(LIB.stat().st_mtime >= d.stat().st_mtime for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *flags(verbose), "-o", str(tmp), *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
