"""K2 A/B timing: one process per libgacq variant (GACQ_LIB=exp/libgacq_<v>.so), device-resident
synthetic batch, CUDA-event kernel times from gacq_stats. Also checks the rows of every variant
against the first one (bit-identical argmax/lag; peaks within 1e-5).
    python tools/k2_ab.py [--config c3] [--batch 256] [--reps 5] v1 v2 ..."""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(args):
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    import bench
    import paper_1309_0052_b200 as g

    c = bench.CONFIGS[args.config]
    be = bench.CudaBackend(0)
    x = be.batch(c, args.batch, seed=1000)
    eng = be.engine(c, argparse.Namespace(scratch_mb=0))
    for _ in range(3):
        rows = eng.run_rows(x)
    torch.cuda.synchronize()
    res = []
    for _ in range(args.reps):
        eng.reset_stats()
        eng.run_rows(x, profile=True)
        st = eng.stats()
        res.append((st["corr_ms"], st["fwd_ms"], st["run_ms"]))
    corr = min(r[0] for r in res)
    f_corr, _ = bench.flops_per_cell(c)
    cells = args.batch * 32 * bench.n_bins_of(c)
    out = {"lib": os.environ.get("GACQ_LIB", "default"), "corr_ms": corr, "fwd_ms": min(r[1] for r in res),
           "run_ms": min(r[2] for r in res), "frac": cells * f_corr / (corr / 1e3) / 74.44992e12,
           "info": eng.info}
    np.save(args.rows_out, rows)
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--rows-out", default="")
    ap.add_argument("variants", nargs="*")
    args = ap.parse_args()
    if args.child:
        return child(args)
    import numpy as np

    base = None
    os.makedirs(ROOT / "gpurun_out", exist_ok=True)
    for v in args.variants or ["default"]:
        env = dict(os.environ)
        if v != "default":
            env["GACQ_LIB"] = str(ROOT / "exp" / f"libgacq_{v}.so")
        rows_out = f"/tmp/rows_{v}.npy"
        p = subprocess.run([sys.executable, __file__, "--child", "--config", args.config, "--batch", str(args.batch),
                            "--reps", str(args.reps), "--rows-out", rows_out], env=env, capture_output=True,
                           text=True, timeout=600)
        line = next((ln for ln in p.stdout.splitlines() if ln.startswith("{")), None)
        if line is None:
            print(v, "FAILED", p.stderr[-2000:], flush=True)
            continue
        d = json.loads(line)
        rows = np.load(rows_out)
        if base is None:
            base = rows
            d["rows"] = "reference"
        else:
            same = (rows["bin"] == base["bin"]) & (rows["lag"] == base["lag"])
            rel = np.abs(rows["peak"] - base["peak"]) / np.maximum(base["peak"], 1e-30)
            d["rows"] = f"{int(same.sum())}/{same.size} same cell, max peak rel {float(rel.max()):.2e}"
        d["variant"] = v
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    sys.exit(main())
