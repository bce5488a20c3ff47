#!/usr/bin/env python
"""Summarise an `ncu --set full` report of the gacq kernels into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep r01 --cells-per-launch 64*32*21
    python tools/ncu_summary.py --launches gpurun_out/launches_r01.csv r01

Writes profiles/<tag>_ncu_summary.md (key metrics per kernel) and, for the corr kernel,
profiles/corr_traffic.json (DRAM bytes per cell) which bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1TEX data-pipe wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.per_cycle_active", "active warps / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "CTA limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall: MIO throttle"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
]


def raw(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("tag")
    ap.add_argument("--cells-per-launch", default=None, help="cells processed by the profiled corr launch")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--launches", default=None, help="ncu --metrics gpu__time_duration.sum csv")
    args = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    if args.launches:
        text = Path(args.launches).read_text().splitlines()
        start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
        rows = list(csv.DictReader(text[start:]))
        rows = [r for r in rows if "gacq" in r["Kernel Name"]]
        tot = {}
        for r in rows:
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            t, n = tot.get(name, (0.0, 0))
            tot[name] = (t + float(r["Metric Value"]), n + 1)
        grand = sum(t for t, _ in tot.values())
        lines = [f"# {args.tag}: gacq launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
                 "| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
        for k, (t, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
            lines.append(f"| {k} | {n} | {t / 1e6:.3f} | {t / n / 1e6:.3f} | {t / grand:.1%} |")
        (prof / f"{args.tag}_launches.md").write_text("\n".join(lines) + "\n")
        with open(prof / f"{args.tag}_launches.csv", "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "grid", "block", "ns"])
            for r in rows:
                w.writerow([r["Kernel Name"].split("(")[0], r["Grid Size"], r["Block Size"], r["Metric Value"]])
        print("\n".join(lines))
        return
    hdr, units, rows = raw(args.report)
    ix = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {args.tag}: ncu --set full summary ({Path(args.report).name})", ""]
    for r in rows:
        name = r[ix["Kernel Name"]]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        vals = {}
        for m, label in METRICS:
            if m in ix:
                lines.append(f"| {label} (`{m}`) | {r[ix[m]]} | {units[ix[m]]} |")
                vals[m] = r[ix[m]]
        lines.append("")
        if "corr" in name and args.cells_per_launch:
            cells = eval(args.cells_per_launch, {}, {})  # noqa: S307 - developer tool, literal arithmetic

            def to_bytes(m):
                v = float(vals[m].replace(",", ""))
                u = units[ix[m]]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]

            traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            (prof / "corr_traffic.json").write_text(json.dumps({
                "source": f"profiles/{args.tag}_ncu_summary.md", "config": args.config,
                "cells_per_profiled_launch": cells, "dram_bytes_per_launch": traffic,
                "dram_bytes_per_cell": traffic / cells}, indent=1) + "\n")
            lines.append(f"DRAM traffic per cell: {traffic / cells:.1f} B "
                         f"({traffic:.3e} B over {cells} cells)")
            lines.append("")
    (prof / f"{args.tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
