#!/usr/bin/env python
"""Benchmark: PRN x Doppler acquisition cells/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config c3] [--impl ours|reference]

A *cell* is one (snapshot, PRN, Doppler bin) searched over all code phases and all
noncoherent rounds. One *step* is one full search of the per-GPU
batch of synthetic snapshots. Snapshots are sharded across ranks (one process per GPU,
weak scaling: the per-GPU batch is fixed) with no data-path collective; the step time
is the device timeline of the library's own stream (CUDA events recorded by libgacq
around each whole gacq_run), max over ranks.

`value`  : batch resident in HBM before the timed region.
`e2e`    : the public API (AcqEngine.search) on a pinned host batch: H2D of the step's
           snapshots + search + D2H of the result rows + host metric, wall-clocked.
`--impl reference` times the CPU path (the pinned oracle restatement of the reference,
oracle/, scipy.fft) on the host cores with one process per core, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
UNIT = "cells/s"

# BASELINE.json configs; c3 is the one the metric is quoted on
CONFIGS = {
    "c1": dict(fs=4.092e6, rounds=1, step=500.0, span_hz=5000.0, batch=1024,
               desc="C1: 1 ms snapshots @4.092 MHz, 32 PRNs x 21 bins (+-5 kHz/500 Hz), 1 x 1 ms"),
    "c2": dict(fs=4.092e6, rounds=10, step=250.0, span_hz=5000.0, batch=512,
               desc="C2: 10 ms snapshots @4.092 MHz, 32 PRNs x 41 bins (+-5 kHz/250 Hz), 10 x 1 ms noncoherent"),
    "c3": dict(fs=4.092e6, rounds=10, step=500.0, span_hz=5000.0, batch=1024,
               desc="C3: 10 ms snapshots @4.092 MHz, 32 PRNs x 21 bins (+-5 kHz/500 Hz), 10 x 1 ms noncoherent"),
    "d8": dict(fs=8.184e6, rounds=10, step=2.0 / 3.0 / 1e-3, span_hz=5000.0, batch=512,
               desc="D8: the reference's default acquisition (8.184 MHz, AcqConfig(): 16 bins of 666.7 Hz, "
                    "10 x 1 ms noncoherent), 32 PRNs"),
    "g5": dict(fs=5.0e6, rounds=10, step=500.0, span_hz=5000.0, batch=64,
               desc="G5: 10 ms snapshots @5 MHz (not chip-aligned: generic power-of-two path), 32 PRNs x 21 bins, "
                    "10 x 1 ms noncoherent"),
    "g8": dict(fs=8.192e6, rounds=10, step=500.0, span_hz=5000.0, batch=64,
               desc="G8: 10 ms snapshots @8.192 MHz (not chip-aligned; n_coh = 8192 runs as the circular "
                    "8192-point transform), 32 PRNs x 21 bins, 10 x 1 ms noncoherent"),
    "c4": dict(fs=16.368e6, rounds=20, step=125.0, span_hz=10000.0, batch=16,
               desc="C4: 20 ms snapshots @16.368 MHz, 32 PRNs x 161 bins (+-10 kHz/125 Hz), 20 x 1 ms noncoherent"),
}


# dominant (K2) kernel of each device path, gacq_info.path
KERNEL_NAMES = {2: "gacq_corr_pfa_kernel (1023-point prime-factor)",
                4: "gacq_gen_corr_kernel (generic power-of-two path)"}


def acq_kwargs(c):
    return dict(doppler_min_hz=-c["span_hz"], doppler_max_hz=c["span_hz"], doppler_step_hz=c["step"],
                noncoherent_rounds=c["rounds"])


def flops_per_cell(c, n_bins):
    """SURVEY.md 8(d) algorithmic FLOPs at the reference's native N (implementation-independent)."""
    n = round(c["fs"] * 1e-3)
    p = n
    corr = c["rounds"] * (6 * n + 5 * n * math.log2(n) + 3 * p + p)
    fwd = c["rounds"] * (6 * n + 5 * n * math.log2(n)) / 32
    return corr, fwd


def bytes_per_cell(c, n_bins):
    n = round(c["fs"] * 1e-3)
    return 8 * n * c["rounds"] / (32 * n_bins) + 16 / n_bins


# ------------------------------------------------------------------ CPU (oracle) legs
def _cpu_worker_init():
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, str(ROOT))


def _cpu_warm(cname):
    import oracle

    c = CONFIGS[cname]
    x, _ = oracle.make_snapshot(0, c["fs"], c["rounds"] * 1e-3, base_seed=1)
    oracle.acquire_all(x[: round(c["fs"] * 1e-3) * 1], c["fs"], range(1, 33),
                       oracle.OracleConfig(**{**acq_kwargs(c), "noncoherent_rounds": 1}))
    return os.getpid()


def _cpu_one(arg):
    import oracle

    cname, x = arg
    c = CONFIGS[cname]
    return len(oracle.acquire_all(x, c["fs"], range(1, 33), oracle.OracleConfig(**acq_kwargs(c))))


def cpu_measure(cname, workers, steps, warmup, per_worker=1):
    """Oracle (restatement of acquisition.py:112-170 on scipy.fft) on `workers` processes,
    one snapshot per worker per step; returns (cells/s per step list, sample description)."""
    import oracle

    c = CONFIGS[cname]
    n_bins = oracle.OracleConfig(**acq_kwargs(c)).doppler_bins_hz().size
    n = workers * per_worker
    snaps = [oracle.make_snapshot(i, c["fs"], c["rounds"] * 1e-3, base_seed=900)[0] for i in range(n)]
    ctx = mp.get_context("spawn")
    rates = []
    with ctx.Pool(workers, initializer=_cpu_worker_init) as pool:
        pool.map(_cpu_warm, [cname] * workers, chunksize=1)
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_cpu_one, [(cname, s) for s in snaps], chunksize=1)
            dt = time.perf_counter() - t0
            if it >= warmup:
                rates.append(n * 32 * n_bins / dt)
    sample = (f"{n} {cname.upper()} snapshots x 32 PRNs x {n_bins} bins per step, {workers} processes "
              f"(oracle/ restatement of acquisition.py:112-170, scipy {__import__('scipy').__version__} fft)")
    return rates, sample


# ------------------------------------------------------------------ GPU helpers
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def synth_batch(torch, n, c, seed, device):
    """Synthetic GPS snapshots generated in HBM by libgacq (gacq_synth):
    8 visible satellites per snapshot (distinct PRNs, Doppler U(-span+250, span-250), integer
    code phase, carrier phase, C/N0 U(38,48) dB-Hz) + AWGN at the 45 dB-Hz reference level.
    Perf input only (parity uses the oracle's synthesis of the reference's PCG64 stream)."""
    import paper_1309_0052_b200 as g

    fs = c["fs"]
    span = round(fs * 1e-3) * c["rounds"]
    sats = g.random_sats(np.random.default_rng(seed), n, fs, doppler_span_hz=c["span_hz"] - 250.0)
    out = torch.empty((n, span), dtype=torch.complex64, device=device)
    sigma = math.sqrt(fs / (2.0 * 10.0 ** (45.0 / 10.0)))
    return g.synthesize_batch(sats, fs, span, out, noise_sigma=sigma, seed=seed,
                              device=device.index if device.index is not None else 0)


# ------------------------------------------------------------------ arms
def _cpu_track(arg):
    """Oracle tracking (restated tracking.py:226-275) of a few channels of one snapshot."""
    import oracle
    from oracle import tracking_oracle as to

    cname, x, prns, epochs = arg
    c = CONFIGS[cname]
    n = round(c["fs"] * 1e-3)
    cfg = to.TrackConfig()
    states = [to.init_from_acquisition(p, 0.0, 0, c["fs"]) for p in prns]
    for k in range(epochs):
        states = [to.track_epoch(x[k * n:(k + 1) * n], s, cfg)[0] for s in states]
    return len(states) * epochs


def measure_tracking(torch, dev, c, epochs, cpu, dist):
    """every PRN of every snapshot in the batch tracked for `epochs`
    1 ms epochs (one device launch for all channels per epoch + vectorised loop closure),
    bit-exact with the reference's tracking (tests/test_gpu_tracking.py)."""
    from paper_1309_0052_b200 import tracking as trk
    from paper_1309_0052_b200.sharding import max_over_ranks

    n_snap, span = dev.shape
    n = round(c["fs"] * 1e-3)
    epochs = max(1, min(epochs, span // n))
    rng = np.random.default_rng(7)
    prns = np.tile(np.arange(1, 33), n_snap)
    states = [trk.TrackState(prn=int(p), code_phase_chips=float(rng.uniform(0, 1023)), carrier_phase_cycles=0.0,
                             doppler_hz=float(d), code_rate_hz=1.023e6 * (1.0 + float(d) / 1575.42e6),
                             sample_rate_hz=c["fs"]) for p, d in zip(prns, rng.uniform(-4750, 4750, prns.size))]
    base = np.repeat(np.arange(n_snap, dtype=np.int64) * span, 32)
    cfg = trk.TrackConfig()
    batch0 = trk.TrackBatch.from_states(states)
    trk.track_step(dev, base, batch0, cfg)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = batch0
    for k in range(epochs):
        batch, outs = trk.track_step(dev, base + k * n, batch, cfg)
    wall = max_over_ranks(time.perf_counter() - t0, dist, "cuda")
    ws = dist.get_world_size() if dist else 1
    res = {"metric": "tracking channel-epochs/s", "value": ws * prns.size * epochs / wall,
           "unit": "channel-epochs/s", "channels_per_gpu": int(prns.size), "epochs": epochs,
           "note": "one gacq_trk_epl launch (all channels) + gacq_trk_chans/gacq_trk_close (multithreaded "
                   "C++ float64 loop closure, bit-exact) per epoch; device-resident samples; wall-clocked"}
    if cpu:
        import oracle

        x = oracle.make_snapshot(0, c["fs"], c["rounds"] * 1e-3, base_seed=900)[0]
        t0 = time.perf_counter()
        m = _cpu_track((next(k for k, v in CONFIGS.items() if v is c), x, list(range(1, 9)), min(4, epochs)))
        res["cpu_baseline"] = {"value": m / (time.perf_counter() - t0), "unit": "channel-epochs/s", "cores": 1,
                               "kind": "port", "sample": f"{m} channel-epochs, oracle/tracking_oracle.py"}
    return res


def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    rates, sample = cpu_measure(args.config, cores, args.steps, args.warmup)
    v = statistics.mean(rates)
    c = CONFIGS[args.config]
    n_bins = len(np.arange(-c["span_hz"], c["span_hz"] + 1e-9, c["step"]))
    ms = cores * 32 * n_bins / v * 1e3  # one step = one snapshot per process
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (oracle.make_snapshot)",
            "impl": "reference",
            "config": {"workload": c["desc"], "parallelism": f"{cores} CPU processes"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    c = CONFIGS[args.config]
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = max(1, min(os.cpu_count() or 1, 16))
        rates, sample = cpu_measure(args.config, workers, 1, 0)
        cpu_baseline = {"value": rates[0], "unit": UNIT, "cores": workers, "kind": "port", "sample": sample}

    torch.cuda.set_device(local_rank)
    if world > 1:  # share the host cores between the ranks of this node (libgacq's OpenMP loops)
        try:
            import ctypes

            per_rank = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", world)))
            ctypes.CDLL("libgomp.so.1").omp_set_num_threads(per_rank)
        except OSError:
            pass
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1309_0052_b200 as g
    from paper_1309_0052_b200.sharding import max_over_ranks

    cfg = g.AcqConfig(**acq_kwargs(c))
    n_bins = cfg.doppler_bins_hz().size
    batch = args.batch or c["batch"]
    eng = g.AcqEngine(c["fs"], list(range(1, 33)), cfg, device=local_rank, scratch_bytes=args.scratch_mb << 20)
    dev = synth_batch(torch, batch, c, seed=1000 + rank, device=torch.device("cuda", local_rank))
    pinned = g.PinnedBuffer(tuple(dev.shape))
    pinned.array[...] = dev.cpu().numpy()
    torch.cuda.synchronize()
    in_bytes = dev.numel() * 8

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        eng.run_rows(dev)
    barrier()
    props = torch.cuda.get_device_properties(local_rank)
    gpu_id = getattr(props, "pci_bus_id", None) or str(local_rank)
    if isinstance(gpu_id, int):
        gpu_id = str(local_rank)
    eng.reset_stats()
    t_wall = time.perf_counter()
    with ClockSampler(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[local_rank]
                      if os.environ.get("CUDA_VISIBLE_DEVICES") else str(local_rank)) as clk:
        for _ in range(args.steps):
            rows = eng.run_rows(dev, profile=True)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    barrier()
    st = eng.stats()
    dev_ms = st["run_ms"]
    if dist:
        t = torch.tensor([dev_ms, t_wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, t_wall_max = float(t[0]), float(t[1])
    else:
        t_wall_max = t_wall
    cells_step = batch * 32 * n_bins
    value = world * cells_step * args.steps / (dev_ms / 1e3)

    # e2e through the public API from pinned host memory
    eng.search(pinned.array)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = eng.search(pinned.array)
        _ = int(res.detected.sum())
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e_value = world * cells_step * args.steps / e2e_s

    # e2e of the IF-ingest path: the same batch as int8 I/Q (the
    # GNSSIF01 payload, quantised against its full scale) in pinned host memory, searched
    # with AcqEngine.search_quantized -- 2 bytes per sample over PCIe instead of 8
    flat = torch.view_as_real(dev).reshape(dev.shape[0], -1)
    scale = float(flat.abs().max())
    q8 = torch.clamp(torch.round(flat / scale * 127.0), -127, 127).to(torch.int8)
    pinned8 = g.PinnedBuffer(tuple(q8.shape), np.int8)
    pinned8.array[...] = q8.cpu().numpy()
    del flat, q8
    eng.search_quantized(pinned8.array, 0, scale)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res8 = eng.search_quantized(pinned8.array, 0, scale)
        _ = int(res8.detected.sum())
    e2e8_s = max_over_ranks(time.perf_counter() - t0, dist, "cuda")
    e2e_int8 = {"value": world * cells_step * args.steps / e2e8_s, "unit": UNIT,
                "h2d_bytes_per_step": pinned8.array.nbytes, "d2h_bytes_per_step": batch * 32 * 16,
                "api": "AcqEngine.search_quantized(pinned int8 I/Q, GNSSIF01 payload)"}
    pinned8.close()

    tracking = measure_tracking(torch, dev, c, args.steps if args.tracking_epochs <= 0 else args.tracking_epochs,
                                rank == 0 and world == 1 and not args.no_cpu_baseline, dist)

    f_corr, f_fwd = flops_per_cell(c, n_bins)
    sm = props.multi_processor_count
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    max_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = sm * 128 * 2 * max_mhz * 1e6 / 1e12
    corr_s = st["corr_ms"] / 1e3
    achieved = st["cells"] * f_corr / corr_s / 1e12 if corr_s > 0 else None
    traffic = None
    prof = ROOT / "profiles" / "corr_traffic.json"
    cells_per_launch = st["cells"] / max(1, st["corr_launches"])
    if prof.exists():
        pj = json.loads(prof.read_text())
        if pj.get("config") == args.config and pj.get("dram_bytes_per_cell"):
            traffic = pj["dram_bytes_per_cell"] * cells_per_launch
    hbm = float(peaks.get("hbm_gbs", 6547.8))
    step_cells_s = cells_step * args.steps / (dev_ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (8 satellites + AWGN per snapshot, generated in HBM by gacq_synth)",
        "config": {"workload": c["desc"], "snapshots_per_gpu": batch, "global_batch": batch * world,
                   "cells_per_step_per_gpu": cells_step, "fs_hz": c["fs"], "prns": 32, "bins": n_bins,
                   "parallelism": f"dp{world} (snapshot shards, no collective)",
                   "l2": f"inputs larger than L2 ({in_bytes / 2**20:.0f} MiB per GPU), no flush"},
        "roofline": {"bound": "fp32", "kernel": KERNEL_NAMES[eng.info["path"]], "achieved": achieved, "peak": fp32_peak,
                     "unit": "TFLOP/s", "frac": achieved / fp32_peak if achieved else None,
                     "traffic": traffic,
                     "peak_source": f"nominal FP32 {sm} SMs x 128 lanes x 2 x {max_mhz:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no FP32 entry)",
                     "flops_per_cell": f_corr,
                     "cells_per_launch": cells_per_launch,
                     "avg_launch_ms": st["corr_ms"] / max(1, st["corr_launches"]),
                     "step_frac": step_cells_s * (f_corr + f_fwd) / 1e12 / fp32_peak},
        "roofline_hbm": {"achieved": step_cells_s * bytes_per_cell(c, n_bins) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": step_cells_s * bytes_per_cell(c, n_bins) / 1e9 / hbm,
                         "note": "compulsory bytes/cell (SURVEY 8(d)); the path is FP32-bound"},
        "kernel_ms": {"fwd": st["fwd_ms"] / args.steps, "corr": st["corr_ms"] / args.steps,
                      "reduce": st["reduce_ms"] / args.steps},
        "cpu_baseline": cpu_baseline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": batch * 32 * 16, "api": "AcqEngine.search(pinned host batch)"},
        "e2e_int8": e2e_int8,
        "tracking": tracking,
        "gpu_launches": st["launches"],
        "wall_ms_per_step": t_wall_max * 1e3 / args.steps,
        "clocks": clk.summary(),
        "detected_per_snapshot": float(rows.shape[0] and eng.finish(rows).detected.sum() / rows.shape[0]),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    pinned.close()
    eng.close()
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="snapshots per GPU (default: config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tracking-epochs", type=int, default=10, help="tracking epochs measured (0: = --steps)")
    ap.add_argument("--scratch-mb", type=int, default=0, help="spectrum scratch (MiB, both halves); 0 = library default")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
