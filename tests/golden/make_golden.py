"""Generate golden fixtures by running the REFERENCE (gnssperf) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.json (case specs, SHA-256 of every reference input
buffer, reference AcqResult fields) and tests/golden/maps.npz (reference float32
power maps for a few small cases, recomputed with an instrumented copy of the
reference loop that calls the reference's own dsp/gnss_signal functions).
The fixtures are committed; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

from gnssperf import dsp
from gnssperf.acquisition import (AcqConfig, acquire_all, acquire_channel,
                                  conjugate_code_spectrum, samples_per_code_period)
from gnssperf.buffers import IqBuffer, Precision
from gnssperf.cacode import CHIP_RATE_HZ, generate_ca_code
from gnssperf.gnss_signal import (NcoState, SignalSpec, add_awgn, carrier_replica,
                                  synthesize_signal)
from gnssperf.harness import sigma_for_cn0_dbhz

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_snapshot(index, fs, duration_s, base_seed=0, n_visible=8, cn0_range=(38.0, 48.0),
                 cn0_ref=45.0, doppler_span_hz=4750.0):
    """Same recipe as oracle.make_snapshot, built from the reference's functions."""
    rng = np.random.default_rng(base_seed + index)
    period = samples_per_code_period(fs)
    prns = rng.choice(np.arange(1, 33), size=n_visible, replace=False)
    acc = np.zeros(round(fs * duration_s), dtype=np.complex64)
    truth = []
    for prn in prns:
        dop = float(rng.uniform(-doppler_span_hz, doppler_span_hz))
        cph = int(rng.integers(0, period))
        carr = float(rng.uniform(0.0, 1.0))
        cn0 = float(rng.uniform(cn0_range[0], cn0_range[1])) if cn0_range[1] > cn0_range[0] \
            else float(cn0_range[0])
        amp = np.float32(10.0 ** ((cn0 - cn0_ref) / 20.0))
        sig = synthesize_signal(SignalSpec(prn=int(prn), doppler_hz=dop, code_phase_samples=cph,
                                           carrier_phase_cycles=carr, sample_rate_hz=fs,
                                           duration_s=duration_s)).samples
        acc = (acc + sig * amp).astype(np.complex64)
        truth.append([int(prn), dop, cph, carr, cn0])
    buf = add_awgn(IqBuffer._wrap(acc, fs, Precision.SINGLE),
                   float(sigma_for_cn0_dbhz(cn0_ref, fs)), base_seed + index)
    return buf, truth


def noise_buffer(seed, n, fs):
    rng = np.random.Generator(np.random.PCG64(seed))
    z = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    return IqBuffer(z, fs)


def ref_power_map(buf, prn, cfg):
    """acquisition.py:128-149 re-run with the reference's own functions, keeping the map."""
    fs = buf.sample_rate_hz
    n_coh = round(fs * cfg.coherent_ms * 1e-3)
    period = samples_per_code_period(fs)
    bins = cfg.doppler_bins_hz()
    cs = conjugate_code_spectrum(prn, fs, n_coh, Precision.SINGLE)
    lag_span = min(period, n_coh)
    pm = np.zeros((bins.size, lag_span), dtype=np.float32)
    blocks = [IqBuffer._wrap(buf.samples[r * n_coh:(r + 1) * n_coh], fs, Precision.SINGLE)
              for r in range(cfg.noncoherent_rounds)]
    for bi, f in enumerate(bins):
        rep, _ = carrier_replica(NcoState(), float(f), fs, n_coh, Precision.SINGLE)
        for b in blocks:
            spec = dsp.fft(dsp.pointwise_multiply(b, rep))
            prod = dsp.pointwise_multiply(spec, dsp.Spectrum._wrap(cs, Precision.SINGLE))
            pm[bi] += dsp.magnitude_sq(dsp.ifft(prod, fs))[:lag_span]
    return pm


def cfg_dict(cfg: AcqConfig) -> dict:
    return dict(doppler_min_hz=cfg.doppler_min_hz, doppler_max_hz=cfg.doppler_max_hz,
                doppler_step_hz=cfg.doppler_step_hz, coherent_ms=cfg.coherent_ms,
                noncoherent_rounds=cfg.noncoherent_rounds,
                detection_threshold=cfg.detection_threshold,
                exclusion_radius_samples=cfg.exclusion_radius_samples)


def res_dict(r) -> dict:
    return dict(prn=r.prn, doppler_hz=r.doppler_hz, code_phase_samples=r.code_phase_samples,
                peak_metric=r.peak_metric, detected=r.detected, bins_searched=r.bins_searched,
                multiplications_performed=r.multiplications_performed)


C1 = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0,
               noncoherent_rounds=1)
C2 = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=250.0,
               noncoherent_rounds=10)
C3 = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0,
               noncoherent_rounds=10)
C4 = AcqConfig(doppler_min_hz=-10000.0, doppler_max_hz=10000.0, doppler_step_hz=125.0,
               noncoherent_rounds=20)
FS8 = 8.184e6


def main():
    if "--generic" in sys.argv:
        return main_generic()
    if "--extra" in sys.argv:
        return main_extra()
    t0 = time.time()
    cases = []
    maps = {}

    def add(name, kind, spec, buf, prns, cfg, keep_map=False):
        prns = [int(p) for p in prns]
        res = acquire_all(buf, prns, cfg)
        cases.append(dict(name=name, kind=kind, spec=spec, fs=buf.sample_rate_hz,
                          n_samples=len(buf), input_sha256=sha(buf.samples), prns=prns,
                          config=cfg_dict(cfg), results=[res_dict(r) for r in res]))
        if keep_map:
            for p in (prns if keep_map is True else keep_map):
                maps[f"{name}__prn{p}"] = ref_power_map(buf, p, cfg)
        print(f"{name}: {len(prns)} prns  ({time.time() - t0:.1f}s)", flush=True)

    def synth(prn, dop, phase, sigma=0.0, seed=7, ms=10.0, fs=FS8, carr=0.0):
        spec = dict(prn=prn, doppler_hz=dop, code_phase_samples=phase, carrier_phase_cycles=carr,
                    fs=fs, duration_s=ms * 1e-3, noise_sigma=float(sigma), seed=seed)
        buf = synthesize_signal(SignalSpec(prn=prn, doppler_hz=dop, code_phase_samples=phase,
                                           carrier_phase_cycles=carr, sample_rate_hz=fs,
                                           duration_s=ms * 1e-3, noise_sigma=float(sigma),
                                           seed=seed))
        return spec, buf

    dflt = AcqConfig()
    # test_acquisition.py known answers (53-66, 88-105, 108-120, 205-236)
    s, b = synth(5, 1500.0, 4000)
    add("ka_prn5_1500_4000", "synth", s, b, [5], dflt)
    s, b = synth(5, 0.0, 0)
    add("aligned_tie_0hz", "synth", s, b, [5], dflt)
    for truth in dflt.doppler_bins_hz()[::4]:
        s, b = synth(5, float(truth), 777)
        add(f"grid_{truth:+.1f}", "synth", s, b, [5], dflt)
    for i, truth in enumerate(np.random.default_rng(12345).uniform(-4500.0, 4500.0, 4)):
        s, b = synth(5, float(truth), 50)
        add(f"offgrid_{i}", "synth", s, b, [5], dflt)
    sig45 = float(sigma_for_cn0_dbhz(45.0, FS8))
    for seed in range(3):
        s, b = synth(9, -2200.0, 1234, sig45, seed)
        add(f"cn45_prn9_seed{seed}", "synth", s, b, [9, 10], dflt)
    for seed in range(3):
        nb = noise_buffer(seed, round(FS8 * 10e-3), FS8)
        add(f"noise_seed{seed}", "noise", dict(seed=seed, n=len(nb), fs=FS8), nb, [11], dflt)
    fs2 = 2.046e6
    s, b = synth(3, 0.0, 411, ms=1.0, fs=fs2)
    add("direct_small_2046k", "synth", s, b, [3],
        AcqConfig(doppler_min_hz=0.0, doppler_max_hz=0.0, noncoherent_rounds=1), keep_map=True)
    s, b = synth(8, 480.0, 333, ms=2.0, fs=fs2)
    add("direct_full_2046k", "synth", s, b, [8, 1, 17],
        AcqConfig(doppler_min_hz=-1000.0, doppler_max_hz=1000.0, doppler_step_hz=500.0,
                  noncoherent_rounds=2), keep_map=True)
    # zero input: peak 0, floor 0 -> metric inf, detected
    zb = IqBuffer(np.zeros(4092, dtype=np.complex64), 4.092e6)
    add("zeros_c1", "zeros", dict(n=4092, fs=4.092e6), zb, [1, 2], C1)
    # BASELINE configs on multi-satellite snapshots
    fs4 = 4.092e6
    all_prns = list(range(1, 33))
    for i in range(16):
        buf, truth = ref_snapshot(i, fs4, 1e-3, base_seed=100)
        add(f"c1_snap{i}", "snapshot", dict(index=i, fs=fs4, duration_s=1e-3, base_seed=100,
                                            truth=truth), buf, all_prns, C1,
            keep_map=([truth[0][0], truth[1][0], 1, 2] if i == 0 else False))
    buf, truth = ref_snapshot(0, fs4, 10e-3, base_seed=200)
    add("c2_snap0", "snapshot", dict(index=0, fs=fs4, duration_s=10e-3, base_seed=200,
                                     truth=truth), buf, all_prns, C2)
    for i in range(8):
        buf, truth = ref_snapshot(i, fs4, 10e-3, base_seed=300)
        add(f"c3_snap{i}", "snapshot", dict(index=i, fs=fs4, duration_s=10e-3, base_seed=300,
                                            truth=truth), buf, all_prns, C3)
    for cn0 in (30.0, 36.0, 42.0):
        buf, truth = ref_snapshot(0, fs4, 10e-3, base_seed=500 + int(cn0),
                                  cn0_range=(cn0, cn0))
        add(f"c5_cn{int(cn0)}", "snapshot",
            dict(index=0, fs=fs4, duration_s=10e-3, base_seed=500 + int(cn0),
                 cn0_range=[cn0, cn0], truth=truth), buf, all_prns, C3)
    # coherent_ms=2 (two code periods folded per block), custom exclusion radius/threshold
    buf, truth = ref_snapshot(0, fs4, 4e-3, base_seed=600)
    add("coh2_snap0", "snapshot", dict(index=0, fs=fs4, duration_s=4e-3, base_seed=600,
                                       truth=truth), buf, [truth[0][0], truth[1][0], 3, 4],
        AcqConfig(coherent_ms=2, noncoherent_rounds=2, doppler_step_hz=250.0))
    buf, truth = ref_snapshot(1, fs4, 2e-3, base_seed=600)
    add("radius10_snap1", "snapshot", dict(index=1, fs=fs4, duration_s=2e-3, base_seed=600,
                                           truth=truth), buf, all_prns,
        AcqConfig(doppler_step_hz=500.0, noncoherent_rounds=2, exclusion_radius_samples=10,
                  detection_threshold=1.8))
    # 8.184 MHz multi-sat (D=8)
    buf, truth = ref_snapshot(0, FS8, 2e-3, base_seed=700)
    add("fs8_snap0", "snapshot", dict(index=0, fs=FS8, duration_s=2e-3, base_seed=700,
                                      truth=truth), buf, all_prns,
        AcqConfig(doppler_step_hz=500.0, noncoherent_rounds=2))
    # C4 large-FFT config: 16.368 MHz, 20 x 1 ms, 161 bins; a few PRNs (reference ~1.5 s/PRN)
    fs16 = 16.368e6
    buf, truth = ref_snapshot(0, fs16, 20e-3, base_seed=800, doppler_span_hz=9750.0)
    add("c4_snap0", "snapshot", dict(index=0, fs=fs16, duration_s=20e-3, base_seed=800,
                                     doppler_span_hz=9750.0, truth=truth), buf,
        [t[0] for t in truth[:5]] + [p for p in all_prns if p not in [t[0] for t in truth]][:3],
        C4)
    # IF files (iffile.py): the reference writes a C3 snapshot as int8 / int16 / float32 and
    # acquires what read_if_file gives back (the cli.py:164-169 acquire path)
    import tempfile

    from gnssperf.iffile import read_if_file, write_if_file

    buf, truth = ref_snapshot(2, fs4, 10e-3, base_seed=300)
    for fmt in ("int8", "int16", "float32"):
        with tempfile.TemporaryDirectory() as td:
            path = Path(td) / f"snap.{fmt}.gnssif"
            write_if_file(path, buf, fmt)
            file_sha = hashlib.sha256(path.read_bytes()).hexdigest()
            back = read_if_file(path)
        add(f"if_{fmt}_c3", "iffile", dict(index=2, fs=fs4, duration_s=10e-3, base_seed=300, fmt=fmt,
                                          file_sha256=file_sha, truth=truth), back, all_prns, C3)

    (OUT / "golden.json").write_text(json.dumps(dict(
        generator="tests/golden/make_golden.py", reference="gnssperf 0.1.0 (/root/reference/pkg)",
        numpy=np.__version__, scipy=__import__("scipy").__version__,
        numba=__import__("gnssperf.kernels").kernels.NUMBA_ENABLED,
        cases=cases), indent=1))
    np.savez_compressed(OUT / "maps.npz", **maps)
    print("wrote", len(cases), "cases,", len(maps), "maps in", round(time.time() - t0, 1), "s")


def main_generic():
    """Sample rates that are not chip-aligned (fs != D * 1.023 MHz): the reference's native
    length is not a multiple of 1023, so the device runs its generic power-of-two path.
    Writes tests/golden/golden_generic.json and maps_generic.npz."""
    t0 = time.time()
    cases = []
    maps = {}

    def add(name, kind, spec, buf, prns, cfg, keep_map=False):
        prns = [int(p) for p in prns]
        res = acquire_all(buf, prns, cfg)
        cases.append(dict(name=name, kind=kind, spec=spec, fs=buf.sample_rate_hz,
                          n_samples=len(buf), input_sha256=sha(buf.samples), prns=prns,
                          config=cfg_dict(cfg), results=[res_dict(r) for r in res]))
        if keep_map:
            for p in keep_map:
                maps[f"{name}__prn{p}"] = ref_power_map(buf, p, cfg)
        print(f"{name}: {len(prns)} prns  ({time.time() - t0:.1f}s)", flush=True)

    all_prns = list(range(1, 33))
    g2 = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0,
                   noncoherent_rounds=2)
    for fs, tag in ((5.0e6, "5M"), (2.5e6, "2M5"), (8.192e6, "8M192"), (3.0e6, "3M")):
        for i in range(2):
            buf, truth = ref_snapshot(i, fs, 2e-3, base_seed=900)
            add(f"gen{tag}_snap{i}", "snapshot", dict(index=i, fs=fs, duration_s=2e-3, base_seed=900,
                                                     truth=truth), buf, all_prns, g2,
                keep_map=([truth[0][0], 5] if i == 0 and fs == 5.0e6 else False))
    # 2 ms coherent (n_coh = 2 P), 6 MHz; and a 10 ms C3-style search at 5 MHz
    buf, truth = ref_snapshot(0, 6.0e6, 4e-3, base_seed=910)
    add("gen6M_coh2", "snapshot", dict(index=0, fs=6.0e6, duration_s=4e-3, base_seed=910, truth=truth),
        buf, all_prns, AcqConfig(coherent_ms=2, noncoherent_rounds=2, doppler_step_hz=250.0),
        keep_map=[truth[0][0]])
    buf, truth = ref_snapshot(1, 5.0e6, 10e-3, base_seed=920)
    add("gen5M_c3", "snapshot", dict(index=1, fs=5.0e6, duration_s=10e-3, base_seed=920, truth=truth),
        buf, all_prns, C3)
    nb = noise_buffer(3, round(5.0e6 * 2e-3), 5.0e6)
    add("gen5M_noise", "noise", dict(seed=3, n=len(nb), fs=5.0e6), nb, [1, 7, 30], g2)
    s = dict(prn=12, doppler_hz=-1750.0, code_phase_samples=2345.0, carrier_phase_cycles=0.25,
             fs=5.0e6, duration_s=2e-3, noise_sigma=0.0, seed=0)
    b = synthesize_signal(SignalSpec(prn=12, doppler_hz=-1750.0, code_phase_samples=2345.0,
                                     carrier_phase_cycles=0.25, sample_rate_hz=5.0e6, duration_s=2e-3))
    add("gen5M_truth", "synth", s, b, [12, 13], g2)
    (OUT / "golden_generic.json").write_text(json.dumps(dict(
        generator="tests/golden/make_golden.py --generic", reference="gnssperf 0.1.0 (/root/reference/pkg)",
        numpy=np.__version__, scipy=__import__("scipy").__version__, cases=cases), indent=1))
    np.savez_compressed(OUT / "maps_generic.npz", **maps)
    print("wrote", len(cases), "generic cases,", len(maps), "maps in", round(time.time() - t0, 1), "s")


def _acq_one(args):
    """One reference channel in a worker process (acquire_all results are bit-identical to
    sequential per-channel calls for any plan, acquisition.py:196-197)."""
    kind, spec, prn, cfg_kw = args
    if kind == "snapshot":
        kw = {k: spec[k] for k in ("doppler_span_hz",) if k in spec}
        buf, _ = ref_snapshot(spec["index"], spec["fs"], spec["duration_s"], spec["base_seed"], **kw)
    else:
        raise ValueError(kind)
    return res_dict(acquire_channel(buf, generate_ca_code(prn), AcqConfig(**cfg_kw)))


def main_extra():
    """Round-2 parity cases (VERDICT r01 "Close the parity holes" and the large-transform
    rates): C4 with all 32 PRNs on 2 snapshots, C2 on 4 more snapshots, and rates whose
    transform exceeds 32768 points or whose chip oversampling D exceeds 16. Channels run in
    parallel worker processes. Writes tests/golden/golden_extra.json."""
    import multiprocessing as mp

    t0 = time.time()
    cases = []
    all_prns = list(range(1, 33))
    specs = []
    fs16 = 16.368e6
    for i in range(2):
        specs.append((f"c4x_snap{i}", dict(index=i, fs=fs16, duration_s=20e-3, base_seed=810,
                                           doppler_span_hz=9750.0), C4))
    fs4 = 4.092e6
    for i in range(1, 5):
        specs.append((f"c2_snap{i}", dict(index=i, fs=fs4, duration_s=10e-3, base_seed=200), C2))
    g2 = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0,
                   noncoherent_rounds=2)
    # generic rates beyond 32768 points (n_coh + P - 1 > 32768, n_coh not a power of two)
    specs.append(("gen20M_snap0", dict(index=0, fs=20.0e6, duration_s=2e-3, base_seed=930), g2))
    specs.append(("gen20M_snap1", dict(index=1, fs=20.0e6, duration_s=2e-3, base_seed=930), g2))
    specs.append(("gen16367k_coh2", dict(index=0, fs=16.367e6, duration_s=4e-3, base_seed=940),
                  AcqConfig(coherent_ms=2, noncoherent_rounds=2, doppler_step_hz=250.0,
                            doppler_min_hz=-2000.0, doppler_max_hz=2000.0)))
    specs.append(("gen8M192_coh5", dict(index=0, fs=8.192e6, duration_s=10e-3, base_seed=950),
                  AcqConfig(coherent_ms=5, noncoherent_rounds=2, doppler_step_hz=100.0,
                            doppler_min_hz=-1000.0, doppler_max_hz=1000.0)))
    # chip-aligned with D > 16 samples per chip
    specs.append(("d20_snap0", dict(index=0, fs=20.46e6, duration_s=2e-3, base_seed=960), g2))
    specs.append(("d32_snap0", dict(index=0, fs=32.736e6, duration_s=2e-3, base_seed=970), g2))
    only = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--only=")]
    if only:
        specs = [sp for sp in specs if sp[0] in only[0].split(",")]
    jobs = [("snapshot", spec, p, cfg_dict(cfg)) for _, spec, cfg in specs for p in all_prns]
    with mp.Pool(min(8, mp.cpu_count())) as pool:
        res = pool.map(_acq_one, jobs, chunksize=1)
    k = 0
    for name, spec, cfg in specs:
        kw = {x: spec[x] for x in ("doppler_span_hz",) if x in spec}
        buf, truth = ref_snapshot(spec["index"], spec["fs"], spec["duration_s"], spec["base_seed"], **kw)
        cases.append(dict(name=name, kind="snapshot", spec=dict(spec, truth=truth), fs=spec["fs"],
                          n_samples=len(buf), input_sha256=sha(buf.samples), prns=all_prns,
                          config=cfg_dict(cfg), results=res[k:k + len(all_prns)]))
        k += len(all_prns)
        print(f"{name}: 32 prns ({time.time() - t0:.1f}s)", flush=True)
    path = OUT / "golden_extra.json"
    if only and path.exists():
        old = [c for c in json.loads(path.read_text())["cases"] if c["name"] not in {c["name"] for c in cases}]
        cases = old + cases
    path.write_text(json.dumps(dict(
        generator="tests/golden/make_golden.py --extra", reference="gnssperf 0.1.0 (/root/reference/pkg)",
        numpy=np.__version__, scipy=__import__("scipy").__version__, cases=cases), indent=1))
    print("wrote", len(cases), "extra cases in", round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    sys.exit(main())
