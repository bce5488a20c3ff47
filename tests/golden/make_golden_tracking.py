"""Tracking golden fixtures from the REFERENCE (gnssperf.tracking) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_tracking.py

Scenarios follow gnssperf's own tests (test_tracking.py: make_scenario / aligned_state,
PULL_IN_CONFIG, _channel_set) plus an acquisition -> tracking chain on a C3 snapshot.
Writes tests/golden/tracking.json: per epoch the six correlators, both discriminators, the
lock metric and the NCO state after the epoch.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

from gnssperf.acquisition import AcqConfig, acquire_all
from gnssperf.buffers import IqBuffer
from gnssperf.cacode import CHIP_RATE_HZ, CODE_LENGTH
from gnssperf.gnss_signal import L1_CARRIER_HZ, SignalSpec, synthesize_signal
from gnssperf.tracking import TrackConfig, TrackState, init_from_acquisition, track_epoch

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import ref_snapshot  # noqa: E402

OUT = Path(__file__).resolve().parent / "tracking.json"


def cfg_dict(c: TrackConfig) -> dict:
    return dict(correlator_spacing_chips=c.correlator_spacing_chips, dll_bandwidth_hz=c.dll_bandwidth_hz,
                pll_bandwidth_hz=c.pll_bandwidth_hz, integration_ms=c.integration_ms)


def state_dict(s: TrackState) -> dict:
    return dict(prn=s.prn, code_phase_chips=s.code_phase_chips, carrier_phase_cycles=s.carrier_phase_cycles,
                doppler_hz=s.doppler_hz, code_rate_hz=s.code_rate_hz, dll_filter_state=list(s.dll_filter_state),
                pll_filter_state=list(s.pll_filter_state), epoch=s.epoch, sample_rate_hz=s.sample_rate_hz,
                lock_nbd=s.lock_nbd, lock_nbp=s.lock_nbp)


def run(blocks, state, config):
    epochs = []
    for b in blocks:
        state, out = track_epoch(b, state, config)
        epochs.append(dict(ie=out.ie, qe=out.qe, ip=out.ip, qp=out.qp, il=out.il, ql=out.ql,
                           dll_error_chips=out.dll_error_chips, pll_error_cycles=out.pll_error_cycles,
                           lock_metric=out.lock_metric, state=state_dict(state)))
    return epochs


def scenario(name, prn, doppler, delay, fs, epochs, config, code_err=0.0, doppler_err=0.0, sigma=0.0, seed=3):
    n = round(fs * 1e-3)
    spec = dict(prn=prn, doppler_hz=doppler, code_phase_samples=delay, carrier_phase_cycles=0.0, fs=fs,
                duration_s=epochs * 1e-3, noise_sigma=sigma, seed=seed)
    buf = synthesize_signal(SignalSpec(prn=prn, doppler_hz=doppler, code_phase_samples=delay, sample_rate_hz=fs,
                                       duration_s=epochs * 1e-3, noise_sigma=sigma, seed=seed))
    blocks = [IqBuffer._wrap(buf.samples[k * n:(k + 1) * n], fs, buf.precision) for k in range(epochs)]
    phase0 = (-delay * (CHIP_RATE_HZ / fs)) % CODE_LENGTH
    d0 = doppler - doppler_err
    state = TrackState(prn=prn, code_phase_chips=(phase0 - code_err) % CODE_LENGTH, carrier_phase_cycles=0.0,
                       doppler_hz=d0, code_rate_hz=CHIP_RATE_HZ * (1.0 + d0 / L1_CARRIER_HZ), sample_rate_hz=fs)
    return dict(name=name, kind="synth", spec=spec, epochs=epochs, config=cfg_dict(config),
                channels=[dict(init=state_dict(state), epochs=run(blocks, state, config))])


def main():
    cases = []
    cases.append(scenario("locked_8184k", 5, 800.0, 3000.0, 8.184e6, 10, TrackConfig()))
    pull = TrackConfig(correlator_spacing_chips=0.5, dll_bandwidth_hz=240.0, pll_bandwidth_hz=240.0,
                       integration_ms=1)
    cases.append(scenario("pullin_8192k", 5, 1200.0, 2000.0, 8.192e6, 50, pull, code_err=0.5, doppler_err=200.0))
    for prn in (2, 9, 17, 30):  # test_tracking.py _channel_set
        cases.append(scenario(f"chset_prn{prn}", prn, 300.0 * prn % 2000, 37 * prn, 8.184e6, 8, TrackConfig(),
                              code_err=0.05))
    cases.append(scenario("noisy45_4092k", 12, -2100.0, 1234.0, 4.092e6, 20, TrackConfig(),
                          sigma=float(np.sqrt(4.092e6 / (2.0 * 10.0 ** 4.5))), seed=11))
    # acquisition -> tracking chain on a C3 snapshot (the receiver's next step)
    fs = 4.092e6
    buf, truth = ref_snapshot(0, fs, 10e-3, base_seed=300)
    cfg = AcqConfig(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0, noncoherent_rounds=10)
    acq = acquire_all(buf, list(range(1, 33)), cfg)
    n = round(fs * 1e-3)
    blocks = [IqBuffer._wrap(buf.samples[k * n:(k + 1) * n], fs, buf.precision) for k in range(10)]
    chans = []
    for r in acq:
        if not r.detected:
            continue
        st = init_from_acquisition(r, fs)
        chans.append(dict(acq=dict(prn=r.prn, doppler_hz=r.doppler_hz, code_phase_samples=r.code_phase_samples),
                          init=state_dict(st), epochs=run(blocks, st, TrackConfig())))
    cases.append(dict(name="chain_c3_snap0", kind="snapshot",
                      spec=dict(index=0, fs=fs, duration_s=10e-3, base_seed=300), epochs=10,
                      config=cfg_dict(TrackConfig()), channels=chans))
    OUT.write_text(json.dumps(dict(generator="tests/golden/make_golden_tracking.py", cases=cases), indent=1))
    print("wrote", len(cases), "tracking cases,", sum(len(c["channels"]) for c in cases), "channels")


if __name__ == "__main__":
    sys.exit(main())
