"""GPU: the reference's acceptance criterion 4 (closed-loop acquisition,
/root/reference/pkg/tests/test_acceptance.py:82-123) run through the drop-in API on the
B200, with inputs regenerated bit-exactly by the oracle's restatement of synthesize_signal.
Same thresholds as the reference test, plus decision-for-decision agreement with the
oracle on a subset."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
FS = 8.184e6


@pytest.fixture(scope="module")
def g():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


def _acq(g, x, prn, cfg):
    return g.acquire_channel(g.IqBuffer(x, FS), g.generate_ca_code(prn), cfg)


def test_criterion_04_closed_loop_acquisition(g):
    cfg = g.AcqConfig()
    ocfg = oracle.OracleConfig()
    bins = cfg.doppler_bins_hz()
    case_rng = np.random.default_rng(40)
    exact_phase = within_half = detected = 0
    for seed in range(100):
        prn = int(case_rng.integers(1, 33))
        truth_doppler = float(case_rng.choice(bins))
        truth_phase = int(case_rng.integers(0, 8184))
        x = oracle.synthesize_signal(prn, truth_doppler, truth_phase, 0.0, FS, 10e-3, 0.0, seed)
        res = _acq(g, x, prn, cfg)
        detected += res.detected
        exact_phase += res.code_phase_samples == truth_phase
        within_half += abs(res.doppler_hz - truth_doppler) <= cfg.doppler_step_hz / 2 + 1e-9
    assert (detected, exact_phase, within_half) == (100, 100, 100)

    sigma = oracle.sigma_for_cn0_dbhz(45.0, FS)
    noisy_hits = agree = 0
    for seed in range(100):
        prn = 1 + seed % 32
        x = oracle.synthesize_signal(prn, -2400.0, 3210, 0.0, FS, 10e-3, sigma, 1000 + seed)
        res = _acq(g, x, prn, cfg)
        noisy_hits += res.detected
        if seed < 10:
            ref = oracle.acquire_channel(x, FS, prn, ocfg)
            agree += (res.detected, res.code_phase_samples, res.doppler_hz) == (
                ref["detected"], ref["code_phase_samples"], ref["doppler_hz"])
    assert noisy_hits >= 95 and agree == 10

    noise_rng = np.random.default_rng(77)
    false_alarms = agree = 0
    for seed in range(100):
        z = (noise_rng.standard_normal(81840) + 1j * noise_rng.standard_normal(81840)).astype(np.complex64)
        res = _acq(g, z, 13, cfg)
        false_alarms += res.detected
        if seed < 10:
            ref = oracle.acquire_channel(z, FS, 13, ocfg)
            agree += (res.detected, res.code_phase_samples, res.doppler_hz) == (
                ref["detected"], ref["code_phase_samples"], ref["doppler_hz"])
            assert res.peak_metric == pytest.approx(ref["peak_metric"], rel=1e-4)
    assert false_alarms <= 1 and agree == 10
