"""GPU: the plan tables built on the device against the oracle --
carrier replicas bit for bit (kernels.py:106-114), C/A chips through the code spectra."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


@pytest.mark.parametrize("fs,dmin,dmax,step,coh", [
    (4.092e6, -5000.0, 5000.0, 500.0, 1),     # C1/C3 grid
    (4.092e6, -5000.0, 5000.0, 250.0, 1),     # C2 grid
    (8.184e6, -5000.0, 5000.0, 666.0, 2),     # reference test rate, 2 ms coherent
    (16.368e6, -10000.0, 10000.0, 125.0, 1),  # C4 grid: 161 bins x 16368 samples
    (2.046e6, -7000.0, 7000.0, 333.3, 1),
])
def test_device_carrier_table_is_bit_identical(pkg, fs, dmin, dmax, step, coh):
    cfg = pkg.AcqConfig(doppler_min_hz=dmin, doppler_max_hz=dmax, doppler_step_hz=step, coherent_ms=coh)
    eng = pkg.AcqEngine(fs, [1, 2], cfg)
    got = eng.carrier_table()
    n = eng.info["n_coh"]
    for b, f in enumerate(cfg.doppler_bins_hz()):
        ref = oracle.carrier_replica(0.0, float(f), fs, n)
        bad = np.flatnonzero(got[b].view(np.uint64) != ref.view(np.uint64))
        assert bad.size == 0, (float(f), bad[:8])
    eng.close()


def test_device_chips_and_spectra_give_reference_maps(pkg):
    # every PRN's conjugate spectrum (built from device LFSR chips) drives a noise-free
    # correlation whose peak sits at the truth lag; an impulse-free check of all 32 codes
    fs = 4.092e6
    cfg = pkg.AcqConfig(doppler_min_hz=-500.0, doppler_max_hz=500.0, doppler_step_hz=500.0, noncoherent_rounds=1)
    eng = pkg.AcqEngine(fs, list(range(1, 33)), cfg)
    for prn in range(1, 33):
        x = oracle.synthesize_signal(prn, 0.0, 1234.0, 0.0, fs, 1e-3)
        res = eng.search(x[None, :]).results()[0][prn - 1]
        assert res.code_phase_samples == 1234 and res.doppler_hz == 0.0 and res.detected, (prn, res)
    eng.close()
