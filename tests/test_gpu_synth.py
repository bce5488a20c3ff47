"""GPU: on-device synthetic batches. The clean signal is bit-identical
to the reference recipe (oracle.synthesize_signal summed in draw order); the Philox AWGN has
the right statistics (it is a performance input, never a parity input)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p, torch


@pytest.mark.parametrize("fs", [4.092e6, 5.0e6, 16.368e6])
def test_noise_free_batch_is_bit_identical_to_reference_recipe(env, fs):
    g, torch = env
    n = round(fs * 2e-3)
    sats = g.random_sats(np.random.default_rng(7), 3, fs)
    out = torch.empty((3, n), dtype=torch.complex64, device="cuda")
    g.synthesize_batch(sats, fs, n, out)
    got = out.cpu().numpy()
    for s in range(3):
        acc = np.zeros(n, dtype=np.complex64)
        for sat in sats[s]:
            sig = oracle.synthesize_signal(int(sat["prn"]), float(sat["doppler_hz"]), float(sat["code_phase_samples"]),
                                           float(sat["carrier_phase_cycles"]), fs, n / fs)
            acc = (acc + sig * np.float32(sat["amplitude"])).astype(np.complex64)
        bad = np.flatnonzero(got[s].view(np.uint64) != acc.view(np.uint64))
        assert bad.size == 0, (s, bad[:8])


def test_awgn_statistics_and_acquisition(env):
    g, torch = env
    fs, n, sigma = 4.092e6, 40920, 8.04
    sats = g.random_sats(np.random.default_rng(3), 16, fs)
    out = torch.empty((16, n), dtype=torch.complex64, device="cuda")
    g.synthesize_batch(sats[:, :0], fs, n, out, noise_sigma=sigma, seed=11)  # noise only
    z = out.cpu().numpy().ravel()
    assert abs(z.real.std() / sigma - 1) < 0.01 and abs(z.imag.std() / sigma - 1) < 0.01
    assert abs(np.mean(z.real * z.imag)) < 0.01 * sigma**2 and abs(z.mean()) < 0.01 * sigma
    g.synthesize_batch(sats, fs, n, out, noise_sigma=sigma, seed=11)
    cfg = g.AcqConfig(doppler_min_hz=-5000, doppler_max_hz=5000, doppler_step_hz=500, noncoherent_rounds=10)
    eng = g.AcqEngine(fs, list(range(1, 33)), cfg)
    res = eng.search(out)
    found = 0
    for s in range(16):
        for sat in sats[s]:
            p = int(sat["prn"]) - 1
            found += res.detected[s, p] and res.code_phase_samples[s, p] == int(sat["code_phase_samples"])
    assert found >= 0.9 * 16 * 8
    eng.close()
