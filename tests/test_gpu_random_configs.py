"""Randomised parity (seeded): the GPU path against the pinned oracle over configurations the
fixed goldens do not enumerate -- every chip-aligned D the prime-factor path instantiates, and
generic rates on both transform forms (native mixed radix, linear power of two) -- with random
Doppler grids (asymmetric, off-centre), coherent_ms 1-3, 1-4 noncoherent rounds, exclusion
radii on both K2 floor forms, thresholds, and PRN subsets in random order. Exact agreement is
required: (bin, lag) and `detected` equal, peak metric within 1e-4; no tie exemption (these
noisy inputs hold no float32-indistinguishable top cells, and a tie would fail loudly)."""

import numpy as np
import pytest

import oracle
from parity import compare

pytestmark = pytest.mark.gpu

# (fs, which path): D = 1, 2, 4, 5, 6, 8, 13, 14, 16 (prime-factor K1/K2 variants) and
# generic rates: 2.5 / 3 / 6 MHz (native 2^a 3^b 5^c), 7 MHz x 1 ms (7000 = 2^3 5^3 7: linear)
RATES = [1.023e6 * d for d in (1, 2, 4, 5, 6, 8, 13, 14, 16)] + [2.5e6, 3.0e6, 6.0e6, 7.0e6]
N_CASES = 52  # four per rate


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


def draw(i):
    rng = np.random.default_rng(20260 + i)
    fs = RATES[i % len(RATES)]
    big = fs > 9e6
    coh = int(rng.integers(1, 2 if big else 4))
    rounds = int(rng.integers(1, 3 if big else 5))
    step = float(rng.choice([250.0, 333.0, 500.0, 750.0]))
    lo = -float(rng.integers(2, 9)) * step
    hi = float(rng.integers(1, 9)) * step + float(rng.uniform(0, step))
    d_chip = fs / 1.023e6
    radius = int(rng.choice([0, 1, int(np.ceil(d_chip)), int(8 * d_chip), int(40 * d_chip)]))
    thr = float(rng.choice([1.8, 2.5, 3.0]))
    prns = [int(p) for p in rng.permutation(np.arange(1, 33))[:int(rng.integers(3, 9))]]
    kw = dict(doppler_min_hz=lo, doppler_max_hz=hi, doppler_step_hz=step, coherent_ms=coh,
              noncoherent_rounds=rounds, detection_threshold=thr, exclusion_radius_samples=radius)
    return fs, kw, prns, 777 + i


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_config_matches_oracle(pkg, i):
    fs, kw, prns, seed = draw(i)
    ocfg = oracle.OracleConfig(**kw)
    x, _ = oracle.make_snapshot(0, fs, kw["coherent_ms"] * kw["noncoherent_rounds"] * 1e-3, base_seed=seed,
                                doppler_span_hz=min(4750.0, max(abs(kw["doppler_min_hz"]), kw["doppler_max_hz"])))
    eng = pkg.AcqEngine(fs, prns, pkg.AcqConfig(**kw))
    got = eng.search(x).results()[0]
    bins = ocfg.doppler_bins_hz()
    for g, prn in zip(got, prns):
        r = oracle.acquire_channel(x, fs, prn, ocfg)
        assert g.prn == prn and g.bins_searched == bins.size
        gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples, peak_metric=g.peak_metric,
                  detected=g.detected)
        v = compare(gd, r, kw["detection_threshold"])
        if v != "exact":
            pm = oracle.acquire_channel(x, fs, prn, ocfg, want_map=True)["power_map"]
            v = compare(gd, r, kw["detection_threshold"], pm, bins)
        assert v == "exact", (fs, kw, prn, v, eng.info)
    eng.close()


@pytest.mark.parametrize("i", range(10))
def test_random_batches_chunks_and_prn_sets(pkg, i):
    # random batch sizes, PRN subsets (any order and count), strides and small spectrum scratch
    # (many chunks, partial 4-pair groups in K2, short first chunk): every batch row equals the
    # same snapshot searched alone, and the first snapshot equals the oracle
    rng = np.random.default_rng(3300 + i)
    fs = [4.092e6, 8.184e6, 5.0e6, 2.046e6, 6.0e6][i % 5]
    kw = dict(doppler_min_hz=-1500.0, doppler_max_hz=1500.0, doppler_step_hz=500.0,
              noncoherent_rounds=int(rng.integers(1, 3)))
    prns = [int(p) for p in rng.permutation(np.arange(1, 33))[:int(rng.integers(1, 33))]]
    n_snap = int(rng.integers(1, 14))
    span = round(fs * 1e-3) * kw["noncoherent_rounds"]
    pad = int(rng.integers(0, 9))
    xs = np.zeros((n_snap, span + pad), dtype=np.complex64)
    for s in range(n_snap):
        xs[s, :span] = oracle.make_snapshot(s, fs, span / fs, base_seed=6100 + i)[0]
    scratch = int(rng.integers(1, 6)) << 20  # 1-5 MiB: a few pairs per chunk
    eng = pkg.AcqEngine(fs, prns, pkg.AcqConfig(**kw), scratch_bytes=scratch)
    rows = eng.run_rows(xs)
    one = pkg.AcqEngine(fs, prns, pkg.AcqConfig(**kw))
    for s in range(n_snap):
        np.testing.assert_array_equal(rows[s], one.run_rows(np.ascontiguousarray(xs[s:s + 1, :span]))[0])
    ocfg = oracle.OracleConfig(**kw)
    bins = ocfg.doppler_bins_hz()
    for g, prn in zip(eng.search(xs[:1]).results()[0], prns):
        r = oracle.acquire_channel(xs[0, :span], fs, prn, ocfg)
        gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples, peak_metric=g.peak_metric,
                  detected=g.detected)
        v = compare(gd, r, ocfg.detection_threshold)
        if v != "exact":
            v = compare(gd, r, ocfg.detection_threshold,
                        oracle.acquire_channel(xs[0, :span], fs, prn, ocfg, want_map=True)["power_map"], bins)
        assert v == "exact", (fs, prn, v)
    eng.close()
    one.close()
