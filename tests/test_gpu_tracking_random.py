"""Randomised tracking parity (seeded): the GPU drop-in `track_epoch` and the batched
`track_epoch_batch` against the oracle's restatement of tracking.py:226-275, bit for bit, on
random channels (PRN, code phase, Doppler, carrier phase, initial loop-filter states) at
chip-aligned and generic sample rates, random loop bandwidths / correlator spacing /
integration length, over several epochs of a noisy multi-satellite snapshot. The oracle is
pinned to the reference's own tracking goldens by tests/test_tracking_oracle.py."""

import numpy as np
import pytest

import oracle
from oracle import tracking_oracle as to

pytestmark = pytest.mark.gpu
RATES = [2.046e6, 4.092e6, 5.0e6, 8.184e6, 16.368e6, 3.0e6]
OUT_KEYS = ("ie", "qe", "ip", "qp", "il", "ql", "dll_error_chips", "pll_error_cycles", "lock_metric")
STATE_KEYS = ("code_phase_chips", "carrier_phase_cycles", "doppler_hz", "code_rate_hz", "dll_filter_state",
              "pll_filter_state", "epoch", "lock_nbd", "lock_nbp")


@pytest.fixture(scope="module")
def trk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    from paper_1309_0052_b200 import tracking

    return tracking


def draw(i):
    rng = np.random.default_rng(5150 + i)
    fs = RATES[i % len(RATES)]
    ms = int(rng.integers(1, 3))
    cfg = dict(correlator_spacing_chips=float(rng.choice([0.25, 0.5, 1.0])),
               dll_bandwidth_hz=float(rng.uniform(0.5, 5.0)), pll_bandwidth_hz=float(rng.uniform(5.0, 30.0)),
               integration_ms=ms)
    x, truth = oracle.make_snapshot(i, fs, 12 * ms * 1e-3, base_seed=9100)
    chans = []
    for prn, dop, code_samples, _carr, _cn0 in truth[:4]:
        dop_err = float(rng.uniform(-60.0, 60.0))
        st = to.init_from_acquisition(int(prn), float(dop) + dop_err, int(code_samples) + int(rng.integers(-1, 2)), fs)
        st = to.replace(st, carrier_phase_cycles=float(rng.uniform(0, 1)),
                        pll_filter_state=(float(rng.normal(0, 2)), float(rng.normal(0, 1))),
                        dll_filter_state=(float(rng.normal(0, 0.01)), 0.0))
        chans.append(st)
    chans.append(to.init_from_acquisition(int(rng.integers(1, 33)), float(rng.uniform(-4000, 4000)),
                                          int(rng.integers(0, round(fs * 1e-3))), fs))  # likely not visible
    return fs, cfg, x, chans


def to_gpu_state(trk, st):
    return trk.TrackState(**{f: getattr(st, f) for f in st.__dataclass_fields__})


@pytest.mark.parametrize("i", range(12))
def test_random_channels_bit_exact(trk, i):
    fs, cfg_kw, x, chans = draw(i)
    ocfg, gcfg = to.TrackConfig(**cfg_kw), trk.TrackConfig(**cfg_kw)
    n = round(fs * cfg_kw["integration_ms"] * 1e-3)
    epochs = 6
    g_states = [to_gpu_state(trk, s) for s in chans]
    o_states = list(chans)
    for k in range(epochs):
        blk = x[k * n:(k + 1) * n]
        g_batch, g_outs = trk.track_epoch_batch(blk, [0] * len(g_states), g_states, gcfg)
        for c in range(len(chans)):
            o_states[c], o_out = to.track_epoch(blk, o_states[c], ocfg)
            g_single, g1 = trk.track_epoch(blk, g_states[c], gcfg)
            for key in OUT_KEYS:
                assert getattr(g1, key) == o_out[key], (i, k, c, key, getattr(g1, key), o_out[key])
                assert getattr(g_outs[c], key) == o_out[key], (i, k, c, "batch", key)
            for key in STATE_KEYS:
                assert getattr(g_single, key) == getattr(o_states[c], key), (i, k, c, key)
                assert getattr(g_batch[c], key) == getattr(o_states[c], key), (i, k, c, "batch", key)
        g_states = g_batch
