"""Robustness of the device path at the boundary: non-finite samples, producer
streams of device inputs (__cuda_array_interface__ v3), mixed-rate tracking batches, refused
double precision, and the lifetime of pinned host buffers."""

import gc

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


FS = 4.092e6
CFG = dict(doppler_min_hz=-2000.0, doppler_max_hz=2000.0, doppler_step_hz=500.0, noncoherent_rounds=2)


def batch(n=4):
    return np.stack([oracle.make_snapshot(i, FS, 2e-3, base_seed=21)[0] for i in range(n)])


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_snapshot_is_refused_and_other_rows_stay_valid(pkg, bad):
    """The reference refuses non-finite samples (IqBuffer, buffers.py:62-63). The batch call
    raises InvalidInputError naming the snapshot; it neither hangs nor faults, and the same
    engine then searches clean input exactly."""
    x = batch()
    eng = pkg.AcqEngine(FS, [1, 2, 3, 9], pkg.AcqConfig(**CFG))
    clean = eng.run_rows(x)
    y = x.copy()
    y[2, 777] = complex(bad, 0.0) if np.isnan(bad) else complex(0.0, bad)
    with pytest.raises(pkg.InvalidInputError, match="snapshot 2"):
        eng.run_rows(y)
    np.testing.assert_array_equal(eng.run_rows(x), clean)  # the context survives
    with pytest.raises(pkg.InvalidInputError):
        pkg.acquire_all(pkg.IqBuffer._wrap(y[2], FS, pkg.Precision.SINGLE), [1, 2], pkg.AcqConfig(**CFG))
    eng.close()


def test_non_finite_on_every_path(pkg):
    """Per-bin rows, the power map, the generic path and a float32-overflowing IF scale."""
    x = batch(2)
    y = x.copy()
    y[1, 5] = np.nan
    eng = pkg.AcqEngine(FS, [4], pkg.AcqConfig(**CFG))
    with pytest.raises(pkg.InvalidInputError):
        eng.run_rows(y, per_bin=True)
    with pytest.raises(pkg.InvalidInputError):
        eng.power_map(y[1])
    q = np.zeros((2, 2 * x.shape[1]), dtype=np.int8)
    q[:, ::3] = 100
    with pytest.raises(pkg.InvalidInputError):
        eng.run_rows_quantized(q, 0, 1e308)  # float32(q * 1e308 / 127) = inf
    eng.close()
    gen = pkg.AcqEngine(5.0e6, [4], pkg.AcqConfig(**CFG))
    assert gen.info["path"] == 4
    z = np.stack([oracle.make_snapshot(i, 5.0e6, 2e-3, base_seed=3)[0] for i in range(2)])
    z[0, 9] = np.inf
    with pytest.raises(pkg.InvalidInputError, match="snapshot 0"):
        gen.run_rows(z)
    gen.close()


class _V3:
    """A CAI v3 view of a torch tensor that names the stream its producer wrote on."""

    def __init__(self, t, stream):
        self.t = t
        self.__cuda_array_interface__ = dict(t.__cuda_array_interface__, version=3, stream=stream)


def test_device_input_waits_for_its_producer_stream(pkg):
    """Device inputs are read only after their producer's queued work: the CAI v3 "stream"
    key (a side stream), and the legacy default stream for v2 producers such as torch (no
    key). The producer stream is kept busy with a long sleep kernel ahead of the copy that
    fills the tensor; without the wait the search would read zeros."""
    import torch

    x = batch(8)
    eng = pkg.AcqEngine(FS, list(range(1, 33)), pkg.AcqConfig(**CFG))
    want = eng.run_rows(x)
    src = torch.from_numpy(x).pin_memory()
    # v2 producer on the legacy default stream
    dev = torch.zeros(x.shape, dtype=torch.complex64, device="cuda")
    torch.cuda.synchronize()
    assert "stream" not in dev.__cuda_array_interface__
    torch.cuda._sleep(200_000_000)
    dev.copy_(src, non_blocking=True)
    np.testing.assert_array_equal(eng.run_rows(dev), want)
    # v3 producer on a side stream
    side = torch.cuda.Stream()
    dev2 = torch.zeros(x.shape, dtype=torch.complex64, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)
        dev2.copy_(src, non_blocking=True)
    np.testing.assert_array_equal(eng.run_rows(_V3(dev2, side.cuda_stream)), want)
    eng.close()


def test_tracking_refuses_double_precision_and_mixed_rates(pkg):
    from paper_1309_0052_b200 import tracking as trk

    st = trk.TrackState(prn=3, code_phase_chips=100.0, carrier_phase_cycles=0.0, doppler_hz=200.0,
                        code_rate_hz=1.023e6, sample_rate_hz=FS)
    cfg = trk.TrackConfig()
    blk = oracle.make_snapshot(0, FS, 1e-3, base_seed=3)[0]
    with pytest.raises(pkg.UnsupportedError):
        trk.epl_correlate(blk.astype(np.complex128), st, cfg)
    with pytest.raises(pkg.UnsupportedError):
        trk.epl_correlate(pkg.IqBuffer(blk, FS, pkg.Precision.DOUBLE), st, cfg)
    st8 = trk.TrackState(prn=4, code_phase_chips=10.0, carrier_phase_cycles=0.0, doppler_hz=0.0,
                         code_rate_hz=1.023e6, sample_rate_hz=2 * FS)
    b = trk.TrackBatch.from_states([st, st8])
    x = np.concatenate([blk, oracle.make_snapshot(1, 2 * FS, 1e-3, base_seed=3)[0]])
    with pytest.raises(pkg.InvalidInputError, match="block length"):
        trk.track_step(x, [0, blk.size], b, cfg)


def test_pinned_array_outlives_its_buffer_object(pkg):
    """PinnedBuffer.array owns the page-locked allocation (a bare from_address view
    did not), so a view taken from a temporary buffer stays valid and usable for H2D."""
    a = pkg.PinnedBuffer((4, 8184)).array
    gc.collect()
    a[:] = batch(4)
    eng = pkg.AcqEngine(FS, [1, 2], pkg.AcqConfig(**CFG))
    np.testing.assert_array_equal(eng.run_rows(a), eng.run_rows(np.array(a)))
    buf = pkg.PinnedBuffer((2, 8184))
    view = buf.array[1]
    buf.close()
    del buf
    gc.collect()
    view[:] = 1.0
    assert view.sum() == 8184
    eng.close()
