"""Tracking channels -- drop-in for gnssperf/tracking.py.

The receiver's step after acquisition. The O(N) per-epoch work -- carrier wipe-off plus
the early / prompt / late dot products (tracking.py:126-165) -- runs on the GPU for a whole
batch of channels in one launch (libgacq ``gacq_trk_epl``); the scalar loop math
(discriminators, second-order loop filters, fixed-point NCO advance, lock detector,
tracking.py:168-275) stays on the host in float64 with the reference's formulas: per channel
in Python (``track_epoch``) or for a struct-of-arrays batch in libgacq's multithreaded C++
(``gacq_trk_close`` / ``gacq_trk_chans``, used by ``track_step``).

Replicas are bit-identical to the reference's (the fixed-point NCO words use kernels.py's
exact expressions), the dot products follow the reference's left-to-right complex64 sums,
and the loop closure keeps its float64 operation order, so every epoch's state equals the
reference's bit for bit (tests/golden/tracking.json).
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .cacode import CHIP_RATE_HZ, CODE_LENGTH
from .errors import DegenerateInputError, InvalidConfigError, InvalidInputError, UnsupportedError

L1_CARRIER_HZ = 1575.42e6  # gnss_signal.py:34
LOOP_DAMPING = 0.7071067811865476  # tracking.py:44
LOCK_SMOOTHING_EPOCHS = 20  # tracking.py:45

CARRIER_SCALE = 1 << 48  # kernels.py:47-50
CODE_SCALE = 1 << 42  # kernels.py:52-53
CODE_MODULUS = CODE_LENGTH * CODE_SCALE


def carrier_phase_to_fixed(phase_cycles: float) -> int:  # kernels.py:56-58
    return int(round((phase_cycles % 1.0) * CARRIER_SCALE)) % CARRIER_SCALE


def carrier_step_to_fixed(freq_hz: float, fs: float) -> int:  # kernels.py:61-62
    return int(round((freq_hz / fs) * CARRIER_SCALE)) % CARRIER_SCALE


def code_phase_to_fixed(phase_chips: float) -> int:  # kernels.py:65-66
    return int(round((phase_chips % 1023.0) * CODE_SCALE)) % CODE_MODULUS


def code_step_to_fixed(chip_rate_hz: float, fs: float) -> int:  # kernels.py:69-70
    return int(round((chip_rate_hz / fs) * CODE_SCALE))


@dataclass(frozen=True)
class TrackConfig:
    """tracking.py:48-67 (same validation and messages)."""

    correlator_spacing_chips: float = 0.5
    dll_bandwidth_hz: float = 2.0
    pll_bandwidth_hz: float = 15.0
    integration_ms: int = 1

    def __post_init__(self):
        if not 0 < self.correlator_spacing_chips <= 1:
            raise InvalidConfigError("correlator spacing must be in (0, 1] chips")
        if self.dll_bandwidth_hz <= 0 or self.pll_bandwidth_hz <= 0:
            raise InvalidConfigError("loop bandwidths must be > 0")
        if self.integration_ms < 1:
            raise InvalidConfigError("integration_ms must be >= 1")
        t = self.integration_ms * 1e-3
        for bw in (self.dll_bandwidth_hz, self.pll_bandwidth_hz):
            if bw * t >= 0.25:
                raise InvalidConfigError(f"stability guard violated: bandwidth {bw} Hz x {t} s >= 0.25")


@dataclass(frozen=True)
class TrackState:
    """tracking.py:70-82."""

    prn: int
    code_phase_chips: float
    carrier_phase_cycles: float
    doppler_hz: float
    code_rate_hz: float
    dll_filter_state: tuple = (0.0, 0.0)
    pll_filter_state: tuple = (0.0, 0.0)
    epoch: int = 0
    sample_rate_hz: float = 8.184e6
    lock_nbd: float = 0.0
    lock_nbp: float = 0.0


@dataclass(frozen=True)
class TrackOutput:
    """tracking.py:85-97."""

    ie: float
    qe: float
    ip: float
    qp: float
    il: float
    ql: float
    dll_error_chips: float = 0.0
    pll_error_cycles: float = 0.0
    lock_metric: float = 0.0
    multiplications: int = 0
    direct_equivalent_multiplications: int = 0


def init_from_acquisition(acq, fs: float) -> TrackState:
    """tracking.py:100-119: code delay -> prompt replica start phase (nominal chip rate)."""
    if not acq.detected:
        raise InvalidInputError(f"PRN {acq.prn} was not detected; nothing to track")
    cps = CHIP_RATE_HZ / fs
    return TrackState(prn=acq.prn, code_phase_chips=(-acq.code_phase_samples * cps) % CODE_LENGTH,
                      carrier_phase_cycles=0.0, doppler_hz=acq.doppler_hz,
                      code_rate_hz=CHIP_RATE_HZ * (1.0 + acq.doppler_hz / L1_CARRIER_HZ), sample_rate_hz=fs)


def block_length(state: TrackState, config: TrackConfig) -> int:  # tracking.py:122-123
    return round(state.sample_rate_hz * config.integration_ms * 1e-3)


def dll_discriminator(out: TrackOutput, spacing_chips: float = 0.5) -> float:  # tracking.py:168-176
    e = out.ie * out.ie + out.qe * out.qe
    l = out.il * out.il + out.ql * out.ql
    if e + l == 0:
        if out.ip == 0 and out.qp == 0:
            raise DegenerateInputError("all correlators zero")
        return 0.0
    return (e - l) / (e + l) * (1.0 - spacing_chips / 2.0) / 2.0


def pll_discriminator(out: TrackOutput) -> float:  # tracking.py:179-185
    if out.ip == 0.0 and out.qp == 0.0:
        raise DegenerateInputError("prompt correlator is zero")
    if out.ip == 0.0:
        return math.copysign(0.25, out.qp)
    return math.atan(out.qp / out.ip) / (2.0 * math.pi)


def loop_gains(bandwidth_hz: float) -> tuple:  # tracking.py:188-190
    w0 = bandwidth_hz / 0.53
    return 2.0 * LOOP_DAMPING * w0, w0 * w0


def loop_filter(error: float, state: tuple, bandwidth_hz: float, integration_s: float) -> tuple:
    """tracking.py:193-208: second-order PI; returns (rate correction, new state)."""
    if bandwidth_hz * integration_s >= 0.25:
        raise InvalidConfigError(f"stability guard violated: {bandwidth_hz} Hz x {integration_s} s >= 0.25")
    g1, g2 = loop_gains(bandwidth_hz)
    acc, prev = state
    acc_new = acc + g2 * integration_s * (error + prev) / 2.0
    return g1 * error + acc_new, (acc_new, error)


def _advance_carrier(phase, doppler, fs, n, step_cycles):  # tracking.py:211-215
    p0 = carrier_phase_to_fixed(phase)
    step = carrier_step_to_fixed(doppler, fs)
    return ((p0 + n * step + carrier_phase_to_fixed(step_cycles)) % CARRIER_SCALE) / CARRIER_SCALE


def _advance_code(phase, rate, fs, n, step_chips):  # tracking.py:218-223
    p0 = code_phase_to_fixed(phase)
    step = code_step_to_fixed(rate, fs)
    nudge = int(round((step_chips % CODE_LENGTH) * CODE_SCALE))
    return ((p0 + n * step + nudge) % CODE_MODULUS) / CODE_SCALE


class _EplChan(C.Structure):
    _fields_ = [("block_offset", C.c_int64), ("carrier_p0", C.c_uint64), ("carrier_step", C.c_uint64),
                ("code_p0", C.c_uint64 * 3), ("code_step", C.c_uint64), ("prn", C.c_int32),
                ("reserved", C.c_int32)]


def _samples_arg(samples, trk):
    """(total, pointer, flags, owner) of a sample buffer for gacq_trk_*: a CUDA array
    (__cuda_array_interface__; the tracker's stream then waits for its producer) or a host
    array. Only complex64 is implemented on the device: complex128 (Precision.DOUBLE) and
    other dtypes are refused rather than silently rounded."""
    cai = getattr(samples, "__cuda_array_interface__", None)
    if cai is not None:
        if cai["typestr"] != "<c8":
            raise InvalidInputError("device samples must be complex64")
        _lib.wait_for_producer(_lib.lib.gacq_trk_wait_stream, trk, cai)
        return int(np.prod(cai["shape"])), cai["data"][0], _lib.SNAPS_ON_DEVICE, samples
    arr = np.asarray(getattr(samples, "samples", samples))
    if arr.dtype == np.complex128:
        raise UnsupportedError("Precision.DOUBLE (complex128) is not implemented on the GPU path")
    if arr.dtype != np.complex64:
        raise InvalidInputError(f"samples must be complex64, got {arr.dtype}")
    arr = np.ascontiguousarray(arr).reshape(-1)
    return arr.size, arr.ctypes.data, 0, arr


class TrackEngine:
    """Batched E/P/L correlators on one device (gacq_trk_*)."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        self._trk = C.c_void_p()
        _lib.check(_lib.lib.gacq_trk_create(C.byref(self._trk), self.device))

    def correlate(self, samples, offsets, states, config: TrackConfig) -> np.ndarray:
        """E/P/L sums [C, 6] = (ie, qe, ip, qp, il, ql) for channel c over the block starting at
        samples[offsets[c]] (complex64; host array, or CUDA array via __cuda_array_interface__)."""
        states = list(states)
        n = block_length(states[0], config)
        for s in states:
            if block_length(s, config) != n:
                raise InvalidInputError("all channels of a batch need the same block length")
        d = config.correlator_spacing_chips
        chans = (_EplChan * len(states))()
        for i, (st, off) in enumerate(zip(states, offsets)):
            fs = st.sample_rate_hz
            c = chans[i]
            c.block_offset = int(off)
            c.carrier_p0 = carrier_phase_to_fixed(st.carrier_phase_cycles)
            c.carrier_step = carrier_step_to_fixed(st.doppler_hz, fs)
            for j, o in enumerate((+d / 2, 0.0, -d / 2)):  # tracking.py:148-156
                c.code_p0[j] = code_phase_to_fixed((st.code_phase_chips + o) % CODE_LENGTH)
            c.code_step = code_step_to_fixed(st.code_rate_hz, fs)
            c.prn = int(st.prn)
        total, ptr, flags, _keep = _samples_arg(samples, self._trk)
        out = np.empty((len(states), 6), dtype=np.float32)
        _lib.check(_lib.lib.gacq_trk_epl(self._trk, ptr, total, n, chans, len(states), flags, out.ctypes.data))
        return out

    def pinned(self, n_chan: int):
        """Page-locked (chans [n], sums [n, 6]) views reused across epochs (fast H2D/D2H)."""
        from .acquisition import PinnedBuffer

        if getattr(self, "_pin_n", 0) < n_chan:
            self._pin_chans = PinnedBuffer((n_chan,), EPL_CHAN_DTYPE)
            self._pin_sums = PinnedBuffer((n_chan, 6), np.float32)
            self._pin_n = n_chan
        return self._pin_chans.array[:n_chan], self._pin_sums.array[:n_chan]

    def correlate_chans(self, samples, chans: np.ndarray, n: int, out: np.ndarray | None = None) -> np.ndarray:
        """Like correlate() but from prepared gacq_epl_chan records (tracking.EPL_CHAN_DTYPE)."""
        chans = np.ascontiguousarray(chans)
        total, ptr, flags, _keep = _samples_arg(samples, self._trk)
        if out is None:
            out = np.empty((chans.size, 6), dtype=np.float32)
        _lib.check(_lib.lib.gacq_trk_epl(self._trk, ptr, total, int(n), chans.ctypes.data, chans.size, flags,
                                         out.ctypes.data))
        return out

    def close(self):
        if self._trk:
            _lib.lib.gacq_trk_destroy(self._trk)
            self._trk = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_engines: dict = {}
_lock = threading.Lock()


def get_track_engine(device: int = 0) -> TrackEngine:
    with _lock:
        if device not in _engines:
            _engines[device] = TrackEngine(device)
        return _engines[device]


def _outputs(sums: np.ndarray, n: int) -> list:
    return [TrackOutput(ie=float(r[0]), qe=float(r[1]), ip=float(r[2]), qp=float(r[3]), il=float(r[4]),
                        ql=float(r[5]), multiplications=4 * n, direct_equivalent_multiplications=n * n)
            for r in sums]


def epl_correlate(block, state: TrackState, config: TrackConfig, device: int = 0) -> TrackOutput:
    """tracking.py:126-165 on the GPU."""
    n = block_length(state, config)
    samples = getattr(block, "samples", block)
    if len(samples) != n:
        raise InvalidInputError(f"block must hold {n} samples, got {len(samples)}")
    return _outputs(get_track_engine(device).correlate(samples, [0], [state], config), n)[0]


def _close_loops(out: TrackOutput, state: TrackState, config: TrackConfig):
    """tracking.py:231-275 after the correlators: discriminators, loops, NCO advance, lock."""
    ed = dll_discriminator(out, config.correlator_spacing_chips)
    ep = pll_discriminator(out)
    t = config.integration_ms * 1e-3
    n = block_length(state, config)
    g1p, _ = loop_gains(config.pll_bandwidth_hz)
    g1d, _ = loop_gains(config.dll_bandwidth_hz)
    _, pll_state = loop_filter(ep, state.pll_filter_state, config.pll_bandwidth_hz, t)
    _, dll_state = loop_filter(ed, state.dll_filter_state, config.dll_bandwidth_hz, t)
    doppler = state.doppler_hz + (pll_state[0] - state.pll_filter_state[0])
    code_rate = CHIP_RATE_HZ * (1.0 + doppler / L1_CARRIER_HZ) + dll_state[0]
    carrier_phase = _advance_carrier(state.carrier_phase_cycles, state.doppler_hz, state.sample_rate_hz, n,
                                     t * g1p * ep)
    code_phase = _advance_code(state.code_phase_chips, state.code_rate_hz, state.sample_rate_hz, n, t * g1d * ed)
    nbd = out.ip * out.ip - out.qp * out.qp
    nbp = out.ip * out.ip + out.qp * out.qp
    if state.epoch == 0:
        nbd_s, nbp_s = nbd, nbp
    else:
        alpha = 1.0 / LOCK_SMOOTHING_EPOCHS
        nbd_s = state.lock_nbd + alpha * (nbd - state.lock_nbd)
        nbp_s = state.lock_nbp + alpha * (nbp - state.lock_nbp)
    lock = nbd_s / nbp_s if nbp_s > 0 else 0.0
    new_state = replace(state, code_phase_chips=code_phase, carrier_phase_cycles=carrier_phase, doppler_hz=doppler,
                        code_rate_hz=code_rate, dll_filter_state=dll_state, pll_filter_state=pll_state,
                        epoch=state.epoch + 1, lock_nbd=nbd_s, lock_nbp=nbp_s)
    return new_state, replace(out, dll_error_chips=ed, pll_error_cycles=ep, lock_metric=lock)


def track_epoch(block, state: TrackState, config: TrackConfig, device: int = 0):
    """tracking.py:226-275: one loop iteration (GPU correlators, host loop closure)."""
    return _close_loops(epl_correlate(block, state, config, device), state, config)


# ---- struct-of-arrays batch path ------------------------------------------------------

EPL_CHAN_DTYPE = np.dtype([("block_offset", "<i8"), ("carrier_p0", "<u8"), ("carrier_step", "<u8"),
                           ("code_p0", "<u8", (3,)), ("code_step", "<u8"), ("prn", "<i4"), ("reserved", "<i4")])
assert EPL_CHAN_DTYPE.itemsize == C.sizeof(_EplChan)


def _carrier_phase_fixed_v(phase):  # kernels.py:56-58, vectorised (np.mod == Python %, rint == round)
    return (np.rint(np.mod(phase, 1.0) * float(CARRIER_SCALE)).astype(np.int64) % CARRIER_SCALE).astype(np.uint64)


def _carrier_step_fixed_v(freq, fs):  # kernels.py:61-62
    return (np.rint((freq / fs) * float(CARRIER_SCALE)).astype(np.int64) % CARRIER_SCALE).astype(np.uint64)


def _code_phase_fixed_v(phase):  # kernels.py:65-66
    return (np.rint(np.mod(phase, 1023.0) * float(CODE_SCALE)).astype(np.int64) % CODE_MODULUS).astype(np.uint64)


def _code_step_fixed_v(rate, fs):  # kernels.py:69-70
    return np.rint((rate / fs) * float(CODE_SCALE)).astype(np.int64).astype(np.uint64)


@dataclass
class TrackBatch:
    """TrackState fields as float64/int arrays over channels (struct of arrays)."""

    prn: np.ndarray
    code_phase_chips: np.ndarray
    carrier_phase_cycles: np.ndarray
    doppler_hz: np.ndarray
    code_rate_hz: np.ndarray
    dll_acc: np.ndarray
    dll_prev: np.ndarray
    pll_acc: np.ndarray
    pll_prev: np.ndarray
    epoch: np.ndarray
    sample_rate_hz: np.ndarray
    lock_nbd: np.ndarray
    lock_nbp: np.ndarray

    @classmethod
    def from_states(cls, states) -> "TrackBatch":
        s = list(states)
        f = lambda k: np.array([getattr(x, k) for x in s], dtype=np.float64)  # noqa: E731
        return cls(prn=np.array([x.prn for x in s], dtype=np.int32), code_phase_chips=f("code_phase_chips"),
                   carrier_phase_cycles=f("carrier_phase_cycles"), doppler_hz=f("doppler_hz"),
                   code_rate_hz=f("code_rate_hz"),
                   dll_acc=np.array([x.dll_filter_state[0] for x in s], dtype=np.float64),
                   dll_prev=np.array([x.dll_filter_state[1] for x in s], dtype=np.float64),
                   pll_acc=np.array([x.pll_filter_state[0] for x in s], dtype=np.float64),
                   pll_prev=np.array([x.pll_filter_state[1] for x in s], dtype=np.float64),
                   epoch=np.array([x.epoch for x in s], dtype=np.int64), sample_rate_hz=f("sample_rate_hz"),
                   lock_nbd=f("lock_nbd"), lock_nbp=f("lock_nbp"))

    def to_states(self) -> list:
        return [TrackState(prn=int(self.prn[i]), code_phase_chips=float(self.code_phase_chips[i]),
                           carrier_phase_cycles=float(self.carrier_phase_cycles[i]), doppler_hz=float(self.doppler_hz[i]),
                           code_rate_hz=float(self.code_rate_hz[i]),
                           dll_filter_state=(float(self.dll_acc[i]), float(self.dll_prev[i])),
                           pll_filter_state=(float(self.pll_acc[i]), float(self.pll_prev[i])), epoch=int(self.epoch[i]),
                           sample_rate_hz=float(self.sample_rate_hz[i]), lock_nbd=float(self.lock_nbd[i]),
                           lock_nbp=float(self.lock_nbp[i]))
                for i in range(self.prn.size)]


def _c_batch(batch: TrackBatch):
    """ctypes view of a TrackBatch whose arrays are contiguous float64 / int64 / int32."""
    d = lambda a: a.ctypes.data_as(_lib._PD)  # noqa: E731
    return _lib.TrkBatch(batch.prn.size, batch.prn.ctypes.data_as(C.POINTER(C.c_int32)), d(batch.code_phase_chips),
                         d(batch.carrier_phase_cycles), d(batch.doppler_hz), d(batch.code_rate_hz), d(batch.dll_acc),
                         d(batch.dll_prev), d(batch.pll_acc), d(batch.pll_prev), d(batch.lock_nbd), d(batch.lock_nbp),
                         batch.epoch.ctypes.data_as(C.POINTER(C.c_int64)), d(batch.sample_rate_hz))


def _c_config(config: TrackConfig):
    return _lib.TrkConfig(float(config.integration_ms), float(config.pll_bandwidth_hz),
                          float(config.dll_bandwidth_hz), float(config.correlator_spacing_chips))


def _owned(batch: TrackBatch) -> TrackBatch:
    """A contiguous copy with the dtypes the C ABI expects."""
    f = lambda a: np.array(a, dtype=np.float64, order="C", copy=True)  # noqa: E731
    return TrackBatch(prn=np.array(batch.prn, dtype=np.int32, copy=True), code_phase_chips=f(batch.code_phase_chips),
                      carrier_phase_cycles=f(batch.carrier_phase_cycles), doppler_hz=f(batch.doppler_hz),
                      code_rate_hz=f(batch.code_rate_hz), dll_acc=f(batch.dll_acc), dll_prev=f(batch.dll_prev),
                      pll_acc=f(batch.pll_acc), pll_prev=f(batch.pll_prev),
                      epoch=np.array(batch.epoch, dtype=np.int64, copy=True), sample_rate_hz=f(batch.sample_rate_hz),
                      lock_nbd=f(batch.lock_nbd), lock_nbp=f(batch.lock_nbp))


def epl_chans(batch: TrackBatch, offsets, config: TrackConfig) -> np.ndarray:
    """gacq_epl_chan records for every channel of the batch (kernels.py:56-70, gacq_trk_chans)."""
    b = _owned(batch)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    if off.shape != (b.prn.size,):
        raise InvalidInputError("one block offset per channel")
    ch = np.zeros(b.prn.size, dtype=EPL_CHAN_DTYPE)
    cb, cc = _c_batch(b), _c_config(config)
    _lib.check(_lib.lib.gacq_trk_chans(C.byref(cb), C.byref(cc), off.ctypes.data, ch.ctypes.data))
    return ch


def close_loops_batch(sums: np.ndarray, batch: TrackBatch, config: TrackConfig):
    """tracking.py:231-275 over a batch, in the reference's float64 operation order
    (bit-identical per channel; libgacq gacq_trk_close, multithreaded C++ with the C library's
    atan, which is what math.atan calls). Returns (new batch, outputs dict)."""
    sums = np.ascontiguousarray(sums, dtype=np.float32)
    new = _owned(batch)
    if sums.shape != (new.prn.size, 6):
        raise InvalidInputError("sums must be [n_channels, 6]")
    out = np.empty((new.prn.size, 3), dtype=np.float64)
    bad = C.c_int64(-1)
    cb, cc = _c_batch(new), _c_config(config)
    rc = _lib.lib.gacq_trk_close(sums.ctypes.data, C.byref(cb), C.byref(cc), out.ctypes.data, C.byref(bad))
    if rc == _lib.ERR_INVALID and bad.value >= 0:
        raise DegenerateInputError((_lib.lib.gacq_last_error() or b"").decode())
    _lib.check(rc)
    s64 = sums.astype(np.float64)
    outs = dict(ie=s64[:, 0], qe=s64[:, 1], ip=s64[:, 2], qp=s64[:, 3], il=s64[:, 4], ql=s64[:, 5],
                dll_error_chips=out[:, 0], pll_error_cycles=out[:, 1], lock_metric=out[:, 2])
    return new, outs


def track_step(samples, offsets, batch: TrackBatch, config: TrackConfig, device: int = 0):
    """One epoch of a struct-of-arrays batch in one native call (libgacq gacq_trk_step): the NCO
    words, the correlator kernel and the loop closure of tracking.py:126-275 for every channel,
    pipelined over channel slices. Returns (new batch, outputs dict) like close_loops_batch; the
    input batch is not modified (a degenerate channel raises before anything is returned)."""
    eng = get_track_engine(device)
    b = _owned(batch)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    if off.shape != (b.prn.size,):
        raise InvalidInputError("one block offset per channel")
    total, ptr, flags, _keep = _samples_arg(samples, eng._trk)
    sums = np.empty((b.prn.size, 6), dtype=np.float32)
    out = np.empty((b.prn.size, 3), dtype=np.float64)
    bad = C.c_int64(-1)
    cb, cc = _c_batch(b), _c_config(config)
    rc = _lib.lib.gacq_trk_step(eng._trk, ptr, total, off.ctypes.data, C.byref(cb), C.byref(cc), flags,
                                sums.ctypes.data, out.ctypes.data, C.byref(bad))
    if rc == _lib.ERR_INVALID and bad.value >= 0:
        raise DegenerateInputError((_lib.lib.gacq_last_error() or b"").decode())
    _lib.check(rc)
    s64 = sums.astype(np.float64)
    outs = dict(ie=s64[:, 0], qe=s64[:, 1], ip=s64[:, 2], qp=s64[:, 3], il=s64[:, 4], ql=s64[:, 5],
                dll_error_chips=out[:, 0], pll_error_cycles=out[:, 1], lock_metric=out[:, 2])
    return b, outs


def track_epoch_batch(samples, offsets, states, config: TrackConfig, device: int = 0):
    """One epoch for many channels in one device launch: channel c correlates
    samples[offsets[c] : offsets[c] + N]. Returns (new_states, outputs), channel order kept."""
    states = list(states)
    if not states:
        raise InvalidInputError("no channels")
    n = block_length(states[0], config)
    sums = get_track_engine(device).correlate(samples, offsets, states, config)
    res = [_close_loops(o, s, config) for o, s in zip(_outputs(sums, n), states)]
    return [r[0] for r in res], [r[1] for r in res]
