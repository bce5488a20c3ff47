"""Parallel code-phase acquisition on B200 -- drop-in for gnssperf/acquisition.py.

Same names, fields, validation and error behaviour as the reference module
(acquisition.py:36-208); the search itself (acquisition.py:128-159) runs in
libgacq.so (hand-written sm_100a kernels, include/gacq.h) and the host only
finishes acquisition.py:160-170 (float64 metric, decision, AcqResult).

New, batch-first API (the paper's proposed batch mode):

* ``AcqEngine``     -- one search plan (fs, config, PRN list) bound to a device;
                      ``search()`` takes a [S, L] batch (host numpy or any CUDA
                      array exposing ``__cuda_array_interface__``) and returns
                      ``BatchResult`` arrays.
* ``acquire_batch`` -- list-of-lists of AcqResult over one or several devices.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .buffers import IqBuffer, Precision
from .cacode import CHIP_RATE_HZ, CODE_LENGTH, CaCode, generate_ca_code
from .errors import InvalidInputError, PipelineError, UnsupportedError

DEFAULT_DOPPLER_SPAN_HZ = 5000.0


def default_doppler_step_hz(coherent_ms: int) -> float:
    """Grid step 2/(3 T_coh), about 667 Hz at 1 ms (acquisition.py:39-41)."""
    return 2.0 / (3.0 * coherent_ms * 1e-3)


@dataclass(frozen=True)
class AcqConfig:
    """acquisition.py:44-70, field for field."""

    doppler_min_hz: float = -DEFAULT_DOPPLER_SPAN_HZ
    doppler_max_hz: float = DEFAULT_DOPPLER_SPAN_HZ
    doppler_step_hz: float = field(default=0.0)
    coherent_ms: int = 1
    noncoherent_rounds: int = 10
    detection_threshold: float = 2.5
    exclusion_radius_samples: int = 0  # 0 means one chip worth of samples at use

    def __post_init__(self):
        if self.doppler_step_hz == 0.0:
            object.__setattr__(self, "doppler_step_hz", default_doppler_step_hz(self.coherent_ms))
        if self.doppler_min_hz > self.doppler_max_hz:
            raise InvalidInputError("doppler_min_hz must be <= doppler_max_hz")
        if self.doppler_step_hz <= 0:
            raise InvalidInputError("doppler_step_hz must be > 0")
        if self.coherent_ms < 1 or self.noncoherent_rounds < 1:
            raise InvalidInputError("coherent_ms and noncoherent_rounds must be >= 1")
        if self.detection_threshold <= 1:
            raise InvalidInputError("detection_threshold must be > 1")
        if self.exclusion_radius_samples < 0:
            raise InvalidInputError("exclusion_radius_samples must be >= 0")

    def doppler_bins_hz(self) -> np.ndarray:
        n = int(math.floor((self.doppler_max_hz - self.doppler_min_hz) / self.doppler_step_hz + 1e-9)) + 1
        return self.doppler_min_hz + self.doppler_step_hz * np.arange(n)


@dataclass(frozen=True)
class AcqResult:
    """acquisition.py:73-81."""

    prn: int
    doppler_hz: float
    code_phase_samples: int
    peak_metric: float
    detected: bool
    bins_searched: int
    multiplications_performed: int


def samples_per_code_period(sample_rate_hz: float) -> int:
    """acquisition.py:108-109."""
    return round(sample_rate_hz * CODE_LENGTH / CHIP_RATE_HZ)


_code_spectrum_cache: dict = {}
_cache_lock = threading.Lock()
_CODE_SCALE = 1 << 42  # kernels.py:51-53: 42-bit code NCO fraction
_CODE_MODULUS = CODE_LENGTH * _CODE_SCALE


def conjugate_code_spectrum(prn: int, sample_rate_hz: float, n: int, precision: Precision = Precision.SINGLE):
    """Drop-in for gnssperf.acquisition.conjugate_code_spectrum (acquisition.py:88-105):
    conj(FFT_n(code replica)) of one PRN, cached immutably per (prn, fs, n, precision).

    The replica is the reference's floor-indexed code NCO from phase 0
    (gnss_signal.py:75-96, kernels.py:65-70: chip index ((k * step) mod 1023*2^42) >> 42), in the
    precision's complex dtype, transformed with scipy.fft as the reference's dsp backend does
    (dsp.py:82-85), so the bins are the reference's bit for bit. This is a host helper for
    callers that use the reference's API directly; the GPU search never calls it (gacq_create
    builds its own code spectra on the device)."""
    key = (int(prn), float(sample_rate_hz), int(n), precision)
    spec = _code_spectrum_cache.get(key)
    if spec is not None:
        return spec
    if n < 1:
        raise InvalidInputError("sample_code_replica needs n >= 1")
    if sample_rate_hz <= 0:
        raise InvalidInputError("rates must be > 0")
    with _cache_lock:
        spec = _code_spectrum_cache.get(key)
        if spec is None:
            from scipy import fft as _sfft  # the reference's FFT dependency (host helper only)

            chips = generate_ca_code(int(prn)).chips
            step = int(round((CHIP_RATE_HZ / sample_rate_hz) * _CODE_SCALE))  # kernels.py:69-70
            # k * step < 2^20 * 2^42 for any n < 2^20 samples: exact in uint64
            if n >= 1 << 20:
                raise InvalidInputError("conjugate_code_spectrum: n must be < 2^20 samples")
            k = np.arange(int(n), dtype=np.uint64)
            idx = (((k * np.uint64(step)) % np.uint64(_CODE_MODULUS)) >> np.uint64(42)).astype(np.int64)
            replica = chips[idx].astype(precision.complex_dtype)
            spec = np.conj(_sfft.fft(replica))
            spec.setflags(write=False)
            _code_spectrum_cache[key] = spec
    return spec


@dataclass
class BatchResult:
    """Vectorised results of a batch: every array is [n_snap, n_prn]."""

    prns: np.ndarray
    bin_index: np.ndarray
    doppler_hz: np.ndarray
    code_phase_samples: np.ndarray
    peak: np.ndarray          # float32 winning-cell power
    floor: np.ndarray         # float32 exclusion floor of the winning row
    peak_metric: np.ndarray   # float64 peak/floor (inf when floor == 0)
    detected: np.ndarray
    bins_searched: int
    multiplications_performed: int

    def results(self) -> list:
        """list (snapshots) of list (PRNs, plan order) of AcqResult."""
        out = []
        for s in range(self.doppler_hz.shape[0]):
            out.append([AcqResult(prn=int(self.prns[p]), doppler_hz=float(self.doppler_hz[s, p]),
                                  code_phase_samples=int(self.code_phase_samples[s, p]),
                                  peak_metric=float(self.peak_metric[s, p]),
                                  detected=bool(self.detected[s, p]),
                                  bins_searched=self.bins_searched,
                                  multiplications_performed=self.multiplications_performed)
                        for p in range(self.prns.shape[0])])
        return out


def _finish(rows: np.ndarray, prns: np.ndarray, bins: np.ndarray, config: AcqConfig, mults: int) -> BatchResult:
    """acquisition.py:160-170 over grid-global rows: metric = float64(peak)/float64(floor)
    (inf when floor == 0), detected = metric >= threshold, doppler = bins[bin]."""
    peak = rows["peak"]
    floor = rows["floor"]
    p64, f64 = peak.astype(np.float64), floor.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        metric = p64 / f64
    metric[~(f64 > 0)] = np.inf  # (8x faster than nested np.where: this is on the e2e path)
    b = rows["bin"]
    return BatchResult(prns=prns.copy(), bin_index=b, doppler_hz=np.take(bins, b),
                       code_phase_samples=rows["lag"].astype(np.int64), peak=peak, floor=floor,
                       peak_metric=metric, detected=metric >= config.detection_threshold,
                       bins_searched=int(bins.size), multiplications_performed=mults)


def _host_array(x) -> np.ndarray:
    arr = np.asarray(x)
    if arr.dtype != np.complex64:
        if arr.dtype == np.complex128:
            raise UnsupportedError("double precision (complex128) is not implemented on the GPU path")
        raise InvalidInputError(f"snapshots must be complex64, got {arr.dtype}")
    if arr.ndim == 1:
        arr = arr[None, :]
    if arr.ndim != 2:
        raise InvalidInputError("snapshots must be [n_snap, n_samples]")
    if arr.strides[1] != 8:
        arr = np.ascontiguousarray(arr)
    if arr.strides[0] % 8:
        arr = np.ascontiguousarray(arr)
    return arr


class _PinnedAlloc:
    """Owner of one page-locked allocation (gacq_host_alloc). Every array view of it keeps
    this object alive through its ``base`` chain, so the memory is freed (cudaFreeHost) only
    when the last view is gone."""

    def __init__(self, nbytes: int):
        self._ptr = C.c_void_p()
        _lib.check(_lib.lib.gacq_host_alloc(max(nbytes, 1), C.byref(self._ptr)))
        self.__array_interface__ = {"shape": (max(nbytes, 1),), "typestr": "|u1", "version": 3,
                                    "data": (self._ptr.value, False)}

    def __del__(self):
        try:
            if self._ptr:
                _lib.lib.gacq_host_free(self._ptr)
                self._ptr = C.c_void_p()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class PinnedBuffer:
    """Page-locked host memory viewed as a numpy array. ``array`` (and any view of it) owns
    the allocation: it stays valid after this object is dropped or closed."""

    def __init__(self, shape, dtype=np.complex64):
        self.shape, self.dtype = tuple(shape), np.dtype(dtype)
        count = int(np.prod(self.shape))
        raw = np.asarray(_PinnedAlloc(count * self.dtype.itemsize))
        self.array = raw[:count * self.dtype.itemsize].view(self.dtype).reshape(self.shape)

    def close(self):
        """Drop this object's reference; the memory is freed with the last array view."""
        self.array = None


class AcqEngine:
    """A search plan bound to one CUDA device (reference: acquire_all's per-call state)."""

    def __init__(self, sample_rate_hz: float, prns, config: AcqConfig | None = None,
                 device: int = 0, scratch_bytes: int = 0, bin_range: tuple | None = None,
                 force_generic: bool = False):
        """``bin_range=(b0, b1)`` searches only bins [b0, b1) of the config's grid (Doppler-bin
        sharding of one snapshot over devices); rows then carry grid-global
        bin indices, so per-shard rows merge with ``merge_bin_shards``. ``force_generic`` takes
        the generic path at a chip-aligned rate too (parity tests of that path)."""
        config = config or AcqConfig()
        prns = [int(p) for p in prns]
        if not prns:
            raise InvalidInputError("prns must be non-empty")
        if len(set(prns)) != len(prns):
            raise InvalidInputError("prns must be distinct")
        for p in prns:
            if not 1 <= p <= 32:
                raise InvalidInputError(f"prn must be an integer in 1..32, got {p!r}")
        fs = float(sample_rate_hz)
        if not fs > 0:
            raise InvalidInputError("sample_rate_hz must be > 0")
        self.sample_rate_hz = fs
        self.config = config
        self.prns = np.asarray(prns, dtype=np.int32)
        self.device = int(device)
        self.bins = config.doppler_bins_hz()
        b0, b1 = (0, self.bins.size) if bin_range is None else (int(bin_range[0]), int(bin_range[1]))
        if not 0 <= b0 < b1 <= self.bins.size:
            raise InvalidInputError(f"bin_range {bin_range} outside the {self.bins.size}-bin grid")
        self.bin0 = b0
        self.n_coh = round(fs * config.coherent_ms * 1e-3)
        self.period = samples_per_code_period(fs)
        if self.n_coh < self.period:
            raise InvalidInputError("coherent window shorter than one code period")
        self.span = self.n_coh * config.noncoherent_rounds
        self.radius = config.exclusion_radius_samples or math.ceil(fs / CHIP_RATE_HZ)
        self._bins_c = np.ascontiguousarray(self.bins[b0:b1], dtype=np.float64)
        params = _lib.Params(fs, config.coherent_ms, config.noncoherent_rounds, self._bins_c.size,
                             self._bins_c.ctypes.data_as(C.POINTER(C.c_double)), self.radius,
                             len(prns), self.prns.ctypes.data_as(C.POINTER(C.c_int32)), self.device,
                             _lib.PLAN_GENERIC if force_generic else 0, int(scratch_bytes))
        self._ctx = C.c_void_p()
        _lib.check(_lib.lib.gacq_create(C.byref(self._ctx), C.byref(params)))
        info = _lib.Info()
        _lib.check(_lib.lib.gacq_info_get(self._ctx, C.byref(info)))
        self.info = {n: getattr(info, n) for n, _ in _lib.Info._fields_}
        self.mults = 2 * self.n_coh * int(self.bins.size) * config.noncoherent_rounds

    # -- raw rows -------------------------------------------------------------------
    def run_rows(self, snapshots, per_bin: bool = False, profile: bool = False,
                 out: np.ndarray | None = None) -> np.ndarray:
        """Search a batch; returns the structured gacq_row array [n_snap, n_prn(, n_bins)]."""
        flags = (_lib.ROWS_PER_BIN if per_bin else 0) | (_lib.PROFILE if profile else 0)
        cai = getattr(snapshots, "__cuda_array_interface__", None)
        if cai is not None:
            if cai["typestr"] not in ("<c8",):
                raise InvalidInputError(f"device snapshots must be complex64, got {cai['typestr']}")
            shape = tuple(cai["shape"])
            if len(shape) == 1:
                shape = (1, shape[0])
            n_snap, n_samp = shape
            strides = cai.get("strides")
            stride = (strides[0] // 8) if strides and len(strides) == 2 else n_samp
            if strides and len(strides) == 2 and strides[1] != 8:
                raise InvalidInputError("device snapshots must be contiguous along samples")
            ptr = cai["data"][0]
            flags |= _lib.SNAPS_ON_DEVICE
            _lib.wait_for_producer(_lib.lib.gacq_wait_stream, self._ctx, cai)
        else:
            arr = _host_array(snapshots)
            n_snap, n_samp = arr.shape
            stride = arr.strides[0] // 8
            ptr = arr.ctypes.data
        if n_samp < self.span:
            raise InvalidInputError(f"buffer holds {n_samp} samples, {self.span} needed for the "
                                    "configured integration")
        shape = (n_snap, self.prns.size) + ((self._bins_c.size,) if per_bin else ())
        if out is None:
            out = np.empty(shape, dtype=_lib.ROW_DTYPE)
        elif out.shape != shape or out.dtype != np.dtype(_lib.ROW_DTYPE) or not out.flags.c_contiguous:
            raise InvalidInputError("bad output row buffer")
        _lib.check(_lib.lib.gacq_run(self._ctx, ptr, n_snap, stride, flags, out.ctypes.data))
        if self.bin0:
            out["bin"] += self.bin0
        return out

    def finish(self, rows: np.ndarray) -> BatchResult:
        """acquisition.py:160-170 over a row array, vectorised (float64 ratio, >= threshold)."""
        return _finish(rows, self.prns, self.bins, self.config, self.mults)

    def search(self, snapshots, profile: bool = False) -> BatchResult:
        return self.finish(self.run_rows(snapshots, profile=profile))

    def run_rows_quantized(self, iq, sample_format: int, scale: float, per_bin: bool = False,
                           profile: bool = False) -> np.ndarray:
        """Search integer I/Q snapshots (the IF-file payload, iffile.py:74-99) without a host
        dequantization: `iq` is int8/int16 [n_snap, 2*L] interleaved I/Q (host array, or a CUDA
        array via __cuda_array_interface__); the device applies float32(float64(q)*scale/limit)."""
        if sample_format not in (_lib.FMT_INT8, _lib.FMT_INT16):
            raise InvalidInputError(f"unknown sample format {sample_format!r}")
        want = np.dtype(np.int8 if sample_format == _lib.FMT_INT8 else np.int16)
        flags = (_lib.ROWS_PER_BIN if per_bin else 0) | (_lib.PROFILE if profile else 0)
        cai = getattr(iq, "__cuda_array_interface__", None)
        if cai is not None:
            if np.dtype(cai["typestr"]) != want:
                raise InvalidInputError(f"device I/Q must be {want}, got {cai['typestr']}")
            shape = tuple(cai["shape"])
            shape = (1, shape[0]) if len(shape) == 1 else shape
            strides = cai.get("strides")
            if strides and len(strides) == 2 and strides[1] != want.itemsize:
                raise InvalidInputError("device I/Q must be contiguous along samples")
            row = strides[0] // want.itemsize if strides and len(strides) == 2 else shape[1]
            ptr = cai["data"][0]
            flags |= _lib.SNAPS_ON_DEVICE
            _lib.wait_for_producer(_lib.lib.gacq_wait_stream, self._ctx, cai)
        else:
            arr = np.asarray(iq)
            if arr.dtype != want:
                raise InvalidInputError(f"I/Q must be {want}, got {arr.dtype}")
            arr = np.ascontiguousarray(arr[None, :] if arr.ndim == 1 else arr)
            shape, row, ptr = arr.shape, arr.shape[1], arr.ctypes.data
        n_snap, n_vals = shape
        if n_vals % 2 or row % 2:
            raise InvalidInputError("interleaved I/Q needs an even number of values per snapshot")
        if n_vals // 2 < self.span:
            raise InvalidInputError(f"buffer holds {n_vals // 2} samples, {self.span} needed for the "
                                    "configured integration")
        out = np.empty((n_snap, self.prns.size) + ((self._bins_c.size,) if per_bin else ()), dtype=_lib.ROW_DTYPE)
        _lib.check(_lib.lib.gacq_run_quantized(self._ctx, ptr, int(sample_format), float(scale), n_snap, row // 2,
                                               flags, out.ctypes.data))
        if self.bin0:
            out["bin"] += self.bin0
        return out

    def search_quantized(self, iq, sample_format: int, scale: float, profile: bool = False) -> BatchResult:
        return self.finish(self.run_rows_quantized(iq, sample_format, scale, profile=profile))

    def carrier_table(self) -> np.ndarray:
        """complex64 [n_bins, n_coh] wipe-off replicas the device built (parity hook)."""
        out = np.empty((self._bins_c.size, self.info["n_coh"]), dtype=np.complex64)
        _lib.check(_lib.lib.gacq_carrier_table(self._ctx, out.ctypes.data))
        return out

    def power_map(self, snapshot) -> np.ndarray:
        """float32 [n_prn, n_bins, P] noncoherent power of one host snapshot (parity hook)."""
        arr = _host_array(snapshot)
        if arr.shape[1] < self.span:
            raise InvalidInputError("snapshot too short for the configured integration")
        x = np.ascontiguousarray(arr[0, :self.span])
        out = np.empty((self.prns.size, self._bins_c.size, self.period), dtype=np.float32)
        _lib.check(_lib.lib.gacq_power_map(self._ctx, x.ctypes.data, out.ctypes.data))
        return out

    def stats(self) -> dict:
        s = _lib.Stats()
        _lib.check(_lib.lib.gacq_stats_get(self._ctx, C.byref(s)))
        return {n: getattr(s, n) for n, _ in _lib.Stats._fields_}

    def reset_stats(self) -> None:
        _lib.check(_lib.lib.gacq_stats_reset(self._ctx))

    def close(self) -> None:
        if self._ctx:
            _lib.lib.gacq_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_engines: "OrderedDict[tuple, AcqEngine]" = OrderedDict()
_engines_lock = threading.Lock()
_MAX_ENGINES = 8


def get_engine(sample_rate_hz: float, prns, config: AcqConfig, device: int = 0) -> AcqEngine:
    """Cached plan per (fs, config, prns, device) -- the analogue of the reference's
    immutable code-spectrum cache (acquisition.py:84-105)."""
    key = (float(sample_rate_hz), config, tuple(int(p) for p in prns), int(device))
    with _engines_lock:
        eng = _engines.get(key)
        if eng is not None:
            _engines.move_to_end(key)
            return eng
    eng = AcqEngine(sample_rate_hz, prns, config, device)
    with _engines_lock:
        _engines[key] = eng
        while len(_engines) > _MAX_ENGINES:
            # drop the cache's reference only: an engine another thread is still searching with
            # stays alive until that call returns, then __del__ releases its device plan
            _engines.popitem(last=False)
    return eng


def _check_buffer(samples, config: AcqConfig):
    """acquisition.py:114-126 (same checks, same order, same messages)."""
    precision = getattr(samples, "precision", Precision.SINGLE)
    if getattr(precision, "value", precision) != "single":
        raise UnsupportedError("Precision.DOUBLE is not implemented on the GPU path")
    fs = float(samples.sample_rate_hz)
    n_coh = round(fs * config.coherent_ms * 1e-3)
    period = samples_per_code_period(fs)
    n = len(samples.samples)
    if n < period:
        raise InvalidInputError("buffer shorter than one code period")
    if n < n_coh * config.noncoherent_rounds:
        raise InvalidInputError(f"buffer holds {n} samples, "
                                f"{n_coh * config.noncoherent_rounds} needed for the configured integration")
    if n_coh < period:
        raise InvalidInputError("coherent window shorter than one code period")
    return fs


def acquire_channel(samples: IqBuffer, code: CaCode, config: AcqConfig, device: int = 0) -> AcqResult:
    """Search the Doppler/code-phase grid for one satellite (acquisition.py:112-170)."""
    fs = _check_buffer(samples, config)
    eng = get_engine(fs, [code.prn], config, device)
    return eng.search(samples.samples).results()[0][0]


def acquire_all(samples: IqBuffer, prns: list, config: AcqConfig, plan=None,
                device: int = 0) -> list:
    """All channels of one snapshot in one device pass (acquisition.py:190-208).

    Results are ordered like ``prns``; ``plan`` (an ExecPlan) is accepted and ignored:
    the GPU batch replaces the thread engine, so results are plan-independent by
    construction. A channel failure raises PipelineError attributed to the first
    failing channel in ``prns`` order, as the reference executor does.
    """
    if not prns:
        raise InvalidInputError("prns must be non-empty")
    if len(set(prns)) != len(prns):
        raise InvalidInputError("prns must be distinct")
    for p in prns:
        try:
            generate_ca_code(p)
        except InvalidInputError as exc:
            raise PipelineError(p, repr(exc)) from exc
    try:
        fs = _check_buffer(samples, config)
    except InvalidInputError as exc:
        raise PipelineError(prns[0], repr(exc)) from exc
    eng = get_engine(fs, prns, config, device)
    return eng.search(samples.samples).results()[0]


def acquire_batch(snapshots, sample_rate_hz: float, prns, config: AcqConfig | None = None,
                  devices=None) -> list:
    """Batch mode: [S, L] snapshots -> S lists of AcqResult (PRN order), sharded over
    ``devices`` (contiguous snapshot ranges, one host thread per device, no collective)."""
    config = config or AcqConfig()
    arr = _host_array(snapshots)
    devices = list(devices) if devices else [0]
    shards = np.array_split(np.arange(arr.shape[0]), len(devices))
    engines = [get_engine(sample_rate_hz, prns, config, d) for d in devices]
    outs: list = [None] * len(devices)
    errs: list = []

    def work(i):
        try:
            idx = shards[i]
            if idx.size:
                outs[i] = engines[i].search(arr[idx[0]:idx[-1] + 1]).results()
            else:
                outs[i] = []
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errs.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(devices))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return [r for o in outs for r in o]


def merge_bin_shards(shard_rows) -> np.ndarray:
    """Merge per-shard rows [n_snap, n_prn] (grid-global bin indices, shards in ascending bin
    order) into the rows of the whole grid: the larger peak wins, ties go to the earlier
    shard, i.e. the lower bin -- the reference's row-major first argmax (acquisition.py:151).
    The winning row's floor travels with it, since the floor is row-local."""
    shard_rows = [np.asarray(r) for r in shard_rows]
    out = shard_rows[0].copy()
    for r in shard_rows[1:]:
        take = r["peak"] > out["peak"]
        out[take] = r[take]
    return out


def acquire_bins_sharded(snapshots, sample_rate_hz: float, prns, config: AcqConfig | None = None,
                         devices=None) -> BatchResult:
    """One (or a few) large snapshots searched with the Doppler grid split into contiguous
    bin ranges, one per device (the C2/C4 single-snapshot case), one host
    thread per device; the per-shard rows are merged exactly (merge_bin_shards)."""
    config = config or AcqConfig()
    arr = _host_array(snapshots)
    devices = list(devices) if devices else [0]
    n_bins = config.doppler_bins_hz().size
    ranges = [r for r in np.array_split(np.arange(n_bins), len(devices)) if r.size]
    engines = [AcqEngine(sample_rate_hz, prns, config, d, bin_range=(int(r[0]), int(r[-1]) + 1))
               for d, r in zip(devices, ranges)]
    outs: list = [None] * len(engines)
    errs: list = []

    def work(i):
        try:
            outs[i] = engines[i].run_rows(arr)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errs.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(engines))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    try:
        if errs:
            raise errs[0]
        e0 = engines[0]
        return _finish(merge_bin_shards(outs), e0.prns, e0.bins, config, e0.mults)
    finally:
        for e in engines:
            e.close()


def acquire_if_file(path, prns, config: AcqConfig | None = None, device: int = 0) -> list:
    """The CLI `acquire` path (cli.py:164-169: read_if_file -> acquire_all) with the
    dequantization fused into the device pipeline for integer formats."""
    from .iffile import FORMAT_FLOAT32, read_if_payload

    config = config or AcqConfig()
    payload = read_if_payload(path)
    if payload.sample_format == FORMAT_FLOAT32:
        return acquire_all(payload.to_iq_buffer(), list(prns), config, device=device)
    if not prns:
        raise InvalidInputError("prns must be non-empty")
    if len(set(prns)) != len(prns):
        raise InvalidInputError("prns must be distinct")
    fs = payload.sample_rate_hz
    n = payload.n_samples
    n_coh = round(fs * config.coherent_ms * 1e-3)
    period = samples_per_code_period(fs)
    try:
        if n < period:
            raise InvalidInputError("buffer shorter than one code period")
        if n < n_coh * config.noncoherent_rounds:
            raise InvalidInputError(f"buffer holds {n} samples, "
                                    f"{n_coh * config.noncoherent_rounds} needed for the configured integration")
    except InvalidInputError as exc:
        raise PipelineError(prns[0], repr(exc)) from exc
    eng = get_engine(fs, list(prns), config, device)
    return eng.search_quantized(payload.iq, payload.sample_format, payload.scale).results()[0]
