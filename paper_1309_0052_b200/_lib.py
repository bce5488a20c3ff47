"""ctypes binding of libgacq.so (include/gacq.h). No fallback: importing this module
without the built extension raises."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import InvalidInputError, ResourceError, UnsupportedError

LIB_PATH = Path(os.environ.get("GACQ_LIB") or Path(__file__).resolve().parent / "libgacq.so")

OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_CUDA, ERR_RESOURCE = 0, -1, -2, -3, -4
SNAPS_ON_DEVICE, ROWS_ON_DEVICE, ROWS_PER_BIN, PROFILE = 1, 2, 4, 8
PLAN_GENERIC = 1
ABI_VERSION = 2


class Params(C.Structure):
    _fields_ = [("sample_rate_hz", C.c_double), ("coherent_ms", C.c_int32),
                ("noncoherent_rounds", C.c_int32), ("n_bins", C.c_int32),
                ("doppler_bins_hz", C.POINTER(C.c_double)),
                ("exclusion_radius_samples", C.c_int32), ("n_prn", C.c_int32),
                ("prns", C.POINTER(C.c_int32)), ("device", C.c_int32), ("plan_flags", C.c_int32),
                ("scratch_bytes", C.c_int64)]


class Row(C.Structure):
    _fields_ = [("bin", C.c_int32), ("lag", C.c_int32), ("peak", C.c_float), ("floor", C.c_float)]


class Info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("samples_per_period", "n_coh", "chip_oversample", "fft_len",
                                         "n_bins", "n_prn", "rounds", "path", "corr_ctas")]


class Sat(C.Structure):
    _fields_ = [("prn", C.c_int32), ("reserved", C.c_int32), ("doppler_hz", C.c_double),
                ("code_phase_samples", C.c_double), ("carrier_phase_cycles", C.c_double),
                ("amplitude", C.c_float), ("reserved2", C.c_float)]


_PD = C.POINTER(C.c_double)


class TrkBatch(C.Structure):
    _fields_ = [("n", C.c_int64), ("prn", C.POINTER(C.c_int32)), ("code_phase_chips", _PD),
                ("carrier_phase_cycles", _PD), ("doppler_hz", _PD), ("code_rate_hz", _PD), ("dll_acc", _PD),
                ("dll_prev", _PD), ("pll_acc", _PD), ("pll_prev", _PD), ("lock_nbd", _PD), ("lock_nbp", _PD),
                ("epoch", C.POINTER(C.c_int64)), ("sample_rate_hz", _PD)]


class TrkConfig(C.Structure):
    _fields_ = [("integration_ms", C.c_double), ("pll_bandwidth_hz", C.c_double), ("dll_bandwidth_hz", C.c_double),
                ("correlator_spacing_chips", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("calls", C.c_int64), ("launches", C.c_int64), ("cells", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("fwd_ms", C.c_double),
                ("corr_ms", C.c_double), ("reduce_ms", C.c_double), ("fwd_launches", C.c_int64),
                ("corr_launches", C.c_int64), ("reduce_launches", C.c_int64),
                ("run_ms", C.c_double)]


ROW_DTYPE = [("bin", "<i4"), ("lag", "<i4"), ("peak", "<f4"), ("floor", "<f4")]

EXPORTS = ("gacq_version", "gacq_last_error", "gacq_create", "gacq_info_get", "gacq_destroy",
           "gacq_run", "gacq_run_quantized", "gacq_power_map", "gacq_stats_get", "gacq_stats_reset",
           "gacq_host_alloc", "gacq_host_free", "gacq_ca_code", "gacq_trk_create", "gacq_trk_destroy",
           "gacq_trk_epl", "gacq_carrier_table", "gacq_synth", "gacq_trk_close", "gacq_trk_chans", "gacq_trk_step",
           "gacq_wait_stream", "gacq_trk_wait_stream", "gacq_fp32_probe")
FMT_INT8, FMT_INT16 = 0, 1


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1309_0052_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))  # CDLL releases the GIL for the duration of each call
    lib.gacq_version.restype = C.c_int
    lib.gacq_last_error.restype = C.c_char_p
    lib.gacq_create.argtypes = [C.POINTER(C.c_void_p), C.POINTER(Params)]
    lib.gacq_info_get.argtypes = [C.c_void_p, C.POINTER(Info)]
    lib.gacq_destroy.argtypes = [C.c_void_p]
    lib.gacq_destroy.restype = None
    lib.gacq_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_uint32, C.c_void_p]
    lib.gacq_run_quantized.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_int64, C.c_int64,
                                       C.c_uint32, C.c_void_p]
    lib.gacq_power_map.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.gacq_carrier_table.argtypes = [C.c_void_p, C.c_void_p]
    lib.gacq_trk_close.argtypes = [C.c_void_p, C.POINTER(TrkBatch), C.POINTER(TrkConfig), C.c_void_p,
                                   C.POINTER(C.c_int64)]
    lib.gacq_trk_chans.argtypes = [C.POINTER(TrkBatch), C.POINTER(TrkConfig), C.c_void_p, C.c_void_p]
    lib.gacq_trk_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(TrkBatch),
                                  C.POINTER(TrkConfig), C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    lib.gacq_synth.argtypes = [C.c_int32, C.c_double, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_double,
                               C.c_uint64, C.c_void_p]
    lib.gacq_stats_get.argtypes = [C.c_void_p, C.POINTER(Stats)]
    lib.gacq_stats_reset.argtypes = [C.c_void_p]
    lib.gacq_host_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
    lib.gacq_host_free.argtypes = [C.c_void_p]
    lib.gacq_ca_code.argtypes = [C.c_int32, C.c_void_p]
    lib.gacq_trk_create.argtypes = [C.POINTER(C.c_void_p), C.c_int32]
    lib.gacq_trk_destroy.argtypes = [C.c_void_p]
    lib.gacq_trk_destroy.restype = None
    lib.gacq_trk_epl.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_uint32,
                                 C.c_void_p]
    lib.gacq_wait_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.gacq_trk_wait_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.gacq_fp32_probe.argtypes = [C.c_int32, C.POINTER(C.c_double)]
    if lib.gacq_version() != ABI_VERSION:
        raise ImportError("libgacq ABI version mismatch")
    return lib


_LIB = None


def __getattr__(name):
    """`_lib.lib` loads libgacq.so on first use (so the in-tree build can run before it)."""
    global _LIB
    if name == "lib":
        if _LIB is None:
            _LIB = _load()
        return _LIB
    raise AttributeError(name)


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (__getattr__("lib").gacq_last_error() or b"").decode()
    if rc == ERR_INVALID:
        raise InvalidInputError(msg)
    if rc == ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise ResourceError(msg or f"libgacq error {rc}")


def cai_stream(cai: dict):
    """The stream a __cuda_array_interface__ producer wrote on, per the CAI v3 contract: None
    when the producer says no synchronisation is needed, else a cudaStream_t handle (1 = the
    legacy default stream, 2 = per-thread default). Producers without a "stream" key (v2) are
    treated as writing on the legacy default stream."""
    if "stream" not in cai:
        return 1
    st = cai["stream"]
    if st is None:
        return None
    st = int(st)
    return 1 if st == 0 else st


def wait_for_producer(fn, handle, cai: dict) -> None:
    """Order the library's device work after the producer's (gacq_wait_stream /
    gacq_trk_wait_stream) before it reads a device array."""
    st = cai_stream(cai)
    if st is not None:
        check(fn(handle, C.c_void_p(st)))
