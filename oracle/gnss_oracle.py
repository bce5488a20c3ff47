"""CPU restatement of the reference acquisition path. TEST INFRASTRUCTURE ONLY.

Restates, with numpy + scipy.fft (the reference's own FFT dependency, scipy
1.18.1 / ducc0 in this image), the arithmetic of:

* ``gnssperf/cacode.py:41-58``          C/A Gold codes (G1 taps 3,10; G2 phase select)
* ``gnssperf/kernels.py:47-70``         48-bit carrier / 42-bit code fixed-point NCO steps
* ``gnssperf/kernels.py:78-90,106-128`` numpy twins: naive complex product, |.|^2,
                                        carrier replica, code chip indices
* ``gnssperf/gnss_signal.py:49-96``     carrier_replica / sample_code_replica
* ``gnssperf/gnss_signal.py:136-186``   gaussian_pairs / add_awgn / synthesize_signal
* ``gnssperf/harness.py:371-373``       sigma_for_cn0_dbhz
* ``gnssperf/acquisition.py:39-70``     AcqConfig defaults + doppler_bins_hz
* ``gnssperf/acquisition.py:84-170``    conjugate code spectrum + acquire_channel
* ``gnssperf/acquisition.py:190-208``   acquire_all (validation + ordering)

Every floating-point operation is performed in the same order and precision as
the reference (complex64 pipeline, float32 power map, float64 metric), so the
outputs are bit-identical to the reference on this image; the golden fixtures
under ``tests/golden`` pin that. Nothing here is imported by the product.

Speed: like the reference (kernels.py:134-196, NUMBA_ENABLED), the per-sample
loops -- complex product, |.|^2, carrier NCO -- run as numba-jitted twins when
numba is importable (it is in this image and on the GPU box), so the CPU
baseline times the reference's own execution model, not a slower numpy port.
Both twins give identical bits (explicit float32 component arithmetic, no
contraction); the golden tests run whichever is active.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import fft as _sfft

try:  # the reference's numba twins (kernels.py:134-196); numpy fallbacks below
    from numba import njit as _njit
except ImportError:  # pragma: no cover - numba is in the image
    _njit = None

CODE_LENGTH = 1023  # cacode.py:18
CHIP_RATE_HZ = 1.023e6  # cacode.py:19

# GPS ICD-200 G2 phase-select stage pairs, PRN 1..32 (cacode.py:22-29)
_G2_SELECT = (
    (2, 6), (3, 7), (4, 8), (5, 9), (1, 9), (2, 10), (1, 8), (2, 9),
    (3, 10), (2, 3), (3, 4), (5, 6), (6, 7), (7, 8), (8, 9), (9, 10),
    (1, 4), (2, 5), (3, 6), (4, 7), (5, 8), (6, 9), (1, 3), (4, 6),
    (5, 7), (6, 8), (7, 9), (8, 10), (1, 6), (2, 7), (3, 8), (4, 9),
)

CARRIER_FRAC_BITS = 48  # kernels.py:47-50
CARRIER_SCALE = 1 << CARRIER_FRAC_BITS
CODE_FRAC_BITS = 42  # kernels.py:52-53
CODE_SCALE = 1 << CODE_FRAC_BITS
CODE_MODULUS = CODE_LENGTH * CODE_SCALE
_TWO_PI = 2.0 * math.pi

_chip_cache: dict = {}


def generate_ca_code(prn: int) -> np.ndarray:
    """1023 chips in {+1,-1} (int8) for PRN 1..32 -- cacode.py:41-58.

    Two 10-stage LFSRs from the all-ones state; output bit = G1[10] xor the two
    selected G2 stages; binary 1 maps to +1.
    """
    if not isinstance(prn, (int, np.integer)) or not 1 <= int(prn) <= 32:
        raise ValueError(f"prn must be an integer in 1..32, got {prn!r}")
    prn = int(prn)
    if prn in _chip_cache:
        return _chip_cache[prn]
    a, b = _G2_SELECT[prn - 1]
    g1 = [1] * 10
    g2 = [1] * 10
    out = np.empty(CODE_LENGTH, dtype=np.int8)
    for i in range(CODE_LENGTH):
        out[i] = 1 if (g1[9] ^ g2[a - 1] ^ g2[b - 1]) else -1
        fb1 = g1[2] ^ g1[9]
        fb2 = g2[1] ^ g2[2] ^ g2[5] ^ g2[7] ^ g2[8] ^ g2[9]
        g1 = [fb1] + g1[:9]
        g2 = [fb2] + g2[:9]
    out.setflags(write=False)
    _chip_cache[prn] = out
    return out


# --- fixed-point NCO (kernels.py:56-70) -------------------------------------

def carrier_phase_to_fixed(phase_cycles: float) -> int:
    return int(round((phase_cycles % 1.0) * CARRIER_SCALE)) % CARRIER_SCALE


def carrier_step_to_fixed(freq_hz: float, fs: float) -> int:
    return int(round((freq_hz / fs) * CARRIER_SCALE)) % CARRIER_SCALE


def code_phase_to_fixed(phase_chips: float) -> int:
    return int(round((phase_chips % 1023.0) * CODE_SCALE)) % CODE_MODULUS


def code_step_to_fixed(chip_rate_hz: float, fs: float) -> int:
    return int(round((chip_rate_hz / fs) * CODE_SCALE))


def carrier_replica(phase_cycles: float, freq_hz: float, fs: float, n: int) -> np.ndarray:
    """exp(-2 pi i (p0 + k*step)/2^48) as complex64 -- gnss_signal.py:49-72 +
    kernels.py:106-114 / 175-185 (float64 cos/sin of the exact phase, then
    rounded to complex64 on assignment)."""
    p0 = carrier_phase_to_fixed(phase_cycles)
    step = carrier_step_to_fixed(freq_hz, fs)
    if _njit is not None:
        out = np.empty(n, dtype=np.complex64)
        _carrier_nb(p0, step, n, out)
        return out
    k = np.arange(n, dtype=np.uint64)
    phases = (np.uint64(p0) + k * np.uint64(step)) & np.uint64(CARRIER_SCALE - 1)
    theta = phases.astype(np.float64) * (_TWO_PI / CARRIER_SCALE)
    out = np.empty(n, dtype=np.complex64)
    out.real = np.cos(theta)
    out.imag = -np.sin(theta)
    return out


def code_chip_indices(phase_fixed: int, step_fixed: int, n: int) -> np.ndarray:
    """kernels.py:116-128: floor((p0 + k*step) mod (1023*2^42) / 2^42), chunked
    so the uint64 product never overflows."""
    idx = np.empty(n, dtype=np.int64)
    max_chunk = max(1, (1 << 62) // max(step_fixed, 1))
    pos, p = 0, phase_fixed
    while pos < n:
        c = min(max_chunk, n - pos)
        k = np.arange(c, dtype=np.uint64)
        ph = (np.uint64(p) + k * np.uint64(step_fixed)) % np.uint64(CODE_MODULUS)
        idx[pos:pos + c] = (ph >> np.uint64(CODE_FRAC_BITS)).astype(np.int64)
        p = (p + c * step_fixed) % CODE_MODULUS
        pos += c
    return idx


def code_replica(chips: np.ndarray, phase_chips: float, fs: float, n: int) -> np.ndarray:
    """Floor-indexed +/-1 code replica as complex64 -- gnss_signal.py:75-96."""
    idx = code_chip_indices(code_phase_to_fixed(phase_chips),
                            code_step_to_fixed(CHIP_RATE_HZ, fs), n)
    return chips[idx].astype(np.complex64)


def _cmul_np(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Naive complex64 product, real planes only -- kernels.py:78-86."""
    out = np.empty_like(a)
    out.real = a.real * b.real - a.imag * b.imag
    out.imag = a.real * b.imag + a.imag * b.real
    return out


def _mag2_np(a: np.ndarray) -> np.ndarray:
    """kernels.py:89-90."""
    return a.real * a.real + a.imag * a.imag


if _njit is not None:
    @_njit(cache=True, nogil=True)
    def _cmul_nb(a, b):
        """kernels.py:137-145: the same float32 component formula, one sample at a time."""
        out = np.empty_like(a)
        for i in range(a.shape[0]):
            ar, ai, br, bi = a[i].real, a[i].imag, b[i].real, b[i].imag
            out[i] = complex(ar * br - ai * bi, ar * bi + ai * br)
        return out

    @_njit(cache=True, nogil=True)
    def _mag2_nb(a):
        """kernels.py:147-152."""
        out = np.empty(a.shape[0], dtype=np.float32)
        for i in range(a.shape[0]):
            out[i] = a[i].real * a[i].real + a[i].imag * a[i].imag
        return out

    @_njit(cache=True, nogil=True)
    def _carrier_nb(phase_fixed, step_fixed, n, out):
        """kernels.py:175-185: 48-bit phase accumulator, float64 cos/sin."""
        mask = np.uint64(CARRIER_SCALE - 1)
        p = np.uint64(phase_fixed)
        s = np.uint64(step_fixed)
        inv = _TWO_PI / CARRIER_SCALE
        for i in range(n):
            theta = np.float64(p) * inv
            out[i] = complex(math.cos(theta), -math.sin(theta))
            p = (p + s) & mask

    _cmul, _mag2 = _cmul_nb, _mag2_nb
else:  # pragma: no cover
    _cmul, _mag2 = _cmul_np, _mag2_np


# --- synthesis (gnss_signal.py:136-186, harness.py:371-373) ----------------

def gaussian_pairs(rng: np.random.Generator, n: int):
    u1 = 1.0 - rng.random(n)
    u2 = rng.random(n)
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u2
    return r * np.cos(th), r * np.sin(th)


def add_awgn(samples: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    if sigma == 0:
        return samples
    rng = np.random.Generator(np.random.PCG64(seed))
    zi, zq = gaussian_pairs(rng, samples.shape[0])
    noisy = samples + (sigma * zi + 1j * (sigma * zq)).astype(np.complex64)
    return noisy.astype(np.complex64)


def synthesize_signal(prn: int, doppler_hz: float = 0.0, code_phase_samples: float = 0.0,
                      carrier_phase_cycles: float = 0.0, fs: float = 8.184e6,
                      duration_s: float = 10e-3, noise_sigma: float = 0.0,
                      seed: int = 0) -> np.ndarray:
    """Delayed code x Doppler-rotated carrier (+ AWGN), complex64 -- gnss_signal.py:157-186."""
    n = round(fs * duration_s)
    chips_per_sample = CHIP_RATE_HZ / fs
    code0 = (-code_phase_samples * chips_per_sample) % CODE_LENGTH
    code = code_replica(generate_ca_code(prn), code0, fs, n)
    carrier = carrier_replica((-carrier_phase_cycles) % 1.0, -doppler_hz, fs, n)
    return add_awgn(_cmul(code, carrier), noise_sigma, seed)


def sigma_for_cn0_dbhz(cn0_dbhz: float, fs: float, amplitude: float = 1.0) -> float:
    return amplitude * np.sqrt(fs / (2.0 * 10.0 ** (cn0_dbhz / 10.0)))


def make_snapshot(index: int, fs: float, duration_s: float, base_seed: int = 0,
                  n_visible: int = 8, cn0_range=(38.0, 48.0), cn0_ref: float = 45.0,
                  doppler_span_hz: float = 4750.0):
    """Multi-satellite synthetic snapshot; returns (samples, truth).

    rng = default_rng(base_seed + index); n_visible PRNs without replacement;
    Doppler ~ U(-span, span); integer code phase ~ U[0, P); carrier phase ~ U[0, 1);
    C/N0 ~ U(cn0_range). Each satellite is synthesize_signal(noise_sigma=0) scaled
    by 10**((cn0-cn0_ref)/20) in complex64 and summed in draw order; then
    add_awgn(sum, sigma_for_cn0_dbhz(cn0_ref, fs), seed=base_seed + index).
    cn0_range=(c, c) gives a fixed-C/N0 sweep point.
    """
    rng = np.random.default_rng(base_seed + index)
    period = samples_per_code_period(fs)
    prns = rng.choice(np.arange(1, 33), size=n_visible, replace=False)
    truth = []
    acc = np.zeros(round(fs * duration_s), dtype=np.complex64)
    for prn in prns:
        dop = float(rng.uniform(-doppler_span_hz, doppler_span_hz))
        cph = int(rng.integers(0, period))
        carr = float(rng.uniform(0.0, 1.0))
        cn0 = float(rng.uniform(cn0_range[0], cn0_range[1])) if cn0_range[1] > cn0_range[0] \
            else float(cn0_range[0])
        amp = np.float32(10.0 ** ((cn0 - cn0_ref) / 20.0))
        sig = synthesize_signal(int(prn), dop, cph, carr, fs, duration_s, 0.0, 0)
        acc = (acc + sig * amp).astype(np.complex64)
        truth.append((int(prn), dop, cph, carr, cn0))
    out = add_awgn(acc, float(sigma_for_cn0_dbhz(cn0_ref, fs)), base_seed + index)
    return out, truth


# --- acquisition (acquisition.py:39-208) ------------------------------------

@dataclass(frozen=True)
class OracleConfig:
    """Field-for-field AcqConfig (acquisition.py:44-66)."""

    doppler_min_hz: float = -5000.0
    doppler_max_hz: float = 5000.0
    doppler_step_hz: float = field(default=0.0)
    coherent_ms: int = 1
    noncoherent_rounds: int = 10
    detection_threshold: float = 2.5
    exclusion_radius_samples: int = 0

    def __post_init__(self):
        if self.doppler_step_hz == 0.0:  # default step 2/(3 T_coh): acquisition.py:39-41
            object.__setattr__(self, "doppler_step_hz", 2.0 / (3.0 * self.coherent_ms * 1e-3))

    def doppler_bins_hz(self) -> np.ndarray:
        return doppler_bins_hz(self.doppler_min_hz, self.doppler_max_hz, self.doppler_step_hz)


def doppler_bins_hz(dmin: float, dmax: float, step: float) -> np.ndarray:
    """acquisition.py:68-70."""
    n = int(math.floor((dmax - dmin) / step + 1e-9)) + 1
    return dmin + step * np.arange(n)


def samples_per_code_period(fs: float) -> int:
    """acquisition.py:108-109."""
    return round(fs * CODE_LENGTH / CHIP_RATE_HZ)


_spec_cache: dict = {}


def conjugate_code_spectrum(prn: int, fs: float, n: int) -> np.ndarray:
    """conj(fft(code replica)) in complex64 -- acquisition.py:88-105."""
    key = (prn, float(fs), int(n))
    if key not in _spec_cache:
        rep = code_replica(generate_ca_code(prn), 0.0, fs, n)
        _spec_cache[key] = np.conj(_sfft.fft(rep))
    return _spec_cache[key]


def acquire_channel(samples: np.ndarray, fs: float, prn: int, cfg: OracleConfig,
                    want_map: bool = False) -> dict:
    """acquisition.py:112-170, returning the AcqResult fields (and optionally the
    float32 power map [bins, lag_span] and the winning row's floor)."""
    samples = np.ascontiguousarray(samples, dtype=np.complex64)
    n_coh = round(fs * cfg.coherent_ms * 1e-3)
    period = samples_per_code_period(fs)
    if samples.shape[0] < period:
        raise ValueError("buffer shorter than one code period")
    if samples.shape[0] < n_coh * cfg.noncoherent_rounds:
        raise ValueError(f"buffer holds {samples.shape[0]} samples, "
                         f"{n_coh * cfg.noncoherent_rounds} needed for the configured integration")
    if n_coh < period:
        raise ValueError("coherent window shorter than one code period")
    bins = cfg.doppler_bins_hz()
    cspec = conjugate_code_spectrum(prn, fs, n_coh)
    lag_span = min(period, n_coh)
    pmap = np.zeros((bins.size, lag_span), dtype=np.float32)
    blocks = [samples[r * n_coh:(r + 1) * n_coh] for r in range(cfg.noncoherent_rounds)]
    for bi, f in enumerate(bins):
        rep = carrier_replica(0.0, float(f), fs, n_coh)
        for blk in blocks:
            spec = _sfft.fft(_cmul(blk, rep))
            corr = _sfft.ifft(_cmul(spec, cspec))
            pmap[bi] += _mag2(corr)[:lag_span]
    flat = int(np.argmax(pmap))
    bin_idx, lag = divmod(flat, lag_span)
    peak = float(pmap[bin_idx, lag])
    radius = cfg.exclusion_radius_samples or math.ceil(fs / CHIP_RATE_HZ)
    row = pmap[bin_idx]
    excl = np.abs((np.arange(lag_span) - lag + lag_span // 2) % lag_span - lag_span // 2) <= radius
    outside = row[~excl]
    floor = float(outside.max()) if outside.size else 0.0
    metric = peak / floor if floor > 0 else float("inf")
    res = dict(prn=int(prn), doppler_hz=float(bins[bin_idx]), code_phase_samples=int(lag),
               peak_metric=metric, detected=bool(metric >= cfg.detection_threshold),
               bins_searched=int(bins.size),
               multiplications_performed=2 * n_coh * int(bins.size) * cfg.noncoherent_rounds,
               bin_index=int(bin_idx), peak=peak, floor=floor)
    if want_map:
        res["power_map"] = pmap
    return res


def acquire_all(samples: np.ndarray, fs: float, prns, cfg: OracleConfig,
                want_map: bool = False) -> list:
    """acquisition.py:190-208 (results ordered like prns)."""
    prns = list(prns)
    if not prns:
        raise ValueError("prns must be non-empty")
    if len(set(prns)) != len(prns):
        raise ValueError("prns must be distinct")
    return [acquire_channel(samples, fs, p, cfg, want_map) for p in prns]


# --- IF sample files (iffile.py:34-99) ---------------------------------------

import struct as _struct  # noqa: E402

_IF_HEADER = _struct.Struct("<8sId2B10sd")  # iffile.py:36
_IF_FORMATS = {"int8": 0, "int16": 1, "float32": 2}
_IF_DTYPES = {0: "<i1", 1: "<i2", 2: "<f4"}
_IF_LIMITS = {0: 127, 1: 32767}


def if_file_bytes(samples: np.ndarray, fs: float, sample_format: str) -> bytes:
    """write_if_file (iffile.py:53-71) to bytes: max-|component| full scale for integers."""
    fmt = _IF_FORMATS[sample_format]
    inter = np.empty(2 * samples.shape[0], dtype=np.float64)
    inter[0::2] = samples.real
    inter[1::2] = samples.imag
    if fmt == 2:
        scale = 1.0
        payload = inter.astype("<f4").tobytes()
    else:
        limit = _IF_LIMITS[fmt]
        peak = float(np.max(np.abs(inter))) if inter.size else 0.0
        scale = peak if peak > 0 else 1.0
        q = np.clip(np.round(inter / scale * limit).astype(np.int64), -limit, limit)
        payload = q.astype(_IF_DTYPES[fmt]).tobytes()
    return _IF_HEADER.pack(b"GNSSIF01", 1, fs, fmt, 0, b"\x00" * 10, scale) + payload


def if_file_decode(raw: bytes):
    """read_if_file (iffile.py:74-99): returns (fs, complex64 samples, fmt, scale, raw ints)."""
    magic, version, fs, fmt, layout, _r, scale = _IF_HEADER.unpack_from(raw)
    if magic != b"GNSSIF01" or version != 1 or layout != 0 or fmt not in _IF_DTYPES:
        raise ValueError("bad GNSSIF01 header")
    ints = np.frombuffer(raw[_IF_HEADER.size:], dtype=_IF_DTYPES[fmt])
    if fmt == 2:
        flat = ints.astype(np.float64)
    else:
        flat = ints.astype(np.float64) * (scale / _IF_LIMITS[fmt])
    return fs, (flat[0::2] + 1j * flat[1::2]).astype(np.complex64), fmt, scale, ints
