"""On-device synthetic snapshot batches through gacq_synth.

The reference builds benchmark inputs on the host, one satellite at a time
(synthesize_signal / add_awgn, gnss_signal.py:136-186; the multi-satellite recipe of
SURVEY.md 8(d)). Here a whole batch is generated in HBM by one kernel:

* the clean signal uses the reference's fixed-point code and carrier NCO words and its
  complex64 rounding, so with ``noise_sigma=0`` each snapshot is bit-identical to summing
  ``synthesize_signal(...) * float32(amp)`` in draw order;
* the AWGN comes from a counter-based Philox stream, not the reference's PCG64 stream, so
  noisy batches are performance inputs only -- never parity inputs.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .acquisition import samples_per_code_period
from .errors import InvalidInputError

SAT_DTYPE = np.dtype([("prn", "<i4"), ("reserved", "<i4"), ("doppler_hz", "<f8"),
                      ("code_phase_samples", "<f8"), ("carrier_phase_cycles", "<f8"),
                      ("amplitude", "<f4"), ("reserved2", "<f4")])
assert SAT_DTYPE.itemsize == C.sizeof(_lib.Sat)


def random_sats(rng: np.random.Generator, n_snap: int, sample_rate_hz: float, n_visible: int = 8,
                cn0_range=(38.0, 48.0), cn0_ref: float = 45.0, doppler_span_hz: float = 4750.0) -> np.ndarray:
    """Satellite draws of the SURVEY.md 8(d) recipe: n_visible distinct PRNs, Doppler
    U(-span, span), integer code phase U[0, P), carrier phase U[0, 1), C/N0 U(cn0_range)
    -> amplitude float32(10**((cn0 - cn0_ref)/20)). Returns a [n_snap, n_visible] SAT_DTYPE array."""
    period = samples_per_code_period(sample_rate_hz)
    sats = np.zeros((n_snap, n_visible), dtype=SAT_DTYPE)
    for s in range(n_snap):
        sats["prn"][s] = rng.choice(np.arange(1, 33), size=n_visible, replace=False)
        sats["doppler_hz"][s] = rng.uniform(-doppler_span_hz, doppler_span_hz, n_visible)
        sats["code_phase_samples"][s] = rng.integers(0, period, n_visible)
        sats["carrier_phase_cycles"][s] = rng.uniform(0.0, 1.0, n_visible)
        cn0 = rng.uniform(cn0_range[0], cn0_range[1], n_visible)
        sats["amplitude"][s] = (10.0 ** ((cn0 - cn0_ref) / 20.0)).astype(np.float32)
    return sats


def synthesize_batch(sats: np.ndarray, sample_rate_hz: float, n_samples: int, out, noise_sigma: float = 0.0,
                     seed: int = 0, device: int = 0):
    """Fill ``out`` (a CUDA complex64 array [n_snap, n_samples], any object with
    ``__cuda_array_interface__``, e.g. a torch tensor) with the snapshots described by
    ``sats`` ([n_snap, n_sat] SAT_DTYPE). Returns ``out``."""
    sats = np.ascontiguousarray(sats, dtype=SAT_DTYPE)
    if sats.ndim != 2:
        raise InvalidInputError("sats must be [n_snap, n_sat]")
    cai = getattr(out, "__cuda_array_interface__", None)
    if cai is None or cai["typestr"] != "<c8":
        raise InvalidInputError("out must be a complex64 CUDA array")
    shape = tuple(cai["shape"])
    strides = cai.get("strides")
    if shape != (sats.shape[0], n_samples) or (strides and tuple(strides) != (8 * n_samples, 8)):
        raise InvalidInputError(f"out must be a contiguous [{sats.shape[0]}, {n_samples}] array")
    _lib.check(_lib.lib.gacq_synth(device, float(sample_rate_hz), sats.shape[0], n_samples, sats.shape[1],
                                   sats.ctypes.data, float(noise_sigma), int(seed) & (2**64 - 1),
                                   cai["data"][0]))
    return out
