"""C-ABI boundary and host logic -- CPU only (no kernel launches)."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def pkg():
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


def declared_symbols():
    hdr = (ROOT / "include" / "gacq.h").read_text()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(gacq_\w+)\(", hdr, re.M)))


def test_library_exports_every_declared_symbol(pkg):
    from paper_1309_0052_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 12
    lib = C.CDLL(str(_lib.LIB_PATH))
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.gacq_version() == _lib.ABI_VERSION == 2


def test_library_is_sm100a_only(pkg):
    import subprocess

    from paper_1309_0052_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_ca_codes_match_oracle(pkg):
    for prn in range(1, 33):
        np.testing.assert_array_equal(pkg.generate_ca_code(prn).chips, oracle.generate_ca_code(prn))
    with pytest.raises(pkg.InvalidInputError):
        pkg.generate_ca_code(0)


def test_config_validation_mirrors_reference(pkg):
    cfg = pkg.AcqConfig()
    assert cfg.doppler_step_hz == pytest.approx(2000.0 / 3.0)
    np.testing.assert_array_equal(cfg.doppler_bins_hz(), oracle.OracleConfig().doppler_bins_hz())
    for bad in (dict(doppler_min_hz=1.0, doppler_max_hz=-1.0), dict(detection_threshold=1.0),
                dict(noncoherent_rounds=0), dict(coherent_ms=0, doppler_step_hz=100.0),
                dict(exclusion_radius_samples=-1),
                dict(doppler_step_hz=-5.0)):
        with pytest.raises(pkg.InvalidInputError):
            pkg.AcqConfig(**bad)
    c = pkg.AcqConfig(doppler_min_hz=-5000, doppler_max_hz=5000, doppler_step_hz=250)
    assert c.doppler_bins_hz().size == 41


def test_buffer_validation_order_and_messages(pkg):
    cfg = pkg.AcqConfig()
    short = pkg.IqBuffer(np.ones(100, dtype=np.complex64), 8.184e6)
    with pytest.raises(pkg.InvalidInputError, match="shorter than one code period"):
        pkg.acquire_channel(short, pkg.CaCode(1, oracle.generate_ca_code(1)), cfg)
    one_ms = pkg.IqBuffer(np.ones(8184, dtype=np.complex64), 8.184e6)
    with pytest.raises(pkg.InvalidInputError, match="8184 samples, 81840 needed"):
        pkg.acquire_channel(one_ms, pkg.CaCode(1, oracle.generate_ca_code(1)), cfg)
    with pytest.raises(pkg.PipelineError, match="channel 7"):
        pkg.acquire_all(one_ms, [7], cfg)
    with pytest.raises(pkg.PipelineError, match="channel 40"):
        pkg.acquire_all(one_ms, [40], cfg)
    with pytest.raises(pkg.InvalidInputError):
        pkg.acquire_all(one_ms, [], cfg)
    with pytest.raises(pkg.InvalidInputError):
        pkg.acquire_all(one_ms, [1, 1], cfg)
    dbl = pkg.IqBuffer(np.ones(81840), 8.184e6, pkg.Precision.DOUBLE)
    with pytest.raises(pkg.UnsupportedError):
        pkg.acquire_channel(dbl, pkg.CaCode(1, oracle.generate_ca_code(1)), cfg)


def test_create_rejects_oversized_generic_rate_before_touching_a_device(pkg):
    # 40.1 MHz: n_coh = 40100 = 4 * 25 * 401 is not 2^a 3^b 5^c, and the power-of-two linear
    # transform (n_coh + P - 1 -> 131072 points) exceeds the 8-CTA cluster (65536): refused
    # loudly, never a CPU path
    with pytest.raises(pkg.UnsupportedError, match="generic path"):
        pkg.AcqEngine(40.1e6, [1], pkg.AcqConfig())
    # 16.367 MHz with 4 ms coherent: 65468 = 4 * 13 * 1259, linear form 81834 points: refused
    # (2 ms, 32734 + 16367 - 1 -> 65536 points, runs)
    with pytest.raises(pkg.UnsupportedError, match="generic path"):
        pkg.AcqEngine(16.367e6, [1], pkg.AcqConfig(coherent_ms=4))


def test_create_without_gpu_raises_resource_error(pkg):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.ResourceError, match="no CUDA device"):
        pkg.AcqEngine(4.092e6, [1, 2], pkg.AcqConfig(noncoherent_rounds=1))


def test_finish_metric_semantics(pkg):
    # acquisition.py:160-161: float64 peak/floor, inf when floor == 0, detected = metric >= thr
    from paper_1309_0052_b200 import _lib
    from paper_1309_0052_b200.acquisition import AcqEngine

    eng = object.__new__(AcqEngine)
    eng.prns = np.array([3, 4], dtype=np.int32)
    eng.bins = np.array([-500.0, 0.0, 500.0])
    eng.config = pkg.AcqConfig(detection_threshold=2.5)
    eng.mults = 123
    rows = np.zeros((1, 2), dtype=_lib.ROW_DTYPE)
    rows[0, 0] = (2, 17, np.float32(5.0), np.float32(2.0))
    rows[0, 1] = (0, 0, np.float32(0.0), np.float32(0.0))
    r = eng.finish(rows).results()[0]
    assert r[0] == pkg.AcqResult(3, 500.0, 17, 2.5, True, 3, 123)
    assert r[1].peak_metric == float("inf") and r[1].detected
    eng._ctx = None


@pytest.mark.parametrize("fs,n", [(4.092e6, 4092), (8.184e6, 16368), (5.0e6, 5000), (2.046e6, 2046)])
def test_conjugate_code_spectrum_drop_in(pkg, fs, n):
    # acquisition.py:88-105: same bins as the pinned oracle (which restates the reference bit for
    # bit), complex64 for SINGLE, read-only and cached; DOUBLE gives the complex128 spectrum
    got = pkg.conjugate_code_spectrum(7, fs, n, pkg.Precision.SINGLE)
    from oracle import gnss_oracle

    want = gnss_oracle.conjugate_code_spectrum(7, fs, n)
    assert got.dtype == np.complex64 and not got.flags.writeable
    np.testing.assert_array_equal(got, want)
    assert pkg.conjugate_code_spectrum(7, fs, n, pkg.Precision.SINGLE) is got
    dbl = pkg.conjugate_code_spectrum(7, fs, n, pkg.Precision.DOUBLE)
    assert dbl.dtype == np.complex128
    np.testing.assert_allclose(dbl, want.astype(np.complex128), rtol=0, atol=1e-3)


def test_conjugate_code_spectrum_equals_reference_itself(pkg):
    # in the build container the reference package is importable: compare with its own function
    import sys
    from pathlib import Path

    src = Path("/root/reference/pkg/src")
    if not src.exists():
        pytest.skip("reference sources not present (GPU box)")
    sys.path.insert(0, str(src))
    try:
        from gnssperf import acquisition as ref_acq
        from gnssperf.buffers import Precision as RefPrecision
    except Exception as exc:  # noqa: BLE001 - optional dependency chain
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(str(src))
    for fs, n, prn in ((4.092e6, 4092, 3), (8.184e6, 8184, 31), (5.0e6, 10000, 12)):
        np.testing.assert_array_equal(pkg.conjugate_code_spectrum(prn, fs, n, pkg.Precision.SINGLE),
                                      ref_acq.conjugate_code_spectrum(prn, fs, n, RefPrecision.SINGLE))
        np.testing.assert_array_equal(pkg.conjugate_code_spectrum(prn, fs, n, pkg.Precision.DOUBLE),
                                      ref_acq.conjugate_code_spectrum(prn, fs, n, RefPrecision.DOUBLE))
