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
