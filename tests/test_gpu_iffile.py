"""GPU parity of the IF-ingest path: integer I/Q payloads are
dequantized on the device (float32(float64(q) * scale/limit), iffile.py:95-98) and must give
the reference's read_if_file -> acquire_all results."""

import tempfile
from pathlib import Path

import numpy as np
import pytest

import oracle
from golden_cases import case, if_bytes, if_decoded, load_cases
from parity import compare

pytestmark = pytest.mark.gpu
IF_CASES = [c["name"] for c in load_cases() if c["kind"] == "iffile"]


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


def check(results, c):
    for g, r in zip(results, c["results"]):
        gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples,
                  peak_metric=g.peak_metric, detected=g.detected)
        assert g.prn == r["prn"]
        assert compare(gd, r, c["config"]["detection_threshold"]) == "exact", (c["name"], g, r)


@pytest.mark.parametrize("name", IF_CASES)
def test_acquire_if_file_matches_reference(pkg, name):
    c = case(name)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "snap.gnssif"
        p.write_bytes(if_bytes(c))
        res = pkg.acquire_if_file(p, c["prns"], pkg.AcqConfig(**c["config"]))
    check(res, c)


@pytest.mark.parametrize("name", [n for n in IF_CASES if "float32" not in n])
def test_quantized_rows_equal_host_dequantized_rows(pkg, name):
    # device dequantization is bit-identical to read_if_file, so the rows must be identical
    c = case(name)
    fs, samples, fmt, scale, ints = if_decoded(c)
    eng = pkg.get_engine(fs, c["prns"], pkg.AcqConfig(**c["config"]))
    rows_q = eng.run_rows_quantized(ints, fmt, scale)
    rows_f = eng.run_rows(samples)
    np.testing.assert_array_equal(rows_q, rows_f)


def test_quantized_batch_strided_and_device(pkg):
    import torch

    c = case("if_int8_c3")
    fs, samples, fmt, scale, ints = if_decoded(c)
    eng = pkg.get_engine(fs, c["prns"], pkg.AcqConfig(**c["config"]))
    one = eng.run_rows_quantized(ints, fmt, scale)
    wide = np.zeros((3, ints.size + 64), dtype=np.int8)
    wide[:, :ints.size] = ints
    np.testing.assert_array_equal(eng.run_rows_quantized(wide, fmt, scale), np.repeat(one, 3, axis=0))
    dev = torch.from_numpy(wide).cuda()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.run_rows_quantized(dev, fmt, scale), np.repeat(one, 3, axis=0))
    st = eng.stats()
    assert st["launches"] > 0
    with pytest.raises(pkg.InvalidInputError):
        eng.run_rows_quantized(ints.astype(np.int16), fmt, scale)


@pytest.mark.parametrize("name", [n for n in IF_CASES if "float32" not in n])
def test_quantized_misaligned_device_and_generic_path(pkg, name):
    # K1 dequantizes in its wipe load: an I/Q buffer whose start is not load-aligned takes the
    # per-sample path, and the generic (non-prime-factor) plan keeps the staging dequant kernel;
    # both must give the rows of the host-dequantized samples
    import torch

    c = case(name)
    fs, samples, fmt, scale, ints = if_decoded(c)
    eng = pkg.get_engine(fs, c["prns"], pkg.AcqConfig(**c["config"]))
    want = eng.run_rows(samples)
    isz = ints.dtype.itemsize
    raw = torch.zeros(ints.size * isz + 64, dtype=torch.uint8, device="cuda")
    off = 2 * isz  # one I/Q pair: aligned to the element, not to the 2-pair load
    raw[off:off + ints.size * isz] = torch.from_numpy(ints.view(np.uint8).copy()).cuda()
    view = raw[off:off + ints.size * isz].view(torch.int8 if isz == 1 else torch.int16)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.run_rows_quantized(view, fmt, scale), want)
    gen = pkg.AcqEngine(fs, c["prns"], pkg.AcqConfig(**c["config"]), force_generic=True)
    np.testing.assert_array_equal(gen.run_rows_quantized(ints, fmt, scale), gen.run_rows(samples))
    gen.close()


@pytest.mark.parametrize("seed", range(6))
def test_quantized_random_scales_equal_host_dequantized(pkg, seed):
    # random full-scale values (1e-3 .. 1e4) and both integer formats: K1's in-register
    # dequantization (int8 via its shared-memory table, int16 by DMUL) gives exactly the rows of
    # the host-side float32(float64(q) * scale / limit) samples (iffile.py:95-98)
    rng = np.random.default_rng(700 + seed)
    fs = [4.092e6, 8.184e6, 2.046e6][seed % 3]
    fmt = seed % 2  # 0: int8, 1: int16
    limit = 127.0 if fmt == 0 else 32767.0
    scale = float(10.0 ** rng.uniform(-3, 4))
    cfg = pkg.AcqConfig(doppler_min_hz=-2000.0, doppler_max_hz=2000.0, doppler_step_hz=500.0, noncoherent_rounds=2)
    x, _ = oracle.make_snapshot(seed, fs, 2e-3, base_seed=4400)
    iq = np.stack([x.real, x.imag], -1).reshape(1, -1) / np.abs(x).max() * limit * 0.9
    q = np.clip(np.round(iq), -limit, limit).astype(np.int8 if fmt == 0 else np.int16)
    host = (q.astype(np.float64) * (scale / limit)).astype(np.float32).reshape(1, -1, 2)
    samples = (host[..., 0] + 1j * host[..., 1]).astype(np.complex64)
    eng = pkg.get_engine(fs, list(range(1, 33)), cfg)
    np.testing.assert_array_equal(eng.run_rows_quantized(q, fmt, scale), eng.run_rows(samples))
