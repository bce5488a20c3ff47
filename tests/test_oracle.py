"""Pin the CPU oracle to the reference's own outputs (golden fixtures). CPU only."""

import math

import numpy as np
import pytest

import oracle
from golden_cases import case, case_input, load_cases, load_maps, oracle_config, sha

FAST = [c["name"] for c in load_cases()]


def test_golden_fixture_shape():
    cases = load_cases()
    assert len(cases) >= 40
    kinds = {c["kind"] for c in cases}
    assert {"synth", "noise", "zeros", "snapshot"} <= kinds


@pytest.mark.parametrize("name", [c["name"] for c in load_cases()])
def test_oracle_regenerates_reference_inputs(name):
    c = case(name)
    x = case_input(c)
    assert x.dtype == np.complex64 and x.shape[0] == c["n_samples"]
    assert sha(x) == c["input_sha256"], "oracle synthesis diverged from the reference"


def _prn_sample(c):
    """The channels the CPU suite re-runs: all of them, except on the C4 cases (1.5 s per
    channel on the oracle), where three planted satellites and one absent PRN stand in; the
    GPU suite checks every channel of those against the same reference results."""
    if c["name"].startswith("c4x_"):
        planted = [t[0] for t in c["spec"]["truth"][:3]]
        absent = [p for p in c["prns"] if p not in {t[0] for t in c["spec"]["truth"]}][:1]
        return [i for i, p in enumerate(c["prns"]) if p in planted + absent]
    return list(range(len(c["prns"])))


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_results_bit_exact(name):
    c = case(name)
    x = case_input(c)
    idx = _prn_sample(c)
    got = oracle.acquire_all(x, c["fs"], [c["prns"][i] for i in idx], oracle_config(c))
    for g, r in zip(got, [c["results"][i] for i in idx]):
        for k in ("prn", "doppler_hz", "code_phase_samples", "detected", "bins_searched",
                  "multiplications_performed"):
            assert g[k] == r[k], (k, g[k], r[k])
        if math.isinf(r["peak_metric"]):
            assert math.isinf(g["peak_metric"])
        else:
            assert g["peak_metric"] == r["peak_metric"]


def test_oracle_power_maps_bit_exact():
    maps = load_maps()
    assert maps
    for key, ref_map in maps.items():
        name, prn = key.rsplit("__prn", 1)
        c = case(name)
        got = oracle.acquire_channel(case_input(c), c["fs"], int(prn), oracle_config(c),
                                     want_map=True)["power_map"]
        np.testing.assert_array_equal(got, ref_map)


def test_known_answer_prn5():
    # PRN 5 / 1500 Hz / 4000 at 8.184 MHz, default config
    r = case("ka_prn5_1500_4000")["results"][0]
    assert r["code_phase_samples"] == 4000 and r["detected"]
    assert r["doppler_hz"] == pytest.approx(1666.666666666666)


def test_ca_codes_balanced_and_distinct():
    codes = [oracle.generate_ca_code(p) for p in range(1, 33)]
    for c in codes:
        assert c.shape == (1023,) and int(c.sum()) in (1, -1)  # Gold code balance
    assert len({c.tobytes() for c in codes}) == 32
    with pytest.raises(ValueError):
        oracle.generate_ca_code(33)


@pytest.mark.parametrize("name", [c["name"] for c in load_cases() if c["kind"] == "iffile"])
def test_if_files_match_reference_bytes(name):
    from golden_cases import if_bytes

    import hashlib

    c = case(name)
    raw = if_bytes(c)
    assert hashlib.sha256(raw).hexdigest() == c["spec"]["file_sha256"]
    # the product's writer / reader mirror the reference byte for byte
    import paper_1309_0052_b200 as g

    _, samples, _, _, _ = oracle.if_file_decode(raw)
    assert sha(samples) == c["input_sha256"]
    import tempfile
    from pathlib import Path

    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "x.gnssif"
        p.write_bytes(raw)
        buf = g.read_if_file(p)
        assert sha(buf.samples) == c["input_sha256"]
        q = Path(td) / "y.gnssif"
        g.write_if_file(q, g.IqBuffer._wrap(oracle.make_snapshot(
            c["spec"]["index"], c["spec"]["fs"], c["spec"]["duration_s"], c["spec"]["base_seed"])[0],
            c["spec"]["fs"], g.Precision.SINGLE), c["spec"]["fmt"])
        assert q.read_bytes() == raw
        with pytest.raises(g.FormatError):
            (Path(td) / "bad").write_bytes(b"NOTGNSS!" + raw[8:])
            g.read_if_file(Path(td) / "bad")
