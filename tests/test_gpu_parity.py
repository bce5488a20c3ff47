"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden outputs and
the pinned CPU oracle. Needs a B200 and the built libgacq.so."""

import math

import numpy as np
import pytest

import oracle
from golden_cases import case, case_input, load_cases, load_maps, oracle_config
from parity import compare, record

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


def to_cfg(pkg, c):
    return pkg.AcqConfig(**c["config"])


def run_case(pkg, c):
    x = case_input(c)
    eng = pkg.get_engine(c["fs"], c["prns"], to_cfg(pkg, c))
    res = eng.search(x).results()[0]
    return [dict(prn=r.prn, doppler_hz=r.doppler_hz, code_phase_samples=r.code_phase_samples,
                 peak_metric=r.peak_metric, detected=r.detected, bins_searched=r.bins_searched,
                 multiplications_performed=r.multiplications_performed) for r in res]


@pytest.mark.parametrize("name", [c["name"] for c in load_cases()])
def test_golden_case(pkg, name):
    # every golden runs, including the 65536-point generic transforms of 20 MHz, 16.367 MHz x
    # 2 ms, 8.192 MHz x 5 ms and the chip-aligned D = 20 / 32 rates (8-CTA clusters)
    c = case(name)
    got = run_case(pkg, c)
    cfg = oracle_config(c)
    bins = cfg.doppler_bins_hz()
    for g, r in zip(got, c["results"]):
        assert g["prn"] == r["prn"]
        assert g["bins_searched"] == r["bins_searched"]
        assert g["multiplications_performed"] == r["multiplications_performed"]
        verdict = compare(g, r, c["config"]["detection_threshold"])
        if verdict not in ("exact", "tie"):
            pmap = oracle.acquire_channel(case_input(c), c["fs"], r["prn"], cfg, want_map=True)["power_map"]
            verdict = compare(g, r, c["config"]["detection_threshold"], pmap, bins)
        assert verdict in ("exact", "tie"), f"{name} prn {r['prn']}: {verdict}"
        record("test_golden_case", name, r["prn"], verdict)  # ties only on ALLOWED_TIES inputs


def test_power_maps_match_reference(pkg):
    for key, ref_map in load_maps().items():
        name, prn = key.rsplit("__prn", 1)
        c = case(name)
        eng = pkg.get_engine(c["fs"], [int(prn)], to_cfg(pkg, c))
        got = eng.power_map(case_input(c))[0]
        assert got.shape == ref_map.shape
        scale = ref_map.max(axis=1, keepdims=True)
        err = np.abs(got - ref_map) / scale
        assert err.max() < 2e-6, (key, float(err.max()))
        assert np.all(np.abs(got - ref_map) <= 1e-4 * np.abs(ref_map) + 2e-6 * scale)


def test_rows_per_bin_merge_equals_reduced_rows(pkg):
    c = case("c3_snap1")
    eng = pkg.get_engine(c["fs"], c["prns"], to_cfg(pkg, c))
    x = case_input(c)
    per_bin = eng.run_rows(x, per_bin=True)[0]
    rows = eng.run_rows(x)[0]
    for p in range(per_bin.shape[0]):
        r = per_bin[p]
        best = max(range(r.shape[0]), key=lambda b: (r[b]["peak"], -b))
        assert tuple(r[best]) == tuple(rows[p])
        assert np.all(r["bin"] == np.arange(r.shape[0]))


def test_batch_equals_single_snapshot_runs(pkg):
    names = [f"c3_snap{i}" for i in range(8)]
    cs = [case(n) for n in names]
    eng = pkg.get_engine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]))
    batch = np.stack([case_input(c) for c in cs])
    rows = eng.run_rows(batch)
    for i, c in enumerate(cs):
        np.testing.assert_array_equal(rows[i], eng.run_rows(case_input(c))[0])
    # a strided view (rows longer than needed) gives the same answer
    wide = np.zeros((len(cs), batch.shape[1] + 1000), dtype=np.complex64)
    wide[:, :batch.shape[1]] = batch
    np.testing.assert_array_equal(eng.run_rows(wide), rows)


def test_device_resident_input(pkg):
    import torch

    cs = [case(f"c3_snap{i}") for i in range(4)]
    eng = pkg.get_engine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]))
    host = np.stack([case_input(c) for c in cs])
    dev = torch.from_numpy(host).cuda()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.run_rows(dev), eng.run_rows(host))


def test_reference_api_semantics(pkg):
    c = case("ka_prn5_1500_4000")
    buf = pkg.IqBuffer(case_input(c), c["fs"])
    r = pkg.acquire_channel(buf, pkg.generate_ca_code(5), pkg.AcqConfig())
    assert r.detected and r.code_phase_samples == 4000 and r.prn == 5
    assert abs(r.doppler_hz - 1500.0) <= pkg.AcqConfig().doppler_step_hz / 2
    assert r.multiplications_performed == r.bins_searched * 10 * 2 * 8184
    prns = list(range(1, 13))
    allr = pkg.acquire_all(buf, prns, pkg.AcqConfig())
    assert [x.prn for x in allr] == prns
    assert allr[4] == r  # channel 5 identical to the single-channel call
    for p, x in zip(prns, allr):
        assert x == pkg.acquire_channel(buf, pkg.generate_ca_code(p), pkg.AcqConfig())


def test_large_batch_properties(pkg):
    """Full C3 batch size (1024 snapshots): size-independent properties. The batch is
    built from 8 golden snapshots tiled with per-row scaling (power scales by a^2, so the
    winning cell is invariant and the metric is scale-free)."""
    cs = [case(f"c3_snap{i}") for i in range(8)]
    eng = pkg.get_engine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]))
    base = np.stack([case_input(c) for c in cs])
    ref = eng.run_rows(base)
    scales = np.float32(2.0) ** np.arange(-4, 4, dtype=np.float32)
    batch = np.concatenate([base * s for s in scales] * 16).astype(np.complex64)
    assert batch.shape[0] == 1024
    rows = eng.run_rows(batch)
    for k in range(1024):
        r, q = rows[k], ref[k % 8]
        np.testing.assert_array_equal(r["bin"], q["bin"])
        np.testing.assert_array_equal(r["lag"], q["lag"])
        s2 = np.float32(scales[(k // 8) % 8]) ** 2
        np.testing.assert_allclose(r["peak"], q["peak"] * s2, rtol=1e-5)


def test_visible_satellites_found(pkg):
    # strong (>= 44 dB-Hz) satellites are acquired at their true code phase within one bin
    hits = total = 0
    misses = []
    for i in range(8):
        c = case(f"c3_snap{i}")
        res = run_case(pkg, c)
        by_prn = {r["prn"]: r for r in res}
        step = c["config"]["doppler_step_hz"]
        for prn, dop, cph, _carr, cn0 in c["spec"]["truth"]:
            if cn0 < 44:
                continue
            total += 1
            r = by_prn[prn]
            ok = (r["detected"] and r["code_phase_samples"] == cph
                  and abs(r["doppler_hz"] - dop) <= step + 1e-9)
            hits += ok
            if not ok:
                misses.append((i, prn, round(dop, 1), cph, round(cn0, 1), r["doppler_hz"],
                               r["code_phase_samples"], round(r["peak_metric"], 2)))
    assert total > 10 and hits >= 0.9 * total, (hits, total, misses)


@pytest.mark.parametrize("cn0", [30.0, 33.0, 36.0, 39.0, 42.0, 45.0])
def test_c5_weak_signal_sweep_decisions(pkg, cn0):
    """BASELINE C5: decisions at C/N0 30-45 dB-Hz vs the CPU oracle on the same inputs
    (C3 grid, 32 PRNs, 4 snapshots per point): (bin, lag) and `detected` exact except
    float32-indistinguishable ties (tests/parity.py)."""
    fs = 4.092e6
    kw = dict(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0, noncoherent_rounds=10)
    ocfg = oracle.OracleConfig(**kw)
    eng = pkg.get_engine(fs, list(range(1, 33)), pkg.AcqConfig(**kw))
    snaps = [oracle.make_snapshot(i, fs, 10e-3, base_seed=7000 + int(cn0) * 10, cn0_range=(cn0, cn0))[0]
             for i in range(4)]
    got = eng.search(np.stack(snaps)).results()
    exact = 0
    for i, (x, res) in enumerate(zip(snaps, got)):
        ref = oracle.acquire_all(x, fs, range(1, 33), ocfg)
        for g, r in zip(res, ref):
            gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples,
                      peak_metric=g.peak_metric, detected=g.detected)
            v = compare(gd, r, ocfg.detection_threshold)
            if v not in ("exact", "tie"):
                pm = oracle.acquire_channel(x, fs, r["prn"], ocfg, want_map=True)["power_map"]
                v = compare(gd, r, ocfg.detection_threshold, pm, ocfg.doppler_bins_hz())
            assert v in ("exact", "tie"), f"cn0 {cn0} prn {r['prn']}: {v}"
            record("test_c5_weak_signal_sweep_decisions", f"c5_cn{int(cn0)}_snap{i}", r["prn"], v)
            exact += v == "exact"
    assert exact == 4 * 32, exact


def test_acquire_batch_over_device_list(pkg):
    """acquire_batch shards snapshots over `devices` (one host thread each); with the one
    visible GPU listed twice the shards run concurrently on two plans of the same device."""
    cs = [case(f"c3_snap{i}") for i in range(5)]
    cfg = pkg.AcqConfig(**cs[0]["config"])
    batch = np.stack([case_input(c) for c in cs])
    got = pkg.acquire_batch(batch, cs[0]["fs"], list(range(1, 33)), cfg, devices=[0, 0])
    assert len(got) == 5
    for res, c in zip(got, cs):
        for g, r in zip(res, c["results"]):
            gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples,
                      peak_metric=g.peak_metric, detected=g.detected)
            assert compare(gd, r, c["config"]["detection_threshold"]) == "exact"


def test_plans_with_different_rates_coexist(pkg):
    """Kernel attributes are process-wide: creating a D=2 plan after a D=4 one must not
    break the D=4 plan (regression: launch 'invalid argument')."""
    cfg = pkg.AcqConfig(doppler_step_hz=500.0, noncoherent_rounds=1)
    rates = (4.092e6, 2.046e6, 16.368e6, 8.184e6)
    engines = [pkg.AcqEngine(fs, [1, 2], cfg) for fs in rates]
    for fs, eng in zip(rates, engines):
        x = oracle.make_snapshot(0, fs, 1e-3, base_seed=31)[0]
        rows = eng.run_rows(x)
        assert rows.shape == (1, 2)
    for eng in engines:
        eng.close()


GENERIC_ON_ALIGNED = ["c1_snap0", "c1_snap1", "c3_snap0", "coh2_snap0", "fs8_snap0", "radius10_snap1",
                      "direct_full_2046k", "zeros_c1", "noise_seed0", "ka_prn5_1500_4000",
                      "c4_snap0"]  # 16.368 MHz: M = 32768, a 4-CTA cluster transform


@pytest.mark.parametrize("name", GENERIC_ON_ALIGNED)
def test_generic_path_on_chip_aligned_cases(pkg, name):
    # the generic path (gacq_generic.cuh) that serves rates which are not chip-aligned,
    # forced onto chip-aligned golden cases: same reference answers as the 1023-point path
    c = case(name)
    eng = pkg.AcqEngine(c["fs"], c["prns"], to_cfg(pkg, c), force_generic=True)
    assert eng.info["path"] == 4 and eng.info["fft_len"] >= eng.info["n_coh"] + eng.info["samples_per_period"] - 1
    res = eng.search(case_input(c)).results()[0]
    cfg = oracle_config(c)
    for g, r in zip(res, c["results"]):
        gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples, peak_metric=g.peak_metric,
                  detected=g.detected)
        verdict = compare(gd, r, c["config"]["detection_threshold"])
        if verdict not in ("exact", "tie"):
            pmap = oracle.acquire_channel(case_input(c), c["fs"], r["prn"], cfg, want_map=True)["power_map"]
            verdict = compare(gd, r, c["config"]["detection_threshold"], pmap, cfg.doppler_bins_hz())
        assert verdict in ("exact", "tie"), f"{name} prn {r['prn']}: {verdict}"
        record("test_generic_path_on_chip_aligned_cases", name, r["prn"], verdict)
    eng.close()


def test_generic_rates_use_the_generic_path(pkg):
    for fs in (5.0e6, 2.5e6, 8.192e6, 3.0e6, 6.0e6):
        eng = pkg.AcqEngine(fs, [1], pkg.AcqConfig(noncoherent_rounds=1))
        assert eng.info["path"] == 4, (fs, eng.info)
        eng.close()
    eng = pkg.AcqEngine(4.092e6, [1], pkg.AcqConfig(noncoherent_rounds=1))
    assert eng.info["path"] == 2
    eng.close()


@pytest.mark.parametrize("coherent_ms,fft_len", [(1, 8192), (2, 16384), (4, 32768), (8, 65536)])
def test_power_of_two_rate_runs_the_circular_transform(pkg, coherent_ms, fft_len):
    # 8.192 MHz: n_coh = 8192 * coherent_ms is a power of two, so the reference's n_coh-point
    # circular correlation is the M = n_coh transform itself (no extension; clusters of M / 8192)
    fs = 8.192e6
    cfg = pkg.AcqConfig(doppler_min_hz=-1000.0, doppler_max_hz=1000.0, doppler_step_hz=250.0,
                        coherent_ms=coherent_ms, noncoherent_rounds=2)
    ocfg = oracle.OracleConfig(doppler_min_hz=-1000.0, doppler_max_hz=1000.0, doppler_step_hz=250.0,
                               coherent_ms=coherent_ms, noncoherent_rounds=2)
    x = oracle.synthesize_signal(7, 430.0, 2222, 0.3, fs, 2 * coherent_ms * 1e-3,
                                 oracle.sigma_for_cn0_dbhz(44.0, fs), 77)
    prns = [7, 12, 30]
    eng = pkg.AcqEngine(fs, prns, cfg)
    assert eng.info["path"] == 4 and eng.info["fft_len"] == fft_len
    res = eng.search(x).results()[0]
    assert res[0].detected and res[0].code_phase_samples == 2222
    for g, prn in zip(res, prns):
        r = oracle.acquire_channel(x, fs, prn, ocfg, want_map=True)
        gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples, peak_metric=g.peak_metric,
                  detected=g.detected)
        verdict = compare(gd, r, ocfg.detection_threshold, r["power_map"], ocfg.doppler_bins_hz())
        assert verdict in ("exact", "tie"), f"{coherent_ms} ms prn {prn}: {verdict}"
        record("test_power_of_two_rate_runs_the_circular_transform", f"p2_8M192_{coherent_ms}ms", prn, verdict)
    eng.close()


@pytest.mark.parametrize("n_snap", [1, 3, 17, 40])
def test_chunked_staging_matches_device_resident(pkg, n_snap):
    # a small spectrum scratch forces many compute chunks (a short first one, then full ones)
    # and 16-snapshot copy events; staged host input and device input give identical rows
    import torch

    cs = [case(f"c3_snap{i}") for i in range(8)]
    host = np.stack([case_input(cs[i % 8]) for i in range(n_snap)])
    small = pkg.AcqEngine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]), scratch_bytes=24 << 20)
    big = pkg.get_engine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]))
    ref = big.run_rows(torch.from_numpy(host).cuda())
    np.testing.assert_array_equal(small.run_rows(host), ref)
    pinned = pkg.PinnedBuffer(host.shape)
    pinned.array[...] = host
    np.testing.assert_array_equal(small.run_rows(pinned.array), ref)
    pinned.close()
    small.close()


@pytest.mark.parametrize("name,n_dev", [("c2_snap0", 3), ("c4_snap0", 2), ("ka_prn5_1500_4000", 4), ("gen5M_snap0", 2)])
def test_doppler_bin_sharding_equals_whole_grid(pkg, name, n_dev):
    # one snapshot, contiguous Doppler-bin ranges per device (here all on device 0),
    # rows merged exactly -- identical to the single-plan search and to the reference
    c = case(name)
    x = case_input(c)
    cfg = to_cfg(pkg, c)
    whole = pkg.get_engine(c["fs"], c["prns"], cfg).search(x)
    shard = pkg.acquire_bins_sharded(x, c["fs"], c["prns"], cfg, devices=[0] * n_dev)
    for k in ("bin_index", "code_phase_samples", "peak", "floor", "peak_metric", "detected"):
        np.testing.assert_array_equal(getattr(shard, k), getattr(whole, k), err_msg=k)
    for g, r in zip(shard.results()[0], c["results"]):
        assert (g.doppler_hz, g.code_phase_samples, g.detected) == (r["doppler_hz"], r["code_phase_samples"],
                                                                    r["detected"])


def test_concurrent_host_threads_on_one_plan(pkg):
    # calls on one context are serialized inside libgacq (the GIL is released by ctypes), so
    # several host threads sharing a plan get exactly the sequential answers
    import threading

    cs = [case(f"c3_snap{i}") for i in range(8)]
    eng = pkg.get_engine(cs[0]["fs"], cs[0]["prns"], to_cfg(pkg, cs[0]))
    xs = [case_input(c) for c in cs]
    want = [eng.run_rows(x) for x in xs]
    got = [None] * 32
    errs = []

    def work(i):
        try:
            got[i] = eng.run_rows(xs[i % 8])
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(32)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs[0]
    for i in range(32):
        np.testing.assert_array_equal(got[i], want[i % 8])


# exclusion radii around the K2 floor's two forms (gacq_pfa.cuh): phase summaries while
# 2 r < 33 D (every window holds <= 33 chip lags), the full per-phase rows beyond; the
# boundary pair at each D, the default one chip, and windows wider than the whole code
RADIUS_CASES = [(4.092e6, r) for r in (1, 4, 10, 64, 65, 66, 67, 200, 2000, 2045, 2046)] + \
               [(8.184e6, r) for r in (8, 131, 132, 500)] + [(16.368e6, r) for r in (16, 263, 264)]


@pytest.mark.parametrize("rounds", [2, 1])  # R = 1 also selects K2's kR1 instantiation (summaries)
@pytest.mark.parametrize("fs,radius", RADIUS_CASES)
def test_exclusion_radius_floor_forms(pkg, fs, radius, rounds):
    kw = dict(doppler_min_hz=-2000.0, doppler_max_hz=2000.0, doppler_step_hz=500.0, noncoherent_rounds=rounds,
              exclusion_radius_samples=radius)
    ocfg = oracle.OracleConfig(**kw)
    bins = ocfg.doppler_bins_hz()
    for snap in range(2):
        x, _ = oracle.make_snapshot(snap, fs, 2e-3, base_seed=8080 + radius)
        eng = pkg.get_engine(fs, list(range(1, 33)), pkg.AcqConfig(**kw))
        got = eng.search(x).results()[0]
        ref = oracle.acquire_all(x, fs, range(1, 33), ocfg)
        for g, r in zip(got, ref):
            gd = dict(doppler_hz=g.doppler_hz, code_phase_samples=g.code_phase_samples, peak_metric=g.peak_metric,
                      detected=g.detected)
            v = compare(gd, r, kw.get("detection_threshold", 2.5))
            if v != "exact":
                pm = oracle.acquire_channel(x, fs, r["prn"], ocfg, want_map=True)["power_map"]
                v = compare(gd, r, 2.5, pm, bins)
            assert v == "exact", (fs, radius, snap, r["prn"], v)
