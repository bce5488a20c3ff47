"""GPU tracking against the reference's tracking goldens.

Replicas are bit-identical to the reference and the E/P/L sums are the reference's own
left-to-right complex64 sums (same float32 addition order), so correlators, discriminators,
NCO states and lock decisions are compared bit for bit, every epoch. A second test keeps
tolerance checks (TRK_RTOL of the epoch's largest correlator) as a readable diagnostic.
"""

import numpy as np
import pytest

from tracking_cases import blocks, case, load

pytestmark = pytest.mark.gpu
TRK_RTOL = 2e-5


@pytest.fixture(scope="module")
def trk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    from paper_1309_0052_b200 import tracking

    return tracking


def to_state(trk, d):
    d = dict(d)
    d["dll_filter_state"] = tuple(d["dll_filter_state"])
    d["pll_filter_state"] = tuple(d["pll_filter_state"])
    return trk.TrackState(**d)


@pytest.mark.parametrize("name", [c["name"] for c in load()])
def test_track_epochs_bit_exact(trk, name):
    """Replicas, wipe-off and the left-to-right complex64 sums are the reference's, and the
    loop closure is the same float64 arithmetic: every epoch must equal the golden bit for bit
    (an ulp difference of the device fp64 cos/sin vs glibc could, rarely, break this; the
    tolerance test below still bounds such cases)."""
    c = case(name)
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    for ch in c["channels"]:
        st = to_state(trk, ch["init"])
        for k, ref in enumerate(ch["epochs"]):
            st, out = trk.track_epoch(bl[k], st, cfg)
            for key in ("ie", "qe", "ip", "qp", "il", "ql", "dll_error_chips", "pll_error_cycles", "lock_metric"):
                assert getattr(out, key) == ref[key], (name, k, key)
            for key in ("code_phase_chips", "carrier_phase_cycles", "doppler_hz", "code_rate_hz", "lock_nbd",
                        "lock_nbp"):
                assert getattr(st, key) == ref["state"][key], (name, k, key)


@pytest.mark.parametrize("name", [c["name"] for c in load()])
def test_track_epochs_match_reference(trk, name):
    c = case(name)
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    for ch in c["channels"]:
        st = to_state(trk, ch["init"])
        for k, ref in enumerate(ch["epochs"]):
            st, out = trk.track_epoch(bl[k], st, cfg)
            got = np.array([out.ie, out.qe, out.ip, out.qp, out.il, out.ql])
            want = np.array([ref[x] for x in ("ie", "qe", "ip", "qp", "il", "ql")])
            scale = np.abs(want).max()
            assert np.all(np.abs(got - want) <= TRK_RTOL * scale), (name, k, got, want)
            assert abs(out.dll_error_chips - ref["dll_error_chips"]) < 1e-4, (name, k)
            assert abs(out.pll_error_cycles - ref["pll_error_cycles"]) < 1e-4, (name, k)
            assert abs(out.lock_metric - ref["lock_metric"]) < 1e-4, (name, k)
            rs = ref["state"]
            assert abs(st.doppler_hz - rs["doppler_hz"]) < 1e-2, (name, k)
            dc = (st.code_phase_chips - rs["code_phase_chips"] + 511.5) % 1023 - 511.5
            assert abs(dc) < 1e-4, (name, k)
            dp = (st.carrier_phase_cycles - rs["carrier_phase_cycles"] + 0.5) % 1.0 - 0.5
            assert abs(dp) < 1e-3, (name, k)
            assert st.epoch == k + 1


def test_batch_epoch_equals_single_channel_epochs(trk):
    """The chain case: every detected PRN of a C3 snapshot in one launch per epoch."""
    c = case("chain_c3_snap0")
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    states = [to_state(trk, ch["init"]) for ch in c["channels"]]
    singles = list(states)
    n = bl[0].size
    for k in range(c["epochs"]):
        # all channels share the epoch's block: offset 0 into the same samples
        states, outs = trk.track_epoch_batch(bl[k], [0] * len(states), states, cfg)
        res = [trk.track_epoch(bl[k], s, cfg) for s in singles]
        singles = [r[0] for r in res]
        for a, (b, ob) in zip(states, res):
            assert a == b
        assert [o.ip for o in outs] == [r[1].ip for r in res]
    # a concatenated buffer with per-channel offsets gives the same first epoch
    cat = np.concatenate([bl[0], bl[1]])
    st0 = [to_state(trk, ch["init"]) for ch in c["channels"]]
    s_a, o_a = trk.track_epoch_batch(cat, [0] * len(st0), st0, cfg)
    s_b, o_b = trk.track_epoch_batch(cat[n:], [0] * len(st0), st0, cfg)
    s_c, o_c = trk.track_epoch_batch(cat, [n] * len(st0), st0, cfg)
    assert [o.ie for o in o_b] == [o.ie for o in o_c]


def test_track_step_struct_of_arrays_bit_exact(trk):
    """The batched path (one launch + vectorised closure per epoch, device-resident samples)
    on the acquisition->tracking chain: every detected PRN of a C3 snapshot, 10 epochs."""
    import torch

    c = case("chain_c3_snap0")
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    dev = torch.from_numpy(np.concatenate(bl)).cuda()
    torch.cuda.synchronize()
    n = bl[0].size
    batch = trk.TrackBatch.from_states([to_state(trk, ch["init"]) for ch in c["channels"]])
    for k in range(c["epochs"]):
        batch, outs = trk.track_step(dev, [k * n] * batch.prn.size, batch, cfg)
        for i, ch in enumerate(c["channels"]):
            ref = ch["epochs"][k]
            assert outs["ip"][i] == ref["ip"] and outs["ql"][i] == ref["ql"], (k, i)
            assert batch.doppler_hz[i] == ref["state"]["doppler_hz"]
            assert batch.code_phase_chips[i] == ref["state"]["code_phase_chips"]


def test_tracking_api_semantics(trk):
    with pytest.raises(trk.InvalidConfigError):
        trk.TrackConfig(pll_bandwidth_hz=300.0)
    from paper_1309_0052_b200 import AcqResult

    st = trk.init_from_acquisition(AcqResult(5, 1000.0, 0, 10.0, True, 1, 0), 8.184e6)
    assert st.code_phase_chips == 0.0 and st.doppler_hz == 1000.0
    with pytest.raises(trk.InvalidInputError):
        trk.init_from_acquisition(AcqResult(5, 1000.0, 0, 1.0, False, 1, 0), 8.184e6)
    with pytest.raises(trk.InvalidInputError):
        trk.epl_correlate(np.ones(100, np.complex64), st, trk.TrackConfig())
    zero = np.zeros(8184, np.complex64)
    with pytest.raises(trk.DegenerateInputError):
        trk.track_epoch(zero, st, trk.TrackConfig())


def test_track_step_slices_equal_separate_calls(trk):
    """gacq_trk_step pipelines > 2048 channels over several slices (kernel of one slice under the
    host work of the others); results equal the three separate calls (NCO words, correlators,
    closure) bit for bit, and the input batch is left untouched."""
    import dataclasses

    import torch

    c = case("chain_c3_snap0")
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    n = bl[0].size
    dev = torch.from_numpy(np.concatenate(bl[:2])).cuda()
    base = [to_state(trk, ch["init"]) for ch in c["channels"]]
    states = [dataclasses.replace(base[i % len(base)], doppler_hz=base[i % len(base)].doppler_hz + 0.5 * (i // len(base)))
              for i in range(5000)]
    batch = trk.TrackBatch.from_states(states)
    before = batch.doppler_hz.copy()
    offs = np.array([(i % 2) * n for i in range(5000)], dtype=np.int64)
    b1, o1 = trk.track_step(dev, offs, batch, cfg)
    np.testing.assert_array_equal(batch.doppler_hz, before)
    eng = trk.get_track_engine(0)
    sums = eng.correlate_chans(dev, trk.epl_chans(batch, offs, cfg), n)
    b2, o2 = trk.close_loops_batch(sums, batch, cfg)
    for k in o1:
        np.testing.assert_array_equal(o1[k], o2[k], err_msg=k)
    for f in ("code_phase_chips", "carrier_phase_cycles", "doppler_hz", "code_rate_hz", "pll_acc", "lock_nbp"):
        np.testing.assert_array_equal(getattr(b1, f), getattr(b2, f), err_msg=f)


def test_track_step_degenerate_channel_in_a_later_slice(trk):
    """A channel whose block is all zeros raises DegenerateInputError naming it (tracking.py:173-175),
    even when earlier slices were already closed; the caller's batch is unchanged."""
    import torch

    c = case("chain_c3_snap0")
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    n = bl[0].size
    dev = torch.from_numpy(np.concatenate([bl[0], np.zeros(n, np.complex64)])).cuda()
    base = [to_state(trk, ch["init"]) for ch in c["channels"]]
    batch = trk.TrackBatch.from_states([base[i % len(base)] for i in range(4100)])
    before = batch.code_phase_chips.copy()
    offs = np.zeros(4100, dtype=np.int64)
    offs[4099] = n
    with pytest.raises(trk.DegenerateInputError, match="all correlators zero on channel 4099"):
        trk.track_step(dev, offs, batch, cfg)
    np.testing.assert_array_equal(batch.code_phase_chips, before)


def test_track_step_host_samples_equal_device_samples(trk):
    """gacq_trk_step from a host buffer (staged H2D) and from a device buffer give identical epochs."""
    import torch

    c = case("chain_c3_snap0")
    bl = blocks(c)
    cfg = trk.TrackConfig(**c["config"])
    n = bl[0].size
    host = np.concatenate(bl[:3])
    dev = torch.from_numpy(host).cuda()
    b_h = b_d = trk.TrackBatch.from_states([to_state(trk, ch["init"]) for ch in c["channels"]])
    for k in range(3):
        offs = [k * n] * b_h.prn.size
        b_h, o_h = trk.track_step(host, offs, b_h, cfg)
        b_d, o_d = trk.track_step(dev, offs, b_d, cfg)
        for key in o_h:
            np.testing.assert_array_equal(o_h[key], o_d[key], err_msg=f"{k} {key}")
    np.testing.assert_array_equal(b_h.carrier_phase_cycles, b_d.carrier_phase_cycles)
