"""Host-side tracking logic (no kernel launches): the vectorised batch loop closure and NCO
word builder must reproduce the reference's per-channel float64 arithmetic bit for bit."""

import numpy as np
import pytest

from tracking_cases import case, load

trk = pytest.importorskip("paper_1309_0052_b200.tracking")


def to_state(d):
    d = dict(d)
    d["dll_filter_state"] = tuple(d["dll_filter_state"])
    d["pll_filter_state"] = tuple(d["pll_filter_state"])
    return trk.TrackState(**d)


def all_channels():
    out = []
    for c in load():
        for ch in c["channels"]:
            out.append((c, ch))
    return out


def test_close_loops_batch_equals_reference_per_channel():
    """Drive the vectorised closure with the reference's own correlator values for every
    channel of every fixture; states and outputs must equal the golden epoch by epoch."""
    groups = {}
    for c, ch in all_channels():
        groups.setdefault(c["name"], []).append((c, ch))
    for name, chans in groups.items():
        cfg = trk.TrackConfig(**chans[0][0]["config"])
        batch = trk.TrackBatch.from_states([to_state(ch["init"]) for _, ch in chans])
        for k in range(chans[0][0]["epochs"]):
            sums = np.array([[ch["epochs"][k][x] for x in ("ie", "qe", "ip", "qp", "il", "ql")]
                             for _, ch in chans], dtype=np.float32)
            batch, outs = trk.close_loops_batch(sums, batch, cfg)
            for i, (_, ch) in enumerate(chans):
                ref = ch["epochs"][k]
                for key in ("dll_error_chips", "pll_error_cycles", "lock_metric"):
                    assert outs[key][i] == ref[key], (name, k, key)
                st = batch.to_states()[i]
                for key in ("code_phase_chips", "carrier_phase_cycles", "doppler_hz", "code_rate_hz", "lock_nbd",
                            "lock_nbp"):
                    assert getattr(st, key) == ref["state"][key], (name, k, key)
                assert st.dll_filter_state == tuple(ref["state"]["dll_filter_state"])
                assert st.pll_filter_state == tuple(ref["state"]["pll_filter_state"])


def test_vectorised_nco_words_equal_scalar():
    rng = np.random.default_rng(5)
    states = [trk.TrackState(prn=int(rng.integers(1, 33)), code_phase_chips=float(rng.uniform(0, 1023)),
                             carrier_phase_cycles=float(rng.uniform(-3, 3)), doppler_hz=float(rng.uniform(-9e3, 9e3)),
                             code_rate_hz=1.023e6 * (1 + float(rng.uniform(-1e-5, 1e-5))),
                             sample_rate_hz=float(rng.choice([4.092e6, 8.184e6, 5e6, 16.368e6])))
              for _ in range(500)]
    cfg = trk.TrackConfig(correlator_spacing_chips=0.37)
    ch = trk.epl_chans(trk.TrackBatch.from_states(states), np.arange(500) * 7, cfg)
    d = cfg.correlator_spacing_chips
    for i, s in enumerate(states):
        assert ch["carrier_p0"][i] == trk.carrier_phase_to_fixed(s.carrier_phase_cycles)
        assert ch["carrier_step"][i] == trk.carrier_step_to_fixed(s.doppler_hz, s.sample_rate_hz)
        for j, o in enumerate((+d / 2, 0.0, -d / 2)):
            assert ch["code_p0"][i, j] == trk.code_phase_to_fixed((s.code_phase_chips + o) % 1023)
        assert ch["code_step"][i] == trk.code_step_to_fixed(s.code_rate_hz, s.sample_rate_hz)
        assert ch["block_offset"][i] == 7 * i and ch["prn"][i] == s.prn


def test_track_batch_round_trip():
    states = [to_state(ch["init"]) for _, ch in all_channels()]
    assert trk.TrackBatch.from_states(states).to_states() == states
    assert case("locked_8184k")["epochs"] == 10


def test_mixed_rate_batch_closes_each_channel_at_its_own_block_length():
    """gacq_trk_close advances every channel's NCOs over that channel's own block length
    (tracking.py:122-123), so a batch mixing sample rates equals the per-channel closure."""
    rng = np.random.default_rng(11)
    rates = [4.092e6, 8.184e6, 5e6, 16.368e6]
    states = [trk.TrackState(prn=1 + i, code_phase_chips=float(rng.uniform(0, 1023)),
                             carrier_phase_cycles=float(rng.uniform(0, 1)), doppler_hz=float(rng.uniform(-4e3, 4e3)),
                             code_rate_hz=1.023e6, sample_rate_hz=rates[i % 4]) for i in range(16)]
    cfg = trk.TrackConfig()
    sums = rng.normal(size=(16, 6)).astype(np.float32) * 100
    batch, outs = trk.close_loops_batch(sums, trk.TrackBatch.from_states(states), cfg)
    for i, s in enumerate(states):
        o = trk._outputs(sums[i:i + 1], trk.block_length(s, cfg))[0]
        ref_state, ref_out = trk._close_loops(o, s, cfg)
        assert batch.to_states()[i] == ref_state, i
        assert outs["pll_error_cycles"][i] == ref_out.pll_error_cycles
