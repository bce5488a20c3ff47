"""Pin the tracking oracle (oracle/tracking_oracle.py) to the reference's outputs. CPU only."""

import pytest

from oracle import tracking_oracle as to
from tracking_cases import blocks, case, config_from, load, state_from

KEYS = ("ie", "qe", "ip", "qp", "il", "ql", "dll_error_chips", "pll_error_cycles", "lock_metric")
STATE_KEYS = ("code_phase_chips", "carrier_phase_cycles", "doppler_hz", "code_rate_hz", "lock_nbd", "lock_nbp")


@pytest.mark.parametrize("name", [c["name"] for c in load()])
def test_tracking_oracle_bit_exact(name):
    c = case(name)
    bl = blocks(c)
    cfg = config_from(c["config"])
    assert c["channels"]
    for ch in c["channels"]:
        st = state_from(ch["init"])
        if "acq" in ch:  # init_from_acquisition restated
            a = ch["acq"]
            assert to.init_from_acquisition(a["prn"], a["doppler_hz"], a["code_phase_samples"],
                                            st.sample_rate_hz) == st
        for k, ref in enumerate(ch["epochs"]):
            st, out = to.track_epoch(bl[k], st, cfg)
            for key in KEYS:
                assert out[key] == ref[key], (name, k, key, out[key], ref[key])
            for key in STATE_KEYS:
                assert getattr(st, key) == ref["state"][key], (name, k, key)
            assert st.epoch == k + 1


def test_chain_case_tracks_detected_channels():
    # every detected PRN of the C3 snapshot is handed to tracking (10 epochs, still pulling in)
    c = case("chain_c3_snap0")
    assert len(c["channels"]) >= 5
    assert all(len(ch["epochs"]) == 10 for ch in c["channels"])
    assert case("locked_8184k")["channels"][0]["epochs"][-1]["lock_metric"] > 0.9
