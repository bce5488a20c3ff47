"""Tracking golden fixtures (tests/golden/tracking.json, written by the reference) and the
regeneration of their input blocks with the pinned oracle synthesis."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

import oracle
from oracle import tracking_oracle as to

GOLDEN = Path(__file__).resolve().parent / "golden" / "tracking.json"


@lru_cache(maxsize=None)
def load() -> tuple:
    return tuple(json.loads(GOLDEN.read_text())["cases"])


def case(name: str) -> dict:
    return next(c for c in load() if c["name"] == name)


def blocks(c: dict) -> list:
    s = c["spec"]
    fs = s["fs"]
    if c["kind"] == "synth":
        x = oracle.synthesize_signal(s["prn"], s["doppler_hz"], s["code_phase_samples"], s["carrier_phase_cycles"],
                                     fs, s["duration_s"], s["noise_sigma"], s["seed"])
    else:
        x, _ = oracle.make_snapshot(s["index"], fs, s["duration_s"], s["base_seed"])
    n = round(fs * 1e-3)
    return [np.ascontiguousarray(x[k * n:(k + 1) * n]) for k in range(c["epochs"])]


def state_from(d: dict) -> "to.TrackState":
    d = dict(d)
    d["dll_filter_state"] = tuple(d["dll_filter_state"])
    d["pll_filter_state"] = tuple(d["pll_filter_state"])
    return to.TrackState(**d)


def config_from(d: dict) -> "to.TrackConfig":
    return to.TrackConfig(**d)
