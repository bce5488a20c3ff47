"""Load the committed golden fixtures and regenerate their inputs with the oracle.

The fixtures (tests/golden/golden.json, maps.npz) were produced by running the
reference itself (tests/golden/make_golden.py); each case records the SHA-256
of the reference's input buffer so a regenerated input can be checked before use.
"""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

import oracle

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load_cases() -> tuple:
    return tuple(json.loads((GOLDEN / "golden.json").read_text())["cases"])


@lru_cache(maxsize=None)
def load_maps() -> dict:
    with np.load(GOLDEN / "maps.npz") as z:
        return {k: z[k] for k in z.files}


def case(name: str) -> dict:
    for c in load_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_inputs: dict = {}


def case_input(c: dict) -> np.ndarray:
    """Regenerate the complex64 input of a golden case with the oracle's synthesis."""
    if c["name"] in _inputs:
        return _inputs[c["name"]]
    s = c["spec"]
    if c["kind"] == "synth":
        x = oracle.synthesize_signal(s["prn"], s["doppler_hz"], s["code_phase_samples"],
                                     s["carrier_phase_cycles"], s["fs"], s["duration_s"],
                                     s["noise_sigma"], s["seed"])
    elif c["kind"] == "noise":
        g = np.random.Generator(np.random.PCG64(s["seed"]))
        x = (g.standard_normal(s["n"]) + 1j * g.standard_normal(s["n"])).astype(np.complex64)
    elif c["kind"] == "zeros":
        x = np.zeros(s["n"], dtype=np.complex64)
    elif c["kind"] == "snapshot":
        kw = {}
        if "cn0_range" in s:
            kw["cn0_range"] = tuple(s["cn0_range"])
        if "doppler_span_hz" in s:
            kw["doppler_span_hz"] = s["doppler_span_hz"]
        x, _ = oracle.make_snapshot(s["index"], s["fs"], s["duration_s"], s["base_seed"], **kw)
    else:
        raise ValueError(c["kind"])
    _inputs[c["name"]] = x
    return x


def oracle_config(c: dict) -> "oracle.OracleConfig":
    return oracle.OracleConfig(**c["config"])
