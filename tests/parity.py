"""Parity rule of SURVEY.md 8(c) shared by the GPU tests, smoke() and bench.py.

(bin, lag) and `detected` must equal the reference's; `peak_metric` within 1e-4 relative.
A (bin, lag) mismatch is an *ambiguous tie* (counted, reported, not a failure) only when
the oracle's own power at the GPU's cell is within TIE_REL of the oracle's peak -- i.e.
the two cells are indistinguishable in float32 (e.g. the symmetric +-f bins of a 0 Hz
truth, SURVEY.md 7 "Hard parts" 5). Likewise a `detected` flip is a tie only when the
reference metric is within TIE_REL of the threshold.
"""

from __future__ import annotations

import math

METRIC_RTOL = 1e-4   # north_star: correlation peak values within 1e-4 relative (fp32)
TIE_REL = 1e-5


def compare(got: dict, ref: dict, threshold: float, pmap=None, bins=None) -> str:
    """Return 'exact', 'tie' or a failure description. `got`/`ref` carry doppler_hz,
    code_phase_samples, peak_metric, detected; `pmap` is the oracle power map [B, P]."""
    same_cell = (got["doppler_hz"] == ref["doppler_hz"]
                 and got["code_phase_samples"] == ref["code_phase_samples"])
    if same_cell:
        rm, gm = ref["peak_metric"], got["peak_metric"]
        if math.isinf(rm) or math.isinf(gm):
            if not (math.isinf(rm) and math.isinf(gm)):
                return f"metric inf mismatch {gm} vs {rm}"
        elif abs(gm - rm) > METRIC_RTOL * abs(rm):
            return f"metric {gm} vs {rm} (rel {abs(gm - rm) / abs(rm):.2e})"
        if got["detected"] != ref["detected"]:
            if abs(rm - threshold) <= TIE_REL * threshold:
                return "tie"
            return f"detected {got['detected']} vs {ref['detected']}"
        return "exact"
    if pmap is None or bins is None:
        return (f"cell ({got['doppler_hz']}, {got['code_phase_samples']}) vs "
                f"({ref['doppler_hz']}, {ref['code_phase_samples']}) and no map to classify")
    import numpy as np

    gb = int(np.flatnonzero(bins == got["doppler_hz"])[0])
    peak = float(pmap.max())
    mine = float(pmap[gb, got["code_phase_samples"]])
    if peak - mine <= TIE_REL * peak:
        return "tie"
    return (f"cell ({got['doppler_hz']}, {got['code_phase_samples']}) vs "
            f"({ref['doppler_hz']}, {ref['code_phase_samples']}): oracle power {mine} vs peak {peak}")
