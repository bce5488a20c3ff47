"""CPU oracle for the acquisition hot path. TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package (``paper_1309_0052_b200``) never
imports it and has no CPU fallback.

Parity status: PINNED. ``tests/golden/make_golden.py`` runs the reference
(``gnssperf``, /root/reference/pkg/src) in the build container and stores its
outputs; ``tests/test_oracle.py`` asserts the oracle reproduces them
bit-for-bit (synthesised buffers by SHA-256, power maps and ``AcqResult``
fields exactly).
"""

from oracle.gnss_oracle import (  # noqa: F401
    CHIP_RATE_HZ,
    CODE_LENGTH,
    OracleConfig,
    acquire_all,
    acquire_channel,
    add_awgn,
    carrier_replica,
    code_replica,
    doppler_bins_hz,
    generate_ca_code,
    if_file_bytes,
    if_file_decode,
    make_snapshot,
    samples_per_code_period,
    sigma_for_cn0_dbhz,
    synthesize_signal,
)
