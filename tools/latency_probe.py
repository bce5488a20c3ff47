"""Per-call latency of the drop-in API on one snapshot (acquire_all, C3 grid), and of the
batched engine at a few batch sizes."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
import paper_1309_0052_b200 as g  # noqa: E402

fs = 4.092e6
cfg = g.AcqConfig(doppler_min_hz=-5000, doppler_max_hz=5000, doppler_step_hz=500, noncoherent_rounds=10)
x, _ = oracle.make_snapshot(0, fs, 10e-3, base_seed=5)
buf = g.IqBuffer(x, fs)
prns = list(range(1, 33))
g.acquire_all(buf, prns, cfg)
for _ in range(3):
    t0 = time.perf_counter()
    n = 50
    for _ in range(n):
        g.acquire_all(buf, prns, cfg)
    dt = (time.perf_counter() - t0) / n
    print(f"acquire_all 1 snapshot x 32 PRNs x 21 bins: {dt * 1e3:.3f} ms/call ({672 / dt / 1e6:.3f} M cells/s)")
eng = g.get_engine(fs, prns, cfg)
for s in (1, 8, 64, 256):
    xb = np.ascontiguousarray(np.broadcast_to(x, (s, x.size)))
    eng.search(xb)
    t0 = time.perf_counter()
    for _ in range(10):
        eng.search(xb)
    dt = (time.perf_counter() - t0) / 10
    print(f"AcqEngine.search batch {s}: {dt * 1e3:.3f} ms ({s * 672 / dt / 1e6:.3f} M cells/s)")
