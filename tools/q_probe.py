"""K1/K2 event times of one device-resident C3 batch as complex64, int8 and int16 I/Q
(gacq_run vs gacq_run_quantized).  python tools/q_probe.py [batch]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = bench.CONFIGS["c3"]
be = bench.CudaBackend(0)
x = be.batch(c, n, seed=1000)
eng = be.engine(c, type("A", (), {"scratch_mb": 0})())
flat = torch.view_as_real(x).reshape(n, -1)
scale = float(flat.abs().max())
q8 = torch.clamp(torch.round(flat / scale * 127.0), -127, 127).to(torch.int8)
q16 = torch.clamp(torch.round(flat / scale * 32767.0), -32767, 32767).to(torch.int16)
torch.cuda.synchronize()
out = {}
for name, fn in (("c64", lambda: eng.run_rows(x, profile=True)),
                 ("int8", lambda: eng.run_rows_quantized(q8, 0, scale, profile=True)),
                 ("int16", lambda: eng.run_rows_quantized(q16, 1, scale, profile=True))):
    fn()
    best = None
    for _ in range(5):
        eng.reset_stats()
        fn()
        st = eng.stats()
        if best is None or st["run_ms"] < best["run_ms"]:
            best = {k: st[k] for k in ("run_ms", "fwd_ms", "corr_ms")}
    out[name] = best
print(json.dumps(out))
