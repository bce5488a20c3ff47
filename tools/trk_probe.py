"""Time the parts of one batched tracking epoch (32768 channels)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1309_0052_b200 import tracking as trk  # noqa: E402

n_snap, fs = 1024, 4.092e6
n = 4092
span = 10 * n
dev = torch.randn((n_snap, span), dtype=torch.complex64, device="cuda") * 8
rng = np.random.default_rng(7)
prns = np.tile(np.arange(1, 33), n_snap)
states = [trk.TrackState(prn=int(p), code_phase_chips=float(rng.uniform(0, 1023)), carrier_phase_cycles=0.0,
                         doppler_hz=float(d), code_rate_hz=1.023e6, sample_rate_hz=fs)
          for p, d in zip(prns, rng.uniform(-4750, 4750, prns.size))]
base = np.repeat(np.arange(n_snap, dtype=np.int64) * span, 32)
cfg = trk.TrackConfig()
batch = trk.TrackBatch.from_states(states)
eng = trk.get_track_engine(0)
batch, _ = trk.track_step(dev, base, batch, cfg)
torch.cuda.synchronize()

def t(f, k=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3, r

ms, chans = t(lambda: trk.epl_chans(batch, base, cfg))
print(f"epl_chans          {ms:.3f} ms")
ms, sums = t(lambda: eng.correlate_chans(dev, chans, n))
print(f"correlate (kernel) {ms:.3f} ms")
ms, _ = t(lambda: trk.close_loops_batch(sums, batch, cfg))
print(f"close_loops_batch  {ms:.3f} ms")
ms, _ = t(lambda: trk._owned(batch))
print(f"_owned copy        {ms:.3f} ms")
ms, _ = t(lambda: trk.track_step(dev, base, batch, cfg))
print(f"track_step         {ms:.3f} ms  -> {prns.size / ms * 1e3 / 1e6:.2f} M channel-epochs/s")
