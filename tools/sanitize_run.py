"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Exercises every device kernel: the table builders, the 1023-point path (K1/K2 at D = 2, 4, 16;
both floor forms; int8 and int16 dequantized in K1), the generic path (native mixed radix at
5, 3 and 20 MHz, the last on 4-CTA clusters; linear power-of-two transforms up to 65536 points on
8-CTA clusters; 8.192 MHz circular transforms), K3, the power-map hook and the tracking correlators.
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
import paper_1309_0052_b200 as g  # noqa: E402
from paper_1309_0052_b200 import tracking as trk  # noqa: E402


def run(fs, rounds, coh=1, generic=False, radius=0):
    cfg = g.AcqConfig(doppler_min_hz=-1000.0, doppler_max_hz=1000.0, doppler_step_hz=500.0,
                      noncoherent_rounds=rounds, coherent_ms=coh, exclusion_radius_samples=radius)
    x = np.stack([oracle.make_snapshot(i, fs, rounds * coh * 1e-3, base_seed=11)[0] for i in range(2)])
    eng = g.AcqEngine(fs, [1, 5, 9], cfg, force_generic=generic)
    r = eng.search(x)
    q = np.clip(np.round(np.stack([x.real, x.imag], -1).reshape(2, -1) / 40.0 * 127), -127, 127).astype(np.int8)
    eng.search_quantized(q, 0, 40.0)
    eng.search_quantized(q.astype(np.int16) * 200, 1, 40.0 * 200 * 32767 / 127)
    eng.power_map(x[0])
    eng.carrier_table()
    print(fs, generic, eng.info["path"], r.code_phase_samples[0].tolist())
    eng.close()


def main():
    for fs, rounds in ((2.046e6, 2), (4.092e6, 2), (16.368e6, 1)):
        run(fs, rounds)
        run(fs, rounds, generic=True)
    run(4.092e6, 2, radius=200)  # K2 floor from full rows (window > 33 chip lags)
    run(5.0e6, 2)  # native mixed radix: 5000 = 8 x 5^4, one CTA
    run(3.0e6, 1)  # native with a radix-3 pass
    run(20.0e6, 1)  # native 20000 points on 4-CTA clusters (DSMEM combine)
    run(6.0e6, 1, coh=2)
    run(8.192e6, 2)  # power-of-two n_coh: circular 8192-point transform, 16 values per thread
    run(8.192e6, 1, coh=4)  # circular 32768-point transform, 4-CTA clusters
    run(16.367e6, 1, coh=2)  # linear 65536-point transform, 8-CTA clusters
    st = [trk.TrackState(prn=p, code_phase_chips=10.0 * p, carrier_phase_cycles=0.0, doppler_hz=100.0 * p,
                         code_rate_hz=1.023e6, sample_rate_hz=4.092e6) for p in (1, 2, 3)]
    blk = oracle.make_snapshot(0, 4.092e6, 1e-3, base_seed=3)[0]
    s2, out = trk.track_epoch_batch(blk, [0, 0, 0], st, trk.TrackConfig())
    print("track", [round(o.ip, 2) for o in out])
    # 40 channels: a full 32-channel CTA and a partial one
    st = [trk.TrackState(prn=1 + i % 32, code_phase_chips=7.0 * i, carrier_phase_cycles=0.1, doppler_hz=50.0 * i,
                         code_rate_hz=1.023e6, sample_rate_hz=4.092e6) for i in range(40)]
    s2, out = trk.track_epoch_batch(blk, [0] * 40, st, trk.TrackConfig())
    print("track40", round(out[39].ip, 2))


if __name__ == "__main__":
    main()
