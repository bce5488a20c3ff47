"""The multi-GPU paths on one B200 (VERDICT r01 "done" bar for the bench launcher): several
ranks / host threads share cuda:0, so the sharding, gather and max-over-ranks logic runs with
the real engine, and every gathered row is checked against the CPU oracle.

- `bench.py --gpus 2 --device-map 0,0`: the self-spawning launcher (torch.distributed.run,
  gloo because both ranks share a device), strong-sharded fixed batch, rank-0 gather; the
  dumped batch and rows are compared with oracle.acquire_all snapshot by snapshot.
- `acquire_batch(devices=[0, 0, 0])`: the one-process, one-thread-per-device batch API.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_0052_b200 import build

    build.build()
    import paper_1309_0052_b200 as p

    return p


C1 = dict(doppler_min_hz=-5000.0, doppler_max_hz=5000.0, doppler_step_hz=500.0, noncoherent_rounds=1)


def oracle_rows(x, fs):
    res = oracle.acquire_all(x, fs, range(1, 33), oracle.OracleConfig(**C1))
    return [(r["bin_index"], r["code_phase_samples"]) for r in res]


def test_bench_launcher_two_ranks_rows_match_oracle(tmp_path):
    dump = tmp_path / "rows.npz"
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--device-map", "0,0",
                        "--config", "c1", "--batch", "6", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--tracking-epochs", "1", "--dump", str(dump)],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-4000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["rows"]["identical_to_single_gpu"] and ln["rows"]["world"] == 2
    assert ln["value"] > 0 and ln["e2e"]["value"] > 0 and ln["gpu_launches"] > 0
    d = np.load(dump)
    batch, rows = d["batch"], d["rows"]
    assert rows.shape == (6, 32)
    for s in range(batch.shape[0]):
        want = oracle_rows(batch[s], 4.092e6)
        got = [(int(r["bin"]), int(r["lag"])) for r in rows[s]]
        assert got == want, s


def test_acquire_batch_three_threads_one_device(pkg):
    fs = 4.092e6
    xs = np.stack([oracle.make_snapshot(i, fs, 1e-3, base_seed=77)[0] for i in range(7)])
    res = pkg.acquire_batch(xs, fs, range(1, 33), pkg.AcqConfig(**C1), devices=[0, 0, 0])
    assert len(res) == 7
    bins = oracle.OracleConfig(**C1).doppler_bins_hz()
    for s in range(7):
        want = oracle_rows(xs[s], fs)
        got = [(int(np.flatnonzero(bins == r.doppler_hz)[0]), r.code_phase_samples) for r in res[s]]
        assert got == want, s
