"""bench.py's multi-rank launcher end to end on CPU (VERDICT r01 "make the BASELINE multi-GPU
configs measurable"): `--gpus N` without a launcher spawns N ranks (torch.distributed.run,
gloo), shards the FIXED global batch, takes the max over ranks, gathers the rows to rank 0 and
checks them against one rank searching the whole batch. A fake engine stands in for libgacq."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def run_bench(*args, env=None, timeout=300):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p, [json.loads(ln) for ln in lines]


@pytest.mark.parametrize("gpus,batch", [(2, 10), (3, 7)])
def test_launcher_spawns_ranks_and_shards_the_fixed_batch(gpus, batch):
    p, lines = run_bench("--fake", "--gpus", str(gpus), "--config", "c1", "--batch", str(batch), "--steps", "3",
                         "--warmup", "3")
    assert p.returncode == 0, p.stderr[-3000:]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    ln = lines[0]
    assert ln["n_gpus"] == gpus and ln["scaling"] == "strong"
    assert ln["config"]["global_batch"] == batch
    assert ln["rows"] == {"world": gpus, "identical_to_single_gpu": True, "n_rows": batch * 32}
    assert ln["weak"]["snapshots_per_gpu"] == batch and ln["weak"]["value"] > 0
    assert ln["value"] > 0 and ln["e2e"]["value"] > 0


def test_world_size_must_match_gpus():
    p, lines = run_bench("--fake", "--gpus", "2", "--config", "c1", "--batch", "4", "--steps", "3",
                         env={"WORLD_SIZE": "1"})
    assert p.returncode == 2 and not lines
    assert "--gpus 2" in p.stderr


def test_reference_arm_prints_the_same_config_keys():
    p, ours = run_bench("--fake", "--gpus", "1", "--config", "c1", "--batch", "4", "--steps", "3", "--warmup", "3")
    assert p.returncode == 0, p.stderr[-3000:]
    p2, ref = run_bench("--impl", "reference", "--config", "c1", "--batch", "4", "--steps", "1", "--warmup", "3",
                        timeout=600)
    assert p2.returncode == 0, p2.stderr[-3000:]
    assert ref[0]["impl"] == "reference" and ref[0]["config"] == ours[0]["config"]
    assert ref[0]["cpu_baseline"]["cores"] >= 1 and ref[0]["e2e"]["h2d_bytes_per_step"] == 0
