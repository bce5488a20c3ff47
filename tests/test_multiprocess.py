"""Multi-GPU host logic on CPU: world_size-2 gloo process group, fake per-rank engine.

The data path has no collective (snapshots are independent); this checks
the shard bounds, the rank-0 gather order of the 16-byte rows and the max-over-ranks timing.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1309_0052_b200 import _lib
from paper_1309_0052_b200.sharding import gather_rows, max_over_ranks, search_sharded, shard_bounds


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


class FakeEngine:
    """Stands in for AcqEngine: row = (bin, lag, peak, floor) derived from the snapshot."""

    prns = [1, 2, 3]

    def run_rows(self, snaps):
        out = np.zeros((snaps.shape[0], 3), dtype=_lib.ROW_DTYPE)
        ids = snaps[:, 0].real.astype(np.int32)
        for p in range(3):
            out["bin"][:, p] = p
            out["lag"][:, p] = ids
            out["peak"][:, p] = ids * 10.0 + p
            out["floor"][:, p] = 1.0
        return out


def _worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    snaps = np.zeros((n, 8), dtype=np.complex64)
    snaps[:, 0] = np.arange(n)
    rows = search_sharded(FakeEngine(), snaps, dist)
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        q.put((rows["lag"].tolist(), rows["peak"].tolist(), t))
    else:
        q.put(("rank1", rows, t))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [5, 64])
def test_gloo_world2_shard_and_gather(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = next(g for g in got if g[0] != "rank1")
    r1 = next(g for g in got if g[0] == "rank1")
    lags, peaks, t0 = r0
    assert [row[0] for row in lags] == list(range(n))  # snapshot order restored on rank 0
    assert peaks[3][2] == 32.0
    assert r1[1] is None  # only rank 0 holds the gathered rows
    assert t0 == 2.0 and r1[2] == 2.0  # max over ranks


def test_single_process_passthrough():
    rows = FakeEngine().run_rows(np.zeros((4, 8), dtype=np.complex64))
    assert gather_rows(rows, 4, None) is rows
    assert max_over_ranks(3.5) == 3.5


def test_merge_bin_shards_is_the_row_major_first_argmax():
    # merging per-shard rows (grid-global bins, ascending shards) equals the argmax over the
    # concatenated grid: larger peak wins, ties go to the lower bin, the floor travels with it
    from paper_1309_0052_b200 import _lib, merge_bin_shards

    rng = np.random.default_rng(3)
    n_snap, n_prn, n_bins = 5, 7, 21
    per_bin = np.zeros((n_snap, n_prn, n_bins), dtype=_lib.ROW_DTYPE)
    per_bin["bin"] = np.arange(n_bins)
    per_bin["lag"] = rng.integers(0, 4092, per_bin.shape)
    per_bin["peak"] = rng.integers(0, 6, per_bin.shape).astype(np.float32)  # many exact ties
    per_bin["floor"] = rng.random(per_bin.shape).astype(np.float32)
    want = per_bin[np.arange(n_snap)[:, None], np.arange(n_prn)[None, :], np.argmax(per_bin["peak"], axis=2)]
    for cuts in ([0, 7, 14, 21], [0, 1, 21], [0, 10, 11, 20, 21]):
        shards = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            sub = per_bin[:, :, a:b]
            k = np.argmax(sub["peak"], axis=2)
            shards.append(sub[np.arange(n_snap)[:, None], np.arange(n_prn)[None, :], k])
        got = merge_bin_shards(shards)
        np.testing.assert_array_equal(got, want)
