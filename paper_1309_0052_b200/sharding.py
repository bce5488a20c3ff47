"""Multi-GPU host logic: one process per GPU, snapshots sharded in contiguous ranges.

Snapshots are independent units, so the data path has no collective:
each rank searches its own shard on its own device. torch.distributed (NCCL on GPUs,
gloo for the CPU tests) is used only for control: barriers, the max-over-ranks step
time and an optional gather of the 16-byte result rows to rank 0.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of n units for `rank` of `world`, sizes differing by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. a device-timed step) across the process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local_rows: np.ndarray, n_total: int, dist=None):
    """Gather every rank's [n_local, n_prn] gacq_row array to rank 0 in snapshot order.
    Returns the full [n_total, n_prn] array on rank 0, None elsewhere."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local_rows
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * world if rank == 0 else None
    dist.gather_object(local_rows.tobytes(), parts, dst=0)
    if rank != 0:
        return None
    n_prn = local_rows.shape[1]
    out = np.empty((n_total, n_prn), dtype=_lib.ROW_DTYPE)
    for r, blob in enumerate(parts):
        a, b = shard_bounds(n_total, world, r)
        out[a:b] = np.frombuffer(blob, dtype=_lib.ROW_DTYPE).reshape(b - a, n_prn)
    return out


def search_sharded(engine, snapshots, dist=None) -> np.ndarray | None:
    """Search this rank's shard of the global [S, L] batch with `engine` (bound to this
    rank's GPU) and gather the rows to rank 0 (None on other ranks)."""
    n = snapshots.shape[0]
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    a, b = shard_bounds(n, world, rank)
    rows = engine.run_rows(snapshots[a:b]) if b > a else np.empty((0, len(engine.prns)), dtype=_lib.ROW_DTYPE)
    return gather_rows(rows, n, dist)
