"""Multi-GPU batch plumbing for the INLA-style batch.

A single factorisation never crosses a device; the batch of independent
problems is partitioned into contiguous blocks, one per rank, and the only
exchange is one all-gather of per-problem result rows (log-determinant and,
optionally, a solution vector) — NCCL over NVLink on the GPU path, gloo in the
CPU tests.  Kept device-agnostic so the rank logic is testable without a GPU.
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_range", "gather_rows", "gather_rows_device", "sharded_rows"]


def shard_range(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of P problems owned by `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return (rank * P) // world, ((rank + 1) * P) // world


def gather_rows(local_rows, P: int, group=None, device=None) -> np.ndarray:
    """All-gather the ranks' result rows (local_rows: float64 [n_local, width],
    in problem order) into the full [P, width] array on every rank.  One
    collective; ranks with fewer rows pad to the common capacity."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    rows = torch.as_tensor(np.asarray(local_rows, dtype=np.float64))
    width = rows.shape[1] if rows.ndim == 2 else 1
    rows = rows.reshape(-1, width)
    lo, hi = shard_range(P, world, rank)
    if rows.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {rows.shape[0]} rows, expected {hi - lo}")
    cap = -(-P // world)
    buf = torch.zeros((cap, width), dtype=torch.float64, device=device)
    buf[: hi - lo] = rows.to(buf.device)
    if world > 1:
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf, group=group)
    else:
        out = [buf]
    parts = []
    for r in range(world):
        a, b = shard_range(P, world, r)
        parts.append(out[r][: b - a])
    return torch.cat(parts).cpu().numpy()


def gather_rows_device(rows, P: int, group=None):
    """gather_rows for result rows that already live on the device (float64
    tensor [n_local, width], problem order): one all_gather straight from the
    device buffers (NCCL over NVLink on GPUs, gloo on CPU tensors), no host
    round trip before the collective.  Returns the [P, width] tensor."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    lo, hi = shard_range(P, world, rank)
    if rows.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {rows.shape[0]} rows, expected {hi - lo}")
    if world == 1:
        return rows
    cap = -(-P // world)
    buf = torch.zeros((cap, rows.shape[1]), dtype=rows.dtype, device=rows.device)
    buf[: hi - lo] = rows
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([out[r][: shard_range(P, world, r)[1] - shard_range(P, world, r)[0]] for r in range(world)])


def sharded_rows(P: int, local_fn, width: int, group=None, device="cuda"):
    """Rank orchestration of a sharded batch: this rank computes the result
    rows of its contiguous block [lo, hi) with ``local_fn(lo, hi)`` (a
    [hi-lo, width] float64 tensor on ``device``) and one all-gather returns
    the full [P, width] tensor on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    lo, hi = shard_range(P, world, rank)
    rows = local_fn(lo, hi) if hi > lo else torch.zeros((0, width), dtype=torch.float64, device=device)
    return gather_rows_device(rows, P, group=group)
