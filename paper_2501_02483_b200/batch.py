"""Multi-GPU batch plumbing for the INLA-style batch.

A single factorisation never crosses a device; the batch of independent
problems is partitioned into contiguous blocks, one per rank, and the only
exchange is one all-gather of per-problem result rows (log-determinant and,
optionally, a solution vector) — NCCL over NVLink on the GPU path, gloo in the
CPU tests.  Kept device-agnostic so the rank logic is testable without a GPU.
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_range", "gather_rows"]


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
