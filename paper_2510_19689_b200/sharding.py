"""Row sharding across GPUs: one process per GPU, contiguous
row blocks, a full weight replica per rank, no collective on the hot path.

``shard_bounds`` is the partition (rank r gets ``[r*B/G, (r+1)*B/G)`` with the
remainder spread over the first ranks).  ``gather_outputs`` is the optional
final gather to rank 0 (NCCL over NVLink/NVSwitch on the GPU box, gloo in the
CPU tests); it is timed separately from the hot path.  Per-row results are
bitwise independent of the shard a row lands in (the batch-invariance
contract), so the gathered outputs equal a single-GPU call bit for bit.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_bounds(rows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, stop) row ranges for each of ``world`` ranks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, rem = divmod(rows, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((start, start + n))
        start += n
    return out


def shard_of(x: np.ndarray, rank: int, world: int) -> np.ndarray:
    a, b = shard_bounds(x.shape[0], world)[rank]
    return x[a:b]


def gather_outputs(local: dict, rows: int, rank: int, world: int, *, dst: int = 0) -> dict | None:
    """Gather per-rank outputs ``{logits (b,C), probabilities (b,C), masks
    (S,b,F), importance (b,F)}`` to rank ``dst`` with torch.distributed.

    Works with any initialized process group (NCCL with CUDA tensors, gloo
    with CPU tensors).  Shards are padded to the largest shard for the
    collective and trimmed afterwards.  Returns the full-batch dict on ``dst``
    and None elsewhere.
    """
    import torch
    import torch.distributed as dist

    bounds = shard_bounds(rows, world)
    maxb = max(b - a for a, b in bounds)
    full = {} if rank == dst else None
    for key in ("logits", "probabilities", "importance", "masks"):
        t = local[key]
        t = torch.as_tensor(t)
        row_dim = 1 if key == "masks" else 0
        pad = maxb - t.shape[row_dim]
        if pad:
            shape = list(t.shape)
            shape[row_dim] = pad
            t = torch.cat([t, t.new_zeros(shape)], dim=row_dim)
        t = t.contiguous()
        parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
        dist.gather(t, parts, dst=dst)
        if rank == dst:
            trimmed = []
            for (a, b), p in zip(bounds, parts):
                trimmed.append(p[:, : b - a] if row_dim == 1 else p[: b - a])
            full[key] = torch.cat(trimmed, dim=row_dim)
    return full


def run_sharded(forward: Callable[[np.ndarray], dict], x: np.ndarray, rank: int, world: int,
                *, gather: bool = True) -> dict | None:
    """Compute this rank's shard with ``forward`` and optionally gather to rank 0."""
    xs = shard_of(x, rank, world)
    local = forward(xs)
    if not gather:
        return local
    return gather_outputs(local, x.shape[0], rank, world)
