"""Signal sharding across GPUs.

Every signal is independent, so P signals split into contiguous per-rank
shards with the dictionary replicated on each GPU; no data crosses GPUs while
coding.  The only collective is the optional gather of the per-rank outputs
(BatchSolve arrays) to one rank -- ``torch.distributed.gather`` (NCCL on
GPUs, gloo on CPU).
"""

from __future__ import annotations

import numpy as np

FIELDS = ("counts", "sel", "alpha", "rnorm", "scans", "flag")


def shard_range(total: int, rank: int, world: int) -> tuple:
    """Contiguous, balanced [start, stop) of ``total`` signals for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(int(total), int(world))
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_solutions(local: dict, total: int, dst: int = 0, group=None, device=None):
    """Gather per-rank solution arrays (dict of ``FIELDS``, shard rows first)
    into full P-row numpy arrays on rank ``dst`` (None elsewhere).

    Shards are padded to the largest shard so one fixed-size collective per
    field suffices; the padding is trimmed on ``dst``.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(total, r, world) for r in range(world)]
    rows = max(b - a for a, b in sizes)
    out = {} if rank == dst else None
    for name in FIELDS:
        arr = local[name]
        t = arr if isinstance(arr, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(arr))
        if device is not None:
            t = t.to(device)
        pad_shape = (rows,) + tuple(t.shape[1:])
        buf = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
        buf[: t.shape[0]] = t
        bufs = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
        dist.gather(buf, bufs, dst=dst, group=group)
        if rank == dst:
            parts = [bufs[r][: sizes[r][1] - sizes[r][0]].cpu().numpy() for r in range(world)]
            out[name] = np.concatenate(parts, axis=0)
    return out
