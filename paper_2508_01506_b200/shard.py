"""Batch sharding across ranks.

Encoder sequences are independent (no cross-batch op anywhere), so a global
batch is split contiguously across ranks -- rank k owns
[k*B/n, (k+1)*B/n) with the remainder spread over the first ranks -- and each
rank runs the whole model on its shard with a full factor replica.  No
collective touches the hot path; the outputs are gathered to rank 0 once
(NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous [start, stop) of sequences owned by `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(global_batch, world)
    start = rank * base + min(rank, rem)
    stop = start + base + (1 if rank < rem else 0)
    return start, stop


def gather_outputs(local, world: int, rank: int, global_batch: int, dst: int = 0):
    """Gathers per-rank [b_k, M, d] outputs into [global_batch, M, d] on `dst`.

    Ragged shards are padded to the largest shard for the collective and
    trimmed afterwards.  Returns the full tensor on `dst`, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    sizes = [shard_range(global_batch, world, r) for r in range(world)]
    biggest = max(b - a for a, b in sizes)
    pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst)
    if rank != dst:
        return None
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(sizes)], dim=0)
