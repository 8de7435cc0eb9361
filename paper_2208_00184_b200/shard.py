"""Multi-GPU sharding of the batched-candidate path.

Only independent work shards: rank r simulates candidates [lo, hi) of the batch, reduces
locally to the first strict minimum, and one collective — an all-reduce MIN over the
packed key (makespan << 20 | candidate index) — picks the global winner with the
reference's tie rule (lowest index among equal makespans, simulator.cpp:292-294).
With NCCL this is a single 8-byte all-reduce over NVLink; with gloo (CPU tests) the
same code path runs on host tensors.
"""
from __future__ import annotations

import numpy as np

INDEX_BITS = 20
MAX_MAKESPAN = (1 << (63 - INDEX_BITS)) - 1


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items for `rank` of `world`."""
    per = (total + world - 1) // world
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def pack(makespan: int, index: int) -> int:
    if not 0 <= index < (1 << INDEX_BITS):
        raise ValueError("candidate index does not fit the packed key")
    if not 0 <= makespan <= MAX_MAKESPAN:
        raise ValueError("makespan does not fit the packed key")
    return (int(makespan) << INDEX_BITS) | int(index)


def unpack(key: int) -> tuple[int, int]:
    return key >> INDEX_BITS, key & ((1 << INDEX_BITS) - 1)


def local_key(makespans: np.ndarray, lo: int) -> int:
    """Packed key of this shard's first strict minimum (or +inf for an empty shard)."""
    if len(makespans) == 0:
        return (1 << 63) - 1
    i = int(np.argmin(makespans))  # numpy argmin returns the first minimum
    return pack(int(makespans[i]), lo + i)


def global_argmin(makespans: np.ndarray, lo: int, device=None) -> tuple[int, int]:
    """One MIN all-reduce of the packed keys across the default process group."""
    import torch
    import torch.distributed as dist
    key = torch.tensor([local_key(makespans, lo)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(key, op=dist.ReduceOp.MIN)
    return unpack(int(key.item()))
