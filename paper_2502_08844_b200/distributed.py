"""Multi-GPU plumbing for the batched env step.

Worlds are independent: rank r of W owns a contiguous block of global world
indices and passes its first index as ``env_index_offset``, so every world
keeps its Philox stream (envkit.py:41-49 keys on the global index) and results
are bit-identical for any GPU count.  There is no collective on the step path;
``torch.distributed`` (NCCL over NVLink between GPUs) only carries the
benchmark barrier / max-over-ranks timing and statistic reductions.
"""

from __future__ import annotations


def shard(num_worlds: int, rank: int, world_size: int) -> tuple[int, int]:
    """(env_index_offset, count) of `rank`'s block; the first num_worlds %
    world_size ranks get one extra world."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    base, extra = divmod(int(num_worlds), world_size)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (bench timing is the slowest rank's)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def sharded_env(config, num_worlds_global: int, rank: int, world_size: int, **kw):
    """DeviceBatchEnv over this rank's shard of the global worlds."""
    from .envkit import DeviceBatchEnv

    offset, count = shard(num_worlds_global, rank, world_size)
    return DeviceBatchEnv(config, count, env_index_offset=offset, **kw)
