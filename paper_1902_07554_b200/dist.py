"""Multi-GPU plumbing for bench.py (one process per GPU, torch.distributed).

The path shards over independent objects: each rank owns a whole instance of
the configuration (its own seeded point set, sample and partial DTs), so the
data path has no collective. The only cross-rank operations are the timing
barrier and the max-over-ranks reduction of the measured time.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def rank_seed(base_seed: int, rank: int, world_size: int) -> int | None:
    """Seed of rank's instance: the config's own seed on a single GPU, a
    distinct derived seed per rank otherwise (independent shards)."""
    if world_size <= 1:
        return None
    return base_seed * 1000 + rank


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: int, world_size: int, max_seconds: float) -> float:
    """Whole-job throughput: all ranks' units over the slowest rank's time."""
    return world_size * units_per_rank / max_seconds
