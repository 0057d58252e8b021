"""Multi-GPU sharding of the TVOLAP lanes.

Lanes (channels / sources) are independent (proj/tests/test_engine.cpp:91-102), so
one process per GPU takes a contiguous lane range and no data-path collective is needed. The
only exchange is config C3's stereo mix: each rank reduces its own sources on the device
(tvolap_mix_device) and the partial mixes are summed with one all-reduce (NCCL on GPUs; the
same code runs on gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple


def weak_lanes(sources_per_rank: int, rank: int) -> Tuple[int, int]:
    """Weak scaling (bench.py): every rank runs its own `sources_per_rank` lanes, seeded lane0 = rank * S."""
    return rank * sources_per_rank, sources_per_rank


def strong_lanes(total_sources: int, rank: int, world: int) -> Tuple[int, int]:
    """Strong scaling: split `total_sources` into contiguous, as-equal-as-possible ranges."""
    base, extra = divmod(total_sources, world)
    lane0 = rank * base + min(rank, extra)
    return lane0, base + (1 if rank < extra else 0)


def mix_allreduce(partial_mix, group=None):
    """Sum the per-rank partial mixes (ears x samples) in place across ranks."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial_mix, op=dist.ReduceOp.SUM, group=group)
    return partial_mix


def max_over_ranks(value: float, device=None) -> float:
    """Max of a timing over ranks (bench.py reports the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
