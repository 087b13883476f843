"""Multi-GPU partitioning of the cross-section batch (config 3).

Sections are independent solves: rank r of W owns a contiguous slice of the
section list and runs it as one batched solver on its own GPU.  There is no
collective on the solve path; torch.distributed is used only for the barrier
around the timed region and the max-over-ranks of the device time.
"""
from __future__ import annotations

from typing import List


def section_shard(n_sections: int, rank: int, world: int) -> List[int]:
    """Contiguous, balanced slice of range(n_sections) owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    base, extra = divmod(n_sections, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return list(range(start, start + count))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank timing over all ranks (identity without a process group)."""
    if dist is None or not dist.is_initialized():
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized():
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
