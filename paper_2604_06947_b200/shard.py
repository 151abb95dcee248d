"""Ensemble sharding across ranks (SURVEY §8(e) "Ensembles"): B independent problems
(BJ north_star "batched ensembles") are split into contiguous ranges of problems, one per
rank, with no data-path communication; each rank steps its range with one batched plan.
The only collective of an ensemble run is the timing reduction (max over ranks), and the
verification flags.  "Structurally parallel at the execution level"."""
from __future__ import annotations


def ensemble_range(batch_total: int, nranks: int, rank: int):
    """(first, count) of rank's contiguous range of problems; ranges differ by at most one."""
    if not (0 <= rank < nranks) or batch_total < nranks:
        raise ValueError("need 0 <= rank < nranks <= batch_total")
    base, rem = divmod(batch_total, nranks)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The one collective of an ensemble run: the slowest rank's time."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])
