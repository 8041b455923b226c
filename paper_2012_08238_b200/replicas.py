"""Multi-GPU replicas: the path shards by signal, so each
rank owns a disjoint slice of the signal queue and runs it with no data-path
collective.  Only the measurement is combined: device time is the MAX over
ranks and the transform count is the SUM."""

from __future__ import annotations


def shard(total: int, rank: int, world: int) -> range:
    """Contiguous, disjoint, covering slice of ``range(total)`` for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} / world {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def combine(ms: float, count: int, device=None):
    """(max over ranks of ms, sum over ranks of count); identity without a
    process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(ms), int(count)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    c = torch.tensor([int(count)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), int(c.item())
