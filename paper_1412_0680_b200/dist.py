"""Multi-GPU plumbing for the encoding path.

Patches are independent, so a multi-GPU run is patch sharding with the
dictionary and tree replicated on every rank; there is no per-iteration
exchange.  The only collectives are the inner-product totals (the reference's
``ScoreCounter.merge``, pkg/src/stmp/dictionary.py:61-63, summed across ranks)
and max-over-ranks timing.
"""

from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) patch range of `rank` (first ranks get the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_counters(local_ip, group=None):
    """Sum per-rank (inner_products, centroid_inner_products) totals.

    ``local_ip`` is a length-2 int64 tensor on the rank's device (CPU tensor with
    gloo).  Returns the global totals as a Python tuple."""
    import torch
    import torch.distributed as dist
    t = local_ip.clone().to(torch.int64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t[0]), int(t[1])


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms): the job time of a weak-scaling step."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
