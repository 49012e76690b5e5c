"""Bin-slab sharding of the likelihood-map path across ranks.

Each rank owns a contiguous slab of bins [k0, k1), builds that slab of the integral
histogram and the slab's partial window statistic (the per-bin terms summed over its
bins), and one reduce adds the partial maps on the destination rank, which then runs
the finalisation.  Everything here is plumbing on torch.distributed (NCCL on GPUs,
gloo in the CPU tests); the computation lives in the CUDA kernels.

The reference has no multi-device path; the decomposition is exact
because every plane depends only on [bin == k] and the window statistic is a sum
over bins (likelihood.cpp:215-219).
"""
from __future__ import annotations


def slab_bounds(nbins: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal bin slab of `rank` (the first nbins % world ranks get one more)."""
    if not (world >= 1 and 0 <= rank < world and nbins >= 1):
        raise ValueError("slab_bounds: need world >= 1, 0 <= rank < world, nbins >= 1")
    base, extra = divmod(nbins, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def reduce_partials(partial, dst: int = 0, group=None, async_op: bool = False):
    """Sum the ranks' partial maps onto `dst` (one collective per frame)."""
    import torch.distributed as dist

    return dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (step time) over all ranks."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
