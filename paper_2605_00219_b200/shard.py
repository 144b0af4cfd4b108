"""View sharding across ranks: Gaussians are replicated, rank r
renders views r, r+N, r+2N, ... of the batch, every view's parameter gradients accumulate into the
rank's flat buffer, and one all-reduce (sum) of that buffer is the only exchange (row a9)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def views_for_rank(rank: int, world: int, n_views: int) -> list[int]:
    """Round-robin assignment of a batch of `n_views` views to `world` ranks."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank, n_views, world))


def allreduce_grads(grad_flat: torch.Tensor, group=None, async_op: bool = False):
    """Sum the flat per-Gaussian gradient buffer over ranks (NCCL on GPUs, gloo on CPU)."""
    if not dist.is_available() or not dist.is_initialized():
        return None
    return dist.all_reduce(grad_flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
