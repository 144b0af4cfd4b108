"""Multi-GPU layer of the view-sharded path.

The path shards by view: every rank holds the full (replicated) Gaussian set, renders its own
views, and accumulates their parameter gradients into one flat fp32 buffer
(`GaussianParams.grad_flat`, group-major).  The only exchange of the path (row a9) is the sum of
that buffer over ranks.  This module provides:

* `partition_views` — which ring views a rank renders per step: strong scaling (a fixed global
  batch split round-robin) or weak scaling (a fixed per-rank batch of distinct views);
* `GradientSync` — the all-reduce of the gradient buffer in Gaussian-row chunks on a
  communication stream, each chunk started as soon as the projection backward has written its
  rows (so the transfer of chunk k overlaps the projection backward of chunk k + 1);
* `ShardedAdam` — the sharded-optimizer variant of row f1 ("Proj Bwd
  + Optimizer"): reduce-scatter of the gradients so each rank owns the summed gradients of 1/N of
  the rows, the Adam step (vks_adam_step) on those rows only, with Adam moments stored for those
  rows only, then an all-gather of the updated parameters.  Same bytes on the wire as the
  all-reduce, 1/N of the optimizer's HBM traffic and moment memory per rank.

Collectives go through torch.distributed (NCCL on GPUs; gloo in the CPU tests).  No arithmetic of
the method happens here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .pipeline import GaussianParams


def views_for_rank(rank: int, world: int, n_views: int) -> list[int]:
    """Round-robin assignment of a batch of `n_views` views to `world` ranks."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank, n_views, world))


def partition_views(rank: int, world: int, views: int, scaling: str = "strong") -> tuple[list[int], int]:
    """(ring view indices rank `rank` renders per step, number of ring cameras).

    strong: one global batch of `views` views (a ring of `views` cameras) split round-robin —
            total work fixed as the world grows (BASELINE config 4: "a batch of 8 views sharded
            across 1/2/4/8").
    weak:   every rank renders `views` distinct views of a ring of `views * world` cameras —
            per-rank work fixed (no view is rendered twice in a step)."""
    if scaling == "strong":
        if views < world:
            raise ValueError(f"strong scaling needs at least one view per rank ({views} < {world})")
        return views_for_rank(rank, world, views), views
    if scaling == "weak":
        return views_for_rank(rank, world, views * world), views * world
    raise ValueError(f"scaling must be 'strong' or 'weak', not {scaling!r}")


def row_chunks(n: int, chunks: int, align: int = 256) -> list[tuple[int, int]]:
    """Split rows [0, n) into `chunks` contiguous ranges whose inner boundaries are multiples of
    `align` (last range takes the remainder); empty ranges are dropped."""
    chunks = max(1, chunks)
    step = -(-n // chunks)
    step = -(-step // align) * align
    out, r = [], 0
    while r < n:
        out.append((r, min(n, r + step)))
        r += step
    return out or [(0, 0)]


def _initialized() -> bool:
    return dist.is_available() and dist.is_initialized()


def allreduce_grads(grad_flat: torch.Tensor, group=None, async_op: bool = False):
    """Sum the flat per-Gaussian gradient buffer over ranks in one call (NCCL on GPUs, gloo on CPU)."""
    if not _initialized():
        return None
    return dist.all_reduce(grad_flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


class GradientSync:
    """Chunked all-reduce of a GaussianParams gradient buffer (row a9).

    Usage per step: for each row chunk (r0, r1) from `chunks()`, enqueue the producer of those
    gradient rows (the projection backward restricted to the rows) on the compute stream, then call
    `launch(r0, r1)`; after the last chunk, `finish()` makes the compute stream wait for the
    transfers.  On CUDA the collectives run on a dedicated stream ordered after an event recorded on
    the compute stream, so chunk k's transfer overlaps the compute of chunk k + 1."""

    def __init__(self, params: GaussianParams, n_chunks: int = 1, group=None, align: int = 256):
        self.params = params
        self.group = group
        self.n_chunks = max(1, n_chunks)
        self.align = align
        self.cuda = params.grad_flat.is_cuda
        self.stream = torch.cuda.Stream(device=params.grad_flat.device) if self.cuda else None
        self.pending = []

    def chunks(self) -> list[tuple[int, int]]:
        return row_chunks(self.params.n, self.n_chunks, self.align)

    def launch(self, r0: int, r1: int):
        if not _initialized():
            return
        groups = self.params.grad_groups(r0, r1)
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.params.grad_flat.device))
            self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                for g in groups:
                    dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)
        else:
            self.pending += [dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
                             for g in groups]

    def finish(self):
        if self.cuda:
            torch.cuda.current_stream(self.params.grad_flat.device).wait_stream(self.stream)
        for w in self.pending:
            w.wait()
        self.pending = []


class ShardedAdam:
    """Sharded optimizer (row f1 variant): reduce-scatter → Adam on this rank's rows → all-gather.

    `params` must be allocated with `GaussianParams.from_host(..., pad_to=world)` so every gradient
    group and parameter tensor splits into `world` equal row shards.  Rank r owns storage rows
    [r * s, (r + 1) * s) with s = n_rows / world, and holds Adam moments for those rows only.
    `adam_fn(step, params, grads, m, v)` updates the five shard groups in place (default:
    vks_adam_step through the C ABI with the learning rates `lrs`)."""

    def __init__(self, params: GaussianParams, lrs: dict, rank: int = 0, world: int = 1, group=None,
                 adam_fn=None, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
        if params.n_rows % world:
            raise ValueError(f"storage rows {params.n_rows} not a multiple of the world size {world}: "
                             "allocate with GaussianParams.from_host(..., pad_to=world)")
        self.p, self.rank, self.world, self.group = params, rank, world, group
        self.s = params.n_rows // world
        self.r0, self.r1 = rank * self.s, (rank + 1) * self.s
        shard_params = params.param_groups(self.r0, self.r1)
        self.m = [torch.zeros_like(t) for t in shard_params]
        self.v = [torch.zeros_like(t) for t in shard_params]
        self.gshard = [torch.zeros(g.numel() // world, dtype=g.dtype, device=g.device) for g in params.grad_groups()]
        if adam_fn is None:
            from . import _vks as V

            def adam_fn(step, prm, grd, m, v):
                V.vks_adam_step(V.make_adam_config(lrs, beta1, beta2, eps, step=step), prm, grd, m, v)
        self.adam_fn = adam_fn

    def step(self, t: int):
        """One optimizer step (t >= 1) on the summed gradients of all ranks."""
        full = self.p.grad_groups()
        if _initialized() and self.world > 1:
            for out, g in zip(self.gshard, full):
                dist.reduce_scatter_tensor(out, g, op=dist.ReduceOp.SUM, group=self.group)
        else:
            for out, g in zip(self.gshard, full):
                out.copy_(g)
        shard_params = self.p.param_groups(self.r0, self.r1)
        grads = [g.view(p.shape) for g, p in zip(self.gshard, shard_params)]
        self.adam_fn(t, shard_params, grads, self.m, self.v)
        if _initialized() and self.world > 1:
            for full_p, sp in zip(self.p.param_groups(), shard_params):
                # NCCL gathers in place (input = this rank's slice of the output); gloo needs a copy
                src = sp if full_p.is_cuda else sp.clone()
                dist.all_gather_into_tensor(full_p, src, group=self.group)
