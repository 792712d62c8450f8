"""Multi-GPU plumbing for the keyframe-batch step (P:284 global optimisation).

A single frame never leaves its GPU.  A batch of views is split across ranks (one process per GPU);
each rank renders its views and accumulates the gradient of the shared unstable-slot parameters,
then ONE collective sums the gradient buffers over ranks (NCCL over NVLink on the GPU box, gloo in
the CPU tests) before the identical Adam step runs on every rank.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0)))


def view_partition(n_views: int, world: int, rank: int) -> list[int]:
    """Contiguous block of views owned by `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def allreduce_grads(grad: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank gradient buffers in place (one collective per optimiser step)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def global_step_distributed(eng, views, group=None, ratio=0.4, lr_scale=0.1):
    """(e) the keyframe batch over ranks: this rank's contiguous block of `views` (every rank passes
    the same full list), the batch-mean loss weights (1 / len(views)), one gradient all-reduce, then
    the identical Adam step on every rank (the parameters stay replicated)."""
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    mine = [views[v] for v in view_partition(len(views), world, rank)]
    return eng.global_step(mine, ratio=ratio, lr_scale=lr_scale, n_total=len(views),
                           reduce_grads=lambda g: allreduce_grads(g, group))
