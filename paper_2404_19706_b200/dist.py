"""Multi-GPU plumbing for the keyframe-batch step (P:284 global optimisation).

A single frame never leaves its GPU.  A batch of views is split across ranks (one process per GPU);
each rank renders its views and accumulates the gradient of the shared slot parameters.  Then
either ONE all-reduce sums the gradient buffers before the identical Adam step runs on every rank
(global_step_distributed), or (global_step_sharded) a reduce-scatter hands every rank
the summed gradient of its block of slots, each rank runs Adam on its block only, and an
all-gather of the updated rows brings every rank's map copy back in sync: the same result with
1/N of the optimiser work per rank.  NCCL over NVLink on the GPU box; gloo in the CPU tests (gloo
has no reduce-scatter, so it is emulated by an all-reduce and a slice there).
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


def shard_rows(n_rows: int, world: int) -> tuple[int, int]:
    """(rows per rank, padded total): the slot rows are split in equal contiguous blocks."""
    per = max(1, -(-n_rows // world))
    return per, per * world


def reduce_scatter_rows(full: torch.Tensor, world: int, rank: int, group=None) -> torch.Tensor:
    """Sum `full` [world * per, ...] over ranks and return this rank's block of rows [per, ...]."""
    per = full.shape[0] // world
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return full[rank * per:(rank + 1) * per]
    if dist.get_backend(group) == "nccl":
        out = torch.empty((per,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=group)
        return out
    dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full[rank * per:(rank + 1) * per]


def all_gather_rows(block: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Concatenate every rank's block of rows in rank order."""
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return block
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * block.shape[0],) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
        dist.all_gather_into_tensor(out, block.contiguous(), group=group)
        return out
    parts = [torch.empty_like(block) for _ in range(world)]
    dist.all_gather(parts, block.contiguous(), group=group)
    return torch.cat(parts, 0)


def global_step_sharded(eng, views, group=None, ratio=0.4, lr_scale=0.1):
    """(e) the keyframe batch over ranks with a sharded optimiser: this rank's views ->
    gradient of every slot -> reduce-scatter (each rank: the summed rows of its slot block) -> Adam
    on the block -> all-gather of the updated rows -> every map copy identical."""
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    mine = [views[v] for v in view_partition(len(views), world, rank)]
    eng.global_backward(mine, ratio=ratio, n_total=len(views))
    S, D = int(eng.g_gid.numel()), eng.g_grad.shape[1]
    per, padded = shard_rows(S, world)
    full = torch.zeros((padded, D), dtype=eng.g_grad.dtype, device=eng.g_grad.device)
    full[:S] = eng.g_grad[:S]
    eng.g_grad.zero_()  # consumed
    block = reduce_scatter_rows(full, world, rank, group)
    packed = eng.global_adam_shard(block, rank * per, (rank + 1) * per, lr_scale=lr_scale)
    eng.global_apply_rows(all_gather_rows(packed, world, group))
    return eng.g_loss
