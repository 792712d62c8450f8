"""Multi-GPU plumbing for the keyframe-batch step (P:284 global optimisation).

A single frame never leaves its GPU.  A batch of views is split across ranks (one process per GPU);
each rank renders its views and accumulates the gradient of every Gaussian (global slot == map
row).  Then either ONE all-reduce sums the gradient buffers before the identical Adam step runs on
every rank (global_step_distributed), or (global_step_sharded) an in-place
reduce-scatter hands every rank the summed gradient of its block of rows, each rank runs Adam on
its block only, and in-place all-gathers of the map arrays bring every rank's copy back in sync:
the same result with 1/N of the optimiser work per rank, no packing, no scatter, no allocation.
NCCL over NVLink on the GPU box; gloo in the CPU tests (gloo has no reduce-scatter, so it is
emulated by an all-reduce there).
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


def _nccl(group) -> bool:
    return dist.get_backend(group) == "nccl"


def reduce_scatter_rows_(full: torch.Tensor, world: int, rank: int, group=None) -> torch.Tensor:
    """IN PLACE: sum `full` [world * per, ...] over ranks into this rank's block of rows of `full`
    (NCCL in-place reduce-scatter: the output is the input at offset rank * per) and return it."""
    per = full.shape[0] // world
    block = full[rank * per:(rank + 1) * per]
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return block
    if _nccl(group):
        dist.reduce_scatter_tensor(block, full, op=dist.ReduceOp.SUM, group=group)
    else:  # gloo has no reduce-scatter: all-reduce, the block is then in place
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return block


def all_gather_rows_(full: torch.Tensor, world: int, rank: int, group=None) -> torch.Tensor:
    """IN PLACE: every rank's block of rows of `full` [world * per, ...] (its own rows already there)
    is copied to every other rank (NCCL in-place all-gather)."""
    per = full.shape[0] // world
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return full
    block = full[rank * per:(rank + 1) * per]
    if _nccl(group):
        dist.all_gather_into_tensor(full, block, group=group)
    else:  # gloo (CPU or CUDA tensors): an all-reduce of the blocks, each rank contributing its own
        tmp = torch.zeros_like(full)
        tmp[rank * per:(rank + 1) * per] = block
        dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
        full.copy_(tmp)
    return full


def global_step_sharded(eng, views, group=None, ratio=0.4, lr_scale=0.1, world=None, rank=None):
    """(e) the keyframe batch over ranks with a sharded optimiser: this rank's views ->
    gradient of every Gaussian (slot == row) -> in-place reduce-scatter (each rank: the summed rows of
    its block) -> Adam on the block -> in-place all-gathers of the block's rows of the map arrays and
    of eta -> every map copy identical.  No host synchronisation and no allocation per step: the
    gradient buffer and the map storage already have `world` equal blocks of rows
    (MappingEngine._global_state).  `views` has one entry per view of the batch (entries of other
    ranks' views are not read); world = rank = None take the process group's, world=1 runs the whole
    batch here without collectives."""
    on = dist.is_available() and dist.is_initialized()
    if world is None:
        world = dist.get_world_size(group) if on else 1
    if rank is None:
        rank = dist.get_rank(group) if (on and world > 1) else 0
    mine = [views[v] for v in view_partition(len(views), world, rank)]
    eng.global_backward(mine, ratio=ratio, n_total=len(views), world=world)
    per, rows = eng.g_per, eng.g_rows
    reduce_scatter_rows_(eng.g_grad[:rows], world, rank, group)
    if world > 1:  # the other blocks held this rank's partial sums: consumed
        eng.g_grad[: rank * per].zero_()
        eng.g_grad[(rank + 1) * per: rows].zero_()
    eng.global_adam_block(rank * per, (rank + 1) * per, lr_scale=lr_scale)
    gm = eng.gm
    for k in ("pos", "log_scale", "rot", "sh"):
        all_gather_rows_(gm.store[k][:rows], world, rank, group)
    all_gather_rows_(eng._state_store["eta"][:rows], world, rank, group)
    return eng.g_loss
