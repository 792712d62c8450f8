"""World-size-2 gloo tests of the multi-GPU host logic (view partition, gradient all-reduce, the
sharded optimiser's row reduce-scatter / all-gather)."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_19706_b200.dist import allreduce_grads, view_partition


def test_view_partition_covers_all_views_once():
    for n in (1, 7, 64, 65):
        for w in (1, 2, 3, 4, 8):
            parts = [view_partition(n, w, r) for r in range(w)]
            flat = [v for p in parts for v in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_views, S, D = 10, 37, 58
    rng = np.random.default_rng(0)
    per_view = rng.normal(size=(n_views, S, D)).astype(np.float32)
    g = torch.zeros((S, D))
    for v in view_partition(n_views, world, rank):
        g += torch.as_tensor(per_view[v])           # each rank accumulates its own views
    allreduce_grads(g)
    q.put((rank, g.numpy(), per_view.sum(0)))
    dist.destroy_process_group()


def test_gloo_allreduce_equals_sum_over_all_views():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for _, g, ref in res:
        np.testing.assert_allclose(g, ref, rtol=1e-5, atol=1e-5)
    np.testing.assert_array_equal(res[0][1], res[1][1])


def _shard_worker(rank, world, port, q):
    from paper_2404_19706_b200.dist import all_gather_rows_, reduce_scatter_rows_, shard_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, D = 37, 5
    rng = np.random.default_rng(rank)
    mine = rng.normal(size=(S, D)).astype(np.float32)      # this rank's gradient of every slot
    per, padded = shard_rows(S, world)
    full = torch.zeros((padded, D))
    full[:S] = torch.as_tensor(mine)
    block = reduce_scatter_rows_(full, world, rank)          # in place: this rank's rows of `full`
    summed = block.numpy().copy()
    block.mul_(2.0).add_(rank)                               # stand-in for the per-block optimiser
    all_gather_rows_(full, world, rank)                      # in place: every rank's block everywhere
    q.put((rank, per, summed, full.numpy().copy()))
    dist.destroy_process_group()


def test_gloo_sharded_rows_round_trip():
    """The in-place reduce-scatter (emulated on gloo) leaves each rank the summed rows of its block in
    place; the in-place all-gather puts every rank's updated block into every rank's buffer in rank
    order (padding rows included)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=60)
    S, D = 37, 5
    total = sum(np.random.default_rng(r).normal(size=(S, D)).astype(np.float32) for r in range(world))
    per = res[0][1]
    assert per == 19
    padded = np.zeros((per * world, D), np.float32)
    padded[:S] = total
    for rank, _, block, gathered in res:
        np.testing.assert_allclose(block, padded[rank * per:(rank + 1) * per], rtol=1e-6, atol=1e-6)
    expect = np.concatenate([res[r][2] * 2.0 + r for r in range(world)], 0)
    for _, _, _, gathered in res:
        np.testing.assert_allclose(gathered, expect, rtol=1e-6)
