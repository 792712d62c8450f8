"""World-size-2 gloo test of the multi-GPU host logic (view partition + gradient all-reduce)."""
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
