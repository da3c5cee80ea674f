"""Multi-rank host logic on CPU: view sharding and the frame gather over gloo, world size 2 and 3."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_19233_b200.dist import (gather_frames, gathered_view_order, run_gather_pipeline, shard_views,
                                        views_for_rank)


def test_views_partition_covers_orbit_once():
    for world in (1, 2, 3, 4, 8):
        seen = []
        for r in range(world):
            seen += shard_views(256, r, world)
        assert sorted(seen) == list(range(256))
        # per-step interleave: 256 / (world * V) steps visit every view once
        V = 4
        steps = 256 // (world * V)
        got = sorted(v for s in range(steps) for r in range(world) for v in views_for_rank(s, V, r, world, 256))
        if 256 % (world * V) == 0:
            assert got == list(range(256))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame(view, H=6, W=5):
    # deterministic synthetic "render" of a view: content encodes the view index
    g = torch.Generator().manual_seed(1000 + view)
    return torch.rand((H, W, 4), generator=g)


def _worker(rank, world, port, V, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for step in range(steps):
            mine = views_for_rank(step, V, rank, world, 256)
            frames = torch.stack([_frame(v) for v in mine])
            recv = torch.empty((world - 1,) + frames.shape) if rank == 0 else None
            for h in gather_frames(frames, recv, rank, world):
                h.wait()
            if rank == 0:
                order = gathered_view_order(step, V, world, 256)
                allf = torch.cat([frames[None], recv])
                for slot, views in enumerate(order):
                    for j, v in enumerate(views):
                        ok &= bool(torch.equal(allf[slot, j], _frame(v)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_frames_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 3, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _pipeline_worker(rank, world, port, V, steps, q):
    """The bench's own step schedule (run_gather_pipeline: double-buffered frames and recv,
    the gather of step k - 1 waited only after step k was enqueued) over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = [torch.full((V, 6, 5, 4), -1.0) for _ in range(2)]
        recv = [torch.full((world - 1, V, 6, 5, 4), -1.0) for _ in range(2)] if rank == 0 else None
        checked, ok = [], True

        def render(k, views, bi):
            for j, v in enumerate(views):
                frames[bi][j] = _frame(v)

        def post(k, bi):
            return gather_frames(frames[bi], recv[bi] if rank == 0 else None, rank, world)

        def on_done(k):
            nonlocal ok
            if rank != 0:
                return
            order = gathered_view_order(k, V, world, 256)
            got = torch.cat([frames[k & 1][None], recv[k & 1]])
            for slot, views in enumerate(order):
                for j, v in enumerate(views):
                    ok &= bool(torch.equal(got[slot, j], _frame(v)))
            checked.append(k)

        run_gather_pipeline(3, steps, V, rank, world, 256, render, post, on_done)
        q.put((rank, ok and (rank != 0 or checked == list(range(3, 3 + steps)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_gather_pipeline_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, world, port, 3, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res
