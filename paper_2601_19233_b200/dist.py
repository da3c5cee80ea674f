"""Camera-view sharding across GPUs and the frame gather.

Views are independent units: view i of an orbit goes to rank i mod N (the
interleave evens out cost along the orbit).  The scene is replicated.  The only
collective is the gather of rendered frames to rank 0, done with grouped
point-to-point send/recv (NCCL has no native gather), issued on a separate
stream so it overlaps the next step's rendering.
"""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def views_for_rank(step: int, views_per_step: int, rank: int, world: int, n_views: int) -> List[int]:
    """Global view indices rendered by `rank` in `step` (view i -> rank i mod world)."""
    return [((step * views_per_step + v) * world + rank) % n_views for v in range(views_per_step)]


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """All views of an n_views batch owned by `rank` (static interleaved partition)."""
    return list(range(rank, n_views, world))


def gather_frames(frames: torch.Tensor, recv: Optional[torch.Tensor], rank: int, world: int, dst: int = 0):
    """Post the gather of every rank's `frames` [V,H,W,C] into `recv` [world-1,V,H,W,C] on `dst`.

    Returns the list of work handles (wait() before reusing the buffers).  On
    CUDA tensors call it inside `torch.cuda.stream(comm_stream)` after the comm
    stream waited for the rendering; with gloo (CPU tensors) it is plain P2P.
    """
    if world == 1:
        return []
    if rank == dst:
        assert recv is not None and recv.shape[0] == world - 1
        src = [p for p in range(world) if p != dst]
        ops = [dist.P2POp(dist.irecv, recv[i], p) for i, p in enumerate(src)]
    else:
        ops = [dist.P2POp(dist.isend, frames, dst)]
    return dist.batch_isend_irecv(ops)


def gathered_view_order(step: int, views_per_step: int, world: int, n_views: int, dst: int = 0):
    """View index of every slot of [dst's own frames] + recv[world-1] after gather_frames."""
    order = [views_for_rank(step, views_per_step, dst, world, n_views)]
    for p in range(world):
        if p != dst:
            order.append(views_for_rank(step, views_per_step, p, world, n_views))
    return order
