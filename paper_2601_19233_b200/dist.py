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


class _DevicePtr:
    """Wraps a raw device pointer as a float32 array (``__cuda_array_interface__``) so
    torch can view it without a copy."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class P2PFrameGather:
    """The fused frame gather (SURVEY §8(e) variant): every rank's blend stores its frames
    straight into rank 0's frame buffer over NVLink P2P, so no separate collective runs.

    Rank 0 ``cudaMalloc``s buf [2][world][V][H][W][4] (double-buffered by step) and
    shares one CUDA IPC handle; rank r maps it and passes ``frames(step)`` -- its
    slot buf[step % 2][r] -- as the ``out`` of ``Renderer.render``, so the blend's
    epilogue writes the remote frame directly.  ``step_done()`` (device sync +
    barrier) makes a step's frames complete on rank 0.  No kernel waits on another
    rank: ranks only store, then meet at a host barrier.
    """

    def __init__(self, V: int, H: int, W: int, rank: int, world: int, group=None):
        from cuda.bindings import runtime as rt
        self.rt, self.rank, self.world, self.group = rt, rank, world, group
        self.shape = (2, world, V, H, W, 4)
        nbytes = 4 * 2 * world * V * H * W * 4
        obj = [None]
        if rank == 0:
            err, ptr = rt.cudaMalloc(nbytes)
            _check(err, "cudaMalloc")
            err, h = rt.cudaIpcGetMemHandle(ptr)
            _check(err, "cudaIpcGetMemHandle")
            self.ptr = int(ptr)
            obj = [bytes(h.reserved)]
        dist.broadcast_object_list(obj, src=0, group=group)
        if rank != 0:
            h = rt.cudaIpcMemHandle_t()
            h.reserved = obj[0]
            err, ptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
            _check(err, "cudaIpcOpenMemHandle")
            self.ptr = int(ptr)
        self.buf = torch.as_tensor(_DevicePtr(self.ptr, self.shape), device="cuda")

    def frames(self, step: int) -> torch.Tensor:
        """This rank's slot of the step: [V, H, W, 4] on rank 0's device memory."""
        return self.buf[step % 2][self.rank]

    def step_done(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)

    def close(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self.buf = None
        if self.rank != 0:  # importers unmap first; the exporter frees after them
            self.rt.cudaIpcCloseMemHandle(self.ptr)
        dist.barrier(group=self.group)
        if self.rank == 0:
            self.rt.cudaFree(self.ptr)


def _check(err, what):
    from cuda.bindings import runtime as rt
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"{what}: {err}")
