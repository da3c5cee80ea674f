"""Camera-view sharding across GPUs and the frame gather.

Views are independent units: view i of an orbit goes to rank i mod N (the
interleave evens out cost along the orbit).  The scene is replicated.  The only
collective is the gather of rendered frames to rank 0, done with grouped
point-to-point send/recv (NCCL has no native gather), issued on a separate
stream so it overlaps the next step's rendering -- or, fused, by the blend
storing into rank 0's buffer over P2P with device-side step flags
(P2PFrameGather).  run_gather_pipeline is the step schedule both bench.py and
the gloo tests drive.
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


def run_gather_pipeline(first: int, steps: int, views_per_step: int, rank: int, world: int, n_views: int,
                        render, post, on_done=None):
    """The multi-view bench's step schedule, shared by bench.py and the
    world-size-2 gloo test: step k renders this rank's views ``views_for_rank(k, ...)``
    into frame buffer ``k & 1`` (``render(k, views, buf)``), then posts its gather
    (``post(k, buf)`` -> work handles); the handles of step k - 1 are waited only after
    step k has been enqueued, so the gather of k - 1 overlaps the rendering of k and
    buffer (k + 1) & 1 is free again before step k + 1 writes it (double buffering).
    ``on_done(k)`` runs once step k's handles completed (rank 0 may then read what it
    received for step k)."""
    pending, prev = [], None
    for k in range(first, first + steps):
        buf = k & 1
        render(k, views_for_rank(k, views_per_step, rank, world, n_views), buf)
        new = post(k, buf)
        for q in pending:
            q.wait()
        if on_done is not None and prev is not None:
            on_done(prev)
        pending, prev = new, k
    for q in pending:
        q.wait()
    if on_done is not None and prev is not None:
        on_done(prev)


class _DevicePtr:
    """Wraps a raw device pointer as an array (``__cuda_array_interface__``) so torch can
    view it without a copy."""

    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def _ipc_export(rt, nbytes):
    err, ptr = rt.cudaMalloc(nbytes)
    _check(err, "cudaMalloc")
    err, h = rt.cudaIpcGetMemHandle(ptr)
    _check(err, "cudaIpcGetMemHandle")
    return int(ptr), bytes(h.reserved)


def _ipc_import(rt, handle: bytes):
    h = rt.cudaIpcMemHandle_t()
    h.reserved = handle
    err, ptr = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
    _check(err, "cudaIpcOpenMemHandle")
    return int(ptr)


class P2PFrameGather:
    """The fused frame gather (SURVEY §8(e) variant): every rank's blend stores its frames
    straight into rank 0's frame buffer over NVLink P2P, so no separate collective runs,
    and steps complete through device-side flags -- no host barrier, no device sync.

    Rank 0 ``cudaMalloc``s buf [2][world][V][H][W][4] (double-buffered by step) plus one
    int32 ``done`` flag per rank, and shares their CUDA IPC handles; rank r > 0 shares
    one int32 ``free`` flag of its own.  Rank r passes ``frames(step)`` -- its slot
    buf[step % 2][r] -- as the ``out`` of ``Renderer.render``, so the blend's epilogue
    writes the remote frame directly.  Per step (stream memory operations, executed by
    the GPU front end, no kernel waits on another rank):
      * ``before_step(k, ...)``: rank r > 0 waits (GEQ) until its ``free`` flag says
        rank 0 has released step k - 2 -- the slot step k overwrites;
      * ``step_done(k, ...)``: rank r > 0 writes done[r] = k + 1 into rank 0's memory
        after its step-k renders; rank 0 waits done[r] >= k + 1 for every r (then
        step k's frames are complete in its buffer) and writes free = k + 1 into every
        rank's flag.
    Both run on flag streams of their own, so a step's renders queue behind the
    previous step's without a join (the pipelining of the 1-GPU bench).
    """

    def __init__(self, V: int, H: int, W: int, rank: int, world: int, group=None):
        from cuda.bindings import driver as drv
        from cuda.bindings import runtime as rt
        self.rt, self.drv, self.rank, self.world, self.group = rt, drv, rank, world, group
        self.shape = (2, world, V, H, W, 4)
        nbytes = 4 * 2 * world * V * H * W * 4
        obj = [None, None]
        if rank == 0:
            self.ptr, h = _ipc_export(rt, nbytes)
            self.done_ptr, hd = _ipc_export(rt, 4 * world)
            _check(rt.cudaMemset(self.done_ptr, 0, 4 * world)[0], "cudaMemset")
            obj = [h, hd]
        dist.broadcast_object_list(obj, src=0, group=group)
        if rank != 0:
            self.ptr = _ipc_import(rt, obj[0])
            self.done_ptr = _ipc_import(rt, obj[1])
        # every rank r > 0: its own free flag, imported by rank 0
        self.free_ptr, hf = _ipc_export(rt, 4)
        _check(rt.cudaMemset(self.free_ptr, 0, 4)[0], "cudaMemset")
        _check(rt.cudaDeviceSynchronize()[0], "cudaDeviceSynchronize")
        handles = [None] * world
        dist.all_gather_object(handles, hf, group=group)
        self.peer_free = {}
        if rank == 0:
            self.peer_free = {r: _ipc_import(rt, handles[r]) for r in range(1, world)}
        self.buf = torch.as_tensor(_DevicePtr(self.ptr, self.shape), device="cuda")
        self.flag_stream = torch.cuda.Stream()  # done-flag writes / waits (rank 0: the release)
        self.free_stream = torch.cuda.Stream()  # waits for the slot of the next step
        dist.barrier(group=group)

    def frames(self, step: int) -> torch.Tensor:
        """This rank's slot of the step: [V, H, W, 4] on rank 0's device memory."""
        return self.buf[step % 2][self.rank]

    def _wait_geq(self, stream, ptr, value):
        r, = self.drv.cuStreamWaitValue32(self.drv.CUstream(stream.cuda_stream), ptr, value,
                                         self.drv.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
        _check_drv(r, "cuStreamWaitValue32")

    def _write(self, stream, ptr, value):
        r, = self.drv.cuStreamWriteValue32(self.drv.CUstream(stream.cuda_stream), ptr, value,
                                          self.drv.CUstreamWriteValue_flags.CU_STREAM_WRITE_VALUE_DEFAULT)
        _check_drv(r, "cuStreamWriteValue32")

    def before_step(self, step: int, streams):
        """Make `streams` (the contexts rendering step `step`) wait until rank 0 has released
        step - 2, whose slot this step overwrites (rank 0 itself never waits)."""
        if self.rank == 0 or step < 2:
            return
        self._wait_geq(self.free_stream, self.free_ptr, step - 1)
        ev = torch.cuda.Event()
        ev.record(self.free_stream)
        for st in streams:
            st.wait_event(ev)

    def step_done(self, step: int, streams):
        """Enqueue the completion of `step` once every stream in `streams` has rendered it."""
        fs = self.flag_stream
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            fs.wait_event(ev)
        if self.rank != 0:
            self._write(fs, self.done_ptr + 4 * self.rank, step + 1)
            return
        for r in range(1, self.world):
            self._wait_geq(fs, self.done_ptr + 4 * r, step + 1)
        for r, fp in self.peer_free.items():
            self._write(fs, fp, step + 1)

    def join(self, stream):
        """`stream` waits for every enqueued completion (rank 0: all ranks' frames landed)."""
        stream.wait_stream(self.flag_stream)
        stream.wait_stream(self.free_stream)

    def close(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self.buf = None
        if self.rank != 0:  # importers unmap first; the exporter frees after them
            self.rt.cudaIpcCloseMemHandle(self.ptr)
            self.rt.cudaIpcCloseMemHandle(self.done_ptr)
        else:
            for fp in self.peer_free.values():
                self.rt.cudaIpcCloseMemHandle(fp)
        dist.barrier(group=self.group)
        self.rt.cudaFree(self.free_ptr)
        if self.rank == 0:
            self.rt.cudaFree(self.ptr)
            self.rt.cudaFree(self.done_ptr)


def _check(err, what):
    from cuda.bindings import runtime as rt
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"{what}: {err}")


def _check_drv(err, what):
    from cuda.bindings import driver as drv
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"{what}: {err}")
