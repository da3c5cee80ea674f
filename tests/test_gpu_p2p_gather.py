"""The fused P2P frame gather (dist.P2PFrameGather; SURVEY §8(e) variant) on one GPU.

Two processes share the GPU (CUDA IPC works between processes of one device); rank 1's
blend writes its frames straight into rank 0's buffer through the IPC mapping, steps
complete through device-side flags (stream memory operations: rank 1 writes done, rank 0
waits for it and writes free, rank 1 waits for free before reusing a slot -- no host
barrier, no kernel waits on another rank), and rank 0 checks every gathered frame of the
last two steps bit-for-bit against its own render of the same view.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result):
    import torch
    import torch.distributed as dist
    from paper_2601_19233_b200 import renderer as R, scenes
    from paper_2601_19233_b200.dist import P2PFrameGather, views_for_rank
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = scenes.make_random(17, n_gauss=3000, n_tris=120, W=160, H=96)
    c0 = sc.cameras[0]
    cams = [scenes.Camera(c0.width, c0.height, c0.fx, c0.fy, c0.cx, c0.cy, c0.R,
                          np.asarray(c0.t, np.float32) + np.float32(0.03 * i)) for i in range(8)]
    V = 2
    g = P2PFrameGather(V, c0.height, c0.width, rank, world)
    r = R.renderer_for(sc)
    ds = R.to_device(sc)
    s = torch.cuda.current_stream()
    steps = 5
    for step in range(steps):  # steps >= 2 reuse a slot: the device-side free flags gate it
        g.before_step(step, [s])
        for j, vi in enumerate(views_for_rank(step, V, rank, world, len(cams))):
            r.render_view(ds, cams[vi], out=g.frames(step)[j])
        g.step_done(step, [s])
    g.join(s)
    torch.cuda.synchronize()
    ok = True
    if rank == 0:
        for step in range(steps - 2, steps):  # the last two steps are still in the buffer
            for src in range(world):
                for j, vi in enumerate(views_for_rank(step, V, src, world, len(cams))):
                    want = r.render_view(ds, cams[vi]).clone()
                    torch.cuda.synchronize()
                    ok = ok and torch.equal(g.buf[step % 2][src][j], want)
        result.put(bool(ok))
    g.close()
    dist.destroy_process_group()


def test_p2p_gather_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=10) is True
