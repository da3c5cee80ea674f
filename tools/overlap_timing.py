"""Multi-view throughput with 1 vs S renderer contexts on S CUDA streams (views round-robin),
to measure how much of preprocess/binning hides under the compute-bound blend of the
previous view.   python tools/overlap_timing.py [--views 32] [--streams 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402


def run(sc, ds, renderers, streams, views, outs):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for s in streams:
        s.wait_stream(main)
    for j, vi in enumerate(views):
        k = j % len(renderers)
        renderers[k].render_view(ds, sc.cameras[vi], out=outs[j], stream=streams[k])
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=32)
    ap.add_argument("--streams", type=int, default=2)
    a = ap.parse_args()
    sc = scenes.make_multiview()
    ds = R.to_device(sc)
    W, H = 1920, 1080
    rs = [R.Renderer(sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H) for _ in range(a.streams)]
    ss = [torch.cuda.Stream() for _ in range(a.streams)]
    outs = [torch.empty((H, W, 4), device="cuda") for _ in range(a.views)]
    views = list(range(a.views))
    res = {}
    for n in (1, a.streams):
        run(sc, ds, rs[:n], ss[:n], views[:4], outs)
        ms = min(run(sc, ds, rs[:n], ss[:n], views, outs) for _ in range(3))
        res[f"streams_{n}"] = {"ms_per_frame": ms / a.views, "fps": 1000 * a.views / ms}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
