"""Where the multi-view bench's frame time goes: the bench's launch configuration
(renderer.ContextPool, 4 contexts, priority streams, 16 views per step) timed
(a) as in the bench, (b) blends only (each context re-renders the bins of its
first view), (c) preprocess + bin only (no blend), each as ms per view.

python tools/bench_diag.py [--steps 10] [--streams 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    sc = scenes.make_multiview()
    W, H = sc.cameras[0].width, sc.cameras[0].height
    pool = R.ContextPool(a.streams, sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H,
                         bg=tuple(float(v) for v in sc.bg), batch=a.batch)
    ds = R.to_device(sc)
    out = torch.empty((a.views, H, W, 4), device="cuda")
    s = torch.cuda.current_stream()
    n = len(pool.rs)

    def full(step):
        cams = [sc.cameras[(step * a.views + j) % 256] for j in range(a.views)]
        pool.render_views(ds, cams, out, after=s)

    def blend_only(step):
        for j in range(a.views):
            pool.rs[j % n].render(out[j], stream=pool.streams[j % n])

    def bin_only(step):
        for j in range(a.views):
            rr, ps = pool.rs[j % n], pool.pstreams[j % n]
            rr.preprocess(ds, sc.cameras[(step * a.views + j) % 256], stream=ps)
            rr.bin(stream=ps)

    def pre_only(step):
        for j in range(a.views):
            rr, ps = pool.rs[j % n], pool.pstreams[j % n]
            rr.preprocess(ds, sc.cameras[(step * a.views + j) % 256], stream=ps)

    def pre_batched(step):
        B = max(1, a.batch)
        for g0 in range(0, a.views, B):
            k = (g0 // B) % (n // B)
            R.preprocess_multi(pool.rs[k * B:(k + 1) * B], ds,
                               [sc.cameras[(step * a.views + g0 + j) % 256] for j in range(B)], stream=pool.bstreams[k])

    res = {}
    modes = [("full", full), ("blend_only", blend_only), ("preprocess_bin_only", bin_only),
             ("preprocess_only", pre_only), ("full2", full)]
    if a.batch > 1:
        modes.append(("preprocess_batched_only", pre_batched))
    for name, fn in modes:
        for k in range(3):
            fn(k)
        for st in pool.streams + pool.pstreams + pool.bstreams:
            s.wait_stream(st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for k in range(a.steps):
            fn(3 + k)
        for st in pool.streams + pool.pstreams + pool.bstreams:
            s.wait_stream(st)
        e1.record(s)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / (a.steps * a.views)
    print(json.dumps({k: round(v, 4) for k, v in res.items()}))


if __name__ == "__main__":
    main()
