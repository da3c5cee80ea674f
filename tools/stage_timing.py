"""Per-stage device timing (CUDA events on the launching stream) for one config.

python tools/stage_timing.py --config mip360 --iters 20 [--sort-mode 0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mip360")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--sort-mode", type=int, default=0)
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--tri-depth", type=int, default=0)
    a = ap.parse_args()
    t0 = time.time()
    sc = scenes.make_scene(a.config)
    gen = time.time() - t0
    cam = sc.cameras[a.view]
    r = R.renderer_for(sc, max_pairs=24 << 20, sort_mode=a.sort_mode, tri_depth=a.tri_depth)
    ds = R.to_device(sc)
    out = torch.empty((cam.height, cam.width, 4), device="cuda")
    for _ in range(3):
        r.render_view(ds, cam, out=out)
    st = r.stats()
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = [0.0, 0.0, 0.0]
    for _ in range(a.iters):
        ev[0].record(s)
        r.preprocess(ds, cam)
        ev[1].record(s)
        r.bin()
        ev[2].record(s)
        r.render(out)
        ev[3].record(s)
        torch.cuda.synchronize()
        for i in range(3):
            acc[i] += ev[i].elapsed_time(ev[i + 1])
    ms = [x / a.iters for x in acc]
    print(json.dumps(dict(config=a.config, sort_mode=a.sort_mode, tri_depth=a.tri_depth, gen_s=round(gen, 2), preprocess_ms=ms[0],
                          bin_ms=ms[1], render_ms=ms[2], frame_ms=sum(ms), fps=1000 / sum(ms), stats=st)))


if __name__ == "__main__":
    main()
