"""Device time of unimgs_bind (LBVH build + traversal) on SPEC's binding workload.

python tools/bind_timing.py [--n 100000] [--lon 250 --lat 100] [--cams 8] [--iters 5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--lon", type=int, default=250)
    ap.add_argument("--lat", type=int, default=100)
    ap.add_argument("--cams", type=int, default=8)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    g, mesh, cams = scenes.make_bind_case(n_gauss=a.n, lon=a.lon, lat=a.lat, n_cams=a.cams)
    dev = lambda x, dt=torch.float32: torch.as_tensor(np.ascontiguousarray(x)).to("cuda", dt)  # noqa: E731
    args = (dev(g.means), dev(g.quats), dev(g.scales), dev(mesh.positions), dev(mesh.faces, torch.int32), cams)
    out = {"gaussians": a.n, "faces": mesh.num_triangles, "cameras": a.cams}
    for mode in (0, 1):
        R.bind(*args, mode)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            face, _ = R.bind(*args, mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        rays = a.n * (1 if mode == 0 else 8) * a.cams
        out[f"mode{mode}"] = {"ms": ms, "rays": rays, "grays_per_s": rays / ms / 1e6,
                              "bound_frac": float((face >= 0).float().mean().item())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
