"""Device timing of the deformation transfer (Eq.12-13); HBM roofline from the algorithmic bytes.

  --bind random   : the mip360 Gaussians with K random nearby faces of the mip360 meshes
  --bind raycast  : n Gaussians on the binding workload's 50k-face sphere (scenes.make_bind_case),
                    bound on the GPU by unimgs_bind (K = 8: bbx8, K = 1: centre), so the anchors
                    are the spatially coherent ones the method produces

python tools/deform_timing.py [--K 8] [--iters 20] [--bind random|raycast]
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
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--n", type=int, default=3_000_000)
    ap.add_argument("--bind", default="random", choices=["random", "raycast"])
    a = ap.parse_args()
    dev = lambda x, dt=None: torch.from_numpy(np.ascontiguousarray(x if dt is None else x.astype(dt))).cuda()
    t0 = time.time()
    bind_ms = None
    if a.bind == "random":
        sc = scenes.make_mip360(n=a.n)
        b = scenes.make_binding(np.random.default_rng(0), sc.gaussians, sc.mesh, a.K, nearest=False)
        face, bary = dev(b.face, np.int32), dev(b.bary, np.float32)
        ds = R.to_device(sc)
    else:
        g, mesh, cams = scenes.make_bind_case(n_gauss=a.n)
        sc = scenes.Scene("bound", g, mesh, cams)
        ds = R.to_device(sc)
        pos, fc = dev(mesh.positions, np.float32), dev(mesh.faces, np.int32)
        R.bind(ds.means, ds.quats, ds.scales, pos, fc, cams, 0 if a.K == 1 else 1)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        face, bary = R.bind(ds.means, ds.quats, ds.scales, pos, fc, cams, 0 if a.K == 1 else 1)
        e1.record()
        torch.cuda.synchronize()
        bind_ms = e0.elapsed_time(e1)
    field = scenes.twist_field(sc.mesh)
    tb = time.time() - t0
    args = (face, bary, dev(sc.mesh.faces, np.int32), dev(field.packed()))
    for _ in range(3):
        R.deform(ds, *args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        R.deform(ds, *args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    N = sc.gaussians.count
    alg = N * (12 + 16 + 12 + a.K * (4 + 12) + 12 + 24)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) if os.path.exists(
        os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
    gbs = alg / (ms * 1e-3) / 1e9
    print(json.dumps(dict(kernel="k_deform", N=N, K=a.K, ms=ms, gaussians_per_s=N / (ms * 1e-3),
                          alg_bytes=alg, achieved_gbs=gbs, peak_gbs=peak, frac=gbs / peak, binding=a.bind,
                          bind_ms=bind_ms, bound_frac=float((face >= 0).float().mean().item()),
                          setup_s=round(tb, 1))))


if __name__ == "__main__":
    main()
