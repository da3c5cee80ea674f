"""Device timing of the deformation transfer (Eq.12-13) on the mip360 Gaussians bound with
K anchors to the mip360 proxy meshes; HBM roofline from the algorithmic bytes.

python tools/deform_timing.py [--K 8] [--iters 20]
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
    a = ap.parse_args()
    sc = scenes.make_mip360(n=a.n)
    t0 = time.time()
    b = scenes.make_binding(np.random.default_rng(0), sc.gaussians, sc.mesh, a.K, nearest=False)
    field = scenes.twist_field(sc.mesh)
    tb = time.time() - t0
    ds = R.to_device(sc)
    dev = lambda x, dt=None: torch.from_numpy(np.ascontiguousarray(x if dt is None else x.astype(dt))).cuda()
    args = (dev(b.face, np.int32), dev(b.bary, np.float32), dev(sc.mesh.faces, np.int32), dev(field.packed()))
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
                          alg_bytes=alg, achieved_gbs=gbs, peak_gbs=peak, frac=gbs / peak, binding_gen_s=round(tb, 1))))


if __name__ == "__main__":
    main()
