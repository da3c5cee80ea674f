"""Memory-safety workload: every kernel of libunimgs.so on small inputs -- the tiny
config (the smoke test), a NeRF-synthetic-like view (300k Gaussians + 10k-triangle
textured sphere, 800x800), the fragment-count variant, sort_mode 1 with per-tile
triangle depth, the whole-pixel mode at M = 16, a capacity overflow, the host-buffer
path on 2 lanes, deformation transfer and ray-cast binding -- each checked for
finite output.  compute-sanitizer is closed on this pool, so the evidence comes from
the checked build (libunimgs_checked.so: bounds checks that trap, guard bands after
every scratch buffer):

  UNIMGS_LIB=paper_2601_19233_b200/libunimgs_checked.so python tools/sanitize.py --check-guards --dump a.npz
  python tools/sanitize.py --dump b.npz        # production library: outputs must be identical
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_19233_b200 import renderer as R, scenes  # noqa: E402

OUT = {}
RENDERERS = []


def run(sc, label, **settings):
    r = R.renderer_for(sc, **settings)
    ds = R.to_device(sc)
    cam = sc.cameras[0]
    img = r.render_view(ds, cam)
    r2 = R.renderer_for(sc, **settings)
    r2.preprocess(ds, cam)
    r2.bin()
    img2, cnt = r2.render_fragments()
    torch.cuda.synchronize()
    st = r.stats()
    assert torch.isfinite(img).all() and torch.equal(img, img2), label
    OUT[label] = img.cpu().numpy()
    OUT[label + "_counts"] = cnt.cpu().numpy()
    RENDERERS.extend([r, r2])
    print(f"{label}: K={st['num_pairs']} fragments={int(cnt[..., 0].sum()) + int(cnt[..., 1].sum())}", flush=True)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nerf-gaussians", type=int, default=300_000)
    ap.add_argument("--check-guards", action="store_true")
    ap.add_argument("--dump", default=None)
    a = ap.parse_args()
    run(scenes.make_tiny(), "tiny")
    nerf = scenes.subsample(scenes.make_nerf(), a.nerf_gaussians)
    r = run(nerf, "nerf")
    run(scenes.make_random(2, n_gauss=3000, n_tris=200, W=211, H=117), "random_ragged_tri_depth", sort_mode=1,
        tri_depth=1)
    run(scenes.make_random(3, n_gauss=2000, n_tris=100), "random_whole_pixel_m16", blend_mode=3, msaa=16)
    run(scenes.make_needles(), "needles", t_eps=0.0)
    # capacity overflow: nothing may be written out of bounds
    sc = scenes.make_random(6, n_gauss=2000, n_tris=50)
    ro = R.renderer_for(sc, max_pairs=64)
    ro.render_view(R.to_device(sc), sc.cameras[0])
    assert ro.stats(check=False)["overflow"] == 1
    RENDERERS.append(ro)
    # host-buffer path on two lanes
    host = R.to_pinned(nerf)
    cams = [nerf.cameras[0]] * 3
    r.set_host_lanes(2)
    out = torch.empty((3, nerf.cameras[0].height, nerf.cameras[0].width, 4), dtype=torch.float32).pin_memory()
    r.render_host_async(host, cams, out)
    r.host_wait()
    assert torch.isfinite(out).all()
    OUT["host_path"] = out.numpy().copy()
    print("render_host_async: ok", flush=True)
    # deformation transfer + ray-cast binding
    sc, b = scenes.make_deform(n_gauss=4000, K=8)
    field = scenes.twist_field(sc.mesh)
    ds = R.to_device(sc)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    mo, co = R.deform(ds, dev(b.face.astype(np.int32)), dev(b.bary.astype(np.float32)),
                      dev(sc.mesh.faces.astype(np.int32)), dev(field.packed()))
    face, bary = R.bind(ds.means, ds.quats, ds.scales, ds.positions, ds.faces, sc.cameras, mode=1)
    torch.cuda.synchronize()
    assert torch.isfinite(mo).all() and torch.isfinite(co).all() and torch.isfinite(bary).all()
    OUT["deform_mu"], OUT["deform_cov"] = mo.cpu().numpy(), co.cpu().numpy()
    OUT["bind_face"], OUT["bind_bary"] = face.cpu().numpy(), bary.cpu().numpy()
    print(f"deform + bind: ok (bound anchors {(face >= 0).float().mean().item():.3f})", flush=True)
    if a.check_guards:
        bad = sum(x.check_guards() for x in RENDERERS)
        print(f"guard bytes overwritten: {bad}", flush=True)
        assert bad == 0
    if a.dump:
        np.savez(a.dump, **OUT)
    print("sanitize workload: ok", flush=True)


if __name__ == "__main__":
    main()
