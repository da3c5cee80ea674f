"""GPU-vs-oracle comparison helpers for the -m gpu parity tests.

Bar (north_star): per-primitive key-relevant records, the key
multiset, the sorted (key, id) array and the tile ranges bit-exact; colour
within 1e-3 max abs per channel (and T within 1e-3).
"""
import numpy as np

COLOUR_TOL = 1e-3


def run_gpu(scene, cam, sort_mode=0, max_pairs=None, renderer=None):
    import torch
    from paper_2601_19233_b200 import renderer as R
    r = renderer or R.renderer_for(scene, max_pairs=max_pairs, sort_mode=sort_mode)
    ds = R.to_device(scene)
    img = r.render_view(ds, cam)
    torch.cuda.synchronize()
    return r, ds, img.cpu().numpy()


def run_oracle(oracle_mod, scene, cam):
    o = oracle_mod.Oracle(scene.gaussians, scene.mesh)
    o.project(cam, **oracle_mod.scene_settings(scene))
    o.bin()
    return o


def compare_records(r, o, scene):
    rec = r.records()
    F = scene.mesh.num_triangles
    og, ot = o.gaussian_records(), o.triangle_records()
    touched_o = np.concatenate([ot["touched"], og["touched"]])
    assert np.array_equal(rec["touched"], touched_o), "tiles_touched differ"
    vis = touched_o > 0
    assert np.array_equal(rec["rect"][vis], np.concatenate([ot["rect"], og["rect"]])[vis]), "tile rects differ"
    depth_o = np.concatenate([ot["depth"], og["rec"][:, 7]]).astype(np.float32).view(np.uint32)
    assert np.array_equal(rec["dkey"][vis], depth_o[vis]), "depth keys differ"
    assert np.all(rec["dkey"][~vis] == 0xFFFFFFFF)
    gv = og["touched"] > 0
    if gv.any():
        g = rec["grec"][gv]
        # u v qmax o ca cb cc: bit-exact (depth is compared through the depth keys above)
        assert np.array_equal(g[:, :7].view(np.uint32), og["rec"][gv][:, :7].view(np.uint32)), "gaussian records differ"
        assert np.abs(g[:, 8:11] - og["rgb"][gv]).max() < 1e-5, "SH colour"
    tv = ot["touched"] > 0
    if tv.any():
        t = rec["trec"][tv]
        xy = np.stack([t[:, 0], t[:, 1], t[:, 2], t[:, 3], t[:, 4], t[:, 5]], -1)
        assert np.array_equal(xy, ot["xy"][tv]), "snapped vertices differ"
        assert np.array_equal(t[:, 11].view(np.uint32), ot["depth"][tv].view(np.uint32))
    del F


def compare_bins(r, o):
    k, v, rg = r.bins()
    ok, ov, orr = o.bins()
    assert len(k) == len(ok), f"K differs: gpu {len(k)} oracle {len(ok)}"
    assert np.array_equal(k, ok), "sorted keys differ"
    assert np.array_equal(v, ov), "sorted ids differ"
    assert np.array_equal(rg, orr), "tile ranges differ"
    return len(k)


def compare_image(img, ref, tol=COLOUR_TOL):
    mask = ~np.isnan(ref[..., 0])
    assert mask.any()
    d = np.abs(img[mask].astype(np.float64) - ref[mask])
    assert np.isfinite(img[mask]).all()
    err = float(d.max())
    assert err <= tol, f"max abs colour/T error {err:.3e} > {tol}"
    return err
