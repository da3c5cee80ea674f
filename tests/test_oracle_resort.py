"""Pins of the per-pixel resort window (tri_depth 2; SURVEY §8(f) row 3's second
variant; SPEC S:235 / S:280: triangle fragments ordered by their plane depth at the
pixel centre; Fig.5b P:511-515 interpenetration).

tri_depth 2 keys the pairs like tri_depth 1 (N8, the tile-centre plane depth) and
then, per pixel, passes the fragments of the tile list through a window of W
entries (a bounded priority queue on (bits(depth at the pixel), id): N9 for a
triangle -- N8's formula at the pixel centre --, the view z for a Gaussian).
Pinned against: the closed-form ray-plane depth at pixel centres (N9); a full
per-pixel sort of the brute-force fragment set when W is at least the number of
fragments (the window is then an exact sort); the tiled path = the brute-force
path at W = 4; and the effect on two interpenetrating opaque quads -- every pixel,
not only every tile, shows the plane nearer at its centre.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

from test_oracle_tri_depth import _plane_z, _tri_scene, _world


def _oracle(oracle_mod, sc, **kw):
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(sc.cameras[0], **oracle_mod.scene_settings(sc, **kw))
    return o


@pytest.mark.parametrize("zs", [(2.0, 5.0, 3.0), (1.0, 1.3, 9.0), (4.0, 2.5, 2.6)])
def test_pixel_depth_matches_ray_plane_intersection(oracle_mod, zs):
    W, H = 96, 64
    cam = scenes.Camera(W, H, 96.0, 96.0, 48.0, 32.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    uv = [(4.0, 3.0), (93.0, 10.0), (20.0, 62.0)]
    P = np.array([_world(cam, u, v, z) for (u, v), z in zip(uv, zs)], np.float32)
    sc = _tri_scene(P, W, H)
    o = _oracle(oracle_mod, sc, tri_depth=2)
    P64 = P.astype(np.float64)
    zmin, zmax = min(zs), max(zs)
    inside = 0
    for y in range(0, H, 3):
        for x in range(0, W, 3):
            zc = _plane_z(P64, cam, x + 0.5, y + 0.5)
            got = float(o.tri_pixel_depth(0, x, y))
            if zc > 0:
                want = min(max(zc, zmin), zmax)
                assert abs(got - want) <= 2e-6 * want, (x, y, got, want)
                inside += zmin < zc < zmax
            else:
                assert got == np.float32(zmax)
    assert inside >= 100


def _full_sort_blend(oracle_mod, o, x, y, st):
    """Every fragment of pixel (x, y) (brute force, C.1 membership), sorted by
    (bits(depth at the pixel), id), blended by the state machine."""
    fr = o.pixel_fragments(x, y)
    if len(fr) == 0:
        return None
    order = np.lexsort((fr["id"], fr["pdepth"].view(np.uint32)))
    out, _ = oracle_mod.blend_fragments(fr[order], **st)
    return out


CASES = [("crossing_g", lambda: scenes.make_crossing(W=136, n_gauss=300, alpha=0.6)),
         ("random0", lambda: scenes.make_random(0)),
         ("nested", lambda: scenes.make_nested(W=64, H=64))]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_wide_window_is_the_full_per_pixel_sort(oracle_mod, name, mk):
    sc = mk()
    st = oracle_mod.scene_settings(sc, tri_depth=2, resort_window=64, t_eps=0.0)
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = o.full(sc.cameras[0], **st)
    n = 0
    H, W = sc.cameras[0].height, sc.cameras[0].width
    for y in range(0, H, 3):
        for x in range(0, W, 3):
            fr = o.pixel_fragments(x, y)
            if len(fr) > 64:
                continue
            ref = _full_sort_blend(oracle_mod, o, x, y, st)
            if ref is None:
                continue
            np.testing.assert_allclose(img[y, x], ref, atol=1e-12)
            n += (fr["kind"] == 1).any()
    assert n > 30


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_tiled_equals_bruteforce_w4(oracle_mod, name, mk):
    sc = mk()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = o.full(sc.cameras[0], **oracle_mod.scene_settings(sc, tri_depth=2))
    assert np.array_equal(img, o.render_bruteforce())


def test_crossing_quads_every_pixel_shows_the_nearer_plane(oracle_mod):
    """Opaque crossing quads (1/z affine across each quad, make_crossing): tri_depth 2
    shows, at every pixel whose 4 samples both quads cover, the quad nearer at the
    pixel centre -- also in the tiles the intersection line crosses, where the per-tile
    order of tri_depth 1 must be wrong on one side of the line."""
    sc = scenes.make_crossing(W=136, alpha=1.0)  # the crossing column x = 68 lies inside tile 4
    cam = sc.cameras[0]
    W = cam.width
    u0, u1 = 6.0, W - 6.0
    res = {}
    for td in (1, 2):
        o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
        img = o.full(cam, **oracle_mod.scene_settings(sc, tri_depth=td))
        good = bad = 0
        for y in range(8, cam.height - 8):
            for x in range(8, W - 8):
                u = x + 0.5
                t = (u - u0) / (u1 - u0)
                za = 1.0 / ((1 - t) / 2.0 + t / 4.0)  # quad A: z 2 -> 4 left to right
                zb = 1.0 / ((1 - t) / 4.0 + t / 2.0)  # quad B: z 4 -> 2
                if abs(za - zb) < 1e-3:
                    continue
                red = za < zb
                pix = img[y, x, :3]
                ok = (pix[0] > 0.9 and pix[1] < 0.2) if red else (pix[1] > 0.9 and pix[0] < 0.2)
                good += ok
                bad += not ok
        res[td] = (good, bad)
    assert res[2][1] == 0 and res[2][0] > 5000
    assert res[1][1] > 0  # the per-tile order misorders the pixels around the crossing column


def test_resort_tracks_the_supersampled_truth(oracle_mod):
    """Against the 16x16 supersampled ground truth that orders each sub-sample by the
    plane depth there: tri_depth 2's error is no larger than tri_depth 1's and smaller
    on the pixels of the tiles the intersection crosses."""
    sc = scenes.make_crossing(alpha=0.6, W=72, H=48)  # crossing column x = 36, inside tile 2
    cam = sc.cameras[0]
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc, tri_depth=2))
    gt = o.render_supersampled(16)  # per sub-sample: the plane depth there orders the fragments
    errs = {}
    for td in (1, 2):
        img = o.full(cam, **oracle_mod.scene_settings(sc, tri_depth=td))
        errs[td] = np.abs(img[..., :3] - gt[..., :3]).mean(-1)
    cx = cam.width // 2
    band = (slice(4, cam.height - 4), slice(16 * (cx // 16), 16 * (cx // 16) + 16))
    assert errs[2].mean() <= errs[1].mean() + 1e-12
    assert errs[2][band].mean() < 0.5 * errs[1][band].mean()
