"""Pins of the per-row ellipse tile spans N5' (tile_cull = 1).

N5' keeps, in each row of a Gaussian's N5 rect, the tiles whose pixel-centre box
meets the padded ellipse {Q <= q_max (1 + 2^-5)}.  Pinned against an independent
formulation (the minimum of the quadratic form over each tile's box, by edge-wise
1-D minimisation -- not the oracle's band x-extent), against the property it must
keep (every pixel with an N6 fragment lies in a kept tile, brute force), its
fallbacks (ill-conditioned conics keep the rect; tile_cull = 0 is the rect), and
its effect (fewer pairs, same image).
"""
import numpy as np

from paper_2601_19233_b200 import scenes


def _oracle(oracle_mod, sc, **kw):
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(sc.cameras[0], **oracle_mod.scene_settings(sc, **kw))
    return o


def _box_min_q(A, B, C, dx0, dx1, dy0, dy1):
    """min of A dx^2 + 2B dx dy + C dy^2 over [dx0,dx1] x [dy0,dy1] (float64, scalar)."""
    if dx0 <= 0 <= dx1 and dy0 <= 0 <= dy1:
        return 0.0
    best = np.inf
    for X in (dx0, dx1):
        dy = min(max(-B * X / C, dy0), dy1)
        best = min(best, A * X * X + 2 * B * X * dy + C * dy * dy)
    for Y in (dy0, dy1):
        dx = min(max(-B * Y / A, dx0), dx1)
        best = min(best, A * dx * dx + 2 * B * dx * Y + C * Y * Y)
    return best


def test_spans_match_box_minimum(oracle_mod):
    sc = scenes.make_random(40, n_gauss=1500, n_tris=0, W=160, H=128)
    o = _oracle(oracle_mod, sc)
    rec = o.gaussian_records()
    checked = 0
    for g in np.nonzero(rec["touched"] > 0)[0][:600]:
        u, v, qmax, _, A, B, C, _ = rec["rec"][g].astype(np.float64)
        x0, y0, x1, y1 = rec["rect"][g]
        det = A * C - B * B
        if (A + C) ** 2 > 1000 * det:
            continue
        Q = qmax * 1.03125
        for ty in range(y0, y1 + 1):
            lo, hi = o.gauss_row_span(g, ty)
            for tx in range(x0, x1 + 1):
                m = _box_min_q(A, B, C, 16 * tx + 0.5 - u, 16 * tx + 15.5 - u, 16 * ty + 0.5 - v, 16 * ty + 15.5 - v)
                if abs(m - Q) <= 1e-9 * Q:
                    continue  # on the boundary: either answer is exact to rounding
                assert (lo <= tx <= hi) == (m <= Q), (g, tx, ty, lo, hi, m, Q)
                checked += 1
    assert checked > 2000


def test_every_fragment_pixel_is_in_a_kept_tile(oracle_mod):
    """Brute force: every (pixel, Gaussian) N6 fragment lies in a tile of its spans,
    including elongated, rotated and large Gaussians."""
    rng = np.random.default_rng(41)
    sc = scenes.make_random(41, n_gauss=800, n_tris=0, W=128, H=96)
    g = sc.gaussians
    g.scales[:200, 0] *= rng.uniform(5, 30, 200).astype(np.float32)  # needles and large splats
    o = _oracle(oracle_mod, sc)
    rec = o.gaussian_records()
    H, W = sc.cameras[0].height, sc.cameras[0].width
    ys, xs = np.mgrid[0:H, 0:W]
    lost = 0
    for gi in np.nonzero(rec["touched"] > 0)[0]:
        r = rec["rec"][gi]
        dx = (xs.astype(np.float32) + np.float32(0.5)) - r[0]
        dy = (ys.astype(np.float32) + np.float32(0.5)) - r[1]
        q = r[4] * (dx * dx) + (r[6] * (dy * dy) + (r[5] + r[5]) * (dx * dy))  # fp32, N6 order up to fma
        frag = q <= r[2] * np.float32(0.999)  # margin for the fma-vs-unfused difference of this check
        x0, y0, x1, y1 = rec["rect"][gi]
        for ty, tx in set(zip((ys[frag] // 16).tolist(), (xs[frag] // 16).tolist())):
            if not (y0 <= ty <= y1 and x0 <= tx <= x1):
                continue  # outside the N5 rect: the documented support truncation, not N5'
            lo, hi = o.gauss_row_span(gi, ty)
            lost += not (lo <= tx <= hi)
    assert lost == 0


def test_ill_conditioned_keeps_rect_and_mode0_is_rect(oracle_mod):
    sc = scenes.make_random(42, n_gauss=400, n_tris=0)
    sc.gaussians.scales[:50] = np.array([0.5, 0.0005, 0.0005], np.float32)  # extreme needles
    o1 = _oracle(oracle_mod, sc, tile_cull=1)
    o0 = _oracle(oracle_mod, sc, tile_cull=0)
    r1, r0 = o1.gaussian_records(), o0.gaussian_records()
    area = (r0["rect"][:, 2] - r0["rect"][:, 0] + 1) * (r0["rect"][:, 3] - r0["rect"][:, 1] + 1)
    vis0 = r0["touched"] > 0
    assert np.array_equal(r0["touched"][vis0], area[vis0])
    assert np.all(r1["touched"] <= r0["touched"])
    for g in np.nonzero(r1["touched"] > 0)[0]:
        _, _, _, _, A, B, C, _ = r1["rec"][g].astype(np.float64)
        if (A + C) ** 2 > 1000 * (A * C - B * B):
            assert r1["touched"][g] == r0["touched"][g]
            x0, y0, x1, y1 = r1["rect"][g]
            assert all(o1.gauss_row_span(g, ty) == (x0, x1) for ty in range(y0, y1 + 1))


def test_fewer_pairs_same_image(oracle_mod):
    sc = scenes.make_nerf()
    cam = sc.cameras[0]
    ks, imgs = {}, {}
    for mode in (0, 1):
        o = _oracle(oracle_mod, sc, tile_cull=mode)
        ks[mode] = o.bin()
        tiles = np.random.default_rng(3).choice(o.tiles_x * o.tiles_y, 150, replace=False)
        imgs[mode] = o.render(tiles)
    assert ks[1] < 0.9 * ks[0], ks
    m = ~np.isnan(imgs[0][..., 0])
    assert np.abs(imgs[0][m] - imgs[1][m]).max() <= 1e-12
    del cam
