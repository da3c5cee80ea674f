"""Pins for the oracle's per-pixel fragment bookkeeping (run with -m "not gpu").

or_render_counts walks each pixel's tile list (the keys/sort/ranges path) and
reports the fragments it blended; with t_eps = 0 nothing terminates, so the
counts must equal the brute-force fragment set of C.1 (every primitive tested at
every pixel: a Gaussian is a fragment iff its tile rect holds the pixel's tile and
q <= q_max, alpha >= 1/255; a triangle iff its coverage mask is non-zero,
P:300), split by kind, and the last id must be the last of the brute-force order
(depth bits, id).  This is what the GPU's unimgs_render_fragments is compared
against bit for bit.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

CASES = [("needles", lambda: scenes.make_needles(n=600, W=96, H=80)),
         ("random0", lambda: scenes.make_random(0)),
         ("nested", lambda: scenes.make_nested(W=64, H=64)),
         ("overflow", lambda: scenes.make_overflow())]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_counts_equal_bruteforce_fragments(oracle_mod, name, mk):
    sc = mk()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(sc.cameras[0], **oracle_mod.scene_settings(sc, t_eps=0.0))
    o.bin()
    cnt = o.fragment_counts()
    H, W = sc.cameras[0].height, sc.cameras[0].width
    nz = 0
    for y in range(0, H, 3):
        for x in range(0, W, 2):
            fr = o.pixel_fragments(x, y)
            ng = int((fr["kind"] == 0).sum())
            nt = int((fr["kind"] == 1).sum())
            assert (cnt[y, x, 0], cnt[y, x, 1]) == (ng, nt), (x, y)
            assert cnt[y, x, 2] == (fr["id"][-1] if len(fr) else 0xFFFFFFFF)
            nz += len(fr) > 0
    assert nz > 100


def test_counts_stop_at_termination(oracle_mod):
    """With t_eps > 0 a pixel stops at the first fragment after which T_eff < t_eps (R16):
    the count is the length of the prefix blend_fragments reports as used."""
    sc = scenes.make_random(9, n_gauss=4000, n_tris=60)
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    st = oracle_mod.scene_settings(sc)
    o.project(sc.cameras[0], **st)
    o.bin()
    cnt = o.fragment_counts()
    stopped = 0
    for y in range(0, sc.cameras[0].height, 4):
        for x in range(0, sc.cameras[0].width, 4):
            fr = o.pixel_fragments(x, y)
            _, trace = oracle_mod.blend_fragments(fr, **st)
            used = fr[:len(trace)]
            assert cnt[y, x, 0] == (used["kind"] == 0).sum() and cnt[y, x, 1] == (used["kind"] == 1).sum()
            stopped += len(trace) < len(fr)
    assert stopped > 20


def test_needles_are_adversarial(oracle_mod):
    """The needle construction really straddles both the blend's culling-exactness
    threshold (cond ~ 1000) and the membership cutoff (pixel centres within 1e-3 q_max)."""
    sc = scenes.make_needles()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(sc.cameras[0])
    r = o.gaussian_records()
    vis = r["touched"] > 0
    ca, cb, cc = r["rec"][vis, 4:7].astype(np.float64).T
    kap = (ca + cc) ** 2 / (ca * cc - cb * cb)
    assert 0.25 < (kap <= 1000).mean() < 0.75
    ys, xs = np.mgrid[0:256, 0:256] + 0.5
    near = 0
    for g in np.nonzero(vis)[0]:
        u, v, qm, _, a, b, c, _ = r["rec"][g].astype(np.float64)
        x0, y0, x1, y1 = r["rect"][g]
        sl = (slice(16 * y0, 16 * (y1 + 1)), slice(16 * x0, 16 * (x1 + 1)))
        dx, dy = xs[sl] - u, ys[sl] - v
        near += int((np.abs(a * dx * dx + 2 * b * dx * dy + c * dy * dy - qm) <= 1e-3 * qm).sum())
    assert near > 300
