"""Pins for the CPU oracle (run with -m "not gpu").

Each test checks the oracle against something other than itself: a worked
example printed in SPEC/derived by hand from the paper's equations (golden
fixtures), a closed form, a textbook/library routine, an invariant, or a brute
force on tiny inputs.  Citations: PAPER.md line numbers (P:L), SPEC.md (S:L).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _frag_list(oracle_mod, items):
    return oracle_mod.frags(*[dict(kind=it["kind"], alpha=it["alpha"], rgb=it["rgb"], mask=it.get("mask", 0))
                              for it in items])


# --------------------------------------------------------------------------
# worked examples (Eq.1-2, 7-11; Fig.3)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("ex", GOLDEN["examples"], ids=lambda e: e["name"])
def test_worked_examples(oracle_mod, ex):
    out, _ = oracle_mod.blend_fragments(_frag_list(oracle_mod, ex["frags"]), t_eps=0.0,
                                        bg=tuple(ex.get("bg", (0, 0, 0))))
    np.testing.assert_allclose(out, ex["out"], atol=1e-12)


def test_fig3_whole_pixel_entity_would_overflow(oracle_mod):
    """a single entity across the Gaussian over-weights the far triangle.
    Computed by hand: whole-pixel entity gives weights summing to 1.25;
    the oracle's depth-adjacent entity stays at partition of unity."""
    ex = [e for e in GOLDEN["examples"] if e["name"] == "fig3_construct_exact_entity"][0]
    white = [dict(it, rgb=[1, 1, 1]) for it in ex["frags"]]
    out, _ = oracle_mod.blend_fragments(_frag_list(oracle_mod, white), t_eps=0.0)
    assert abs(out[0] + out[3] - 1.0) < 1e-12          # weights + T = 1, not 1.25


def test_overflow_scene_end_to_end(oracle_mod):
    """Fig.3 construction through projection, setup, binning and the tiled render."""
    sc = scenes.make_overflow()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = o.full(sc.cameras[0], **oracle_mod.scene_settings(sc, t_eps=0.0))
    fr = o.pixel_fragments(32, 32)
    assert list(fr["kind"]) == [1, 0, 1, 1]
    assert fr[0]["mask"] == 0b0101  # the edge x = 32.5 splits samples with ox < 0 (bits 0, 2)
    np.testing.assert_allclose(img[32, 32], [0.75, 0.25, 0.5, 0.0], atol=2e-7)


# --------------------------------------------------------------------------
# Gaussian alpha and EWA projection
# --------------------------------------------------------------------------

def _one_gaussian(mean, scale, opacity, quat=(1, 0, 0, 0), sh_dc=(0, 0, 0)):
    sh = np.zeros((1, 1, 3), np.float32)
    sh[0, 0] = sh_dc
    return scenes.Gaussians(np.array([mean], np.float32), np.array([quat], np.float32),
                            np.array([scale], np.float32), np.array([opacity], np.float32), sh, 0)


def _cam(W=64, H=64, f=64.0, cx=32.5, cy=32.5, R=None, t=None):
    return scenes.Camera(W, H, f, f, cx, cy, np.eye(3, dtype=np.float32) if R is None else R.astype(np.float32),
                         np.zeros(3, np.float32) if t is None else t.astype(np.float32))


@pytest.mark.parametrize("o", [0.3, 0.995, 1.0])
def test_alpha_at_centre(oracle_mod, o):
    """d = 0 -> alpha = min(0.99, o)."""
    g = _one_gaussian((0, 0, 4.0), (0.2, 0.2, 0.2), o)
    orc = oracle_mod.Oracle(g, scenes.empty_mesh())
    orc.project(_cam())
    fr = orc.pixel_fragments(32, 32)
    assert len(fr) == 1 and fr[0]["q"] == 0.0
    assert fr[0]["alpha"] == pytest.approx(min(float(np.float32(0.99)), float(np.float32(o))), abs=1e-12)


def test_alpha_half_at_2ln2(oracle_mod):
    """Mahalanobis^2 = 2 ln 2 with o = 1 -> alpha = 0.5."""
    g = _one_gaussian((0, 0, 4.0), (0.2, 0.2, 0.2), 1.0)
    orc = oracle_mod.Oracle(g, scenes.empty_mesh())
    orc.project(_cam())
    fr = orc.pixel_fragments(36, 32)  # dx = 4 px
    q = float(fr[0]["q"])
    assert fr[0]["alpha"] == pytest.approx(math.exp(-q / 2), rel=1e-12)
    # alpha = 0.5 exactly where q = 2 ln 2: check the closed-form relation through cov2d
    rec = orc.gaussian_records()
    a = float(rec["cov"][0, 0])
    d_half = math.sqrt(2 * math.log(2) * a)
    assert math.exp(-(d_half ** 2) / a / 2) == pytest.approx(0.5, rel=1e-12)


def test_zero_opacity_is_culled(oracle_mod):
    """o = 0 (and any o < 1/255) produces no fragment (R7)."""
    g = _one_gaussian((0, 0, 4.0), (0.2, 0.2, 0.2), 0.0)
    orc = oracle_mod.Oracle(g, scenes.empty_mesh())
    orc.project(_cam())
    assert orc.gaussian_records()["touched"][0] == 0
    assert len(orc.pixel_fragments(32, 32)) == 0


def test_ewa_isotropic_closed_form(oracle_mod):
    """Isotropic sigma on the optical axis, W = I: cov2d = (fx sigma / z)^2 I + 0.3 I."""
    for sigma, z, f in [(0.1, 4.0, 64.0), (0.02, 2.5, 1111.11), (0.5, 10.0, 300.0)]:
        g = _one_gaussian((0, 0, z), (sigma,) * 3, 0.8)
        orc = oracle_mod.Oracle(g, scenes.empty_mesh())
        orc.project(_cam(f=f))
        r = orc.gaussian_records()
        expect = (f * sigma / z) ** 2 + 0.3
        np.testing.assert_allclose(r["cov"][0], [expect, 0.0, expect], rtol=1e-6, atol=1e-6 * expect)
        np.testing.assert_allclose(r["rec"][0, 4:7], [1 / expect, 0.0, 1 / expect], rtol=1e-6, atol=1e-9)
        assert r["rec"][0, 7] == np.float32(z)


def _rot(axis, ang):
    axis = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K


def _quat_to_R(q):
    w, x, y, z = np.asarray(q, np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def test_ewa_monte_carlo(oracle_mod):
    """Small Gaussians (sigma/z <= 1e-3): the covariance of exactly projected samples
    matches J W Sigma W^T J^T (the EWA local affine approximation) within 1%."""
    rng = np.random.default_rng(11)
    W, H, f = 640, 480, 500.0
    R = _rot([0.3, 1.0, -0.2], 0.4)
    t = np.array([0.1, -0.2, 0.5])
    cam = _cam(W, H, f, 320.3, 240.7, R, t)
    for k in range(6):
        pc = np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.4, 0.4), 1.0]) * rng.uniform(3, 8)
        mean = R.T @ (pc - t)
        s = rng.uniform(0.3e-3, 1e-3, 3) * pc[2]
        q = rng.standard_normal(4)
        g = _one_gaussian(mean, s, 0.9, quat=q)
        orc = oracle_mod.Oracle(g, scenes.empty_mesh())
        orc.project(cam)
        cov = orc.gaussian_records()["cov"][0].astype(np.float64)
        Rg = _quat_to_R(q)
        Sig = Rg @ np.diag(np.asarray(s, np.float64) ** 2) @ Rg.T
        pts = rng.multivariate_normal(np.asarray(g.means[0], np.float64), Sig, 1_000_000)
        pv = pts @ R.T.astype(np.float32).astype(np.float64) + t.astype(np.float32)
        uv = np.stack([f * pv[:, 0] / pv[:, 2], f * pv[:, 1] / pv[:, 2]], -1)
        emp = np.cov(uv.T)
        model = np.array([[cov[0] - 0.3, cov[1]], [cov[1], cov[2] - 0.3]])
        scale = np.linalg.eigvalsh(model).max()
        assert np.abs(emp - model).max() < 0.01 * scale, (k, emp, model)


def test_ewa_projection_centre(oracle_mod):
    """u = fx X/Z + cx, v = fy Y/Z + cy (pinhole, R21) against float64 numpy."""
    rng = np.random.default_rng(3)
    sc = scenes.make_random(seed=3, n_tris=0, quads=0)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    cam = sc.cameras[0]
    orc.project(cam)
    r = orc.gaussian_records()
    vis = r["touched"] > 0
    m = sc.gaussians.means.astype(np.float64)
    u = cam.fx * m[:, 0] / m[:, 2] + cam.cx
    v = cam.fy * m[:, 1] / m[:, 2] + cam.cy
    np.testing.assert_allclose(r["rec"][vis, 0], u[vis], atol=2e-4)
    np.testing.assert_allclose(r["rec"][vis, 1], v[vis], atol=2e-4)
    del rng


def test_rotation_invariance(oracle_mod):
    """Rotating camera and Gaussian jointly leaves the conic unchanged within 1e-5."""
    rng = np.random.default_rng(5)
    for k in range(8):
        q = rng.standard_normal(4)
        s = rng.uniform(0.05, 0.3, 3)
        pc = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 1]) * rng.uniform(3, 6)
        g0 = _one_gaussian(pc, s, 0.9, quat=q)
        o0 = oracle_mod.Oracle(g0, scenes.empty_mesh())
        o0.project(_cam(256, 256, 200.0, 128.2, 127.9))
        r0 = o0.gaussian_records()["rec"][0]
        Q = _rot(rng.standard_normal(3), rng.uniform(0.2, 2.5))
        # world rotated by Q: mean' = Q mean, Gaussian rotation Q R, camera R_w2c = Q^T
        qw = _R_to_quat(Q @ _quat_to_R(q))
        g1 = _one_gaussian(Q @ pc, s, 0.9, quat=qw)
        o1 = oracle_mod.Oracle(g1, scenes.empty_mesh())
        o1.project(_cam(256, 256, 200.0, 128.2, 127.9, R=Q.T))
        r1 = o1.gaussian_records()["rec"][0]
        np.testing.assert_allclose(r1[:2], r0[:2], atol=1e-3)
        np.testing.assert_allclose(r1[4:7], r0[4:7], rtol=1e-5, atol=1e-5 * np.abs(r0[4:7]).max())


def _R_to_quat(R):
    w = math.sqrt(max(0.0, 1 + R[0, 0] + R[1, 1] + R[2, 2])) / 2
    if w > 1e-3:
        return np.array([w, (R[2, 1] - R[1, 2]) / (4 * w), (R[0, 2] - R[2, 0]) / (4 * w), (R[1, 0] - R[0, 1]) / (4 * w)])
    i = int(np.argmax(np.diag(R)))
    j, k = (i + 1) % 3, (i + 2) % 3
    r = math.sqrt(1 + R[i, i] - R[j, j] - R[k, k])
    q = np.zeros(4)
    q[1 + i] = r / 2
    q[0] = (R[k, j] - R[j, k]) / (2 * r)
    q[1 + j] = (R[j, i] + R[i, j]) / (2 * r)
    q[1 + k] = (R[k, i] + R[i, k]) / (2 * r)
    return q


def test_conic_inverts_cov(oracle_mod):
    """conic . cov2d = I within 1e-6 for every visible Gaussian of a random scene."""
    sc = scenes.make_random(seed=4, n_gauss=2000, n_tris=0, quads=0)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    orc.project(sc.cameras[0])
    r = orc.gaussian_records()
    vis = r["touched"] > 0
    a, b, c = r["cov"][vis].astype(np.float64).T
    ca, cb, cc = r["rec"][vis, 4:7].astype(np.float64).T
    i00 = ca * a + cb * b
    i01 = ca * b + cb * c
    i11 = cb * b + cc * c
    assert np.abs(i00 - 1).max() < 1e-5 and np.abs(i11 - 1).max() < 1e-5
    assert (np.abs(i01) / np.sqrt(a * c)).max() < 1e-5


# --------------------------------------------------------------------------
# SH colour
# --------------------------------------------------------------------------

def test_sh_degree0_and_zero(oracle_mod):
    C0 = GOLDEN["sh_examples"]["C0"]
    coef = np.array([[0.7, -0.2, 1.5]], np.float32)
    out = oracle_mod.sh_colour(coef, 0, [0, 0, 1])
    np.testing.assert_allclose(out, np.maximum(0.5 + C0 * coef[0].astype(np.float64), 0), atol=1e-15)
    out = oracle_mod.sh_colour(np.zeros((16, 3), np.float32), 3, [0.6, 0.0, 0.8])
    np.testing.assert_allclose(out, [0.5, 0.5, 0.5], atol=1e-15)


def test_sh_degree1_parity(oracle_mod):
    rng = np.random.default_rng(2)
    coef = np.zeros((4, 3), np.float32)
    coef[1:] = rng.standard_normal((3, 3)) * 0.1
    d = rng.standard_normal(3)
    d /= np.linalg.norm(d)
    a = oracle_mod.sh_colour(coef, 1, d) - 0.5
    b = oracle_mod.sh_colour(coef, 1, -d) - 0.5
    np.testing.assert_allclose(a, -b, atol=1e-15)


def test_sh_basis_matches_scipy(oracle_mod):
    """Each basis function equals the real spherical harmonic built from scipy's complex
    Y_l^m (Condon-Shortley phase kept, the 3DGS convention): sqrt2*Im(Y_l^|m|) for m<0,
    Y_l^0, sqrt2*Re(Y_l^m) for m>0, with the polar axis along +z."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(8)
    for _ in range(20):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        theta = math.acos(d[2])
        phi = math.atan2(d[1], d[0])
        for l in range(4):
            for m in range(-l, l + 1):
                idx = l * l + l + m
                coef = np.zeros((16, 3), np.float32)
                coef[idx] = 1.0
                got = oracle_mod.sh_colour(coef, 3, d)[0] - 0.5
                Y = sph_harm_y(l, abs(m), theta, phi)
                ref = Y.real if m == 0 else math.sqrt(2) * (Y.imag if m < 0 else Y.real)
                if got + 0.5 <= 0:      # clamp at 0 hides the value
                    continue
                assert got == pytest.approx(ref, abs=1e-12), (l, m)


# --------------------------------------------------------------------------
# triangle coverage (N7; M = 4; R10-R11)
# --------------------------------------------------------------------------

def _orient(xy):
    X, Y = xy[0::2], xy[1::2]
    A2 = (X[1] - X[0]) * (Y[2] - Y[0]) - (X[2] - X[0]) * (Y[1] - Y[0])
    if A2 < 0:
        xy = np.array([X[0], Y[0], X[2], Y[2], X[1], Y[1]], np.int64)
    return xy, A2


def test_sample_pattern(oracle_mod):
    """A tiny triangle around each D3D standard sample covers exactly that sample."""
    offs = GOLDEN["sample_pattern"]["offsets"]
    x, y = 5, 7
    for j, (ox, oy) in enumerate(offs):
        PX, PY = 256 * x + 128 + 16 * ox, 256 * y + 128 + 16 * oy
        xy = np.array([PX - 4, PY - 4, PX + 4, PY - 4, PX, PY + 5], np.int64)
        xy, _ = _orient(xy)
        assert oracle_mod.coverage_mask(xy, x, y) == 1 << j


def test_coverage_exact_rational(oracle_mod):
    """Masks equal an exact rational barycentric point-in-triangle test (Cramer's rule in
    Fractions) at every sample not lying on an edge line."""
    rng = np.random.default_rng(21)
    offs = GOLDEN["sample_pattern"]["offsets"]
    checked = 0
    for _ in range(300):
        base = rng.integers(0, 8 * 256, 2)
        xy = np.concatenate([base + rng.integers(-900, 900, 2) for _ in range(3)]).astype(np.int64)
        xy, A2 = _orient(xy)
        if A2 == 0:
            continue
        V = [(Fraction(int(xy[2 * k])), Fraction(int(xy[2 * k + 1]))) for k in range(3)]
        for py in range(0, 10):
            for px in range(0, 10):
                m = oracle_mod.coverage_mask(xy, px, py)
                for j, (ox, oy) in enumerate(offs):
                    P = (Fraction(256 * px + 128 + 16 * ox), Fraction(256 * py + 128 + 16 * oy))
                    # solve P = V0 + s (V1 - V0) + t (V2 - V0)
                    a, b = V[1][0] - V[0][0], V[2][0] - V[0][0]
                    c, d = V[1][1] - V[0][1], V[2][1] - V[0][1]
                    det = a * d - b * c
                    rx, ry = P[0] - V[0][0], P[1] - V[0][1]
                    s = (rx * d - b * ry) / det
                    t = (a * ry - c * rx) / det
                    lam = (1 - s - t, s, t)
                    if any(l == 0 for l in lam):
                        continue
                    inside = all(l > 0 for l in lam)
                    assert bool(m >> j & 1) == inside
                    checked += 1
    assert checked > 10000


def _lattice_mesh(rng, n=6, cell=2.0, z=1.0):
    """A triangulated grid whose vertices sit on the 1/16-px lattice; random diagonals and windings.
    Camera fx = fy = 1, z = 1: screen px == world x, so snapping is exact."""
    gx = np.arange(n + 1) * cell + 4.0
    X, Y = np.meshgrid(gx, gx)
    jit = rng.integers(-7, 8, X.shape + (2,)) / 16.0
    jit[0, :] = jit[-1, :] = jit[:, 0] = jit[:, -1] = 0.0
    P = np.stack([X + jit[..., 0], Y + jit[..., 1], np.full(X.shape, z)], -1).reshape(-1, 3)
    faces = []
    for i in range(n):
        for j in range(n):
            a, b, c, d = i * (n + 1) + j, i * (n + 1) + j + 1, (i + 1) * (n + 1) + j, (i + 1) * (n + 1) + j + 1
            tri = [[a, b, d], [a, d, c]] if rng.uniform() < 0.5 else [[a, b, c], [b, d, c]]
            for t in tri:
                faces.append(t if rng.uniform() < 0.5 else [t[0], t[2], t[1]])
    return P, np.array(faces)


def test_watertight_tiling(oracle_mod):
    """A triangulation of a region covers every interior sample exactly once (R11):
    sum over triangles of the coverage bit = 1, including samples on shared edges."""
    rng = np.random.default_rng(13)
    cam = scenes.Camera(24, 24, 1.0, 1.0, 0.0, 0.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    on_edge = 0
    for rep in range(12):
        P, faces = _lattice_mesh(rng)
        mesh = scenes.Mesh(P.astype(np.float32), faces.astype(np.int32), np.ones(len(faces), np.float32))
        orc = oracle_mod.Oracle(scenes.empty_gaussians(), mesh)
        orc.project(cam)
        for y in range(4, 16):
            for x in range(4, 16):
                fr = orc.pixel_fragments(x, y)
                cnt = np.zeros(4, int)
                for f in fr:
                    for j in range(4):
                        cnt[j] += (int(f["mask"]) >> j) & 1
                assert (cnt == 1).all(), (rep, x, y, cnt)
                on_edge += len(fr) > 1
    assert on_edge > 50


def test_quad_diagonal_exactly_once(oracle_mod):
    """Two triangles sharing an edge cover every sample of the quad once (S:258 quad)."""
    sc = scenes.make_tiny()
    orc = oracle_mod.Oracle(scenes.empty_gaussians(), sc.mesh)
    orc.project(sc.cameras[0])
    tr = orc.triangle_records()
    assert (tr["touched"] > 0).all()
    for y in range(64):
        for x in range(64):
            m = [int(oracle_mod.coverage_mask(tr["xy"][f], x, y)) for f in range(2)]
            assert m[0] & m[1] == 0


# --------------------------------------------------------------------------
# binning, sort, ranges: brute force on tiny inputs
# --------------------------------------------------------------------------

SMALL = [("tiny", lambda: scenes.make_tiny()),
         ("random0", lambda: scenes.make_random(0)),
         ("random1", lambda: scenes.make_random(1, n_gauss=800, n_tris=120, textured=False)),
         ("nested", lambda: scenes.make_nested()),
         ("edge", lambda: scenes.make_edge()),
         ("overflow", lambda: scenes.make_overflow())]


@pytest.mark.parametrize("name,mk", SMALL, ids=[s[0] for s in SMALL])
def test_tiled_equals_bruteforce(oracle_mod, name, mk):
    """Keys/sort/ranges are checked by rendering through them and comparing with the
    brute-force per-pixel renderer (every primitive tested at every pixel, C.1)."""
    sc = mk()
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc))
    bf = orc.render_bruteforce()
    assert np.array_equal(img, bf)
    assert orc.support_truncation() == 0


@pytest.mark.parametrize("name,mk", SMALL[:3], ids=[s[0] for s in SMALL[:3]])
def test_key_layout(oracle_mod, name, mk):
    """key = tile << 32 | bits(depth), sorted ascending, one pair per (prim, tile in rect)."""
    sc = mk()
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    orc.project(sc.cameras[0])
    K = orc.bin()
    keys, vals, ranges = orc.bins()
    g, t = orc.gaussian_records(), orc.triangle_records()
    F = sc.mesh.num_triangles
    assert K == int(g["touched"].sum() + t["touched"].sum())
    assert np.all(keys[1:] >= keys[:-1])
    depth = np.concatenate([t["depth"], g["rec"][:, 7]]).astype(np.float32)
    assert np.array_equal((keys & 0xFFFFFFFF).astype(np.uint32), depth[vals].view(np.uint32))
    rect = np.concatenate([t["rect"], g["rect"]])
    tile = (keys >> 32).astype(np.int64)
    tx, ty = tile % orc.tiles_x, tile // orc.tiles_x
    r = rect[vals]
    assert np.all((tx >= r[:, 0]) & (tx <= r[:, 2]) & (ty >= r[:, 1]) & (ty <= r[:, 3]))
    for tl in range(len(ranges)):
        b, e = ranges[tl]
        assert np.all(tile[b:e] == tl)
    assert ranges[:, 1].max() == K
    del F


# --------------------------------------------------------------------------
# reductions of the entity blend to textbook methods
# --------------------------------------------------------------------------

def _per_sample_resolve(frs, bg):
    """Textbook MSAA resolve: per sample ordered alpha blending of the covering triangles
    (colour shaded once at the pixel centre), then the mean over the M = 4 samples."""
    acc = np.zeros(3)
    Tm = 0.0
    for j in range(4):
        T = 1.0
        c = np.zeros(3)
        for f in frs:
            if int(f["mask"]) >> j & 1:
                c += T * f["alpha"] * f["rgb"]
                T *= 1 - f["alpha"]
        acc += c + T * np.asarray(bg)
        Tm += T
    return np.concatenate([acc / 4, [Tm / 4]])


def _eq12(frs, bg):
    """Eq.1-2: front-to-back alpha blending, T_in = 1."""
    T = 1.0
    c = np.zeros(3)
    for f in frs:
        c += T * f["alpha"] * f["rgb"]
        T *= 1 - f["alpha"]
    return np.concatenate([c + T * np.asarray(bg), [T]])


def test_entity_exactness_mesh_only(oracle_mod):
    """Mesh-only pixel = mean over samples of per-sample ordered blending."""
    sc = scenes.make_random(5, n_gauss=0, n_tris=150, opaque_frac=0.2)
    sc.gaussians = scenes.empty_gaussians()
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    st = oracle_mod.scene_settings(sc, t_eps=0.0)
    img = orc.full(sc.cameras[0], **st)
    n = 0
    for y in range(0, sc.cameras[0].height, 3):
        for x in range(0, sc.cameras[0].width, 3):
            frs = orc.pixel_fragments(x, y)
            np.testing.assert_allclose(img[y, x], _per_sample_resolve(frs, sc.bg.astype(np.float64)), atol=1e-6)
            n += len(frs) > 1
    assert n > 50


def test_entity_random_stacks(oracle_mod):
    """200 random triangle-only stacks (1-8 fragments, random masks, alpha in [0.05, 1])."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = rng.integers(1, 9)
        items = [dict(kind="t", mask=int(rng.integers(1, 16)), alpha=float(rng.uniform(0.05, 1)),
                      rgb=rng.uniform(0, 1, 3)) for _ in range(n)]
        fr = oracle_mod.frags(*items)
        out, _ = oracle_mod.blend_fragments(fr, t_eps=0.0, bg=(0.2, 0.3, 0.4))
        np.testing.assert_allclose(out, _per_sample_resolve(fr, [0.2, 0.3, 0.4]), atol=1e-12)


def test_opaque_msaa_first_cover(oracle_mod):
    """alpha = 1 mesh-only: each sample shows the first covering triangle (Eq.3-4 under R2)."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        n = rng.integers(1, 7)
        items = [dict(kind="t", mask=int(rng.integers(1, 16)), alpha=1.0, rgb=rng.uniform(0, 1, 3))
                 for _ in range(n)]
        fr = oracle_mod.frags(*items)
        out, _ = oracle_mod.blend_fragments(fr, t_eps=0.0)
        ref = np.zeros(3)
        unc = 0
        for j in range(4):
            first = [f for f in fr if int(f["mask"]) >> j & 1]
            if first:
                ref += first[0]["rgb"] / 4
            else:
                unc += 1
        np.testing.assert_allclose(out[:3], ref, atol=1e-12)
        assert out[3] == pytest.approx(unc / 4, abs=1e-12)


def test_full_coverage_reduces_to_eq12(oracle_mod):
    """All masks full -> Eq.1-2 over the mixed list."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        n = rng.integers(1, 10)
        items = [dict(kind="t" if rng.uniform() < 0.5 else "g", mask=15, alpha=float(rng.uniform(0.05, 0.99)),
                      rgb=rng.uniform(0, 1, 3)) for _ in range(n)]
        fr = oracle_mod.frags(*items)
        out, _ = oracle_mod.blend_fragments(fr, t_eps=0.0, bg=(0.5, 0.1, 0.9))
        np.testing.assert_allclose(out, _eq12(fr, [0.5, 0.1, 0.9]), atol=1e-12)


def test_gaussian_only_equals_eq12(oracle_mod):
    """Gaussian-only scene: every pixel equals Eq.1-2 over its fragments."""
    sc = scenes.make_random(6, n_gauss=3000, n_tris=0, quads=0)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    st = oracle_mod.scene_settings(sc, t_eps=0.0)
    img = orc.full(sc.cameras[0], **st)
    for y in range(1, sc.cameras[0].height, 4):
        for x in range(2, sc.cameras[0].width, 4):
            frs = orc.pixel_fragments(x, y)
            np.testing.assert_allclose(img[y, x], _eq12(frs, sc.bg.astype(np.float64)), atol=1e-9)


def test_partition_of_unity_random(oracle_mod):
    """Weights + final T sum to 1: colours 1 / bg 0 -> out = 1 - T; colours 0 / bg 1 -> out = T.
    Only the exit-T reading R3 passes this."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = rng.integers(1, 12)
        items = [dict(kind="t" if rng.uniform() < 0.6 else "g", mask=int(rng.integers(1, 16)),
                      alpha=float(rng.uniform(0.05, 1.0)), rgb=[1, 1, 1]) for _ in range(n)]
        fr = oracle_mod.frags(*items)
        out, _ = oracle_mod.blend_fragments(fr, t_eps=0.0)
        np.testing.assert_allclose(out[:3], 1 - out[3], atol=1e-12)
        fr["rgb"] = 0.0
        out, _ = oracle_mod.blend_fragments(fr, t_eps=0.0, bg=(1, 1, 1))
        np.testing.assert_allclose(out[:3], out[3], atol=1e-12)


def test_partition_of_unity_scene(oracle_mod):
    """Same invariant through the whole oracle path with white texture and white Gaussians."""
    sc = scenes.make_random(8, n_gauss=600, n_tris=80, sh_degree=0)
    sc.gaussians.sh[:] = np.float32(0.5 / scenes.SH_C0)
    sc.mesh.texture[:] = 255
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc, t_eps=0.0, bg=(0, 0, 0)))
    np.testing.assert_allclose(img[..., :3], np.broadcast_to(1 - img[..., 3:4], img[..., :3].shape), atol=1e-6)


def test_monotonic_T(oracle_mod):
    """T_eff trace is non-increasing and in [0, 1]."""
    rng = np.random.default_rng(9)
    for _ in range(300):
        n = rng.integers(1, 16)
        items = [dict(kind="t" if rng.uniform() < 0.5 else "g", mask=int(rng.integers(1, 16)),
                      alpha=float(rng.uniform(0.0, 1.0)), rgb=rng.uniform(0, 1, 3)) for _ in range(n)]
        _, tr = oracle_mod.blend_fragments(oracle_mod.frags(*items), t_eps=0.0)
        full = np.concatenate([[1.0], tr])
        assert np.all(np.diff(full) <= 1e-15) and full.min() >= 0 and full.max() <= 1


def test_empty_scene(oracle_mod):
    sc = scenes.make_tiny()
    orc = oracle_mod.Oracle(scenes.empty_gaussians(), scenes.empty_mesh())
    img = orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc))
    assert np.all(img[..., :3] == sc.bg.astype(np.float64)) and np.all(img[..., 3] == 1.0)


def test_opaque_front_quad(oracle_mod):
    """Screen-filling alpha = 1 quad in front of everything: every pixel = c, T = 0 (also
    watertight along the diagonal)."""
    sc = scenes.make_random(2, n_gauss=500, n_tris=30)
    cam = sc.cameras[0]
    z = 1.0
    hw, hh = (cam.width + 8) / cam.fx * z, (cam.height + 8) / cam.fy * z
    P = np.array([[-hw, -hh, z], [hw, -hh, z], [hw, hh, z], [-hw, hh, z]], np.float32)
    c = np.array([0.3, 0.6, 0.9], np.float32)
    mesh = scenes.Mesh(np.concatenate([P, sc.mesh.positions]),
                       np.concatenate([[[0, 1, 2], [0, 2, 3]], sc.mesh.faces + 4]).astype(np.int32),
                       np.concatenate([[1, 1], sc.mesh.opacity]).astype(np.float32),
                       colors=np.concatenate([np.tile(c, (4, 1)), np.full((len(sc.mesh.positions), 3), 0.5, np.float32)]))
    orc = oracle_mod.Oracle(sc.gaussians, mesh)
    img = orc.full(cam, **oracle_mod.scene_settings(sc))
    np.testing.assert_allclose(img[..., :3], np.broadcast_to(c.astype(np.float64), img[..., :3].shape), atol=1e-6)
    assert np.all(img[..., 3] == 0.0)


def test_termination_bound(oracle_mod):
    """Blend-then-test termination (R16): |out(eps=1e-4) - out(eps=0)| <= 2 eps."""
    sc = scenes.make_random(9, n_gauss=4000, n_tris=60)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    a = orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc, t_eps=0.0))
    b = orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc, t_eps=1e-4))
    assert np.abs(a - b).max() <= 2e-4


def test_determinism_threads(oracle_mod):
    """Identical images regardless of thread count."""
    sc = scenes.make_random(10, n_gauss=1500, n_tris=50)
    imgs = []
    for th in (1, 3, 8):
        orc = oracle_mod.Oracle(sc.gaussians, sc.mesh, threads=th)
        imgs.append(orc.full(sc.cameras[0], **oracle_mod.scene_settings(sc)))
    assert np.array_equal(imgs[0], imgs[1]) and np.array_equal(imgs[0], imgs[2])


# --------------------------------------------------------------------------
# triangle shading at the pixel centre (R12)
# --------------------------------------------------------------------------

def test_texel_aligned_quad_reproduces_texture(oracle_mod):
    """A fronto-parallel quad mapped 1:1 onto a 16x16 texture: each pixel centre lands on a
    texel centre, so bilinear filtering with texel centres at (i+0.5)/W returns the texel."""
    rng = np.random.default_rng(12)
    tex = rng.integers(0, 256, (16, 16, 4)).astype(np.uint8)
    cam = scenes.Camera(32, 32, 1.0, 1.0, 0.0, 0.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    x0, y0 = 8.0, 4.0
    P = np.array([[x0, y0, 1], [x0 + 16, y0, 1], [x0 + 16, y0 + 16, 1], [x0, y0 + 16, 1]], np.float32)
    uv = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], np.float32)
    mesh = scenes.Mesh(P, np.array([[0, 1, 2], [0, 2, 3]], np.int32), np.ones(2, np.float32), uvs=uv, texture=tex)
    orc = oracle_mod.Oracle(scenes.empty_gaussians(), mesh)
    img = orc.full(cam, bg=(0, 0, 0), t_eps=0.0)
    got = img[4:20, 8:24, :3]
    np.testing.assert_allclose(got, tex[:, :, :3] / 255.0, atol=1e-9)


def test_perspective_correct_colour(oracle_mod):
    """Vertex colours on a triangle strongly tilted in depth: the colour at a pixel equals the
    colour of the 3D point the pixel-centre ray hits (ray-plane intersection in float64),
    up to the 1/256-px vertex snap."""
    W = H = 64
    cam = scenes.Camera(W, H, 60.0, 60.0, 32.0, 32.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    P = np.array([[-1.5, -1.2, 2.0], [1.6, -1.0, 7.0], [0.0, 1.4, 3.0]], np.float64)
    C = np.array([[0.9, 0.1, 0.2], [0.1, 0.8, 0.3], [0.2, 0.3, 0.95]], np.float64)
    mesh = scenes.Mesh(P.astype(np.float32), np.array([[0, 1, 2]], np.int32), np.ones(1, np.float32),
                       colors=C.astype(np.float32))
    orc = oracle_mod.Oracle(scenes.empty_gaussians(), mesh)
    img = orc.full(cam, bg=(0, 0, 0), t_eps=0.0)
    n = 0
    nrm = np.cross(P[1] - P[0], P[2] - P[0])
    for y in range(0, H, 2):
        for x in range(0, W, 2):
            fr = orc.pixel_fragments(x, y)
            if len(fr) == 0 or fr[0]["mask"] != 15:
                continue
            d = np.array([(x + 0.5 - 32.0) / 60.0, (y + 0.5 - 32.0) / 60.0, 1.0])
            hit = d * (nrm @ P[0]) / (nrm @ d)
            # barycentrics of the 3D hit point
            A = np.stack([P[1] - P[0], P[2] - P[0]], 1)
            st = np.linalg.lstsq(A, hit - P[0], rcond=None)[0]
            lam = np.array([1 - st.sum(), st[0], st[1]])
            np.testing.assert_allclose(img[y, x, :3], lam @ C, atol=2e-3)
            n += 1
    assert n > 100


def test_triangle_depth_is_centroid_z(oracle_mod):
    """Triangle sort depth = view z of the centroid (reading R9), vs float64 numpy."""
    sc = scenes.make_random(11, n_gauss=10, n_tris=200)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    orc.project(sc.cameras[0])
    t = orc.triangle_records()
    vis = t["touched"] > 0
    z = sc.mesh.positions[:, 2].astype(np.float64)  # identity camera: view z = world z
    cz = z[sc.mesh.faces].mean(1)
    np.testing.assert_allclose(t["depth"][vis], cz[vis], rtol=1e-6)


def test_gaussian_membership_is_alpha_cutoff(oracle_mod):
    """A Gaussian is a fragment of a pixel iff o*exp(-q/2) >= 1/255 (R7/R17), with q
    recomputed in float64 from the projected record; pairs within 1e-6 of the cutoff skipped."""
    sc = scenes.make_random(12, n_gauss=300, n_tris=0, quads=0, W=48, H=40)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    orc.project(sc.cameras[0])
    r = orc.gaussian_records()
    F = 0
    checked = 0
    for y in range(40):
        for x in range(48):
            ids = set(int(f["id"]) - F for f in orc.pixel_fragments(x, y))
            for g in np.nonzero(r["touched"])[0]:
                u, v, qmax, o, ca, cb, cc, _ = r["rec"][g].astype(np.float64)
                dx, dy = x + 0.5 - u, y + 0.5 - v
                q = ca * dx * dx + 2 * cb * dx * dy + cc * dy * dy
                a = o * math.exp(-q / 2)
                if abs(a - 1 / 255) < 1e-6:
                    continue
                assert (g in ids) == (a >= 1 / 255), (x, y, g, a)
                checked += 1
    assert checked > 10000
