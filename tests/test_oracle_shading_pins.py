"""Pins for the oracle's shading steps that the round-1 pins left open (run with
-m "not gpu"): the bilinear texel weights, the SH view direction and the 1.3x
tan-FoV Jacobian clamp, plus SPEC acceptance #6 (nested transparency against
the supersampled ground truth).

Each expected value comes from mathematics independent of the oracle's code:
  * bilinear interpolation reproduces an affine function exactly (R12: texel
    centres at (i+0.5)/W, clamp-to-edge, row 0 at v = 0);
  * the degree-1 real SH basis is sqrt(3/(4 pi)) * (-y, z, -x) (3DGS sign
    convention, already pinned against scipy) at dir = normalize(mu - eye), with
    the eye taken from the look-at construction, not from -R^T t;
  * the EWA Jacobian is the derivative of (fx X/Z, fy Y/Z) -- textbook calculus --
    evaluated at the point clamped to the 1.3x half-FoV cone (R18, the 3DGS
    forward convention the paper cites at P:72).
"""
import math

import numpy as np
import pytest

from paper_2601_19233_b200 import scenes


# --------------------------------------------------------------------------
# bilinear texel weights (R12; triangle colour at the pixel centre)
# --------------------------------------------------------------------------

def affine_texture_expectation(x0, y0, wq, hq, W, H):
    """Expected RGB at every pixel centre of make_texture_quad from the affine texel law:
    uv at the centre is affine in (x, y) on a fronto-parallel quad, texel coordinate
    s = u*tw - 0.5, and bilinear interpolation of c0 + ci*i + cj*j is exact at (s, t)
    wherever no clamp is involved (0 <= s <= tw-1, 0 <= t <= th-1)."""
    tw, th = scenes.AFFINE_TEX["tw"], scenes.AFFINE_TEX["th"]
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    u = (xs + 0.5 - x0) / wq
    v = (ys + 0.5 - y0) / hq
    s, t = u * tw - 0.5, v * th - 0.5
    inside = (s >= 0) & (s <= tw - 1) & (t >= 0) & (t <= th - 1)
    rgb = np.stack([(scenes.AFFINE_TEX[k][0] + scenes.AFFINE_TEX[k][1] * s + scenes.AFFINE_TEX[k][2] * t) / 255.0
                    for k in "rgb"], -1)
    # pixels whose 4 samples are all inside the quad (interior, away from the quad edges)
    full = (xs >= x0 + 1) & (xs + 1 <= x0 + wq - 1) & (ys >= y0 + 1) & (ys + 1 <= y0 + hq - 1)
    return rgb, inside & full


@pytest.mark.parametrize("geom", [(5.0, 3.0, 37.0, 29.0, 48, 40), (2.0, 1.0, 61.0, 21.0, 72, 28)])
def test_bilinear_affine_texture_exact(oracle_mod, geom):
    """An affine texture is reproduced exactly at arbitrary texel fractions.  Swapping the
    two off-diagonal taps (t10 <-> t01), the axes, or the texel-centre offset breaks it."""
    x0, y0, wq, hq, W, H = geom
    sc = scenes.make_texture_quad(x0, y0, wq, hq, W, H)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = orc.full(sc.cameras[0], bg=(0, 0, 0), t_eps=0.0)
    exp, sel = affine_texture_expectation(x0, y0, wq, hq, W, H)
    assert sel.sum() > 300
    # fractions really vary: both weights take many distinct values over the checked pixels
    tw = scenes.AFFINE_TEX["tw"]
    fr = ((np.mgrid[0:H, 0:W][1] + 0.5 - x0) / wq * tw - 0.5) % 1.0
    assert len(np.unique(np.round(fr[sel], 6))) > 10
    np.testing.assert_allclose(img[sel][:, :3], exp[sel], atol=1e-9)
    assert np.all(img[sel][:, 3] == 0.0)


def test_bilinear_half_texel_shift_is_four_texel_mean(oracle_mod):
    """A 1:1 quad shifted by half a pixel puts every interior pixel centre on a texel
    corner: the bilinear result is the mean of the 4 surrounding texels (random texture)."""
    rng = np.random.default_rng(31)
    tex = rng.integers(0, 256, (16, 16, 4)).astype(np.uint8)
    sc = scenes.make_texture_quad(8.5, 4.5, 16.0, 16.0, 32, 32, texture=tex)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = orc.full(sc.cameras[0], bg=(0, 0, 0), t_eps=0.0)
    t = tex[..., :3].astype(np.float64) / 255.0
    mean4 = 0.25 * (t[:-1, :-1] + t[:-1, 1:] + t[1:, :-1] + t[1:, 1:])  # [15, 15]
    # pixel (x, y) centre x + 0.5 = 8.5 + i + 1  ->  texel corner between i and i + 1
    got = img[5:20, 9:24, :3]
    np.testing.assert_allclose(got, mean4, atol=1e-9)


def test_bilinear_clamp_to_edge(oracle_mod):
    """uv beyond the outermost texel centres clamps to the edge texels (the quad is mapped
    with uv spanning [0, 1] and pixels near the quad border fall outside [0.5, tw - 0.5])."""
    x0, y0, wq, hq, W, H = 5.0, 3.0, 37.0, 29.0, 48, 40
    sc = scenes.make_texture_quad(x0, y0, wq, hq, W, H)
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    img = orc.full(sc.cameras[0], bg=(0, 0, 0), t_eps=0.0)
    tw, th = scenes.AFFINE_TEX["tw"], scenes.AFFINE_TEX["th"]
    n = 0
    for y in range(H):
        for x in range(W):
            fr = orc.pixel_fragments(x, y)
            if len(fr) != 1 or fr[0]["mask"] != 15:
                continue
            s = (x + 0.5 - x0) / wq * tw - 0.5
            t = (y + 0.5 - y0) / hq * th - 0.5
            if 0 <= s <= tw - 1 and 0 <= t <= th - 1:
                continue
            sc_, tc = min(max(s, 0.0), tw - 1.0), min(max(t, 0.0), th - 1.0)
            exp = [(scenes.AFFINE_TEX[k][0] + scenes.AFFINE_TEX[k][1] * sc_ + scenes.AFFINE_TEX[k][2] * tc) / 255
                   for k in "rgb"]
            np.testing.assert_allclose(img[y, x, :3], exp, atol=1e-9)
            n += 1
    assert n > 20


# --------------------------------------------------------------------------
# SH view direction (dir = normalize(mu - campos))
# --------------------------------------------------------------------------

def sh_probe_expectation(means, eye):
    """0.5 + C1 * K * (-y, z, -x) of the unit direction from the eye to each mean."""
    C1 = math.sqrt(3.0 / (4.0 * math.pi))
    d = np.asarray(means, np.float64) - eye
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    k = scenes.SH_PROBE_K
    return np.maximum(0.5 + C1 * k * np.stack([-d[:, 1], d[:, 2], -d[:, 0]], -1), 0.0)


def test_sh_view_direction(oracle_mod):
    """Each projected Gaussian's colour equals the degree-1 SH evaluated at the direction
    from the camera eye (as placed by the look-at construction) to the mean; cameras on
    opposite sides give mirrored colours.  d = campos - mu, a wrong campos (R t, -t) or a
    swapped basis axis fails."""
    sc = scenes.make_sh_probe()
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    spread = []
    for cam, eye in zip(sc.cameras, sc.eyes):
        orc.project(cam)
        r = orc.gaussian_records()
        vis = r["touched"] > 0
        assert vis.sum() >= 20
        exp = sh_probe_expectation(sc.gaussians.means, eye)
        np.testing.assert_allclose(r["rgb"][vis], exp[vis], atol=2e-6)
        spread.append(exp[vis].mean(0))
    spread = np.array(spread)
    # the six viewpoints really exercise both signs of every basis axis
    assert (spread.max(0) - spread.min(0)).min() > 0.5


# --------------------------------------------------------------------------
# N4: 1.3x tan-FoV Jacobian clamp (R18)
# --------------------------------------------------------------------------

def _quat_to_R(q):
    w, x, y, z = np.asarray(q, np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def fov_clamp_expectation(g, cam, dilation=0.3, clamp=True):
    """cov2d = J W Sigma W^T J^T + dilation I, J = d(fx X/Z, fy Y/Z)/d(X, Y, Z) evaluated at
    (X', Y', Z) with X'/Z, Y'/Z clamped to 1.3 x the half-FoV tangents W/(2 fx), H/(2 fy)."""
    R = np.asarray(cam.R, np.float64)
    t = np.asarray(cam.t, np.float64)
    out = []
    for i in range(g.count):
        X, Y, Z = R @ g.means[i].astype(np.float64) + t
        if clamp:
            lx, ly = 1.3 * cam.width / (2 * cam.fx), 1.3 * cam.height / (2 * cam.fy)
            X = min(max(X / Z, -lx), lx) * Z
            Y = min(max(Y / Z, -ly), ly) * Z
        J = np.array([[cam.fx / Z, 0.0, -cam.fx * X / Z ** 2], [0.0, cam.fy / Z, -cam.fy * Y / Z ** 2]])
        Rg = _quat_to_R(g.quats[i])
        Sig = Rg @ np.diag(g.scales[i].astype(np.float64) ** 2) @ Rg.T
        cov = J @ R @ Sig @ R.T @ J.T + dilation * np.eye(2)
        out.append([cov[0, 0], cov[0, 1], cov[1, 1]])
    return np.array(out)


def test_fov_clamp_jacobian(oracle_mod):
    """Gaussians inside the 1.3x cone get the exact EWA Jacobian; those outside get it at
    the cone boundary (x and y clamped independently, each against its own axis)."""
    sc = scenes.make_fov_clamp()
    cam = sc.cameras[0]
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    orc.project(cam)
    r = orc.gaussian_records()
    assert (r["touched"] > 0).all(), "every probe Gaussian must reach the image"
    exp = fov_clamp_expectation(sc.gaussians, cam)
    unclamped = fov_clamp_expectation(sc.gaussians, cam, clamp=False)
    cov = r["cov"].astype(np.float64)
    scale = np.abs(exp).max(1, keepdims=True)
    assert (np.abs(cov - exp) / scale).max() < 2e-5
    # the clamp is active exactly for the five probes outside the cone, and matters there
    rel = (np.abs(unclamped - exp) / scale).max(1)
    assert rel[0] == 0.0 and (rel[1:] > 0.02).all(), rel


# --------------------------------------------------------------------------
# SPEC acceptance #6: nested transparency vs the supersampled ground truth
# --------------------------------------------------------------------------

def test_nested_transparency_vs_supersampled(oracle_mod):
    """Splats inside a semi-transparent closed sphere (lego in a transparent bowl):
    (a) they are visible through the mesh -- removing them changes the pixels inside the
    sphere's silhouette; (b) the exact-entity image is within mean abs error 0.01 of the
    16x16 supersampled per-sample ground truth."""
    sc = scenes.make_nested()
    cam = sc.cameras[0]
    orc = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    st = oracle_mod.scene_settings(sc)
    img = orc.full(cam, **st)
    ss = orc.render_supersampled(16)
    mae = np.abs(img[..., :3] - ss[..., :3]).mean()
    assert mae < 0.01, mae
    shell_only = oracle_mod.Oracle(scenes.empty_gaussians(sc.gaussians.sh_degree), sc.mesh).full(cam, **st)
    inside = shell_only[..., 3] < 0.99            # pixels covered by the sphere
    changed = np.abs(img - shell_only)[..., :3].max(-1) > 0.02
    assert inside.sum() > 2000 and (changed & inside).sum() > 0.3 * inside.sum()
