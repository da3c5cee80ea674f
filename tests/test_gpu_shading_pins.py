"""The CUDA path on the shading pin constructions (run on a B200 with -m gpu),
through the C ABI: the same closed-form expectations the oracle is pinned to
(tests/test_oracle_shading_pins.py) -- bilinear texel weights on an affine
texture, the SH view direction, the 1.3x FoV Jacobian clamp -- plus the bit-exact
record/bin parity and the SPEC #6 nested-transparency bar on the GPU image.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

from parity_util import compare_bins, compare_image, compare_records, run_gpu, run_oracle
from test_oracle_shading_pins import (affine_texture_expectation, fov_clamp_expectation,
                                      sh_probe_expectation)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2601_19233_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()
    return True


@pytest.mark.parametrize("geom", [(5.0, 3.0, 37.0, 29.0, 48, 40), (2.0, 1.0, 61.0, 21.0, 72, 28)])
def test_gpu_bilinear_affine_texture(built, oracle_mod, geom):
    x0, y0, wq, hq, W, H = geom
    sc = scenes.make_texture_quad(x0, y0, wq, hq, W, H)
    r, ds, img = run_gpu(sc, sc.cameras[0])
    exp, sel = affine_texture_expectation(x0, y0, wq, hq, W, H)
    # fp32 barycentrics and filter: well inside the 1e-3 colour bar
    assert np.abs(img[sel][:, :3] - exp[sel]).max() < 2e-4
    o = run_oracle(oracle_mod, sc, sc.cameras[0])
    compare_records(r, o, sc)
    compare_bins(r, o)
    compare_image(img, o.render())


def test_gpu_bilinear_half_texel_shift(built):
    rng = np.random.default_rng(31)
    tex = rng.integers(0, 256, (16, 16, 4)).astype(np.uint8)
    sc = scenes.make_texture_quad(8.5, 4.5, 16.0, 16.0, 32, 32, texture=tex)
    _, _, img = run_gpu(sc, sc.cameras[0])
    t = tex[..., :3].astype(np.float64) / 255.0
    mean4 = 0.25 * (t[:-1, :-1] + t[:-1, 1:] + t[1:, :-1] + t[1:, 1:])
    assert np.abs(img[5:20, 9:24, :3] - mean4).max() < 2e-4


def test_gpu_sh_view_direction(built, oracle_mod):
    sc = scenes.make_sh_probe()
    for cam, eye in zip(sc.cameras, sc.eyes):
        r, ds, img = run_gpu(sc, cam)
        rec = r.records()
        vis = rec["touched"] > 0
        assert vis.sum() >= 20
        exp = sh_probe_expectation(sc.gaussians.means, eye)
        assert np.abs(rec["grec"][vis, 8:11] - exp[vis]).max() < 1e-5
        o = run_oracle(oracle_mod, sc, cam)
        compare_records(r, o, sc)
        compare_image(img, o.render())


def test_gpu_fov_clamp(built, oracle_mod):
    sc = scenes.make_fov_clamp()
    cam = sc.cameras[0]
    r, ds, img = run_gpu(sc, cam)
    rec = r.records()
    assert (rec["touched"] > 0).all()
    exp = fov_clamp_expectation(sc.gaussians, cam)
    a, b, c = exp.T
    det = a * c - b * b
    conic = np.stack([c / det, -b / det, a / det], -1)
    got = rec["grec"][:, 4:7].astype(np.float64)
    assert (np.abs(got - conic) / np.abs(conic).max(1, keepdims=True)).max() < 5e-5
    o = run_oracle(oracle_mod, sc, cam)
    compare_records(r, o, sc)
    compare_bins(r, o)
    compare_image(img, o.render())


def test_gpu_nested_transparency_vs_supersampled(built, oracle_mod):
    """SPEC acceptance #6 on the GPU image: mean abs error < 0.01 against the
    oracle's 16x16 supersampled per-sample ground truth."""
    sc = scenes.make_nested()
    cam = sc.cameras[0]
    _, _, img = run_gpu(sc, cam)
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc))
    ss = o.render_supersampled(16)
    assert np.abs(img[..., :3] - ss[..., :3]).mean() < 0.01
