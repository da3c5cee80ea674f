"""Deformation transfer on the GPU (Eq.12-13) vs the oracle, and rendering deformed Gaussians."""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

pytestmark = pytest.mark.gpu


def _dev(a, dt=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else a.astype(dt))).cuda()


def _gpu_deform(sc, b, field):
    from paper_2601_19233_b200 import renderer as R
    ds = R.to_device(sc)
    mo, co = R.deform(ds, _dev(b.face, np.int32), _dev(b.bary, np.float32), _dev(sc.mesh.faces, np.int32),
                      _dev(field.packed()))
    return ds, mo.cpu().numpy(), co.cpu().numpy()


@pytest.mark.parametrize("K", [1, 8])
def test_deform_parity(oracle_mod, K):
    sc, b = scenes.make_deform(n_gauss=20000, K=K)
    field = scenes.twist_field(sc.mesh, shear_eps=0.1)
    _, mo, co = _gpu_deform(sc, b, field)
    om, oc = oracle_mod.Oracle(sc.gaussians, sc.mesh).deform(b, field, sc.mesh.faces)
    assert np.abs(mo - om).max() < 2e-6
    scale = np.abs(oc).max(1, keepdims=True)
    assert (np.abs(co - oc) / scale).max() < 2e-5


def test_deform_identity_and_unbound(oracle_mod):
    sc, b = scenes.make_deform(n_gauss=5000, K=8)
    _, mo, co = _gpu_deform(sc, b, scenes.uniform_field(sc.mesh.num_vertices))
    om, oc = oracle_mod.Oracle(sc.gaussians, sc.mesh).deform(b, scenes.uniform_field(sc.mesh.num_vertices),
                                                            sc.mesh.faces)
    np.testing.assert_allclose(mo, sc.gaussians.means, atol=1e-6)
    assert (np.abs(co - oc) / np.abs(oc).max(1, keepdims=True)).max() < 2e-6
    b0 = scenes.Binding(np.full_like(b.face, -1), b.bary)
    _, mo0, _ = _gpu_deform(sc, b0, scenes.twist_field(sc.mesh))
    assert np.array_equal(mo0, sc.gaussians.means)


def test_render_deformed_scene(oracle_mod):
    """GPU: deform -> render (cov3d path); oracle: its own deform -> render.  The two inputs
    differ by fp32 rounding only, so colours agree to 1e-3 except where a Gaussian sits on
    the alpha = 1/255 membership boundary (<= 0.1% of pixels, bounded by 1e-2)."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc, b = scenes.make_deform(n_gauss=20000, K=8)
    field = scenes.twist_field(sc.mesh)
    ds, mo, co = _gpu_deform(sc, b, field)
    ds.means, ds.cov3d = _dev(mo), _dev(co)
    r = R.renderer_for(sc)
    img = r.render_view(ds, sc.cameras[0]).cpu().numpy()
    om, oc = oracle_mod.Oracle(sc.gaussians, sc.mesh).deform(b, field, sc.mesh.faces)
    g2 = scenes.Gaussians(om.astype(np.float32), sc.gaussians.quats, sc.gaussians.scales, sc.gaussians.opacities,
                          sc.gaussians.sh, sc.gaussians.sh_degree)
    g2.cov3d = oc.astype(np.float32)
    o = oracle_mod.Oracle(g2, sc.mesh)
    ref = o.full(sc.cameras[0], **oracle_mod.scene_settings(sc))
    d = np.abs(img - ref).max(-1)
    assert d.max() < 1e-2 and (d > 1e-3).mean() < 1e-3, (d.max(), (d > 1e-3).mean())
    torch.cuda.synchronize()


def test_cov3d_render_bit_exact_keys(oracle_mod):
    """With identical cov3d inputs the keys and sort stay bit-exact (cov3d replaces N3)."""
    from paper_2601_19233_b200 import renderer as R
    from parity_util import compare_bins, compare_image
    sc = scenes.make_random(31, n_gauss=2000, n_tris=50)
    q = sc.gaussians.quats.astype(np.float64)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    from scipy.spatial.transform import Rotation
    Rm = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
    S = np.einsum("nij,nj,nkj->nik", Rm, sc.gaussians.scales.astype(np.float64) ** 2, Rm)
    sc.gaussians.cov3d = np.stack([S[:, 0, 0], S[:, 0, 1], S[:, 0, 2], S[:, 1, 1], S[:, 1, 2], S[:, 2, 2]], -1).astype(np.float32)
    r = R.renderer_for(sc)
    img = r.render_view(R.to_device(sc), sc.cameras[0]).cpu().numpy()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(sc.cameras[0], **oracle_mod.scene_settings(sc))
    o.bin()
    compare_bins(r, o)
    compare_image(img, o.render())
