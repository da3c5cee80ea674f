"""GPU ray-cast binding (unimgs_bind, LBVH) vs the exhaustive CPU oracle.

The bar: face ids and squared hit distances identical, barycentrics equal to
the oracle's double values rounded to float32 (bit-exact): the decision
arithmetic is the same IEEE double sequence on both sides, and the BVH only
prunes, so its result equals exhaustive search.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

from test_oracle_bind import _cam, _gauss, _icosphere

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2601_19233_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()
    return True


def _gpu_bind(g, P, F, cams, mode, k=3.0):
    import torch
    from paper_2601_19233_b200 import renderer as R
    dev = lambda a, dt=torch.float32: torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)  # noqa: E731
    face, bary, d2 = R.bind(dev(g.means), dev(g.quats), dev(g.scales), dev(P), dev(F, torch.int32), cams, mode, k,
                            with_dist=True)
    torch.cuda.synchronize()
    return face.cpu().numpy(), bary.cpu().numpy(), d2.cpu().numpy()


def _compare(oracle_mod, g, P, F, cams, mode, rows=None, k=3.0):
    gf, gb, gd = _gpu_bind(g, P, F, cams, mode, k)
    if rows is not None:
        sub = scenes.Gaussians(g.means[rows], g.quats[rows], g.scales[rows], g.opacities[rows], g.sh[rows], g.sh_degree)
        gf, gb, gd = gf[rows], gb[rows], gd[rows]
    else:
        sub = g
    of, ob, od = oracle_mod.bind(sub, P, F, cams, mode=mode, k_sigma=k)
    assert np.array_equal(gf, of), f"faces differ at {np.argwhere(gf != of)[:5]}"
    assert np.array_equal(gb.view(np.uint32), ob.astype(np.float32).view(np.uint32)), "barycentrics differ"
    assert np.array_equal(gd, od), "hit distances differ"
    return float((of >= 0).mean())


def _ring(n=6, r=3.0):
    return [_cam(r * np.array([np.sin(a), 0.3 * np.cos(3 * a), np.cos(a)]))
            for a in np.linspace(0, 2 * np.pi, n, endpoint=False)]


@pytest.mark.parametrize("mode", [0, 1])
def test_icosphere(built, oracle_mod, mode):
    P, F = _icosphere(3)
    rng = np.random.default_rng(10)
    n = 400
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    g = _gauss(d * rng.normal(1.0, 0.03, (n, 1)), np.exp(rng.normal(np.log(0.03), 0.5, (n, 3))),
               rng.normal(size=(n, 4)))
    assert _compare(oracle_mod, g, P, F, _ring(), mode) > 0.9


@pytest.mark.parametrize("mode", [0, 1])
def test_uv_sphere_with_seam_and_poles(built, oracle_mod, mode):
    """Duplicated seam vertices and zero-area pole triangles (det = 0)."""
    g, mesh, cams = scenes.make_bind_case(seed=11, n_gauss=1500, lon=64, lat=32)
    assert _compare(oracle_mod, g, mesh.positions, mesh.faces, cams, mode) > 0.9


def test_occluder_and_invalid_faces(built, oracle_mod):
    P = np.array([[-2, -2, 1], [2, -2, 1], [2, 2, 1], [-2, 2, 1],
                  [-2, -2, 2], [2, -2, 2], [2, 2, 2], [-2, 2, 2]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3], [4, 5, 6], [4, 6, 7], [0, 1, 99], [-1, 2, 3]], np.int32)
    rng = np.random.default_rng(2)
    g = _gauss(np.c_[rng.uniform(-1.5, 1.5, (200, 2)), rng.uniform(0.5, 2.5, 200)])
    cams = [_cam((0.0, 0.0, -3.0), (0.0, 0.0, 1.0)), _cam((0.5, 0.2, 6.0), (0.0, 0.0, 1.5))]
    for mode in (0, 1):
        _compare(oracle_mod, g, P, F, cams, mode)


def test_single_face_and_empty_mesh(built, oracle_mod):
    P = np.array([[-1, -1, 0], [2, -1, 0], [-1, 2, 0]], np.float32)
    g = _gauss(np.random.default_rng(3).uniform(-0.5, 0.5, (50, 3)))
    cams = [_cam((0.3, 0.2, -3.0)), _cam((0.1, -0.2, 3.0))]
    _compare(oracle_mod, g, P, np.array([[0, 1, 2]], np.int32), cams, 1)
    gf, gb, gd = _gpu_bind(g, P, np.zeros((0, 3), np.int32), cams, 1)
    assert np.all(gf == -1) and np.all(gb == 0) and np.all(gd == -1)


def test_spec_workload_sampled(built, oracle_mod):
    """SPEC's throughput workload (100k Gaussians, bbx8, 8 cameras, 50k faces):
    the GPU binds all of them; 256 sampled Gaussians are checked exhaustively."""
    g, mesh, cams = scenes.make_bind_case()
    rows = np.random.default_rng(4).choice(g.count, 256, replace=False)
    assert _compare(oracle_mod, g, mesh.positions, mesh.faces, cams, 1, rows=rows) > 0.9


def test_bind_then_deform_identity(built):
    """The table feeds unimgs_deform directly; an identity field leaves mu unchanged."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    g, mesh, cams = scenes.make_bind_case(seed=12, n_gauss=5000, lon=64, lat=32)
    dev = lambda a, dt=torch.float32: torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)  # noqa: E731
    face, bary = R.bind(dev(g.means), dev(g.quats), dev(g.scales), dev(mesh.positions), dev(mesh.faces, torch.int32),
                        cams, 1)
    sc = scenes.Scene("b", g, mesh, cams)
    ds = R.to_device(sc)
    vdata = dev(scenes.uniform_field(mesh.num_vertices).packed())
    mu, cov = R.deform(ds, face, bary, dev(mesh.faces, torch.int32), vdata)
    torch.cuda.synchronize()
    assert (face >= 0).float().mean().item() > 0.9
    assert torch.allclose(mu, ds.means, atol=1e-6)
