"""ABI call-order, capacity and culling-as-values rules (include/unimgs.h), on a
B200 (-m gpu):

* unimgs_bin exactly once per unimgs_preprocess (a second bin is UNIMGS_ERR_STATE
  and leaves the bins intact);
* unimgs_host_wait reports a capacity overflow of ANY view of the batch, not only
  the last one (the earlier views' frames would otherwise be stale);
* unimgs_render_host_async validates every host pointer before enqueuing;
  a cov3d scene renders through the host path like through the device path;
* unimgs_deform culls anchors whose face has an out-of-range vertex id (the ABI's
  error-as-value rule), matching the oracle.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2601_19233_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()
    return True


def test_bin_twice_is_a_state_error(built, oracle_mod):
    from paper_2601_19233_b200 import renderer as R, _lib
    from parity_util import compare_bins, run_oracle
    sc = scenes.make_random(3, n_gauss=1500, n_tris=100)
    r = R.renderer_for(sc)
    ds = R.to_device(sc)
    r.preprocess(ds, sc.cameras[0])
    r.bin()
    with pytest.raises(_lib.UnimgsError) as e:
        r.bin()
    assert e.value.code == _lib.ERR_STATE
    compare_bins(r, run_oracle(oracle_mod, sc, sc.cameras[0]))  # the rejected call changed nothing
    r.render()
    r.render()  # rendering the same bins twice is allowed
    r.preprocess(ds, sc.cameras[0])
    r.bin()  # a new preprocess re-arms bin


def _overflow_pair():
    """Two views of one scene: a close-up that needs many pairs and a far view that needs few."""
    sc = scenes.make_random(6, n_gauss=3000, n_tris=60, W=128, H=96)
    near = sc.cameras[0]
    far = scenes.Camera(near.width, near.height, near.fx * 0.15, near.fy * 0.15, near.cx, near.cy, near.R, near.t)
    return sc, near, far


@pytest.mark.parametrize("lanes", [1, 2])
def test_host_wait_reports_overflow_of_any_view(built, lanes):
    import torch
    from paper_2601_19233_b200 import renderer as R, _lib
    sc, near, far = _overflow_pair()
    probe = R.renderer_for(sc)
    K_near = (probe.render_view(R.to_device(sc), near), probe.stats()["num_pairs"])[1]
    K_far = (probe.render_view(R.to_device(sc), far), probe.stats()["num_pairs"])[1]
    assert K_far < K_near
    r = R.renderer_for(sc, max_pairs=(K_far + K_near) // 2)
    if lanes > 1:
        r.set_host_lanes(lanes)
    host = R.to_pinned(sc)
    cams = [near, far, far, far]  # only the first view overflows; the last one fits
    out = torch.empty((len(cams), near.height, near.width, 4), dtype=torch.float32).pin_memory()
    r.render_host_async(host, cams, out)
    with pytest.raises(_lib.UnimgsError) as e:
        r.host_wait()
    assert e.value.code == _lib.ERR_CAPACITY
    # the flag is cleared by the wait that reported it: a batch that fits is clean again
    r.render_host_async(host, [far, far], out[:2])
    r.host_wait()


def test_render_host_rejects_null_host_arrays(built):
    import ctypes as C
    import torch
    from paper_2601_19233_b200 import renderer as R, _lib
    sc = scenes.make_random(8, n_gauss=500, n_tris=40)
    r = R.renderer_for(sc)
    host = R.to_pinned(sc)
    out = torch.empty((1, sc.cameras[0].height, sc.cameras[0].width, 4), dtype=torch.float32).pin_memory()
    arr = (_lib.Camera * 1)(R.c_camera(sc.cameras[0]))
    for field, which in (("sh", "g"), ("opacities", "g"), ("means", "g"), ("faces", "m"), ("opacity", "m")):
        g, m = R.c_gaussians(host), R.c_mesh(host)
        setattr(g if which == "g" else m, field, None)
        rc = r.L.unimgs_render_host_async(r._h, C.byref(g), C.byref(m), arr, 1, C.c_void_p(out.data_ptr()), None)
        assert rc == _lib.ERR_INVALID_ARGUMENT, field
    big = scenes.Camera(4096, 64, 64.0, 64.0, 32.0, 32.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    arr2 = (_lib.Camera * 2)(R.c_camera(sc.cameras[0]), R.c_camera(big))
    g, m = R.c_gaussians(host), R.c_mesh(host)
    assert r.L.unimgs_render_host_async(r._h, C.byref(g), C.byref(m), arr2, 2, C.c_void_p(out.data_ptr()),
                                        None) == _lib.ERR_INVALID_ARGUMENT
    r.host_wait()  # nothing was enqueued by the rejected calls
    r.render_host(host, [sc.cameras[0]], out)  # and the context still works


def test_render_host_uploads_cov3d(built):
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(31, n_gauss=2000, n_tris=50)
    q = sc.gaussians.quats.astype(np.float64)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    from scipy.spatial.transform import Rotation
    Rm = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
    S = np.einsum("nij,nj,nkj->nik", Rm, sc.gaussians.scales.astype(np.float64) ** 2, Rm)
    sc.gaussians.cov3d = np.stack([S[:, 0, 0], S[:, 0, 1], S[:, 0, 2], S[:, 1, 1], S[:, 1, 2], S[:, 2, 2]],
                                  -1).astype(np.float32)
    r = R.renderer_for(sc)
    dev = r.render_view(R.to_device(sc), sc.cameras[0]).cpu()
    host = R.to_pinned(sc)
    host.quats = host.scales = None  # cov3d replaces them (include/unimgs.h)
    out = torch.empty((2, sc.cameras[0].height, sc.cameras[0].width, 4), dtype=torch.float32).pin_memory()
    r.render_host(host, [sc.cameras[0]] * 2, out)
    assert torch.equal(out[0], dev) and torch.equal(out[1], dev)


def test_deform_junk_vertex_ids_are_culled(built, oracle_mod):
    from paper_2601_19233_b200 import renderer as R
    import torch
    sc, b = scenes.make_deform(n_gauss=4000, K=8)
    field = scenes.twist_field(sc.mesh)
    faces = sc.mesh.faces.copy()
    V = sc.mesh.num_vertices
    rng = np.random.default_rng(3)
    junk = rng.choice(len(faces), 200, replace=False)
    faces[junk[:100], rng.integers(0, 3, 100)] = -5
    faces[junk[100:], rng.integers(0, 3, 100)] = V + 17
    ds = R.to_device(sc)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    mo, co = R.deform(ds, dev(b.face.astype(np.int32)), dev(b.bary.astype(np.float32)), dev(faces.astype(np.int32)),
                      dev(field.packed()))
    torch.cuda.synchronize()
    om, oc = oracle_mod.Oracle(sc.gaussians, sc.mesh).deform(b, field, faces)
    assert np.abs(mo.cpu().numpy() - om).max() < 2e-6
    assert (np.abs(co.cpu().numpy() - oc) / np.abs(oc).max(1, keepdims=True)).max() < 2e-5
    hit = np.isin(b.face, junk).any(1)
    assert hit.sum() > 100  # the junk faces really are referenced
