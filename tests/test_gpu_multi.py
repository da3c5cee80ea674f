"""unimgs_preprocess_multi (several views of one scene preprocessed in one pass, the
scene read once) on a B200 (-m gpu): every context's records, sorted bins and image
are bit-identical to a single-view unimgs_preprocess of its view, for 1..4 views,
with Gaussians from quaternions and from cov3d; the batched ContextPool renders the
multiview config bit-identically to single-context renders."""
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


def _cams(sc, k):
    c0 = sc.cameras[0]
    return [scenes.Camera(c0.width, c0.height, c0.fx * (1 + 0.05 * i), c0.fy * (1 + 0.05 * i), c0.cx, c0.cy, c0.R,
                          np.asarray(c0.t, np.float32) + np.float32(0.04 * i)) for i in range(k)]


@pytest.mark.parametrize("nviews", [1, 2, 3, 4])
@pytest.mark.parametrize("cov", [False, True])
def test_preprocess_multi_bit_identical(built, nviews, cov):
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(5, n_gauss=5000, n_tris=300, W=300, H=200)
    if cov:
        q = sc.gaussians.quats.astype(np.float64)
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        from scipy.spatial.transform import Rotation
        Rm = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()
        S = np.einsum("nij,nj,nkj->nik", Rm, sc.gaussians.scales.astype(np.float64) ** 2, Rm)
        sc.gaussians.cov3d = np.stack([S[:, 0, 0], S[:, 0, 1], S[:, 0, 2], S[:, 1, 1], S[:, 1, 2], S[:, 2, 2]],
                                      -1).astype(np.float32)
    cams = _cams(sc, nviews)
    ds = R.to_device(sc)
    rs = [R.renderer_for(sc) for _ in range(nviews)]
    R.preprocess_multi(rs, ds, cams)
    for r in rs:
        r.bin()
    imgs = [r.render().clone() for r in rs]
    torch.cuda.synchronize()
    for r, cam, img in zip(rs, cams, imgs):
        ref = R.renderer_for(sc)
        want = ref.render_view(ds, cam)
        torch.cuda.synchronize()
        assert torch.equal(img, want)
        a, b = r.records(), ref.records()
        for k in ("touched", "dkey"):
            assert np.array_equal(a[k], b[k]), k
        vis = b["touched"] > 0  # (a culled primitive's record is never written or read)
        F = sc.mesh.num_triangles
        assert np.array_equal(a["rect"][vis], b["rect"][vis])
        assert np.array_equal(a["grec"][vis[F:]], b["grec"][vis[F:]])
        assert np.array_equal(a["trec"][vis[:F]], b["trec"][vis[:F]])
        for x, y in zip(r.bins(), ref.bins()):
            assert np.array_equal(x, y)
        assert r.stats()["visible_gaussians"] == ref.stats()["visible_gaussians"]


def test_preprocess_multi_validation(built):
    from paper_2601_19233_b200 import renderer as R, _lib
    sc = scenes.make_tiny()
    ds = R.to_device(sc)
    r = R.renderer_for(sc)
    with pytest.raises(_lib.UnimgsError):
        R.preprocess_multi([r, r], ds, [sc.cameras[0]] * 2)  # one context twice
    with pytest.raises(_lib.UnimgsError):
        R.preprocess_multi([R.renderer_for(sc) for _ in range(5)], ds, [sc.cameras[0]] * 5)  # > 4 views


def test_batched_pool_multiview_bit_identical(built):
    """The bench's batched configuration (8 contexts in two sets of 4, one
    unimgs_preprocess_multi per group of 4 views) at full size, two steps queued."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_multiview()
    ds = R.to_device(sc)
    W, H = sc.cameras[0].width, sc.cameras[0].height
    views = [3, 4, 5, 6, 40, 41, 42, 43, 150, 151]
    pool = R.ContextPool(8, sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H, batch=4,
                         bg=tuple(float(v) for v in sc.bg), bg_alpha=float(sc.bg_alpha))
    out = torch.empty((len(views), H, W, 4), device="cuda")
    s = torch.cuda.current_stream()
    pool.render_views(ds, [sc.cameras[v] for v in views[:6]], out[:6], after=s)
    pool.render_views(ds, [sc.cameras[v] for v in views[6:]], out[6:])
    pool.join(s)
    torch.cuda.synchronize()
    single = R.Renderer(sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H,
                        bg=tuple(float(v) for v in sc.bg), bg_alpha=float(sc.bg_alpha))
    for j, vi in enumerate(views):
        ref = single.render_view(ds, sc.cameras[vi])
        torch.cuda.synchronize()
        assert torch.equal(out[j], ref), vi
