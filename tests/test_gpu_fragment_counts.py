"""Per-pixel fragment membership on the GPU, bit for bit (run on a B200 with -m gpu).

unimgs_render_fragments reports, per pixel, the Gaussian and triangle fragments
the blend applied and the id of the last one; the oracle's or_render_counts
walks the same tile lists with the C.1 membership ("fragments overlapping
the pixel"; S:173 alpha >= 1/255 as q <= q_max, N6; non-zero 4-sample masks).
With t_eps = 0 nothing terminates, so the counts must match EXACTLY at every
pixel -- this is what proves the blend's per-warp culling (conservative extents
for cond(Q) <= ~1000, never culling needles beyond it) drops no boundary
fragment.  With the default t_eps the termination decision is taken in fp32 on
the GPU and fp64 in the oracle, so a pixel may stop one fragment apart.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

from parity_util import compare_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2601_19233_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()
    return True


def _gpu_counts(sc, cam, **settings):
    import torch
    from paper_2601_19233_b200 import renderer as R
    r = R.renderer_for(sc, max_pairs=max(R.estimate_pairs(sc), 24 << 20 if sc.gaussians.count > 10 ** 6 else 0),
                       **settings)
    ds = R.to_device(sc)
    r.preprocess(ds, cam)
    r.bin()
    img, cnt = r.render_fragments()
    torch.cuda.synchronize()
    return img.cpu().numpy(), cnt.cpu().numpy().view(np.uint32)


def _oracle(oracle_mod, sc, cam, **settings):
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc, **settings))
    o.bin()
    return o


SMALL = {"needles": lambda: scenes.make_needles(),
         "random2_ragged": lambda: scenes.make_random(2, n_gauss=3000, n_tris=200, W=211, H=117),
         "nested": lambda: scenes.make_nested(),
         "degenerate": lambda: scenes.make_degenerate()[0]}


@pytest.mark.parametrize("name", list(SMALL))
def test_fragment_counts_bit_exact(built, oracle_mod, name):
    sc = SMALL[name]()
    cam = sc.cameras[0]
    img, cnt = _gpu_counts(sc, cam, t_eps=0.0)
    o = _oracle(oracle_mod, sc, cam, t_eps=0.0)
    ref = o.fragment_counts()
    bad = np.argwhere((cnt[..., :3] != ref[..., :3]).any(-1))
    assert len(bad) == 0, f"{len(bad)} pixels differ, first {bad[:5].tolist()}: gpu {cnt[tuple(bad[0])][:3]} oracle {ref[tuple(bad[0])][:3]}"
    assert ref[..., 0].sum() > 1000
    compare_image(img, o.render())


def test_fragment_counts_with_termination(built, oracle_mod):
    sc = scenes.make_needles()
    cam = sc.cameras[0]
    img, cnt = _gpu_counts(sc, cam)
    o = _oracle(oracle_mod, sc, cam)
    ref = o.fragment_counts()
    d = np.abs(cnt[..., :2].astype(np.int64) - ref[..., :2].astype(np.int64)).sum(-1)
    assert (d > 0).mean() <= 1e-3 and d.max() <= 1
    compare_image(img, o.render())


def test_fragment_counts_mip360_sampled_tiles(built, oracle_mod):
    """BASELINE's mip360 config (3M Gaussians, 200k triangles, 1080p), the bench's view 0:
    every fragment of 64 sampled tiles (t_eps = 0: the whole tile lists) bit-exact, and with
    the default t_eps the counts of 300 sampled tiles agree up to the fp32/fp64 stop."""
    sc = scenes.make_mip360()
    cam = sc.cameras[0]
    rng = np.random.default_rng(5)
    tiles_x, tiles_y = (cam.width + 15) // 16, (cam.height + 15) // 16
    _, cnt = _gpu_counts(sc, cam, t_eps=0.0)
    o = _oracle(oracle_mod, sc, cam, t_eps=0.0)
    tl = rng.choice(tiles_x * tiles_y, 64, replace=False)
    ref = o.fragment_counts(tl)
    mask = np.zeros(cnt.shape[:2], bool)
    for t in tl:
        ty, tx = divmod(int(t), tiles_x)
        mask[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16] = True
    assert np.array_equal(cnt[mask][:, :3], ref[mask][:, :3])
    assert ref[mask][:, 0].sum() > 10 ** 5
    img, cnt = _gpu_counts(sc, cam)
    o = _oracle(oracle_mod, sc, cam)
    tl = rng.choice(tiles_x * tiles_y, 300, replace=False)
    ref = o.fragment_counts(tl)
    mask[:] = False
    for t in tl:
        ty, tx = divmod(int(t), tiles_x)
        mask[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16] = True
    d = np.abs(cnt[mask][:, :2].astype(np.int64) - ref[mask][:, :2].astype(np.int64)).sum(-1)
    assert (d > 0).mean() <= 1e-3 and d.max() <= 1
    compare_image(img, o.render(tl))
