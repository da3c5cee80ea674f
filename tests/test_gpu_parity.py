"""CUDA path vs the CPU oracle (run on a B200 with -m gpu), through the C ABI.

Small scenes span several tiles with ragged image borders; the full-size
configs run at BASELINE.json's sizes in the bench's launch configuration.
"""
import numpy as np
import pytest

from paper_2601_19233_b200 import scenes

from parity_util import compare_bins, compare_image, compare_records, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

SMALL = {
    "tiny": lambda: scenes.make_tiny(),
    "random0": lambda: scenes.make_random(0),
    "random1_colors": lambda: scenes.make_random(1, n_gauss=800, n_tris=120, textured=False),
    "random2_ragged": lambda: scenes.make_random(2, n_gauss=3000, n_tris=200, W=211, H=117),
    "nested": lambda: scenes.make_nested(),
    "edge": lambda: scenes.make_edge(),
    "overflow": lambda: scenes.make_overflow(),
    "degenerate": lambda: scenes.make_degenerate()[0],
}


@pytest.fixture(scope="module")
def built():
    from paper_2601_19233_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()
    return True


@pytest.mark.parametrize("sort_mode", [0, 1])
@pytest.mark.parametrize("name", list(SMALL))
def test_small_scene_parity(built, oracle_mod, name, sort_mode):
    sc = SMALL[name]()
    cam = sc.cameras[0]
    r, ds, img = run_gpu(sc, cam, sort_mode=sort_mode)
    o = run_oracle(oracle_mod, sc, cam)
    compare_records(r, o, sc)
    compare_bins(r, o)
    compare_image(img, o.render())


def test_gaussians_only_and_mesh_only(built, oracle_mod):
    base = scenes.make_random(3, n_gauss=1500, n_tris=100)
    for sc in (scenes.Scene("g", base.gaussians, scenes.empty_mesh(), base.cameras, base.bg),
               scenes.Scene("m", scenes.empty_gaussians(3), base.mesh, base.cameras, base.bg)):
        r, ds, img = run_gpu(sc, sc.cameras[0])
        o = run_oracle(oracle_mod, sc, sc.cameras[0])
        compare_bins(r, o)
        compare_image(img, o.render())


def test_empty_scene(built, oracle_mod):
    sc = scenes.Scene("empty", scenes.empty_gaussians(0), scenes.empty_mesh(), scenes.make_tiny().cameras,
                      np.array([0.1, 0.2, 0.3], np.float32))
    r, ds, img = run_gpu(sc, sc.cameras[0])
    assert np.allclose(img[..., :3], sc.bg) and np.all(img[..., 3] == 1.0)
    assert r.stats()["num_pairs"] == 0


def test_determinism_bit_identical(built):
    import torch
    sc = scenes.make_random(4, n_gauss=5000, n_tris=300)
    from paper_2601_19233_b200 import renderer as R
    r = R.renderer_for(sc)
    ds = R.to_device(sc)
    a = r.render_view(ds, sc.cameras[0]).clone()
    b = r.render_view(ds, sc.cameras[0]).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_sort_modes_agree(built):
    import torch
    sc = scenes.make_random(5, n_gauss=6000, n_tris=300, W=300, H=200)
    from paper_2601_19233_b200 import renderer as R
    outs = []
    for mode in (0, 1):
        r = R.renderer_for(sc, sort_mode=mode)
        img = r.render_view(R.to_device(sc), sc.cameras[0]).clone()
        outs.append((img, r.bins()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


def test_capacity_overflow(built):
    import torch
    from paper_2601_19233_b200 import renderer as R, _lib
    sc = scenes.make_random(6, n_gauss=2000, n_tris=50)
    r = R.renderer_for(sc, max_pairs=64)
    out = torch.full((sc.cameras[0].height, sc.cameras[0].width, 4), -7.0, device="cuda")
    r.render_view(R.to_device(sc), sc.cameras[0], out=out)
    st = r.stats(check=False)
    assert st["status"] == _lib.ERR_CAPACITY and st["overflow"] == 1 and st["needed_pairs"] > 64
    torch.cuda.synchronize()
    assert torch.all(out == -7.0)  # render leaves out untouched on overflow
    # grow and retry
    r2 = R.renderer_for(sc, max_pairs=st["needed_pairs"])
    r2.render_view(R.to_device(sc), sc.cameras[0])
    assert r2.stats()["num_pairs"] == st["needed_pairs"]


def test_invalid_arguments(built):
    from paper_2601_19233_b200 import renderer as R, _lib
    sc = scenes.make_tiny()
    r = R.renderer_for(sc)
    with pytest.raises(_lib.UnimgsError) as e:
        r.bin()
    assert e.value.code == _lib.ERR_STATE
    big = scenes.Camera(4096, 64, 64.0, 64.0, 32.0, 32.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    with pytest.raises(_lib.UnimgsError) as e:
        r.preprocess(R.to_device(sc), big)
    assert e.value.code == _lib.ERR_INVALID_ARGUMENT
    with pytest.raises(_lib.UnimgsError) as e:
        R.Renderer(10, 10, 100, 64, 64, sort_mode=7)
    for bad in (-1, 5):  # persistent sort CTAs per SM: 0 (auto) .. 4
        with pytest.raises(_lib.UnimgsError) as e:
            R.Renderer(10, 10, 100, 64, 64, sort_ctas_per_sm=bad)
        assert e.value.code == _lib.ERR_INVALID_ARGUMENT


def test_cuda_graph_replay_matches_eager(built):
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(7, n_gauss=4000, n_tris=200)
    r = R.renderer_for(sc)
    ds = R.to_device(sc)
    cam = sc.cameras[0]
    eager = r.render_view(ds, cam).clone()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        r.render_view(ds, cam, out=out)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r.render_view(ds, cam, out=out)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)


def test_render_host_matches_device(built):
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(8, n_gauss=3000, n_tris=150)
    cams = [sc.cameras[0]] * 3
    r = R.renderer_for(sc)
    dev = r.render_view(R.to_device(sc), sc.cameras[0]).cpu()
    host = R.to_pinned(sc)
    out = torch.empty((3, sc.cameras[0].height, sc.cameras[0].width, 4), dtype=torch.float32).pin_memory()
    r.render_host(host, cams, out)
    for v in range(3):
        assert torch.equal(out[v], dev)


# ---------------------------------------------------------------------------
# BASELINE.json configs at full size
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["tiny", "nerf", "mip360", "stress"])
def test_config_parity(built, oracle_mod, name):
    sc = scenes.make_scene(name)
    cam = sc.cameras[0]
    r, ds, img = run_gpu(sc, cam)
    o = run_oracle(oracle_mod, sc, cam)
    compare_records(r, o, sc)
    K = compare_bins(r, o)
    err = compare_image(img, o.render())
    print(f"{name}: K={K} max_err={err:.2e}")


def test_multiview_parity(built, oracle_mod):
    sc = scenes.make_multiview()
    from paper_2601_19233_b200 import renderer as R
    r = R.renderer_for(sc, max_pairs=16 << 20)
    ds = R.to_device(sc)
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    rng = np.random.default_rng(0)
    for i in range(0, 256, 32):  # the 8 views i in {0, 32, ..., 224}
        cam = sc.cameras[i]
        img = r.render_view(ds, cam).cpu().numpy()
        o.project(cam, **oracle_mod.scene_settings(sc))
        o.bin()
        compare_bins(r, o)
        tiles = rng.choice(o.tiles_x * o.tiles_y, 600, replace=False)
        compare_image(img, o.render(tiles))


# ---------------------------------------------------------------------------
# blend-mode ablation and sample counts
# ---------------------------------------------------------------------------

MODE_SCENES = {
    "random0": lambda: scenes.make_random(0),
    "overflow": lambda: scenes.make_overflow(),
    "nested": lambda: scenes.make_nested(),
    "edge": lambda: scenes.make_edge(),
}


@pytest.mark.parametrize("M", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("name", list(MODE_SCENES))
def test_blend_modes_parity(built, oracle_mod, name, mode, M):
    from paper_2601_19233_b200 import renderer as R
    sc = MODE_SCENES[name]()
    cam = sc.cameras[0]
    r = R.renderer_for(sc, blend_mode=mode, msaa=M)
    img = r.render_view(R.to_device(sc), cam).cpu().numpy()
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc, blend_mode=mode, msaa=M))
    o.bin()
    compare_bins(r, o)
    compare_image(img, o.render())


def test_fig3_overflow_on_gpu(built, oracle_mod):
    """The whole-pixel entity's overflow on the Fig.3 construction is reproduced by the GPU
    (P:370-372): its overshoot over the 16x16 supersampled oracle exceeds 5x the exact one's."""
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_overflow()
    cam = sc.cameras[0]
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc, t_eps=0.0))
    ss = o.render_supersampled(16)
    ov = {}
    for mode in (0, 3):
        r = R.renderer_for(sc, blend_mode=mode, t_eps=0.0)
        img = r.render_view(R.to_device(sc), cam).cpu().numpy()
        sel = (slice(14, 51), 32)
        ov[mode] = float(np.clip(img[sel][..., :3] - ss[sel][..., :3], 0, None).max())
    assert ov[0] < 0.02 and ov[3] >= 5 * ov[0] and ov[3] > 0.2, ov


@pytest.mark.parametrize("lanes", [1, 3])
def test_render_host_async_pipeline(built, lanes):
    """Three overlapping pipelined calls (double-buffered device scene, views on 1 or 3
    render lanes): every frame equals the device-resident render of its camera."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(9, n_gauss=3000, n_tris=150)
    cam0 = sc.cameras[0]
    cams = []
    for k in range(6):  # camera k: cam0 translated slightly
        t = np.asarray(cam0.t, np.float32) + np.float32(0.02 * k)
        cams.append(scenes.Camera(cam0.width, cam0.height, cam0.fx, cam0.fy, cam0.cx, cam0.cy, cam0.R, t))
    r = R.renderer_for(sc)
    ds = R.to_device(sc)
    want = [r.render_view(ds, c).cpu() for c in cams]
    host = R.to_pinned(sc)
    r.set_host_lanes(lanes)
    outs = [torch.full((2, cam0.height, cam0.width, 4), -1.0).pin_memory() for _ in range(3)]
    for k in range(3):
        r.render_host_async(host, cams[2 * k:2 * k + 2], outs[k])
    r.host_wait()
    for k in range(3):
        for j in range(2):
            assert torch.equal(outs[k][j], want[2 * k + j])
    one = torch.empty((6, cam0.height, cam0.width, 4)).pin_memory()
    r.render_host(host, cams, one)  # synchronous form, all six views over the lanes
    for j in range(6):
        assert torch.equal(one[j], want[j])


def test_junk_is_invisible_on_gpu(built):
    """NaN / inf / out-of-range primitives are culled as values on the GPU too: the
    frame equals the frame of the valid scene alone; stats count only valid ones."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc, base = scenes.make_degenerate()
    cam = sc.cameras[0]
    r = R.renderer_for(sc)
    img = r.render_view(R.to_device(sc), cam).clone()
    st = r.stats()
    rb = R.renderer_for(base)
    ref = rb.render_view(R.to_device(base), cam).clone()
    stb = rb.stats()
    torch.cuda.synchronize()
    assert torch.isfinite(img).all()
    assert torch.equal(img, ref)
    assert st["num_pairs"] == stb["num_pairs"]
    assert st["visible_gaussians"] == stb["visible_gaussians"]
    assert st["visible_triangles"] == stb["visible_triangles"]
    assert st["culled_guard_band"] > stb["culled_guard_band"]


@pytest.mark.parametrize("mode", [0, 1])
def test_sort_ctas_per_sm_agree(built, mode):
    """settings.sort_ctas_per_sm only schedules: 1..4 persistent sort CTAs per SM
    give bit-identical bins and images (K ~1.8M: several sort tiles per persistent CTA)."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_random(7, n_gauss=60000, n_tris=2000, W=640, H=360)
    ds = R.to_device(sc)
    outs = []
    for spm in (0, 1, 2, 3, 4):
        r = R.renderer_for(sc, max_pairs=4 << 20, sort_mode=mode, sort_ctas_per_sm=spm)
        img = r.render_view(ds, sc.cameras[0]).clone()
        outs.append((img, r.bins()))
    torch.cuda.synchronize()
    assert outs[0][1][0].size > 148 * 2048  # several sort tiles per persistent CTA
    for img, bins in outs[1:]:
        assert torch.equal(outs[0][0], img)
        for a, b in zip(outs[0][1], bins):
            assert np.array_equal(a, b)


def test_multiview_bench_launch_configuration(built, oracle_mod):
    """The bench's launch configuration at full size (bench.py's defaults through the same
    renderer.ContextPool): the 3M-Gaussian multiview scene, views round-robin on 4
    contexts concurrently, one sort CTA per SM, preprocess + bin on high-priority
    streams, blends on normal ones, two steps queued back to back without a join.
    Every frame equals the single-context render of its view bit for bit, and two of
    them match the oracle on sampled tiles."""
    import torch
    from paper_2601_19233_b200 import renderer as R
    sc = scenes.make_multiview()
    ds = R.to_device(sc)
    cam0 = sc.cameras[0]
    W, H = cam0.width, cam0.height
    views = [3, 40, 77, 114, 151, 188, 225, 6]
    pool = R.ContextPool(4, sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H,
                         bg=tuple(float(v) for v in sc.bg), bg_alpha=float(sc.bg_alpha))
    assert all(r._settings.sort_ctas_per_sm == 1 for r in pool.rs)
    out = torch.empty((len(views), H, W, 4), device="cuda")
    s = torch.cuda.current_stream()
    pool.render_views(ds, [sc.cameras[v] for v in views[:4]], out[:4], after=s)
    pool.render_views(ds, [sc.cameras[v] for v in views[4:]], out[4:])  # the next step, no join
    pool.join(s)
    torch.cuda.synchronize()
    single = R.Renderer(sc.gaussians.count, sc.mesh.num_triangles, 20 << 20, W, H,
                        bg=tuple(float(v) for v in sc.bg), bg_alpha=float(sc.bg_alpha))
    for j, vi in enumerate(views):
        ref = single.render_view(ds, sc.cameras[vi])
        torch.cuda.synchronize()
        assert torch.equal(out[j], ref), vi
    for j in (1, 6):
        o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
        o.project(sc.cameras[views[j]], **oracle_mod.scene_settings(sc))
        o.bin()
        tiles = np.random.default_rng(2 + j).choice(o.tiles_x * o.tiles_y, 300, replace=False)
        compare_image(out[j].cpu().numpy(), o.render(tiles))


def test_8k_image_full_keys(built, oracle_mod):
    """7680x4320 = 129,600 tiles: more than the 16-bit tile keys of sort_mode 0 hold,
    which is refused (UNSUPPORTED); sort_mode 1 (and tri_depth 1, which always uses
    it) bins bit-exactly with 17-bit tile ids and renders within the tolerance."""
    from paper_2601_19233_b200 import renderer as R, _lib
    sc = scenes.make_random(21, n_gauss=2500, n_tris=300, W=7680, H=4320)
    cam = sc.cameras[0]
    r0 = R.renderer_for(sc, sort_mode=0)
    with pytest.raises(_lib.UnimgsError) as e:
        r0.preprocess(R.to_device(sc), cam)
    assert e.value.code == _lib.ERR_UNSUPPORTED
    for settings in ({"sort_mode": 1}, {"tri_depth": 1}):
        r = R.renderer_for(sc, max_pairs=16 << 20, **settings)
        img = r.render_view(R.to_device(sc), cam).cpu().numpy()
        o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
        o.project(cam, **oracle_mod.scene_settings(sc, tri_depth=settings.get("tri_depth", 0)))
        o.bin()
        assert o.tiles_x * o.tiles_y > 65536
        compare_bins(r, o)
        tiles = np.random.default_rng(5).choice(o.tiles_x * o.tiles_y, 400, replace=False)
        compare_image(img, o.render(tiles))


@pytest.mark.parametrize("wh", [(1, 1), (17, 3), (16, 16)])
@pytest.mark.parametrize("sort_mode", [0, 1])
def test_tiny_images(built, oracle_mod, wh, sort_mode):
    """One tile (zero tile-key bits: no tile passes), a ragged 2-tile strip, exactly one full tile."""
    sc = scenes.make_random(30 + wh[0], n_gauss=300, n_tris=30, W=wh[0], H=wh[1])
    cam = sc.cameras[0]
    r, ds, img = run_gpu(sc, cam, sort_mode=sort_mode)
    o = run_oracle(oracle_mod, sc, cam)
    compare_bins(r, o)
    compare_image(img, o.render())


def test_mip360_at_4k(built, oracle_mod):
    """Maximum-size case: the 3M-Gaussian mip360 scene at 3840x2160 (~18M pairs, 2.4x
    the bench's 1080p frame; 32,400 tiles = 15 tile-key bits): all sorted pairs
    bit-exact, colour on sampled tiles."""
    sc = scenes.make_scene("mip360")
    c = sc.cameras[0]
    cam = scenes.Camera(3840, 2160, c.fx * 2, c.fy * 2, c.cx * 2, c.cy * 2, c.R, c.t, c.near, c.far)
    from paper_2601_19233_b200 import renderer as R
    r4 = R.Renderer(sc.gaussians.count, sc.mesh.num_triangles, 48 << 20, 3840, 2160,
                    bg=tuple(float(v) for v in sc.bg), bg_alpha=float(sc.bg_alpha))
    r, ds, img = run_gpu(sc, cam, renderer=r4)
    o = run_oracle(oracle_mod, sc, cam)
    K = compare_bins(r, o)
    assert K > 15_000_000
    tiles = np.random.default_rng(6).choice(o.tiles_x * o.tiles_y, 400, replace=False)
    compare_image(img, o.render(tiles))
