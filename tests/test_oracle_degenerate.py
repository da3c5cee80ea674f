"""Invalid device data is culled as a value (include/unimgs.h; N1-N7): the oracle
culls every junk primitive of scenes.make_degenerate (tiles_touched = 0) and the
image equals the image of the valid scene alone -- junk is invisible, not fatal."""
import numpy as np

from paper_2601_19233_b200 import scenes


def test_junk_is_culled_and_invisible(oracle_mod):
    sc, base = scenes.make_degenerate()
    cam = sc.cameras[0]
    o = oracle_mod.Oracle(sc.gaussians, sc.mesh)
    o.project(cam, **oracle_mod.scene_settings(sc))
    o.bin()
    g, t = o.gaussian_records(), o.triangle_records()
    assert np.all(g["touched"][base.gaussians.count:] == 0)
    assert np.all(t["touched"][base.mesh.num_triangles:] == 0)
    ob = oracle_mod.Oracle(base.gaussians, base.mesh)
    ob.project(cam, **oracle_mod.scene_settings(base))
    ob.bin()
    assert o.K == ob.K
    img, ref = o.render(), ob.render()
    assert np.isfinite(img).all()
    assert np.abs(img - ref).max() <= 1e-12
    # the valid primitives keep their records
    assert np.array_equal(g["touched"][:base.gaussians.count], ob.gaussian_records()["touched"])
