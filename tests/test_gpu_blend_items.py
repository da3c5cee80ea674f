"""k_blend's work items -- (tile, 8x4 sub-tile) pairs dealt to CTAs in runs, each warp
taking the next item of its CTA's run (blend.cu) -- must not change any pixel: the image
is bit-identical for runs of 1, 5 (ragged: runs straddle tiles), 16 (the default) and 64
items per CTA.  The run length is read once per process (UNIMGS_BLEND_ITEMS), so each
setting renders in its own subprocess."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2601_19233_b200 import renderer as R, scenes
out = []
for sc in (scenes.make_random(5, n_gauss=3000, n_tris=120, W=211, H=117), scenes.make_scene("nerf")):
    r = R.renderer_for(sc)
    img = r.render_view(R.to_device(sc), sc.cameras[0])
    torch.cuda.synchronize()
    out.append(img.cpu().numpy())
np.savez(sys.argv[2], *out)
"""


def _render(tmp_path, items):
    env = dict(os.environ)
    env["UNIMGS_BLEND_ITEMS"] = str(items)
    dst = str(tmp_path / f"items{items}.npz")
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, dst], env=env, check=True, timeout=600)
    z = np.load(dst)
    return [z[k] for k in sorted(z.files)]


def test_blend_item_runs_do_not_change_pixels(tmp_path):
    ref = _render(tmp_path, 16)
    for items in (1, 5, 64):
        got = _render(tmp_path, items)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b), items
