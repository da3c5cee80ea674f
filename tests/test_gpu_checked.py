"""Memory safety of the CUDA path (compute-sanitizer is
closed on this pool): the whole sanitize workload (tools/sanitize.py -- every kernel,
capacity overflow, host lanes, deform, bind) runs through the CHECKED build
(libunimgs_checked.so: device bounds checks on every scatter index that trap the
kernel, a 4 KiB guard band after every context scratch buffer) without a trap and
without a single guard byte overwritten, and its outputs are bit-identical to the
production library's -- so the checks observe the same execution.  Fault injection
shows both mechanisms are live."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib, dump, *extra):
    env = dict(os.environ, UNIMGS_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py"), "--dump", dump, *extra],
                       env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    return p.stdout


def test_checked_build_is_clean_and_identical(tmp_path):
    from paper_2601_19233_b200 import build
    lib = build.build()
    chk = build.build(checked=True)
    out = _run(chk, str(tmp_path / "checked.npz"), "--check-guards")
    assert "guard bytes overwritten: 0" in out and "UNIMGS_CHECK failed" not in out
    _run(lib, str(tmp_path / "prod.npz"))
    a, b = np.load(tmp_path / "checked.npz"), np.load(tmp_path / "prod.npz")
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


PROBE = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2601_19233_b200 import renderer as R, scenes, _lib
sc = scenes.make_random(3, n_gauss=500, n_tris=20)
r = R.renderer_for(sc)
try:
    r.render_view(R.to_device(sc), sc.cameras[0])
    torch.cuda.synchronize()
    print("guards", r.check_guards())
except (RuntimeError, _lib.UnimgsError) as e:
    print("error", type(e).__name__, str(e)[:200])
'''


@pytest.mark.parametrize("fault", ["UNIMGS_FAULT_TILES", "UNIMGS_FAULT_GUARD"])
def test_checked_build_detects_injected_faults(fault):
    from paper_2601_19233_b200 import build
    chk = build.build(checked=True)
    p = subprocess.run([sys.executable, "-c", PROBE % ROOT], env=dict(os.environ, UNIMGS_LIB=chk, **{fault: "1"}),
                       capture_output=True, text=True, timeout=300)
    if fault == "UNIMGS_FAULT_TILES":  # a tile index beyond the (forged) capacity traps the kernel
        assert "UNIMGS_CHECK failed" in p.stdout + p.stderr and "guards" not in p.stdout, p.stdout + p.stderr[-2000:]
    else:  # the cleared guard byte is reported
        assert p.returncode == 0 and "guards 1" in p.stdout, p.stdout + p.stderr[-2000:]
