"""The C-ABI library builds, loads and exports every symbol include/unimgs.h declares (CPU only)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "unimgs.h")).read()
    return sorted(set(re.findall(r"UNIMGS_API[^;(]*?\b(unimgs_\w+)\s*\(", src)))


def test_header_declares_the_pipeline():
    syms = declared_symbols()
    for s in ("unimgs_preprocess", "unimgs_bin", "unimgs_render", "unimgs_reserve", "unimgs_create"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2601_19233_b200 import build, _lib
    path = build.build()
    lib = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_struct_layouts_match_header():
    """ctypes mirrors of the ABI structs have the sizes a C compiler gives them."""
    import subprocess
    import tempfile
    from paper_2601_19233_b200 import _lib
    code = r'''
#include <stdio.h>
#include "unimgs.h"
int main(void){printf("%zu %zu %zu %zu %zu\n", sizeof(unimgs_camera), sizeof(unimgs_gaussians),
 sizeof(unimgs_mesh), sizeof(unimgs_settings), sizeof(unimgs_stats)); return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(code)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        sizes = list(map(int, subprocess.check_output([exe]).split()))
    mine = [ctypes.sizeof(x) for x in (_lib.Camera, _lib.Gaussians, _lib.Mesh, _lib.Settings, _lib.Stats)]
    assert sizes == mine


def test_no_device_calls_fail_cleanly_without_gpu():
    """Host-side validation works without a device: bad settings are rejected, not crashed."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2601_19233_b200 import _lib
    L = _lib.load()
    s = _lib.Settings()
    L.unimgs_default_settings(ctypes.byref(s))
    assert s.msaa_samples == 4 and s.tile_size == 16 and abs(s.alpha_max - 0.99) < 1e-7
    s.msaa_samples = 3  # only 1, 2, 4, 8, 16
    h = ctypes.c_void_p()
    assert L.unimgs_create(ctypes.byref(h), ctypes.byref(s)) == _lib.ERR_UNSUPPORTED
