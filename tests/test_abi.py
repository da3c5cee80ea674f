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
    """Every ctypes mirror of an ABI struct has the size and the field offsets a C
    compiler gives the header's struct (catches drift between include/unimgs.h and
    the Python binding)."""
    import subprocess
    import tempfile
    from paper_2601_19233_b200 import _lib
    pairs = [("unimgs_camera", _lib.Camera), ("unimgs_gaussians", _lib.Gaussians), ("unimgs_binding", _lib.Binding),
             ("unimgs_vertex_field", _lib.VertexField), ("unimgs_mesh", _lib.Mesh), ("unimgs_settings", _lib.Settings),
             ("unimgs_stats", _lib.Stats), ("unimgs_bind_settings", _lib.BindSettings)]
    lines, want = [], []
    for cname, py in pairs:
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        want.append(ctypes.sizeof(py))
        for fname, _ in py._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {fname}));')
            want.append(getattr(py, fname).offset)
    code = "#include <stdio.h>\n#include <stddef.h>\n#include \"unimgs.h\"\nint main(void){" + "".join(lines) + "return 0;}"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(code)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        got = list(map(int, subprocess.check_output([exe]).split()))
    assert got == want


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


@pytest.mark.parametrize("field,value,code", [
    ("msaa_samples", 3, "ERR_UNSUPPORTED"), ("blend_mode", 5, "ERR_UNSUPPORTED"),
    ("tile_size", 8, "ERR_UNSUPPORTED"), ("sort_mode", 2, "ERR_UNSUPPORTED"),
    ("tri_depth", 3, "ERR_UNSUPPORTED"), ("sort_ctas_per_sm", 5, "ERR_INVALID_ARGUMENT"),
    ("sort_ctas_per_sm", -1, "ERR_INVALID_ARGUMENT"), ("alpha_max", 0.0, "ERR_INVALID_ARGUMENT"),
    ("t_eps", 1.0, "ERR_INVALID_ARGUMENT"), ("dilation", -0.1, "ERR_INVALID_ARGUMENT"),
])
def test_create_rejects_invalid_settings(field, value, code):
    """unimgs_create validates the settings on the host before touching the GPU
    (include/unimgs.h settings contract): no context, the documented status."""
    from paper_2601_19233_b200 import _lib
    L = _lib.load()
    s = _lib.Settings()
    L.unimgs_default_settings(ctypes.byref(s))
    setattr(s, field, value)
    h = ctypes.c_void_p()
    assert L.unimgs_create(ctypes.byref(h), ctypes.byref(s)) == getattr(_lib, code)
    assert not h.value
