"""ctypes view of libunimgs.so (include/unimgs.h).  Argument marshalling only.

The library is built in-tree (``python -m paper_2601_19233_b200.build``).  There
is no fallback: if the shared object is missing, importing the renderer fails.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UNIMGS_LIB") or os.path.join(HERE, "libunimgs.so")  # override: experiments only

OK, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED, ERR_CAPACITY, ERR_CUDA, ERR_STATE = range(6)
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "UNSUPPORTED", 3: "CAPACITY", 4: "CUDA", 5: "STATE"}

# every symbol include/unimgs.h declares
EXPORTS = ("unimgs_default_settings", "unimgs_create", "unimgs_set_settings", "unimgs_reserve", "unimgs_reserve2",
           "unimgs_preprocess", "unimgs_bin", "unimgs_render", "unimgs_render_counted", "unimgs_get_stats", "unimgs_get_bins",
           "unimgs_get_records", "unimgs_render_host", "unimgs_launch_count", "unimgs_error_string",
           "unimgs_destroy", "unimgs_deform", "unimgs_bind", "unimgs_render_host_async", "unimgs_host_wait",
           "unimgs_set_host_lanes", "unimgs_render_fragments", "unimgs_debug_check_guards",
           "unimgs_preprocess_multi")


class BindSettings(C.Structure):
    _fields_ = [("mode", C.c_int32), ("k_sigma", C.c_float)]


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("near_z", C.c_float), ("far_z", C.c_float)]


class Gaussians(C.Structure):
    _fields_ = [("count", C.c_int64), ("means", C.c_void_p), ("quats", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("sh", C.c_void_p), ("sh_degree", C.c_int32), ("cov3d", C.c_void_p)]


class Binding(C.Structure):
    _fields_ = [("count", C.c_int64), ("anchors", C.c_int32), ("face", C.c_void_p), ("bary", C.c_void_p)]


class VertexField(C.Structure):
    _fields_ = [("num_vertices", C.c_int64), ("num_faces", C.c_int64), ("faces", C.c_void_p), ("data", C.c_void_p)]


class Mesh(C.Structure):
    _fields_ = [("num_vertices", C.c_int64), ("num_triangles", C.c_int64), ("positions", C.c_void_p),
                ("uvs", C.c_void_p), ("colors", C.c_void_p), ("faces", C.c_void_p), ("opacity", C.c_void_p),
                ("texture", C.c_void_p), ("tex_width", C.c_int32), ("tex_height", C.c_int32)]


class Settings(C.Structure):
    _fields_ = [("msaa_samples", C.c_int32), ("tile_size", C.c_int32), ("alpha_min", C.c_float),
                ("alpha_max", C.c_float), ("t_eps", C.c_float), ("dilation", C.c_float), ("bg", C.c_float * 3),
                ("bg_alpha", C.c_float), ("sort_mode", C.c_int32), ("blend_mode", C.c_int32),
                ("tri_depth", C.c_int32), ("sort_ctas_per_sm", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("num_pairs", C.c_int64), ("needed_pairs", C.c_int64), ("visible_gaussians", C.c_int64),
                ("visible_triangles", C.c_int64), ("culled_guard_band", C.c_int64), ("overflow", C.c_int32),
                ("max_tile_pairs", C.c_int32), ("max_tile_id", C.c_int32), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32)]


_lib = None


def load():
    """Load the in-tree libunimgs.so; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2601_19233_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.unimgs_default_settings.argtypes = [C.POINTER(Settings)]
    L.unimgs_default_settings.restype = None
    L.unimgs_create.argtypes = [C.POINTER(vp), C.POINTER(Settings)]
    L.unimgs_set_settings.argtypes = [vp, C.POINTER(Settings)]
    L.unimgs_reserve.argtypes = [vp, i64, i64, i32, i32]
    L.unimgs_reserve2.argtypes = [vp, i64, i64, i64, i32, i32]
    L.unimgs_preprocess.argtypes = [vp, C.POINTER(Gaussians), C.POINTER(Mesh), C.POINTER(Camera), vp]
    L.unimgs_bin.argtypes = [vp, vp]
    L.unimgs_preprocess_multi.argtypes = [vp, C.c_int32, C.POINTER(Gaussians), C.POINTER(Mesh), C.POINTER(Camera), vp]
    L.unimgs_render.argtypes = [vp, vp, vp]
    L.unimgs_render_counted.argtypes = [vp, vp, vp, vp]
    L.unimgs_render_fragments.argtypes = [vp, vp, vp, vp]
    L.unimgs_debug_check_guards.argtypes = [vp, vp]
    L.unimgs_get_stats.argtypes = [vp, C.POINTER(Stats), vp]
    L.unimgs_get_bins.argtypes = [vp, vp, vp, vp, vp]
    L.unimgs_get_records.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.unimgs_render_host.argtypes = [vp, C.POINTER(Gaussians), C.POINTER(Mesh), C.POINTER(Camera), i32, vp, vp]
    L.unimgs_render_host_async.argtypes = [vp, C.POINTER(Gaussians), C.POINTER(Mesh), C.POINTER(Camera), i32, vp, vp]
    L.unimgs_render_host_async.restype = C.c_int
    L.unimgs_host_wait.argtypes = [vp]
    L.unimgs_host_wait.restype = C.c_int
    L.unimgs_set_host_lanes.argtypes = [vp, C.c_int32]
    L.unimgs_set_host_lanes.restype = C.c_int
    L.unimgs_deform.argtypes = [C.POINTER(Gaussians), C.POINTER(Binding), C.POINTER(VertexField), vp, vp, vp]
    L.unimgs_deform.restype = C.c_int
    L.unimgs_bind.argtypes = [C.POINTER(Gaussians), C.POINTER(Mesh), C.POINTER(Camera), C.c_int32,
                              C.POINTER(BindSettings), vp, vp, vp, vp]
    L.unimgs_bind.restype = C.c_int
    L.unimgs_launch_count.argtypes = [vp]
    L.unimgs_launch_count.restype = i64
    L.unimgs_error_string.argtypes = [vp]
    L.unimgs_error_string.restype = C.c_char_p
    L.unimgs_destroy.argtypes = [vp]
    L.unimgs_destroy.restype = None
    for name in ("unimgs_create", "unimgs_set_settings", "unimgs_reserve", "unimgs_reserve2", "unimgs_preprocess",
                 "unimgs_bin", "unimgs_render", "unimgs_render_counted", "unimgs_get_stats", "unimgs_get_bins", "unimgs_get_records",
                 "unimgs_render_host", "unimgs_render_fragments", "unimgs_debug_check_guards",
                 "unimgs_preprocess_multi"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


class UnimgsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"unimgs {STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
