"""CPU oracle for the UniMGS single-pass rasterizer -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps
``oracle/unimgs_oracle.c`` (plain C, see its header for the passages each step
follows) through ctypes and shares no code with ``paper_2601_19233_b200``.

Parity-unpinned parts: absolute appearance of realistic scenes,
the triangle sort depth (R9) and per-tile ordering (R8).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "unimgs_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "bind_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, no fast-math, SSE2 scalar floats)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class CCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("near_z", C.c_float), ("far_z", C.c_float)]


class CSettings(C.Structure):
    _fields_ = [("alpha_max", C.c_float), ("t_eps", C.c_float), ("dilation", C.c_float),
                ("bg", C.c_float * 3), ("bg_alpha", C.c_float), ("blend_mode", C.c_int32), ("msaa", C.c_int32),
                ("tri_depth", C.c_int32), ("resort_window", C.c_int32)]


# blend modes: the paper's ablation (Fig.3 / Fig.4)
EXACT, NAIVE, MSAA_PIXEL, WHOLE_PIXEL, PAPER_LITERAL = range(5)


class CFrag(C.Structure):
    _fields_ = [("id", C.c_uint32), ("kind", C.c_int32), ("mask", C.c_uint32), ("q", C.c_float),
                ("depth", C.c_float), ("pdepth", C.c_float), ("alpha", C.c_double), ("rgb", C.c_double * 3)]


FRAG_DTYPE = np.dtype([("id", np.uint32), ("kind", np.int32), ("mask", np.uint32), ("q", np.float32),
                       ("depth", np.float32), ("pdepth", np.float32), ("alpha", np.float64), ("rgb", np.float64, (3,))],
                      align=True)
assert FRAG_DTYPE.itemsize == C.sizeof(CFrag)

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        L.or_create.restype = vp
        L.or_destroy.argtypes = [vp]
        L.or_set_scene.argtypes = [vp, i64, vp, vp, vp, vp, vp, i32, i64, i64, vp, vp, vp, vp, vp, vp, i32, i32]
        L.or_project.argtypes = [vp, C.POINTER(CCamera), C.POINTER(CSettings), i32]
        L.or_project.restype = i32
        L.or_bin.argtypes = [vp]
        L.or_bin.restype = i64
        L.or_render.argtypes = [vp, vp, vp, i64, i32]
        L.or_render.restype = i32
        L.or_render_counts.argtypes = [vp, vp, vp, i64, i32]
        L.or_render_counts.restype = i32
        L.or_render_bruteforce.argtypes = [vp, vp, i32]
        L.or_render_bruteforce.restype = i32
        L.or_pixel_fragments.argtypes = [vp, i32, i32, vp, i64]
        L.or_pixel_fragments.restype = i64
        L.or_support_truncation.argtypes = [vp]
        L.or_support_truncation.restype = i64
        L.or_blend_fragments.argtypes = [vp, i32, C.POINTER(CSettings), vp, vp]
        L.or_blend_fragments.restype = i32
        L.or_num_pairs.argtypes = [vp]
        L.or_num_pairs.restype = i64
        L.or_tiles_x.argtypes = [vp]
        L.or_tiles_y.argtypes = [vp]
        L.or_get_gaussian_records.argtypes = [vp, vp, vp, vp, vp, vp]
        L.or_get_triangle_records.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.or_get_bins.argtypes = [vp, vp, vp, vp]
        L.or_coverage_mask.argtypes = [vp, i32, i32]
        L.or_coverage_mask.restype = C.c_uint32
        L.or_coverage_mask_m.argtypes = [vp, i32, i32, i32]
        L.or_coverage_mask_m.restype = C.c_uint32
        L.or_render_supersampled.argtypes = [vp, vp, i32, i32]
        L.or_render_supersampled.restype = i32
        L.or_sh_basis_colour.argtypes = [vp, i32, vp, vp]
        L.or_set_cov3d.argtypes = [vp, vp]
        L.or_set_cov3d.restype = None
        L.or_deform.argtypes = [vp, i32, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp]
        L.or_deform.restype = i32
        L.or_rodrigues_public.argtypes = [vp, vp]
        L.or_rodrigues_public.restype = None
        L.or_tri_tile_depth.argtypes = [vp, i64, i32, i32]
        L.or_tri_tile_depth.restype = C.c_float
        L.or_tri_pixel_depth.argtypes = [vp, i64, i32, i32]
        L.or_tri_pixel_depth.restype = C.c_float
        L.or_ray_cast.argtypes = [vp, vp, i64, vp, i64, vp, vp, vp, vp]
        L.or_ray_cast.restype = i64
        L.or_bind_targets.argtypes = [vp, vp, vp, i32, C.c_float, vp]
        L.or_bind_targets.restype = None
        L.or_bind.argtypes = [i64, vp, vp, vp, i64, vp, i64, vp, i32, vp, i32, C.c_float, vp, vp, vp, i32]
        L.or_bind.restype = i32
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def make_settings(alpha_max=0.99, t_eps=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), bg_alpha=1.0, blend_mode=EXACT,
                  msaa=4, tri_depth=0, resort_window=4) -> CSettings:
    """tri_depth: 0 = centroid sort depth (R9), 1 = plane depth at the tile centre (N8), 2 = N8 keys and a
    per-pixel resort window of resort_window fragments over the depth at the pixel (N9)."""
    s = CSettings()
    s.alpha_max, s.t_eps, s.dilation, s.bg_alpha = alpha_max, t_eps, dilation, bg_alpha
    s.blend_mode, s.msaa, s.tri_depth, s.resort_window = blend_mode, msaa, tri_depth, resort_window
    for i in range(3):
        s.bg[i] = float(bg[i])
    return s


def make_camera(cam) -> CCamera:
    c = CCamera()
    c.width, c.height = cam.width, cam.height
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    R = np.asarray(cam.R, np.float32).ravel()
    t = np.asarray(cam.t, np.float32).ravel()
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(t[i])
    c.near_z, c.far_z = cam.near, cam.far
    return c


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dt)


class Oracle:
    """One scene, one view at a time.  Arrays are float32/int32/uint8 numpy, borrowed."""

    def __init__(self, gaussians, mesh, threads: int = 0):
        self.threads = threads
        L = lib()
        self._h = L.or_create()
        g, m = gaussians, mesh
        self._keep = [
            _c(g.means, np.float32), _c(g.quats, np.float32), _c(g.scales, np.float32),
            _c(g.opacities, np.float32), _c(g.sh, np.float32),
            _c(m.positions, np.float32), _c(m.uvs, np.float32), _c(m.colors, np.float32),
            _c(m.faces, np.int32), _c(m.opacity, np.float32), _c(m.texture, np.uint8)]
        k = self._keep
        tex = m.texture
        self.N, self.F = int(g.means.shape[0]), int(m.faces.shape[0])
        L.or_set_scene(self._h, self.N, _ptr(k[0]), _ptr(k[1]), _ptr(k[2]), _ptr(k[3]), _ptr(k[4]),
                       int(g.sh_degree), int(m.positions.shape[0]), self.F, _ptr(k[5]), _ptr(k[6]),
                       _ptr(k[7]), _ptr(k[8]), _ptr(k[9]), _ptr(k[10]),
                       0 if tex is None else int(tex.shape[1]), 0 if tex is None else int(tex.shape[0]))
        self.cam = None
        cov = getattr(g, "cov3d", None)
        if cov is not None:
            self._cov = np.ascontiguousarray(cov, np.float32)
            L.or_set_cov3d(self._h, _ptr(self._cov))

    def deform(self, binding, field, faces):
        """Eq.12-13: deformed (means [N,3], covariances [N,6] xx xy xz yy yz zz) in float64.
        V = number of per-vertex field rows; faces with a vertex id outside [0, V) are skipped."""
        face = np.ascontiguousarray(binding.face, np.int32)
        bary = np.ascontiguousarray(binding.bary, np.float32)
        fc = np.ascontiguousarray(faces, np.int32)
        d = np.ascontiguousarray(field.delta, np.float32)
        lr = np.ascontiguousarray(field.log_rot, np.float32)
        sh = np.ascontiguousarray(field.shear, np.float32)
        mu = np.zeros((self.N, 3), np.float64)
        cv = np.zeros((self.N, 6), np.float64)
        K = int(face.shape[1])
        if lib().or_deform(self._h, K, _ptr(face), _ptr(bary), _ptr(fc), int(fc.shape[0]), int(d.shape[0]),
                           _ptr(d), _ptr(lr),
                           _ptr(sh), _ptr(mu), _ptr(cv)):
            raise ValueError("anchors per Gaussian must be 1..8")
        return mu, cv

    def __del__(self):
        try:
            lib().or_destroy(self._h)
        except Exception:
            pass

    # -- stages --------------------------------------------------------------
    def project(self, cam, **settings):
        self.cam = cam
        self._cs = make_settings(**settings)
        self._cc = make_camera(cam)
        rc = lib().or_project(self._h, C.byref(self._cc), C.byref(self._cs), self.threads)
        if rc:
            raise MemoryError("oracle projection allocation failed")
        self.tiles_x = lib().or_tiles_x(self._h)
        self.tiles_y = lib().or_tiles_y(self._h)
        return self

    def bin(self) -> int:
        K = lib().or_bin(self._h)
        if K < 0:
            raise MemoryError("oracle binning allocation failed")
        self.K = int(K)
        return self.K

    def gaussian_records(self):
        N = self.N
        out = dict(rec=np.zeros((N, 8), np.float32), cov=np.zeros((N, 3), np.float32),
                   rgb=np.zeros((N, 3), np.float64), rect=np.zeros((N, 4), np.int32),
                   touched=np.zeros(N, np.uint32))
        lib().or_get_gaussian_records(self._h, _ptr(out["rec"]), _ptr(out["cov"]), _ptr(out["rgb"]),
                                      _ptr(out["rect"]), _ptr(out["touched"]))
        return out

    def triangle_records(self):
        F = self.F
        out = dict(xy=np.zeros((F, 6), np.int32), vid=np.zeros((F, 3), np.int32), z=np.zeros((F, 3), np.float32),
                   depth=np.zeros(F, np.float32), rect=np.zeros((F, 4), np.int32), touched=np.zeros(F, np.uint32))
        lib().or_get_triangle_records(self._h, _ptr(out["xy"]), _ptr(out["vid"]), _ptr(out["z"]),
                                      _ptr(out["depth"]), _ptr(out["rect"]), _ptr(out["touched"]))
        return out

    def tri_tile_depth(self, f: int, tx: int, ty: int) -> np.float32:
        """N8: sort depth of triangle f in tile (tx, ty) (after project())."""
        return np.float32(lib().or_tri_tile_depth(self._h, int(f), int(tx), int(ty)))

    def tri_pixel_depth(self, f: int, x: int, y: int) -> np.float32:
        """N9: triangle f's plane depth at the centre of pixel (x, y), clamped (after project())."""
        return np.float32(lib().or_tri_pixel_depth(self._h, int(f), int(x), int(y)))

    def bins(self):
        keys = np.zeros(self.K, np.uint64)
        vals = np.zeros(self.K, np.uint32)
        ranges = np.zeros((self.tiles_x * self.tiles_y, 2), np.uint32)
        lib().or_get_bins(self._h, _ptr(keys), _ptr(vals), _ptr(ranges))
        return keys, vals, ranges

    def render(self, tiles: Optional[Sequence[int]] = None) -> np.ndarray:
        """Tiled oracle render; pixels of tiles not listed stay NaN."""
        H, W = self.cam.height, self.cam.width
        out = np.full((H, W, 4), np.nan, np.float64)
        tl = None if tiles is None else np.ascontiguousarray(tiles, np.int32)
        rc = lib().or_render(self._h, _ptr(out), _ptr(tl), 0 if tl is None else len(tl), self.threads)
        if rc:
            raise RuntimeError("oracle render before bin()")
        return out

    def fragment_counts(self, tiles: Optional[Sequence[int]] = None) -> np.ndarray:
        """Per pixel [H, W, 4] uint32: Gaussian fragments blended, triangle fragments blended,
        id of the last fragment blended (0xFFFFFFFF none), 0 -- over the listed tiles (others 0)."""
        H, W = self.cam.height, self.cam.width
        out = np.zeros((H, W, 4), np.uint32)
        tl = None if tiles is None else np.ascontiguousarray(tiles, np.int32)
        if lib().or_render_counts(self._h, _ptr(out), _ptr(tl), 0 if tl is None else len(tl), self.threads):
            raise RuntimeError("oracle counts before bin()")
        return out

    def render_bruteforce(self) -> np.ndarray:
        H, W = self.cam.height, self.cam.width
        out = np.zeros((H, W, 4), np.float64)
        lib().or_render_bruteforce(self._h, _ptr(out), self.threads)
        return out

    def pixel_fragments(self, x: int, y: int) -> np.ndarray:
        cap = 256
        while True:
            buf = np.zeros(cap, FRAG_DTYPE)
            n = lib().or_pixel_fragments(self._h, x, y, _ptr(buf), cap)
            if n <= cap:
                return buf[:n]
            cap = int(n)

    def render_supersampled(self, S: int = 16) -> np.ndarray:
        """Ground truth: mean of S x S sub-samples of exact per-sample ordered blending."""
        H, W = self.cam.height, self.cam.width
        out = np.zeros((H, W, 4), np.float64)
        if lib().or_render_supersampled(self._h, _ptr(out), S, self.threads):
            raise RuntimeError("supersampled render needs project() and 256 % S == 0")
        return out

    def support_truncation(self) -> int:
        return int(lib().or_support_truncation(self._h))

    def full(self, cam, **settings):
        """project + bin + render: the whole oracle path for one view."""
        self.project(cam, **settings)
        self.bin()
        return self.render()


def blend_fragments(frags: np.ndarray, **settings):
    """Run the unified state machine on an explicit ordered fragment list."""
    frags = np.ascontiguousarray(frags, FRAG_DTYPE)
    s = make_settings(**settings)
    out = np.zeros(4, np.float64)
    trace = np.zeros(max(len(frags), 1), np.float64)
    used = lib().or_blend_fragments(_ptr(frags), len(frags), C.byref(s), _ptr(out), _ptr(trace))
    return out, trace[:used]


def frags(*items) -> np.ndarray:
    """Build a fragment array: items are dicts with kind ('g'|'t'), alpha, rgb, mask, depth, id."""
    a = np.zeros(len(items), FRAG_DTYPE)
    for i, it in enumerate(items):
        a[i]["id"] = it.get("id", i)
        a[i]["kind"] = 0 if it["kind"] == "g" else 1
        a[i]["mask"] = it.get("mask", 0)
        a[i]["alpha"] = it["alpha"]
        a[i]["rgb"] = it["rgb"]
        a[i]["depth"] = it.get("depth", float(i + 1))
    return a


def coverage_mask(xy6, x: int, y: int) -> int:
    xy = np.ascontiguousarray(xy6, np.int32)
    return int(lib().or_coverage_mask(_ptr(xy), x, y))


def rodrigues(w) -> np.ndarray:
    R = np.zeros(9, np.float64)
    w = np.ascontiguousarray(w, np.float64)  # keep the array alive across the call
    lib().or_rodrigues_public(_ptr(w), _ptr(R))
    return R.reshape(3, 3)


def coverage_mask_m(xy6, x: int, y: int, M: int) -> int:
    xy = np.ascontiguousarray(xy6, np.int32)
    return int(lib().or_coverage_mask_m(_ptr(xy), x, y, M))


def sh_colour(coef: np.ndarray, degree: int, direction) -> np.ndarray:
    coef = np.ascontiguousarray(coef, np.float32)
    d = np.ascontiguousarray(direction, np.float64)
    out = np.zeros(3, np.float64)
    lib().or_sh_basis_colour(_ptr(coef), degree, _ptr(d), _ptr(out))
    return out


def scene_settings(scene, **over):
    """Default render settings for a synthetic scene (bg from the scene)."""
    s = dict(alpha_max=0.99, t_eps=1e-4, dilation=0.3, bg=tuple(float(v) for v in scene.bg),
             bg_alpha=float(scene.bg_alpha))
    s.update(over)
    return s


# ---------------------------------------------------------------------------
# Gaussian-centric ray-cast binding (oracle/bind_oracle.c, readings B1-B6)
# ---------------------------------------------------------------------------

def ray_cast(origin, direction, positions, faces):
    """Nearest hit of one ray over all faces: (face or -1, t, u, v)."""
    o = np.ascontiguousarray(origin, np.float64)
    d = np.ascontiguousarray(direction, np.float64)
    P = np.ascontiguousarray(positions, np.float32)
    Fc = np.ascontiguousarray(faces, np.int32)
    t, u, v = C.c_double(), C.c_double(), C.c_double()
    f = lib().or_ray_cast(_ptr(o), _ptr(d), len(P), _ptr(P), len(Fc), _ptr(Fc), C.byref(t), C.byref(u), C.byref(v))
    return int(f), t.value, u.value, v.value


def bind_targets(mean, quat, scale, mode: int, k_sigma: float = 3.0) -> np.ndarray:
    out = np.zeros((8, 3), np.float64)
    m = np.ascontiguousarray(mean, np.float32)
    q = np.ascontiguousarray(quat, np.float32)
    s = np.ascontiguousarray(scale, np.float32)
    lib().or_bind_targets(_ptr(m), _ptr(q), _ptr(s), mode, float(k_sigma), _ptr(out))
    return out[:1] if mode == 0 else out


def camera_array(cams) -> np.ndarray:
    """[C, 12] float32: R (row-major, world->camera) then t."""
    return np.ascontiguousarray(np.stack([np.concatenate([np.asarray(c.R, np.float32).ravel(),
                                                          np.asarray(c.t, np.float32).ravel()]) for c in cams]),
                                np.float32)


def bind(gaussians, positions, faces, cams, mode: int = 1, k_sigma: float = 3.0, threads: int = 0):
    """Exhaustive binding table: face [N, K] int32 (-1 = no hit), bary [N, K, 3] float64,
    squared hit distance to the centre [N, K] (-1 = no hit); K = 1 (centre) or 8 (bbx8)."""
    N = gaussians.count
    K = 1 if mode == 0 else 8
    mu = np.ascontiguousarray(gaussians.means, np.float32)
    q = np.ascontiguousarray(gaussians.quats, np.float32)
    s = np.ascontiguousarray(gaussians.scales, np.float32)
    P = np.ascontiguousarray(positions, np.float32)
    Fc = np.ascontiguousarray(faces, np.int32)
    ca = camera_array(cams)
    face = np.zeros((N, K), np.int32)
    bary = np.zeros((N, K, 3), np.float64)
    d2 = np.zeros((N, K), np.float64)
    rc = lib().or_bind(N, _ptr(mu), _ptr(q), _ptr(s), len(P), _ptr(P), len(Fc), _ptr(Fc), len(ca), _ptr(ca), mode,
                       float(k_sigma), _ptr(face), _ptr(bary), _ptr(d2), threads)
    if rc:
        raise ValueError("bind: need >= 1 camera and mode 0 or 1")
    return face, bary, d2
