"""Seeded synthetic scene generators (SURVEY.md §8(d) recipes).

This module is shared by the CUDA path (tests, bench, smoke) and by the CPU
oracle's tests.  It holds NONE of the method's arithmetic: it only draws
Gaussians, builds UV-sphere / torus meshes with procedural textures and places
OpenCV look-at cameras.  Everything is float32 / int32 / uint8 numpy, generated
from ``numpy.random.default_rng(seed)``, so both sides read identical bytes.

Shapes follow the paper's workloads (§4 / Table 1 scale, P:485, P:536,
P:507-515):

  tiny      64 G + 2-triangle opaque quad, 64x64              (seed 1)
  nerf      300k G + 10k-triangle textured sphere, 800x800    (seed 2)
  mip360    3M G + 200k-triangle sphere+torus, 1920x1080      (seed 3)
  stress    3M G + 998,784 semi-transparent nested spheres    (seed 4)
  multiview mip360 scene + 256 orbit cameras at 1080p         (seed 5)
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

SH_C0 = 0.28209479177387814  # only used to map a target DC colour to a coefficient

CONFIGS = ("tiny", "nerf", "mip360", "stress", "multiview")


@dataclass
class Camera:
    """Pinhole camera, OpenCV convention (+z forward, y down), world->camera."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray  # float32 [3,3] row-major world->camera
    t: np.ndarray  # float32 [3]
    near: float = 0.2
    far: float = 1000.0

    def campos(self) -> np.ndarray:
        return (-(self.R.astype(np.float64).T @ self.t.astype(np.float64))).astype(np.float32)


@dataclass
class Gaussians:
    means: np.ndarray      # f32 [N,3]
    quats: np.ndarray      # f32 [N,4] (w,x,y,z), not necessarily normalised
    scales: np.ndarray     # f32 [N,3] linear
    opacities: np.ndarray  # f32 [N] in [0,1]
    sh: np.ndarray         # f32 [N,(D+1)^2,3]
    sh_degree: int

    @property
    def count(self) -> int:
        return int(self.means.shape[0])


@dataclass
class Mesh:
    positions: np.ndarray             # f32 [V,3]
    faces: np.ndarray                 # i32 [F,3]
    opacity: np.ndarray               # f32 [F] in [0,1]
    uvs: Optional[np.ndarray] = None  # f32 [V,2]
    colors: Optional[np.ndarray] = None  # f32 [V,3]
    texture: Optional[np.ndarray] = None  # u8 [Ht,Wt,4]

    @property
    def num_vertices(self) -> int:
        return int(self.positions.shape[0])

    @property
    def num_triangles(self) -> int:
        return int(self.faces.shape[0])


@dataclass
class Scene:
    name: str
    gaussians: Gaussians
    mesh: Mesh
    cameras: List[Camera]
    bg: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))
    bg_alpha: float = 1.0


# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------

def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), *, width, height, fx, fy,
            cx, cy, near=0.2, far=1000.0) -> Camera:
    """OpenCV look-at: rows of R are (right, down, forward)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ eye
    return Camera(int(width), int(height), float(fx), float(fy), float(cx), float(cy),
                  R.astype(np.float32), t.astype(np.float32), float(near), float(far))


def empty_mesh() -> Mesh:
    return Mesh(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.int32),
                np.zeros((0,), np.float32))


def empty_gaussians(sh_degree: int = 0) -> Gaussians:
    k = (sh_degree + 1) ** 2
    return Gaussians(np.zeros((0, 3), np.float32), np.zeros((0, 4), np.float32),
                     np.zeros((0, 3), np.float32), np.zeros((0,), np.float32),
                     np.zeros((0, k, 3), np.float32), sh_degree)


def _unit_vectors(rng, n):
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _quats(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _opacities(rng, n):
    hi = rng.uniform(0.6, 1.0, n)
    lo = rng.uniform(0.02, 0.4, n)
    return np.where(rng.uniform(0, 1, n) < 0.7, hi, lo)


def _sh(rng, n, degree):
    k = (degree + 1) ** 2
    sh = np.empty((n, k, 3), np.float32)
    c = rng.uniform(0.15, 0.85, (n, 3))
    sh[:, 0, :] = ((c - 0.5) / SH_C0).astype(np.float32)
    if k > 1:
        sh[:, 1:, :] = rng.standard_normal((n, k - 1, 3), dtype=np.float32) * np.float32(0.03)
    return sh


def _lognormal_scales(rng, n, median, sigma_ln):
    median = np.broadcast_to(np.asarray(median, np.float64), (n,))
    s = np.exp(np.log(median)[:, None] + sigma_ln * rng.standard_normal((n, 3)))
    s[:, 2] *= 0.3  # trained splats are mostly flat
    return s


def _shell_points(rng, n, base_r):
    d = _unit_vectors(rng, n)
    theta = np.arccos(np.clip(d[:, 1], -1, 1))
    phi = np.arctan2(d[:, 2], d[:, 0])
    r = base_r * (1.0 + 0.2 * np.sin(3 * theta) * np.cos(2 * phi)) + rng.normal(0, 0.02, n)
    return d * r[:, None]


def _pack_gaussians(means, quats, scales, opac, sh, degree) -> Gaussians:
    return Gaussians(np.ascontiguousarray(means, np.float32), np.ascontiguousarray(quats, np.float32),
                     np.ascontiguousarray(scales, np.float32), np.ascontiguousarray(opac, np.float32),
                     np.ascontiguousarray(sh, np.float32), degree)


def procedural_texture(rng, size=1024, checks=16) -> np.ndarray:
    """Checker + value noise RGBA8 texture."""
    g = rng.uniform(0, 1, (33, 33, 3))
    xs = np.linspace(0, 32, size, endpoint=False)
    i0 = np.floor(xs).astype(np.int64)
    f = (xs - i0)[:, None]
    # separable bilinear upsample of the value-noise lattice
    rows = g[i0] * (1 - f)[:, :, None] + g[i0 + 1] * f[:, :, None]          # [size,33,3]
    noise = rows[:, i0] * (1 - f.T)[:, :, None] + rows[:, i0 + 1] * f.T[:, :, None]
    cell = (np.arange(size) * checks // size)
    checker = ((cell[:, None] + cell[None, :]) % 2).astype(np.float64)
    base = np.where(checker[:, :, None] > 0, np.array([0.85, 0.75, 0.35]), np.array([0.2, 0.35, 0.7]))
    rgb = np.clip(0.65 * base + 0.35 * noise, 0, 1)
    tex = np.empty((size, size, 4), np.uint8)
    tex[:, :, :3] = np.round(rgb * 255).astype(np.uint8)
    tex[:, :, 3] = 255
    return tex


def uv_sphere(center, r, n_lon, n_lat):
    """Grid sphere with duplicated seam column and kept pole rows (degenerate triangles)."""
    th = np.linspace(0, np.pi, n_lat + 1)
    ph = np.linspace(0, 2 * np.pi, n_lon + 1)
    T, P = np.meshgrid(th, ph, indexing="ij")
    pos = np.stack([np.sin(T) * np.cos(P), np.cos(T), np.sin(T) * np.sin(P)], -1) * r
    pos = pos.reshape(-1, 3) + np.asarray(center, np.float64)
    uv = np.stack(np.meshgrid(np.arange(n_lat + 1) / n_lat, np.arange(n_lon + 1) / n_lon,
                              indexing="ij")[::-1], -1).reshape(-1, 2)
    faces = _grid_faces(n_lat, n_lon)
    return pos, uv, faces


def torus(center, R, r, n_u, n_v):
    u = np.linspace(0, 2 * np.pi, n_u + 1)
    v = np.linspace(0, 2 * np.pi, n_v + 1)
    V, U = np.meshgrid(v, u, indexing="ij")
    pos = np.stack([(R + r * np.cos(V)) * np.cos(U), r * np.sin(V), (R + r * np.cos(V)) * np.sin(U)], -1)
    pos = pos.reshape(-1, 3) + np.asarray(center, np.float64)
    uv = np.stack(np.meshgrid(np.arange(n_v + 1) / n_v, np.arange(n_u + 1) / n_u,
                              indexing="ij")[::-1], -1).reshape(-1, 2)
    return pos, uv, _grid_faces(n_v, n_u)


def _grid_faces(rows, cols):
    i, j = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    a = (i * (cols + 1) + j).ravel()
    b = a + 1
    c = a + (cols + 1)
    d = c + 1
    f = np.empty((rows * cols * 2, 3), np.int64)
    f[0::2] = np.stack([a, c, b], -1)
    f[1::2] = np.stack([b, c, d], -1)
    return f


def merge_meshes(parts, texture) -> Mesh:
    pos, uv, faces, opac = [], [], [], []
    base = 0
    for (p, u, f, alpha) in parts:
        pos.append(p)
        uv.append(u)
        faces.append(f + base)
        opac.append(np.full(len(f), alpha))
        base += len(p)
    return Mesh(np.concatenate(pos).astype(np.float32), np.concatenate(faces).astype(np.int32),
                np.concatenate(opac).astype(np.float32), uvs=np.concatenate(uv).astype(np.float32),
                texture=texture)


# ----------------------------------------------------------------------------
# the five configs
# ----------------------------------------------------------------------------

def make_tiny(seed=1) -> Scene:
    rng = np.random.default_rng(seed)
    n = 64
    means = rng.normal((0.0, 0.0, 3.0), 0.25, (n, 3))
    scales = rng.uniform(0.03, 0.12, (n, 3))
    opac = rng.uniform(0.2, 0.99, n)
    g = _pack_gaussians(means, _quats(rng, n), scales, opac, _sh(rng, n, 0), 0)
    ang = np.deg2rad(20.0)
    c, s = np.cos(ang), np.sin(ang)
    corners = np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], np.float64) * 0.35
    xy = corners @ np.array([[c, s], [-s, c]])
    pos = np.concatenate([xy, np.full((4, 1), 3.0)], 1)
    uv = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], np.float64)
    faces = np.array([[0, 1, 2], [0, 2, 3]])
    cell = np.arange(8)
    chk = ((cell[:, None] + cell[None, :]) % 2).astype(bool)
    tex = np.empty((8, 8, 4), np.uint8)
    tex[chk] = (230, 230, 230, 255)
    tex[~chk] = (30, 60, 200, 255)
    mesh = merge_meshes([(pos, uv, faces, 1.0)], tex)
    cam = Camera(64, 64, 64.0, 64.0, 32.0, 32.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    return Scene("tiny", g, mesh, [cam], bg=np.array([0.1, 0.2, 0.3], np.float32))


def make_nerf(seed=2, n=300_000) -> Scene:
    rng = np.random.default_rng(seed)
    n_shell = int(n * 0.8)
    means = np.concatenate([_shell_points(rng, n_shell, 0.9),
                            rng.uniform(-0.7, 0.7, (n - n_shell, 3))])
    scales = _lognormal_scales(rng, n, 0.006, 0.5)
    g = _pack_gaussians(means, _quats(rng, n), scales, _opacities(rng, n), _sh(rng, n, 3), 3)
    tex = procedural_texture(rng)
    mesh = merge_meshes([uv_sphere((0, 0, 0.9), 0.4, 100, 50) + (1.0,)], tex)
    cam = look_at((0.0, 2.0, 3.46), width=800, height=800, fx=1111.11, fy=1111.11, cx=400, cy=400)
    return Scene("nerf", g, mesh, [cam], bg=np.ones(3, np.float32))


def _mip360_gaussians(rng, n):
    n_obj = int(n * 0.4)
    n_gnd = int(n * 0.3)
    n_far = n - n_obj - n_gnd
    obj = _shell_points(rng, n_obj, 1.0)
    rad = 15.0 * np.sqrt(rng.uniform(0, 1, n_gnd)) + 0.5
    ang = rng.uniform(0, 2 * np.pi, n_gnd)
    gnd = np.stack([rad * np.cos(ang), -1.0 + rng.uniform(-0.05, 0.05, n_gnd), rad * np.sin(ang)], -1)
    d = _unit_vectors(rng, n_far)
    d[:, 1] = np.abs(d[:, 1])
    far = d * rng.uniform(8, 30, n_far)[:, None]
    means = np.concatenate([obj, gnd, far])
    med = 0.004 * np.maximum(np.linalg.norm(means, axis=1), 1.0)
    scales = _lognormal_scales(rng, n, med, 0.6)
    return _pack_gaussians(means, _quats(rng, n), scales, _opacities(rng, n), _sh(rng, n, 3), 3)


def _hd_camera(eye):
    return look_at(eye, width=1920, height=1080, fx=1662.8, fy=1662.8, cx=960, cy=540)


def make_mip360(seed=3, n=3_000_000) -> Scene:
    rng = np.random.default_rng(seed)
    g = _mip360_gaussians(rng, n)
    tex = procedural_texture(rng)
    mesh = merge_meshes([uv_sphere((0.9, -0.3, 0.6), 0.45, 250, 200) + (1.0,),
                         torus((-0.7, -0.5, 0.3), 0.5, 0.12, 250, 200) + (1.0,)], tex)
    return Scene("mip360", g, mesh, [_hd_camera((0.0, 0.78, 2.9))], bg=np.zeros(3, np.float32))


def make_stress(seed=4, n=3_000_000) -> Scene:
    rng = np.random.default_rng(seed)
    g = _mip360_gaussians(rng, n)
    tex = procedural_texture(rng)
    mesh = merge_meshes([uv_sphere((0, 0, 0), r, 408, 408) + (a,)
                         for r, a in ((0.6, 0.35), (0.9, 0.5), (1.2, 0.65))], tex)
    return Scene("stress", g, mesh, [_hd_camera((0.0, 0.78, 2.9))], bg=np.zeros(3, np.float32))


def orbit_cameras(n_views=256, r=3.0):
    cams = []
    for i in range(n_views):
        phi = 2 * np.pi * i / n_views
        el = np.deg2rad(15.0 + 10.0 * np.sin(4 * np.pi * i / n_views))
        eye = (r * np.cos(el) * np.sin(phi), r * np.sin(el), r * np.cos(el) * np.cos(phi))
        cams.append(_hd_camera(eye))
    return cams


def make_multiview(seed=5, n=3_000_000, n_views=256) -> Scene:
    del seed  # cameras are a deterministic orbit; the scene is mip360 seed 3
    sc = make_mip360(3, n)
    sc.name = "multiview"
    sc.cameras = orbit_cameras(n_views)
    return sc


def make_scene(name: str, **kw) -> Scene:
    return {"tiny": make_tiny, "nerf": make_nerf, "mip360": make_mip360,
            "stress": make_stress, "multiview": make_multiview}[name](**kw)


def subsample(scene: Scene, n_gauss: int, seed: int = 0) -> Scene:
    """Keep the first n_gauss Gaussians (the shells are drawn in random order)."""
    g = scene.gaussians
    k = min(n_gauss, g.count)
    g2 = Gaussians(g.means[:k], g.quats[:k], g.scales[:k], g.opacities[:k], g.sh[:k], g.sh_degree)
    return Scene(scene.name + f"-sub{k}", g2, scene.mesh, scene.cameras, scene.bg, scene.bg_alpha)


# ----------------------------------------------------------------------------
# small constructions for tests (SPEC testscenes S:542-584 analogues)
# ----------------------------------------------------------------------------

def _plain_camera(W, H, f=None, cx=None, cy=None):
    f = float(W) if f is None else f
    return Camera(W, H, f, f, W / 2 + 0.173 if cx is None else cx, H / 2 - 0.291 if cy is None else cy,
                  np.eye(3, dtype=np.float32), np.zeros(3, np.float32))


def make_random(seed=0, n_gauss=400, n_tris=60, W=96, H=80, textured=True, sh_degree=3,
                opaque_frac=0.3, quads=4) -> Scene:
    """Random splats + random (partly semi-transparent) triangles in front of an identity camera."""
    rng = np.random.default_rng(seed)
    cam = _plain_camera(W, H)
    z = rng.uniform(2.0, 6.0, n_gauss)
    x = rng.uniform(-0.55, 0.55, n_gauss) * z * W / cam.fx
    y = rng.uniform(-0.55, 0.55, n_gauss) * z * H / cam.fy
    means = np.stack([x, y, z], -1)
    scales = _lognormal_scales(rng, n_gauss, 0.06, 0.7)
    g = _pack_gaussians(means, _quats(rng, n_gauss), scales, _opacities(rng, n_gauss),
                        _sh(rng, n_gauss, sh_degree), sh_degree)
    pos, faces, uv, col, op = [], [], [], [], []
    for k in range(n_tris):
        cz = rng.uniform(1.5, 7.0)
        c = np.array([rng.uniform(-0.6, 0.6) * cz * W / cam.fx, rng.uniform(-0.6, 0.6) * cz * H / cam.fy, cz])
        v = c + rng.normal(0, 0.25 * cz / 3, (3, 3))
        if k % 17 == 5:      # crosses the near plane -> culled
            v[0, 2] = 0.1
        base = len(pos) * 3
        pos.append(v)
        faces.append([base, base + 1, base + 2] if rng.uniform() < 0.5 else [base, base + 2, base + 1])
        uv.append(rng.uniform(0, 1, (3, 2)))
        col.append(rng.uniform(0, 1, (3, 3)))
        op.append(1.0 if rng.uniform() < opaque_frac else rng.uniform(0.2, 0.95))
    P = np.concatenate(pos).reshape(-1, 3) if pos else np.zeros((0, 3))
    Fc = np.asarray(faces, np.int64).reshape(-1, 3)
    UV = np.concatenate(uv).reshape(-1, 2) if uv else np.zeros((0, 2))
    COL = np.concatenate(col).reshape(-1, 3) if col else np.zeros((0, 3))
    OP = np.asarray(op, np.float64)
    # a few quads (shared diagonal) to exercise watertight edges
    for _ in range(quads):
        cz = rng.uniform(2.0, 6.0)
        c = np.array([rng.uniform(-0.4, 0.4) * cz * W / cam.fx, rng.uniform(-0.4, 0.4) * cz * H / cam.fy, cz])
        hw = rng.uniform(0.1, 0.4) * cz / 3
        qv = c + np.array([[-hw, -hw, 0], [hw, -hw, 0.05], [hw, hw, 0.1], [-hw, hw, 0.05]])
        b = len(P)
        P = np.concatenate([P, qv])
        UV = np.concatenate([UV, [[0, 0], [1, 0], [1, 1], [0, 1]]])
        COL = np.concatenate([COL, rng.uniform(0, 1, (4, 3))])
        Fc = np.concatenate([Fc, [[b, b + 1, b + 2], [b, b + 2, b + 3]]])
        a = 1.0 if rng.uniform() < 0.5 else rng.uniform(0.3, 0.9)
        OP = np.concatenate([OP, [a, a]])
    mesh = Mesh(P.astype(np.float32), Fc.astype(np.int32), OP.astype(np.float32),
                uvs=UV.astype(np.float32) if textured else None,
                colors=None if textured else COL.astype(np.float32),
                texture=procedural_texture(rng, 64, 4) if textured else None)
    return Scene(f"random{seed}", g, mesh, [cam], bg=rng.uniform(0, 1, 3).astype(np.float32))


def make_overflow(W=64, H=64) -> Scene:
    """Fig.3 construction: near triangle covering the left half of the
    centre pixel, an interposed Gaussian, and a far full-screen white triangle pair."""
    cam = Camera(W, H, 1.0, 1.0, 0.0, 0.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    # fx = 1, z = 1 maps world x (in px) to screen x exactly; the near triangle edge runs
    # vertically through x = 32.5 (pixel 32 centre): samples with ox < 0 are covered.
    z1, z3 = 1.0, 1.0
    near = np.array([[20.0, 10.0, z1], [32.5, 10.0, z1], [32.5, 54.0, z1]]) * [1, 1, 1]
    # put the far quad at z = 3 with fx=1 scaling: world = screen * z
    far = np.array([[-1, -1], [W + 1, -1], [W + 1, H + 1], [-1, H + 1]], np.float64) * z3
    far = np.concatenate([far * 3.0 / z3, np.full((4, 1), 3.0)], 1)
    P = np.concatenate([near, far])
    faces = np.array([[0, 1, 2], [3, 4, 5], [3, 5, 6]])
    colors = np.array([[1, 0, 0]] * 3 + [[1, 1, 1]] * 4, np.float64)
    mesh = Mesh(P.astype(np.float32), faces.astype(np.int32), np.array([1, 1, 1], np.float32),
                colors=colors.astype(np.float32))
    # one large blue Gaussian at depth 2 centred on pixel (32, 32)
    sh = np.zeros((1, 1, 3), np.float32)
    sh[0, 0] = ((np.array([0.0, 0.0, 1.0]) - 0.5) / SH_C0).astype(np.float32)
    g = Gaussians(np.array([[32.5 * 2.0, 32.5 * 2.0, 2.0]], np.float32), np.array([[1, 0, 0, 0]], np.float32),
                  np.array([[20.0, 20.0, 20.0]], np.float32), np.array([0.5], np.float32), sh, 0)
    return Scene("overflow", g, mesh, [cam], bg=np.zeros(3, np.float32))


def make_nested(seed=7, W=128, H=128) -> Scene:
    """Splat cluster inside a semi-transparent closed sphere (P:511-515 lego-in-bowl analogue)."""
    rng = np.random.default_rng(seed)
    n = 300
    means = rng.normal(0, 0.25, (n, 3)) + [0, 0, 4.0]
    scales = _lognormal_scales(rng, n, 0.08, 0.3)
    g = _pack_gaussians(means, _quats(rng, n), scales, _opacities(rng, n), _sh(rng, n, 1), 1)
    p, uv, f = uv_sphere((0, 0, 4.0), 0.9, 24, 12)
    mesh = merge_meshes([(p, uv, f, 0.4)], procedural_texture(rng, 64, 8))
    return Scene("nested", g, mesh, [_plain_camera(W, H)], bg=np.array([0.05, 0.05, 0.05], np.float32))


def make_edge(W=64, H=64) -> Scene:
    """Thin triangles at sub-pixel slopes (S:567 edge scene)."""
    cam = Camera(W, H, 1.0, 1.0, 0.0, 0.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    tris = []
    for k in range(6):
        y0 = 6 + 9 * k
        slope = 0.07 * (k + 1)
        tris.append([[2.0, y0, 2.0], [62.0, y0 + 60 * slope, 2.0], [2.0, y0 + 0.6 + 0.4 * k, 2.0]])
    P = (np.array(tris, np.float64).reshape(-1, 3) * [2.0, 2.0, 1.0])
    faces = np.arange(len(P)).reshape(-1, 3)
    colors = np.tile(np.array([[1.0, 0.9, 0.2]]), (len(P), 1))
    mesh = Mesh(P.astype(np.float32), faces.astype(np.int32), np.ones(len(faces), np.float32),
                colors=colors.astype(np.float32))
    return Scene("edge", empty_gaussians(0), mesh, [cam], bg=np.array([0.0, 0.0, 0.3], np.float32))


def make_crossing(W=128, H=96, n_gauss=0, alpha=1.0, seed=11) -> Scene:
    """Two interpenetrating tilted quads (SURVEY §8(f) row 3, P:511-515 nested
    relations): quad A (red) recedes from left to right, quad B (green) the
    other way, so each is in front on one side of the crossing column x = W/2.
    1/z is affine in screen space on each (planar) quad: 1/z_A = 0.5 - u/(2W)
    ... (z from 2 to 4), B mirrored.  Optional random Gaussians in the frustum."""
    fx = fy = float(W)
    cam = Camera(W, H, fx, fy, W / 2.0, H / 2.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    u0, u1, v0, v1 = 6.0, W - 6.0, 6.0, H - 6.0

    def world(u, v, z):
        return [(u - W / 2.0) / fx * z, (v - H / 2.0) / fy * z, z]

    def inv_z(u, left, right):  # 1/z affine in u between the quad's left and right edge depths
        t = (u - u0) / (u1 - u0)
        return (1.0 - t) / left + t / right

    P, cols = [], []
    for (zl, zr, c) in ((2.0, 4.0, (1.0, 0.1, 0.1)), (4.0, 2.0, (0.1, 1.0, 0.1))):
        for (u, v) in ((u0, v0), (u1, v0), (u1, v1), (u0, v1)):
            P.append(world(u, v, 1.0 / inv_z(u, zl, zr)))
            cols.append(c)
    faces = np.array([[0, 1, 2], [0, 2, 3], [4, 5, 6], [4, 6, 7]], np.int32)
    mesh = Mesh(np.array(P, np.float32), faces, np.full(4, alpha, np.float32), colors=np.array(cols, np.float32))
    g = empty_gaussians(0)
    if n_gauss:
        rng = np.random.default_rng(seed)
        z = rng.uniform(1.5, 5.0, n_gauss)
        uv = np.stack([rng.uniform(0, W, n_gauss), rng.uniform(0, H, n_gauss)], -1)
        means = np.stack([(uv[:, 0] - W / 2) / fx * z, (uv[:, 1] - H / 2) / fy * z, z], -1)
        q = rng.normal(size=(n_gauss, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        sh = np.zeros((n_gauss, 1, 3))
        sh[:, 0, :] = (rng.uniform(0.15, 0.85, (n_gauss, 3)) - 0.5) / 0.28209479
        g = Gaussians(means.astype(np.float32), q.astype(np.float32),
                      np.exp(rng.normal(np.log(0.03), 0.4, (n_gauss, 3))).astype(np.float32),
                      rng.uniform(0.2, 0.95, n_gauss).astype(np.float32), sh.astype(np.float32), 0)
    return Scene("crossing", g, mesh, [cam], bg=np.array([0.0, 0.0, 0.0], np.float32))


def make_degenerate(seed=13, W=96, H=80):
    """(scene_with_junk, base_scene): a valid random scene plus primitives the ABI
    promises to cull as values (include/unimgs.h; N1-N7): NaN / inf means,
    NaN and zero quaternions, inf scales, opacity 0, < 1/255 or NaN, a mean exactly
    on the near plane or behind the camera; triangles with a NaN or inf vertex, a
    vertex behind the near plane or beyond the 32768-px guard band, collinear
    vertices, and out-of-range face indices.  Junk Gaussians are appended after the
    valid ones and junk triangles after the valid triangles."""
    base = make_random(seed, n_gauss=600, n_tris=40, W=W, H=H, textured=False, sh_degree=1)
    g, m, cam = base.gaussians, base.mesh, base.cameras[0]
    nan, inf = np.float32(np.nan), np.float32(np.inf)
    R = np.asarray(cam.R, np.float64)
    t = np.asarray(cam.t, np.float64)

    def world(u, v, z):  # camera (u, v, z) -> world
        pc = np.array([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, z])
        return R.T @ (pc - t)

    ok = world(W / 2, H / 2, 3.0)
    jm, jq, js, jo = [], [], [], []

    def add(mu, q=(1, 0, 0, 0), s=(0.05, 0.05, 0.05), o=0.8):
        jm.append(mu); jq.append(q); js.append(s); jo.append(o)
    add([nan, ok[1], ok[2]])
    add([ok[0], ok[1], inf])
    add(ok, q=(nan, 0, 0, 0))
    add(ok, q=(0, 0, 0, 0))
    add(ok, s=(inf, 0.05, 0.05))
    add(ok, o=0.0)
    add(ok, o=0.99 / 255.0)
    add(ok, o=nan)
    add(world(W / 2, H / 2, cam.near * (1 - 1e-4)))        # just in front of the near plane
    add(world(W / 2, H / 2, -2.0))                         # behind the camera
    k = g.sh.shape[1]
    junk_g = Gaussians(np.asarray(jm, np.float32), np.asarray(jq, np.float32), np.asarray(js, np.float32),
                       np.asarray(jo, np.float32), np.zeros((len(jm), k, 3), np.float32), g.sh_degree)
    gall = Gaussians(np.concatenate([g.means, junk_g.means]), np.concatenate([g.quats, junk_g.quats]),
                     np.concatenate([g.scales, junk_g.scales]), np.concatenate([g.opacities, junk_g.opacities]),
                     np.concatenate([g.sh, junk_g.sh]), g.sh_degree)
    V0 = m.num_vertices
    a, b, c = world(20, 20, 2.0), world(60, 25, 2.5), world(30, 60, 2.2)
    jp = [a, b, c,                                   # reused by the index-junk faces below
          [nan, a[1], a[2]], b, c,                   # NaN vertex
          [a[0], inf, a[2]], b, c,                   # inf vertex
          world(20, 20, 0.1), b, c,                  # a vertex in front of the near plane
          world(40000, 20, 3.0), b, c,               # beyond the guard band
          world(20, 20, 2.0), world(40, 30, 2.0), world(60, 40, 2.0)]  # collinear on screen
    jp = np.asarray(jp, np.float64)
    jf = [[V0 + 3 * i, V0 + 3 * i + 1, V0 + 3 * i + 2] for i in range(1, 6)]
    jf += [[V0, V0 + 1, -1], [V0, V0 + 1, V0 + len(jp) + 7]]  # out-of-range indices
    pos = np.concatenate([m.positions, jp.astype(np.float32)])
    faces = np.concatenate([m.faces, np.asarray(jf, np.int32)])
    cols = np.concatenate([m.colors, np.full((len(jp), 3), 0.5, np.float32)])
    mall = Mesh(pos, faces, np.concatenate([m.opacity, np.ones(len(jf), np.float32)]), colors=cols)
    return Scene("degenerate", gall, mall, base.cameras, base.bg, base.bg_alpha), base


def make_needles(seed=17, n=2000, W=256, H=256, kappa=(850.0, 1150.0)) -> Scene:
    """Adversarial membership scene (P:300 / S:173 fragment membership; blend.cu's
    per-warp culling): needle Gaussians whose projected conic condition number
    straddles the culling-exactness threshold (~1000), i.e. cov2d eigenvalues
    lambda_2 ~ 0.31 px^2 (dilation 0.3 dominated) and lambda_1 = kappa lambda_2 with
    kappa ~ U(850, 1150): ~115 px long, ~3.5 px wide, random in-plane angle,
    positions and opacities (so q_max varies), crossing 8x4 warp sub-tile edges
    everywhere.  Identity camera, f = W."""
    rng = np.random.default_rng(seed)
    f = float(W)
    cam = Camera(W, H, f, f, W / 2.0 + 0.137, H / 2.0 - 0.219, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    z = rng.uniform(2.0, 6.0, n)
    u = rng.uniform(-20.0, W + 20.0, n)
    v = rng.uniform(-20.0, H + 20.0, n)
    means = np.stack([(u - cam.cx) / f * z, (v - cam.cy) / f * z, z], -1)
    lam2 = 0.31
    lam1 = rng.uniform(kappa[0], kappa[1], n) * lam2
    s1 = z / f * np.sqrt(lam1 - 0.3)
    s2 = z / f * 0.1
    scales = np.stack([s1, s2, np.full(n, 1e-4)], -1)
    th = rng.uniform(0.0, np.pi, n)  # rotation about the view axis
    quats = np.stack([np.cos(th / 2), np.zeros(n), np.zeros(n), np.sin(th / 2)], -1)
    opac = rng.uniform(0.05, 1.0, n)
    sh = ((rng.uniform(0.1, 0.9, (n, 1, 3)) - 0.5) / SH_C0)
    g = _pack_gaussians(means, quats, scales, opac, sh, 0)
    return Scene("needles", g, empty_mesh(), [cam], bg=np.array([0.02, 0.03, 0.05], np.float32))


# ----------------------------------------------------------------------------
# pin constructions for the shading steps (bilinear texture, SH view direction,
# 1.3x FoV Jacobian clamp).  Geometry and inputs only; the expected values are
# derived in the tests.
# ----------------------------------------------------------------------------

AFFINE_TEX = dict(tw=16, th=12, r=(10, 14, 0), g=(7, 0, 20), b=(100, 5, -6))  # value = c0 + ci*i + cj*j


def affine_texture(seed=21) -> np.ndarray:
    """[th, tw, 4] RGBA8 whose RGB is affine in the texel index (i, j): c0 + ci*i + cj*j."""
    tw, th = AFFINE_TEX["tw"], AFFINE_TEX["th"]
    j, i = np.meshgrid(np.arange(th), np.arange(tw), indexing="ij")
    tex = np.empty((th, tw, 4), np.uint8)
    for ch, key in enumerate("rgb"):
        c0, ci, cj = AFFINE_TEX[key]
        tex[..., ch] = c0 + ci * i + cj * j
    tex[..., 3] = np.random.default_rng(seed).integers(0, 256, (th, tw))  # ignored (R13)
    return tex


def make_texture_quad(x0=5.0, y0=3.0, wq=37.0, hq=29.0, W=48, H=40, texture=None, z=1.0) -> Scene:
    """Fronto-parallel 2-triangle quad covering pixels [x0, x0+wq] x [y0, y0+hq] with
    uv (0,0) at (x0, y0) and (1,1) at the far corner (fx = fy = 1 camera at the origin,
    so one world unit at z = 1 is one pixel and vertices on the 1/256 grid snap exactly).
    Default: the affine texture stretched by a non-integer factor, so pixel centres land
    at arbitrary texel fractions."""
    cam = Camera(W, H, 1.0, 1.0, 0.0, 0.0, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    P = np.array([[x0, y0, 1], [x0 + wq, y0, 1], [x0 + wq, y0 + hq, 1], [x0, y0 + hq, 1]], np.float64) * [z, z, z]
    uv = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], np.float32)
    tex = affine_texture() if texture is None else texture
    mesh = Mesh(P.astype(np.float32), np.array([[0, 1, 2], [0, 2, 3]], np.int32), np.ones(2, np.float32),
                uvs=uv, texture=tex)
    return Scene("texquad", empty_gaussians(0), mesh, [cam], bg=np.zeros(3, np.float32))


SH_PROBE_K = 0.8  # the degree-1 coefficient: channel r <- basis 1 (y), g <- basis 2 (z), b <- basis 3 (x)


def make_sh_probe(seed=22, n=24) -> Scene:
    """Degree-1 Gaussians whose only non-zero SH coefficients are SH_PROBE_K on the three
    degree-1 basis functions (one per channel, DC = 0), seen by look-at cameras from
    above, below, left, right, in front and behind (eyes recorded in the scene name
    order).  Each camera looks at the cluster centre."""
    rng = np.random.default_rng(seed)
    centre = np.array([0.3, -0.2, 0.5])
    means = centre + rng.uniform(-0.35, 0.35, (n, 3))
    sh = np.zeros((n, 4, 3), np.float32)
    sh[:, 1, 0] = sh[:, 2, 1] = sh[:, 3, 2] = SH_PROBE_K
    g = _pack_gaussians(means, _quats(rng, n), np.full((n, 3), 0.05), np.full(n, 0.9), sh, 1)
    eyes = [centre + d for d in ([0, 3.0, 0.4], [0, -3.0, 0.4], [-3.0, 0.2, 0.3], [3.0, -0.1, 0.2],
                                 [0.2, 0.3, -3.0], [-0.3, 0.1, 3.0])]
    cams = [look_at(e, centre, up=(0, 0, 1) if abs(e[1] - centre[1]) > 1 else (0, 1, 0),
                    width=96, height=80, fx=80.0, fy=80.0, cx=48.3, cy=39.6) for e in eyes]
    sc = Scene("sh_probe", g, empty_mesh(), cams, bg=np.zeros(3, np.float32))
    sc.eyes = [np.asarray(e, np.float64) for e in eyes]
    return sc


FOV_CAM = dict(W=96, H=64, f=64.0)  # 1.3 x half-FoV: |x/z| <= 0.975, |y/z| <= 0.65 (not equal: a W/H swap shows)


def make_fov_clamp(seed=23) -> Scene:
    """Large Gaussians whose centres lie inside and outside the 1.3x tan-FoV cone
    (R18, the 3DGS Jacobian clamp) yet whose footprints reach the image: camera-space
    (x/z, y/z) = (0.9, 0) [inside x, outside a height-based limit], (1.1, 0.1), (-1.2, -0.2)
    [clamped in x], (0.1, 0.75), (-0.3, -0.8) [clamped in y], (1.05, 0.7) [both].  The
    camera is rotated and translated so W = R_w2c is not the identity."""
    rng = np.random.default_rng(seed)
    W, H, f = FOV_CAM["W"], FOV_CAM["H"], FOV_CAM["f"]
    ang = 0.35
    ax = np.array([0.2, 1.0, -0.3]) / np.linalg.norm([0.2, 1.0, -0.3])
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    Rc = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K
    t = np.array([0.2, -0.1, 0.4])
    cam = Camera(W, H, f, f, W / 2.0, H / 2.0, Rc.astype(np.float32), t.astype(np.float32))
    dirs = [(0.9, 0.0), (1.1, 0.1), (-1.2, -0.2), (0.1, 0.75), (-0.3, -0.8), (1.05, 0.7)]
    z = 3.0
    pc = np.array([[a * z, b * z, z] for a, b in dirs])
    Rf, tf = Rc.astype(np.float32).astype(np.float64), t.astype(np.float32).astype(np.float64)
    means = (pc - tf) @ Rf  # R^T (pc - t), row-wise
    n = len(dirs)
    sh = np.zeros((n, 1, 3), np.float32)
    g = _pack_gaussians(means, _quats(rng, n), rng.uniform(0.3, 0.6, (n, 3)), np.full(n, 0.9), sh, 0)
    return Scene("fov_clamp", g, empty_mesh(), [cam], bg=np.zeros(3, np.float32))


# ----------------------------------------------------------------------------
# deformation inputs (Eq.12-13): a bound proxy mesh
# and a per-vertex transform field.  Synthetic: random nearby faces with Dirichlet
# barycentrics stand in for the ray-cast binding; a twist/bend field stands in for
# ACAP (out of scope).
# ----------------------------------------------------------------------------

@dataclass
class Binding:
    face: np.ndarray   # i32 [N, K]; < 0 = unbound anchor
    bary: np.ndarray   # f32 [N, K, 3] (u, v, w)

    @property
    def anchors(self) -> int:
        return int(self.face.shape[1])


@dataclass
class VertexField:
    delta: np.ndarray    # f32 [V, 3]  V' - V
    log_rot: np.ndarray  # f32 [V, 3]  axis-angle log of the vertex rotation
    shear: np.ndarray    # f32 [V, 6]  symmetric shear: xx xy xz yy yz zz

    def packed(self) -> np.ndarray:
        """[V, 12] float32: delta xyz, log_rot xyz, shear xx xy xz yy yz zz (the C ABI layout)."""
        return np.ascontiguousarray(np.concatenate([self.delta, self.log_rot, self.shear], 1), np.float32)


def make_binding(rng, gaussians: Gaussians, mesh: Mesh, K: int = 8, unbound_frac: float = 0.02,
                 spread: int = 8, nearest: bool = True) -> Binding:
    """Each anchor: the face nearest to the Gaussian (by centroid) shifted by a random index
    offset in [-spread, spread] (grid meshes: index neighbours are spatial neighbours).
    nearest=False draws the base face uniformly (large scenes whose Gaussians lie far from
    the mesh, where exact nearest-face queries are slow; timing only)."""
    n = gaussians.count
    P = mesh.positions.astype(np.float64)
    cent = P[mesh.faces].mean(1)
    if nearest:
        from scipy.spatial import cKDTree
        _, nn = cKDTree(cent).query(gaussians.means.astype(np.float64), k=1)
    else:
        nn = rng.integers(0, len(cent), n)
    face = np.clip(nn[:, None] + rng.integers(-spread, spread + 1, (n, K)), 0, len(cent) - 1).astype(np.int32)
    face[rng.uniform(0, 1, (n, K)) < unbound_frac] = -1
    bary = rng.dirichlet(np.ones(3), (n, K)).astype(np.float32)
    return Binding(face, bary)


def twist_field(mesh: Mesh, twist: float = 0.8, bend: float = 0.3, shear_eps: float = 0.05) -> VertexField:
    """Rotation about +y by twist * y plus a bend about +z by bend * x; small smooth shear."""
    P = mesh.positions.astype(np.float64)
    w = np.stack([np.zeros(len(P)), twist * P[:, 1], bend * P[:, 0]], -1)
    from scipy.spatial.transform import Rotation
    Rm = Rotation.from_rotvec(w).as_matrix()
    Pn = np.einsum("nij,nj->ni", Rm, P)
    s = shear_eps * np.stack([np.sin(P[:, 0]), 0.3 * np.cos(P[:, 1]), 0.2 * np.sin(P[:, 2]),
                              np.cos(P[:, 2]), 0.1 * np.sin(P[:, 0] + P[:, 1]), np.sin(P[:, 1])], -1)
    shear = np.array([1, 0, 0, 1, 0, 1], np.float64) + s
    return VertexField((Pn - P).astype(np.float32), w.astype(np.float32), shear.astype(np.float32))


def uniform_field(V: int, delta=(0, 0, 0), log_rot=(0, 0, 0), shear=(1, 0, 0, 1, 0, 1)) -> VertexField:
    return VertexField(np.tile(np.asarray(delta, np.float32), (V, 1)), np.tile(np.asarray(log_rot, np.float32), (V, 1)),
                       np.tile(np.asarray(shear, np.float32), (V, 1)))


def make_deform(seed=6, n_gauss=20000, K=8, W=160, H=120, lon=48, lat=24):
    """Gaussians on a sphere shell bound to a UV-sphere proxy mesh (K anchors each)."""
    rng = np.random.default_rng(seed)
    p, uv, f = uv_sphere((0, 0, 0), 1.0, lon, lat)
    mesh = merge_meshes([(p, uv, f, 1.0)], procedural_texture(rng, 64, 8))
    means = _shell_points(rng, n_gauss, 1.0) * 0.98
    scales = _lognormal_scales(rng, n_gauss, 0.02, 0.4)
    g = _pack_gaussians(means, _quats(rng, n_gauss), scales, _opacities(rng, n_gauss), _sh(rng, n_gauss, 1), 1)
    cam = look_at((0.0, 0.6, 3.4), width=W, height=H, fx=W * 0.9, fy=W * 0.9, cx=W / 2, cy=H / 2)
    binding = make_binding(rng, g, mesh, K)
    return Scene("deform", g, mesh, [cam], bg=np.array([0.1, 0.1, 0.1], np.float32)), binding


# ----------------------------------------------------------------------------
# ray-cast binding inputs: Gaussians on and
# around a proxy-mesh shell seen by a ring of "training" cameras (SPEC's
# workload: 100k Gaussians, bbx8, 8 cameras, 50k faces).
# ----------------------------------------------------------------------------

def make_bind_case(seed=8, n_gauss=100_000, lon=250, lat=100, n_cams=8, shell_sigma=0.01):
    """(gaussians, mesh, cameras): UV sphere r = 1 with 2 lon lat faces, Gaussians at
    radius ~ N(1, shell_sigma) with log-normal scales (median 0.01), cameras on an
    orbit of radius 3 at alternating elevations looking at the origin."""
    rng = np.random.default_rng(seed)
    p, uv, f = uv_sphere((0, 0, 0), 1.0, lon, lat)
    mesh = Mesh(p.astype(np.float32), f.astype(np.int32), np.ones(len(f), np.float32))
    dirs = _unit_vectors(rng, n_gauss)
    means = dirs * rng.normal(1.0, shell_sigma, (n_gauss, 1))
    scales = _lognormal_scales(rng, n_gauss, 0.01, 0.5)
    g = _pack_gaussians(means, _quats(rng, n_gauss), scales, _opacities(rng, n_gauss), _sh(rng, n_gauss, 0), 0)
    cams = []
    for i in range(n_cams):
        phi = 2 * np.pi * i / n_cams
        el = np.deg2rad(25.0 if i % 2 else -20.0)
        eye = (3.0 * np.cos(el) * np.sin(phi), 3.0 * np.sin(el), 3.0 * np.cos(el) * np.cos(phi))
        cams.append(look_at(eye, width=800, height=800, fx=900.0, fy=900.0, cx=400.0, cy=400.0))
    return g, mesh, cams
