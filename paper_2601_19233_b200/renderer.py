"""Thin Python binding over the C ABI (include/unimgs.h).

PyTorch supplies device memory and the stream; every step of the path runs in
libunimgs.so's kernels.  No CPU fallback exists: a missing library raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .scenes import Camera as SceneCamera


@dataclass
class DeviceScene:
    """Scene arrays resident in device memory (torch tensors)."""
    means: torch.Tensor
    quats: torch.Tensor
    scales: torch.Tensor
    opacities: torch.Tensor
    sh: torch.Tensor
    sh_degree: int
    positions: torch.Tensor
    faces: torch.Tensor
    opacity: torch.Tensor
    uvs: Optional[torch.Tensor] = None
    colors: Optional[torch.Tensor] = None
    texture: Optional[torch.Tensor] = None
    cov3d: Optional[torch.Tensor] = None  # [N, 6]: replaces quats/scales when set

    @property
    def num_gaussians(self) -> int:
        return int(self.means.shape[0])

    @property
    def num_triangles(self) -> int:
        return int(self.faces.shape[0])

    def nbytes(self) -> int:
        ts = [self.means, self.quats, self.scales, self.opacities, self.sh, self.positions, self.faces,
              self.opacity, self.uvs, self.colors, self.texture, self.cov3d]
        return int(sum(t.numel() * t.element_size() for t in ts if t is not None))


def to_device(scene, device="cuda") -> DeviceScene:
    g, m = scene.gaussians, scene.mesh

    def t(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)

    return DeviceScene(t(g.means), t(g.quats), t(g.scales), t(g.opacities), t(g.sh), int(g.sh_degree),
                       t(m.positions), t(m.faces.astype(np.int32)), t(m.opacity), t(m.uvs), t(m.colors), t(m.texture),
                       t(getattr(g, "cov3d", None)))


def to_pinned(scene) -> DeviceScene:
    """Host copies in page-locked memory (inputs of the end-to-end path)."""
    ds = to_device(scene, "cpu")
    for k, v in list(ds.__dict__.items()):
        if isinstance(v, torch.Tensor):
            setattr(ds, k, v.pin_memory())
    return ds


def c_camera(cam: SceneCamera) -> _lib.Camera:
    c = _lib.Camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    R = np.asarray(cam.R, np.float32).ravel()
    t = np.asarray(cam.t, np.float32).ravel()
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(t[i])
    c.near_z, c.far_z = float(cam.near), float(cam.far)
    return c


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_contiguous()
    return t.data_ptr()


def c_gaussians(s: DeviceScene) -> _lib.Gaussians:
    g = _lib.Gaussians()
    g.count = s.num_gaussians
    g.means, g.quats, g.scales = _ptr(s.means), _ptr(s.quats), _ptr(s.scales)
    g.opacities, g.sh, g.sh_degree = _ptr(s.opacities), _ptr(s.sh), int(s.sh_degree)
    g.cov3d = _ptr(s.cov3d)
    return g


def c_mesh(s: DeviceScene) -> _lib.Mesh:
    m = _lib.Mesh()
    m.num_vertices, m.num_triangles = int(s.positions.shape[0]), s.num_triangles
    m.positions, m.uvs, m.colors = _ptr(s.positions), _ptr(s.uvs), _ptr(s.colors)
    m.faces, m.opacity, m.texture = _ptr(s.faces), _ptr(s.opacity), _ptr(s.texture)
    if s.texture is not None:
        m.tex_height, m.tex_width = int(s.texture.shape[0]), int(s.texture.shape[1])
    return m


EXACT, NAIVE, MSAA_PIXEL, WHOLE_PIXEL, PAPER_LITERAL = range(5)  # blend modes (include/unimgs.h)


def make_settings(alpha_max=0.99, t_eps=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), bg_alpha=1.0,
                  sort_mode=0, blend_mode=EXACT, msaa=4, tri_depth=0, sort_ctas_per_sm=0) -> _lib.Settings:
    s = _lib.Settings()
    _lib.load().unimgs_default_settings(C.byref(s))
    s.alpha_max, s.t_eps, s.dilation, s.bg_alpha, s.sort_mode = alpha_max, t_eps, dilation, bg_alpha, sort_mode
    s.blend_mode, s.msaa_samples, s.tri_depth = blend_mode, msaa, tri_depth
    s.sort_ctas_per_sm = sort_ctas_per_sm
    for i in range(3):
        s.bg[i] = float(bg[i])
    return s


def _stream_handle(stream: Optional[torch.cuda.Stream]):
    st = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(st.cuda_stream)


class Renderer:
    """One unimgs context: reserve once, then preprocess -> bin -> render per view."""

    def __init__(self, max_gaussians: int, max_triangles: int, max_pairs: int, max_w: int, max_h: int, **settings):
        self.L = _lib.load()
        self._h = C.c_void_p()
        self._settings = make_settings(**settings)
        self._check(self.L.unimgs_create(C.byref(self._h), C.byref(self._settings)), create=True)
        self._check(self.L.unimgs_reserve2(self._h, max_gaussians, max_triangles, max_pairs, max_w, max_h))
        self.max_w, self.max_h = max_w, max_h
        self._cam = None
        self._scene = None

    def _check(self, rc: int, create: bool = False):
        if rc != _lib.OK:
            msg = "create failed" if create else self.L.unimgs_error_string(self._h).decode()
            raise _lib.UnimgsError(rc, msg)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.L.unimgs_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_settings(self, **settings):
        self._settings = make_settings(**settings)
        self._check(self.L.unimgs_set_settings(self._h, C.byref(self._settings)))

    # ---- the three calls -------------------------------------------------
    def preprocess(self, scene: DeviceScene, cam: SceneCamera, stream=None):
        self._g, self._m, self._cam_c = c_gaussians(scene), c_mesh(scene), c_camera(cam)
        self._cam, self._scene = cam, scene
        self._check(self.L.unimgs_preprocess(self._h, C.byref(self._g), C.byref(self._m), C.byref(self._cam_c),
                                             _stream_handle(stream)))

    def bin(self, stream=None):
        self._check(self.L.unimgs_bin(self._h, _stream_handle(stream)))

    def render(self, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self._cam.height, self._cam.width, 4), dtype=torch.float32, device="cuda")
        assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous()
        self._check(self.L.unimgs_render(self._h, C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def render_counted(self, out: Optional[torch.Tensor] = None, stream=None):
        """Render through the work-counting kernel variant; returns (out, work dict)."""
        if out is None:
            out = torch.empty((self._cam.height, self._cam.width, 4), dtype=torch.float32, device="cuda")
        w = (C.c_int64 * 4)()
        self._check(self.L.unimgs_render_counted(self._h, C.c_void_p(out.data_ptr()), w, _stream_handle(stream)))
        return out, dict(gauss_tests=w[0], gauss_frags=w[1], tri_tests=w[2], tri_frags=w[3])

    def render_fragments(self, out: Optional[torch.Tensor] = None, stream=None):
        """Render through the counting kernel (unimgs_render_fragments); returns (out, counts)
        with counts [H, W, 4] int32: Gaussian fragments blended, triangle fragments blended,
        id of the last fragment blended (-1 = none), Gaussian entries tested."""
        if out is None:
            out = torch.empty((self._cam.height, self._cam.width, 4), dtype=torch.float32, device="cuda")
        counts = torch.empty((self._cam.height, self._cam.width, 4), dtype=torch.int32, device="cuda")
        self._check(self.L.unimgs_render_fragments(self._h, C.c_void_p(out.data_ptr()), C.c_void_p(counts.data_ptr()),
                                                   _stream_handle(stream)))
        return out, counts

    def render_view(self, scene: DeviceScene, cam: SceneCamera, out=None, stream=None) -> torch.Tensor:
        self.preprocess(scene, cam, stream)
        self.bin(stream)
        return self.render(out, stream)

    # ---- host-buffer end-to-end path ---------------------------------------
    def render_host(self, host_scene: DeviceScene, cams: Sequence[SceneCamera], out: torch.Tensor, stream=None):
        """host_scene tensors on the CPU (pinned for async copies); out: pinned CPU [V,H,W,4] float32."""
        g, m = c_gaussians(host_scene), c_mesh(host_scene)
        arr = (_lib.Camera * len(cams))(*[c_camera(c) for c in cams])
        assert not out.is_cuda and out.is_contiguous()
        self._check(self.L.unimgs_render_host(self._h, C.byref(g), C.byref(m), arr, len(cams),
                                              C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def render_host_async(self, host_scene: DeviceScene, cams: Sequence[SceneCamera], out: torch.Tensor,
                          stream=None):
        """Pipelined render_host (unimgs_render_host_async): returns once enqueued; this call's
        scene upload overlaps the previous call's rendering.  Keep host_scene, the camera list
        and out alive until host_wait()."""
        g, m = c_gaussians(host_scene), c_mesh(host_scene)
        arr = (_lib.Camera * len(cams))(*[c_camera(c) for c in cams])
        assert not out.is_cuda and out.is_contiguous()
        self._keep = getattr(self, "_keep", [])[-3:] + [(g, m, arr)]  # ctypes structs stay referenced
        self._check(self.L.unimgs_render_host_async(self._h, C.byref(g), C.byref(m), arr, len(cams),
                                                    C.c_void_p(out.data_ptr()), _stream_handle(stream)))
        return out

    def host_wait(self):
        self._check(self.L.unimgs_host_wait(self._h))

    def set_host_lanes(self, lanes: int):
        """Views of the host path render round-robin on `lanes` contexts/streams."""
        self._check(self.L.unimgs_set_host_lanes(self._h, int(lanes)))

    # ---- stats / debug --------------------------------------------------------
    def stats(self, stream=None, check: bool = True) -> dict:
        st = _lib.Stats()
        rc = self.L.unimgs_get_stats(self._h, C.byref(st), _stream_handle(stream))
        if check:
            self._check(rc)
        d = {k: getattr(st, k) for k, _ in _lib.Stats._fields_}
        d["status"] = rc
        return d

    def bins(self, stream=None):
        st = self.stats(stream)
        K = st["num_pairs"]
        tiles = st["tiles_x"] * st["tiles_y"]
        keys = torch.empty(max(K, 1), dtype=torch.int64, device="cuda")
        vals = torch.empty(max(K, 1), dtype=torch.int32, device="cuda")
        ranges = torch.empty((tiles, 2), dtype=torch.int32, device="cuda")
        self._check(self.L.unimgs_get_bins(self._h, C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()),
                                           C.c_void_p(ranges.data_ptr()), _stream_handle(stream)))
        torch.cuda.synchronize()
        k = keys[:K].cpu().numpy().view(np.uint64)
        v = vals[:K].cpu().numpy().view(np.uint32)
        r = ranges.cpu().numpy().view(np.uint32)
        return k, v, r

    def records(self, stream=None) -> dict:
        s = self._scene
        N, F = s.num_gaussians, s.num_triangles
        P = N + F
        grec = torch.empty((max(N, 1), 12), dtype=torch.float32, device="cuda")
        trec = torch.empty((max(F, 1), 24), dtype=torch.int32, device="cuda")
        rects = torch.empty((max(P, 1), 2), dtype=torch.int32, device="cuda")
        touched = torch.empty(max(P, 1), dtype=torch.int32, device="cuda")
        dkeys = torch.empty(max(P, 1), dtype=torch.int32, device="cuda")
        self._check(self.L.unimgs_get_records(self._h, C.c_void_p(grec.data_ptr()), C.c_void_p(trec.data_ptr()),
                                              C.c_void_p(rects.data_ptr()), C.c_void_p(touched.data_ptr()),
                                              C.c_void_p(dkeys.data_ptr()), _stream_handle(stream)))
        torch.cuda.synchronize()
        rect = rects[:P].cpu().numpy().view(np.uint32)
        unpacked = np.stack([rect[:, 0] & 0xFFFF, rect[:, 0] >> 16, rect[:, 1] & 0xFFFF, rect[:, 1] >> 16], -1)
        return dict(grec=grec[:N].cpu().numpy(), trec=trec[:F].cpu().numpy(),
                    rect=unpacked.astype(np.int32), touched=touched[:P].cpu().numpy().view(np.uint32),
                    dkey=dkeys[:P].cpu().numpy().view(np.uint32))

    def check_guards(self) -> int:
        """Checked build only: guard-band bytes overwritten (unimgs_debug_check_guards)."""
        bad = C.c_int64()
        self._check(self.L.unimgs_debug_check_guards(self._h, C.byref(bad)))
        return int(bad.value)

    def launch_count(self) -> int:
        return int(self.L.unimgs_launch_count(self._h))


def preprocess_multi(renderers: Sequence["Renderer"], scene: DeviceScene, cams: Sequence[SceneCamera], stream=None):
    """unimgs_preprocess_multi: view v of one scene into renderers[v] (<= 4), the scene read once."""
    L = _lib.load()
    n = len(renderers)
    hs = (C.c_void_p * n)(*[r._h.value for r in renderers])
    g, m = c_gaussians(scene), c_mesh(scene)
    arr = (_lib.Camera * n)(*[c_camera(c) for c in cams])
    rc = L.unimgs_preprocess_multi(hs, n, C.byref(g), C.byref(m), arr, _stream_handle(stream))
    if rc != _lib.OK:
        raise _lib.UnimgsError(rc, L.unimgs_error_string(renderers[0]._h).decode())
    for r, cam in zip(renderers, cams):
        r._g, r._m, r._cam, r._scene = g, m, cam, scene


class ContextPool:
    """Several renderer contexts rendering consecutive views concurrently (the bench's
    launch configuration): view j of a batch goes to context j % n on its
    own stream, so the compute-bound blend of one view overlaps the latency-bound
    binning of the next.  With prio, each context's preprocess + bin run on a
    highest-priority stream and its blend on the normal one; sort_ctas_per_sm = 1 leaves
    most of each SM to the other contexts' blends.  With batch > 1, consecutive groups
    of `batch` views are preprocessed together (unimgs_preprocess_multi: the scene
    crosses HBM once per group) into one of n / batch context sets, alternating, so a
    group's preprocess waits only for the blends of the group two back."""

    def __init__(self, n: int, max_gaussians: int, max_triangles: int, max_pairs: int, max_w: int, max_h: int,
                 prio: bool = True, device=None, batch: int = 1, **settings):
        assert batch >= 1 and n % batch == 0
        settings.setdefault("sort_ctas_per_sm", 1 if n > 1 else 0)
        self.batch = batch
        self.rs = [Renderer(max_gaussians, max_triangles, max_pairs, max_w, max_h, **settings) for _ in range(n)]
        self.streams = [torch.cuda.Stream(device=device) for _ in range(n)]
        # (torch maps a priority beyond the device's range to its highest priority)
        self.pstreams = [torch.cuda.Stream(device=device, priority=-100) for _ in range(n)] if prio else self.streams
        self.bstreams = [torch.cuda.Stream(device=device, priority=-100 if prio else 0) for _ in range(n // batch)]
        self.next_set = 0

    def render_views(self, scene: DeviceScene, cams: Sequence[SceneCamera], out: torch.Tensor, after=None,
                     ev_pairs=None):
        """Enqueue cams[j] -> out[j] on context j % n.  `after`: a stream every context waits
        on first.  ev_pairs (list): collects (start, end) CUDA events around each blend.
        No join at the end: the caller joins `streams` when it needs the frames."""
        if self.batch > 1:
            return self._render_batched(scene, cams, out, after, ev_pairs)
        n = len(self.rs)
        if after is not None:
            for st in self.streams:
                st.wait_stream(after)
        for j, cam in enumerate(cams):
            rr, ss, ps = self.rs[j % n], self.streams[j % n], self.pstreams[j % n]
            if ps is not ss:
                ps.wait_stream(ss)  # the context's previous blend has released its buffers
            rr.preprocess(scene, cam, stream=ps)
            rr.bin(stream=ps)
            if ps is not ss:
                ss.wait_stream(ps)
            if ev_pairs is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(ss)
                rr.render(out[j], stream=ss)
                e1.record(ss)
                ev_pairs.append((e0, e1))
            else:
                rr.render(out[j], stream=ss)

    def _render_batched(self, scene, cams, out, after, ev_pairs):
        B, nsets = self.batch, len(self.rs) // self.batch
        if after is not None:
            for st in self.streams:
                st.wait_stream(after)
        for g0 in range(0, len(cams), B):
            k = self.next_set
            self.next_set = (k + 1) % nsets
            idx = list(range(k * B, k * B + min(B, len(cams) - g0)))
            bs = self.bstreams[k]
            for i in idx:
                bs.wait_stream(self.streams[i])  # the set's previous blends have released its buffers
            preprocess_multi([self.rs[i] for i in idx], scene, cams[g0:g0 + len(idx)], stream=bs)
            for jj, i in enumerate(idx):
                rr, ss, ps = self.rs[i], self.streams[i], self.pstreams[i]
                ps.wait_stream(bs)
                rr.bin(stream=ps)
                ss.wait_stream(ps)
                if ev_pairs is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(ss)
                    rr.render(out[g0 + jj], stream=ss)
                    e1.record(ss)
                    ev_pairs.append((e0, e1))
                else:
                    rr.render(out[g0 + jj], stream=ss)

    def join(self, stream):
        for st in self.streams:
            stream.wait_stream(st)

    def launch_count(self) -> int:
        return sum(r.launch_count() for r in self.rs)


def deform(scene: DeviceScene, face: torch.Tensor, bary: torch.Tensor, faces: torch.Tensor, vdata: torch.Tensor,
           stream=None):
    """Eq.12-13 on the device: returns (means' [N,3], cov' [N,6]) CUDA tensors.
    face [N,K] int32, bary [N,K,3], faces [F,3] int32, vdata [V,12] (VertexField.packed())."""
    L = _lib.load()
    N = scene.num_gaussians
    mo = torch.empty((N, 3), dtype=torch.float32, device=scene.means.device)
    co = torch.empty((N, 6), dtype=torch.float32, device=scene.means.device)
    b = _lib.Binding()
    b.count, b.anchors, b.face, b.bary = N, int(face.shape[1]), _ptr(face), _ptr(bary)
    f = _lib.VertexField()
    f.num_vertices, f.num_faces = int(vdata.shape[0]), int(faces.shape[0])
    f.faces, f.data = _ptr(faces), _ptr(vdata)
    rc = L.unimgs_deform(C.byref(c_gaussians(scene)), C.byref(b), C.byref(f), C.c_void_p(mo.data_ptr()),
                         C.c_void_p(co.data_ptr()), _stream_handle(stream))
    if rc != _lib.OK:
        raise _lib.UnimgsError(rc, "deform")
    return mo, co


def bind(means: torch.Tensor, quats: torch.Tensor, scales: torch.Tensor, positions: torch.Tensor,
         faces: torch.Tensor, cams, mode: int = 1, k_sigma: float = 3.0, with_dist: bool = False, stream=None):
    """Gaussian-centric ray-cast binding on the device (unimgs_bind):
    returns face [N,K] int32 (-1 = unbound), bary [N,K,3] float32 and, with
    with_dist, the squared hit distance [N,K] float64; K = 1 (mode 0) or 8."""
    L = _lib.load()
    N = int(means.shape[0])
    K = 1 if mode == 0 else 8
    dev = means.device
    g = _lib.Gaussians()
    g.count, g.means, g.quats, g.scales = N, _ptr(means), _ptr(quats), _ptr(scales)
    m = _lib.Mesh()
    m.num_vertices, m.num_triangles = int(positions.shape[0]), int(faces.shape[0])
    m.positions, m.faces = _ptr(positions), _ptr(faces)
    ca = (_lib.Camera * len(cams))(*[c_camera(c) for c in cams])
    s = _lib.BindSettings(mode, k_sigma)
    face = torch.empty((N, K), dtype=torch.int32, device=dev)
    bary = torch.empty((N, K, 3), dtype=torch.float32, device=dev)
    d2 = torch.empty((N, K), dtype=torch.float64, device=dev) if with_dist else None
    rc = L.unimgs_bind(C.byref(g), C.byref(m), ca, len(cams), C.byref(s), _ptr(face), _ptr(bary), _ptr(d2),
                       _stream_handle(stream))
    if rc != _lib.OK:
        raise _lib.UnimgsError(rc, "bind")
    return (face, bary, d2) if with_dist else (face, bary)


def estimate_pairs(scene, slack: float = 2.0, minimum: int = 1 << 16) -> int:
    """A generous max_pairs for a scene (the caller may also size from get_stats)."""
    n = scene.gaussians.count + scene.mesh.num_triangles
    return int(max(minimum, n * 4 * slack))


def renderer_for(scene, max_pairs: Optional[int] = None, **settings) -> Renderer:
    W = max(c.width for c in scene.cameras)
    H = max(c.height for c in scene.cameras)
    settings.setdefault("bg", tuple(float(v) for v in scene.bg))
    settings.setdefault("bg_alpha", float(scene.bg_alpha))
    return Renderer(max(scene.gaussians.count, 1), max(scene.mesh.num_triangles, 1),
                    max_pairs or estimate_pairs(scene), W, H, **settings)
