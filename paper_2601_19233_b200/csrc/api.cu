// api.cu -- the C ABI of libunimgs.so (include/unimgs.h): host-side validation,
// context / scratch ownership, stream-ordered launches, stats and debug copies.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/unimgs.h"
#include "internal.cuh"

using namespace unimgs;

struct unimgs_ctx {
    unimgs_settings set;
    Buffers buf;
    int64_t max_g = 0, max_t = 0, max_prims = 0, max_pairs = 0;
    int max_w = 0, max_h = 0;
    bool reserved = false;
    int stage = 0;  // 0 none, 1 preprocessed, 2 binned
    GaussInput g{};
    MeshInput m{};
    CamParams cam{};
    int64_t P = 0;
    int sort_mode_used = 0;
    int sort_per_sm_auto = 4;  // sort_ctas_per_sm = 0: 4 alone, 1 with several host lanes
    int sm_count = 148;
    int64_t launches = 0;
    std::string err;
    // end-to-end staging (unimgs_render_host[_async]): two device copies of the
    // scene, so the upload of call i + 1 overlaps the rendering of call i
    void *stage_buf[2] = {nullptr, nullptr};
    size_t stage_bytes[2] = {0, 0};
    float *frames[2] = {nullptr, nullptr};
    size_t frame_bytes = 0;
    cudaStream_t copy_stream = nullptr, up_stream = nullptr;
    cudaEvent_t ev_render[2] = {nullptr, nullptr}, ev_copy[2] = {nullptr, nullptr};
    cudaEvent_t ev_uploaded[2] = {nullptr, nullptr}, ev_stage_free[2] = {nullptr, nullptr};
    int64_t host_calls = 0;
    cudaStream_t host_stream = nullptr;  // compute stream of the last async call
    // extra render lanes of the host path (unimgs_set_host_lanes): child contexts with
    // their own scratch, stream and frame buffers; views go round-robin over the lanes
    static constexpr int kMaxLanes = 8;
    int lanes = 1;
    unimgs_ctx *child[kMaxLanes] = {};
    cudaStream_t lane_stream[kMaxLanes] = {};
    cudaEvent_t ev_lane_free[2][kMaxLanes] = {};  // lane l done with scene slot i
    // per lane context: preprocess + bin on a high-priority stream, so the
    // latency-bound sort passes of one lane get SMs ahead of the queued CTAs of
    // another lane's compute-bound blend (DESIGN.md §5 history)
    cudaStream_t bin_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_binned = nullptr;
    // checked build only: every scratch buffer is followed by a guard band of kGuardBytes
    // filled with kGuardByte (unimgs_debug_check_guards counts the bytes overwritten)
    std::vector<std::pair<void *, size_t>> guards;
};

[[maybe_unused]] static constexpr size_t kGuardBytes = 4096;
[[maybe_unused]] static constexpr unsigned char kGuardByte = 0x5A;

// cudaMalloc of a context scratch buffer (+ the guard band in the checked build)
static cudaError_t dev_alloc(unimgs_ctx *c, void **p, size_t bytes) {
#ifdef UNIMGS_CHECKED
    cudaError_t e = cudaMalloc(p, bytes + kGuardBytes);
    if (e != cudaSuccess) return e;
    c->guards.push_back({*p, bytes});
    return cudaMemset(static_cast<char *>(*p) + bytes, kGuardByte, kGuardBytes);
#else
    (void)c;
    return cudaMalloc(p, bytes);
#endif
}
template <typename T>
static cudaError_t dev_alloc(unimgs_ctx *c, T **p, size_t bytes) {
    return dev_alloc(c, reinterpret_cast<void **>(p), bytes);
}

extern "C" void unimgs_destroy(unimgs_ctx *c);

static int fail(unimgs_ctx *c, int code, const char *fmt, ...) __attribute__((format(printf, 3, 4)));
static int fail(unimgs_ctx *c, int code, const char *fmt, ...) {
    if (c) {
        char b[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(b, sizeof b, fmt, ap);
        va_end(ap);
        c->err = b;
    }
    return code;
}

#define CUDA_TRY(c, x)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) return fail(c, UNIMGS_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

static int check_launch(unimgs_ctx *c, const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, UNIMGS_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return UNIMGS_OK;
}

extern "C" void unimgs_default_settings(unimgs_settings *s) {
    if (!s) return;
    memset(s, 0, sizeof *s);
    s->msaa_samples = 4;
    s->tile_size = 16;
    s->alpha_min = 1.0f / 255.0f;
    s->alpha_max = 0.99f;
    s->t_eps = 1e-4f;
    s->dilation = 0.3f;
    s->bg_alpha = 1.0f;
    s->sort_mode = 0;
    s->blend_mode = 0;
    s->tri_depth = 0;
    s->sort_ctas_per_sm = 0;
}

static int validate_settings(unimgs_ctx *c, const unimgs_settings *s) {
    if (s->msaa_samples != 1 && s->msaa_samples != 2 && s->msaa_samples != 4 && s->msaa_samples != 8 &&
        s->msaa_samples != 16)
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "msaa_samples must be 1, 2, 4, 8 or 16 (got %d)", s->msaa_samples);
    if (s->blend_mode < 0 || s->blend_mode > 4)
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "blend_mode must be 0..4 (got %d)", s->blend_mode);
    if (s->tile_size != 16) return fail(c, UNIMGS_ERR_UNSUPPORTED, "tile_size must be 16 (got %d)", s->tile_size);
    if (!(fabs((double)s->alpha_min - 1.0 / 255.0) < 1e-9))
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "alpha_min must be 1/255 (got %g)", (double)s->alpha_min);
    if (!(s->alpha_max > 0.f && s->alpha_max <= 1.f)) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "alpha_max not in (0,1]");
    if (!(s->t_eps >= 0.f && s->t_eps < 1.f)) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "t_eps not in [0,1)");
    if (!(s->dilation >= 0.f && std::isfinite(s->dilation))) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "dilation < 0");
    if (s->sort_mode != 0 && s->sort_mode != 1) return fail(c, UNIMGS_ERR_UNSUPPORTED, "sort_mode must be 0 or 1");
    if (s->tri_depth < 0 || s->tri_depth > 2) return fail(c, UNIMGS_ERR_UNSUPPORTED, "tri_depth must be 0, 1 or 2");
    if (s->tri_depth == 2 && (s->blend_mode != 0 || s->msaa_samples != 4))
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "tri_depth 2 (per-pixel resort) needs blend_mode 0 and msaa_samples 4");
    if (s->sort_ctas_per_sm < 0 || s->sort_ctas_per_sm > 4)
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "sort_ctas_per_sm must be 0..4");
    for (int i = 0; i < 3; i++)
        if (!std::isfinite(s->bg[i])) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "bg not finite");
    if (!std::isfinite(s->bg_alpha)) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "bg_alpha not finite");
    return UNIMGS_OK;
}

extern "C" int unimgs_create(unimgs_ctx **out, const unimgs_settings *s) {
    if (!out) return UNIMGS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    unimgs_ctx *c = new (std::nothrow) unimgs_ctx();
    if (!c) return UNIMGS_ERR_CUDA;
    unimgs_default_settings(&c->set);
    if (s) {
        int rc = validate_settings(c, s);
        if (rc) { delete c; return rc; }
        c->set = *s;
    }
    memset(&c->buf, 0, sizeof c->buf);
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0) c->sm_count = n;
    }
    *out = c;
    return UNIMGS_OK;
}

extern "C" int unimgs_set_settings(unimgs_ctx *c, const unimgs_settings *s) {
    if (!c || !s) return UNIMGS_ERR_INVALID_ARGUMENT;
    int rc = validate_settings(c, s);
    if (rc) return rc;
    c->set = *s;
    c->stage = 0;
    for (int l = 1; l < c->lanes; l++) {
        c->child[l]->set = *s;
        c->child[l]->stage = 0;
    }
    return UNIMGS_OK;
}

static void free_buffers(unimgs_ctx *c) {
    Buffers &b = c->buf;
    void *ptrs[] = {b.rect, b.touched, b.dkey, b.grec, b.trec, b.pk[0], b.pk[1], b.pv[0], b.pv[1], b.tk[0], b.tk[1],
                    b.tv[0], b.tv[1], b.ranges, b.order, b.bcnt, b.dcnt, b.rstart, b.lookback, b.tcnt, b.gsum, b.st};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    memset(&b, 0, sizeof b);
    c->guards.clear();
    c->reserved = false;
}

extern "C" int unimgs_reserve2(unimgs_ctx *c, int64_t max_gaussians, int64_t max_triangles, int64_t max_pairs,
                               int32_t max_w, int32_t max_h) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (max_gaussians < 0 || max_triangles < 0 || max_pairs < 1 || max_w < 1 || max_h < 1)
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "reserve: bad sizes");
    if (max_gaussians + max_triangles > 0xFFFFFFFFll)
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "reserve: more than 2^32-1 primitives");
    if (max_pairs > (1ll << 30)) return fail(c, UNIMGS_ERR_UNSUPPORTED, "reserve: max_pairs above 2^30");
    free_buffers(c);
    Buffers &b = c->buf;
    const int64_t P = max_gaussians + max_triangles + 1;
    const int64_t tiles = (int64_t)((max_w + 15) / 16) * ((max_h + 15) / 16);
    const int64_t lb_tiles = sort_lookback_tiles(max_pairs, P);
    const int64_t n_rstart = max_pairs / 1024 + 2;
    CUDA_TRY(c, dev_alloc(c, &b.rect, sizeof(uint2) * P));
    CUDA_TRY(c, dev_alloc(c, &b.touched, sizeof(uint32_t) * P));
    CUDA_TRY(c, dev_alloc(c, &b.dkey, sizeof(uint32_t) * P));
    CUDA_TRY(c, dev_alloc(c, &b.grec, sizeof(GaussRecord) * (max_gaussians + 1)));
    CUDA_TRY(c, dev_alloc(c, &b.trec, sizeof(TriRecord) * (max_triangles + 1)));
    for (int i = 0; i < 2; i++) {
        CUDA_TRY(c, dev_alloc(c, &b.pk[i], sizeof(uint32_t) * P));
        CUDA_TRY(c, dev_alloc(c, &b.pv[i], sizeof(uint32_t) * P));
        CUDA_TRY(c, dev_alloc(c, &b.tk[i], sizeof(uint64_t) * max_pairs));
        CUDA_TRY(c, dev_alloc(c, &b.tv[i], sizeof(uint32_t) * max_pairs));
    }
    CUDA_TRY(c, dev_alloc(c, &b.ranges, sizeof(uint2) * tiles));
    CUDA_TRY(c, dev_alloc(c, &b.order, sizeof(uint32_t) * tiles));
    CUDA_TRY(c, dev_alloc(c, &b.bcnt, sizeof(uint32_t) * (size_t)(max_gaussians / 256 + max_triangles / 256 + 4)));
    CUDA_TRY(c, dev_alloc(c, &b.dcnt, sizeof(uint32_t) * (size_t)(P / 2048 + 4)));
    CUDA_TRY(c, dev_alloc(c, &b.rstart, sizeof(uint32_t) * (size_t)n_rstart));
    CUDA_TRY(c, dev_alloc(c, &b.lookback, sizeof(unsigned long long) * 256 * lb_tiles));
    CUDA_TRY(c, dev_alloc(c, &b.tcnt, sizeof(uint32_t) * 256 * lb_tiles));
    CUDA_TRY(c, dev_alloc(c, &b.gsum, sizeof(uint32_t) * 256 * (lb_tiles / 32 + 3)));
    CUDA_TRY(c, dev_alloc(c, &b.st, sizeof(DevState)));
    CUDA_TRY(c, cudaMemset(b.lookback, 0, sizeof(unsigned long long) * 256 * lb_tiles));
    CUDA_TRY(c, cudaMemset(b.st, 0, sizeof(DevState)));
    {
        unsigned caps[4] = {(unsigned)P, (unsigned)max_pairs, (unsigned)tiles, (unsigned)n_rstart};
#ifdef UNIMGS_CHECKED
        // fault injection for the checked build's self-test (tests/test_gpu_checked.py):
        // a 1-tile capacity makes every tile index >= 1 trip UNIMGS_CHECK; a cleared guard
        // byte must be reported by unimgs_debug_check_guards
        if (getenv("UNIMGS_FAULT_TILES")) caps[2] = 1;
        if (getenv("UNIMGS_FAULT_GUARD") && !c->guards.empty())
            CUDA_TRY(c, cudaMemset(static_cast<char *>(c->guards[0].first) + c->guards[0].second, 0, 1));
#endif
        CUDA_TRY(c, cudaMemcpy(&b.st->cap_prims, caps, sizeof caps, cudaMemcpyHostToDevice));
    }
    CUDA_TRY(c, cudaMemset(b.ranges, 0, sizeof(uint2) * tiles));
    CUDA_TRY(c, cudaDeviceSynchronize());
    b.max_prims = P - 1;
    b.max_pairs = max_pairs;
    b.max_tiles = tiles;
    b.max_lb_tiles = lb_tiles;
    b.sorted_vals = b.tv[0];
    b.sorted_keys = b.tk[0];
    b.key_bytes = 2;
    c->max_g = max_gaussians;
    c->max_t = max_triangles;
    c->max_prims = P - 1;
    c->max_pairs = max_pairs;
    c->max_w = max_w;
    c->max_h = max_h;
    c->reserved = true;
    c->stage = 0;
    return UNIMGS_OK;
}

extern "C" int unimgs_reserve(unimgs_ctx *c, int64_t max_prims, int64_t max_pairs, int32_t max_w, int32_t max_h) {
    return unimgs_reserve2(c, max_prims, max_prims, max_pairs, max_w, max_h);
}

static int make_cam(unimgs_ctx *c, const unimgs_camera *cam, CamParams &cp) {
    if (!cam) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "camera is NULL");
    if (cam->width < 1 || cam->height < 1) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "camera size < 1");
    if (cam->width > c->max_w || cam->height > c->max_h)
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "camera %dx%d above reserved %dx%d", cam->width, cam->height,
                    c->max_w, c->max_h);
    if (!(std::isfinite(cam->fx) && std::isfinite(cam->fy) && cam->fx != 0.f && cam->fy != 0.f))
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "camera focal lengths must be finite and non-zero");
    cp.W = cam->width;
    cp.H = cam->height;
    cp.tiles_x = (cam->width + kTile - 1) / kTile;
    cp.tiles_y = (cam->height + kTile - 1) / kTile;
    cp.fx = cam->fx; cp.fy = cam->fy; cp.cx = cam->cx; cp.cy = cam->cy;
    memcpy(cp.R, cam->R, sizeof cp.R);
    memcpy(cp.t, cam->t, sizeof cp.t);
    cp.near_z = cam->near_z;
    cp.far_z = cam->far_z;
    {   // N4's per-camera clamp limits, in the same IEEE single operations as B1 would
        // (round-to-nearest mul and div, no contraction possible): bit-identical
        const float hw = 0.5f * (float)cam->width, hh = 0.5f * (float)cam->height;
        const float qx = hw / cam->fx, qy = hh / cam->fy;
        cp.lx = 1.3f * qx;
        cp.ly = 1.3f * qy;
    }
    for (int a = 0; a < 3; a++)
        cp.campos[a] = (float)(-((double)cam->R[a] * cam->t[0] + (double)cam->R[3 + a] * cam->t[1] +
                                 (double)cam->R[6 + a] * cam->t[2]));
    if ((int64_t)cp.tiles_x * cp.tiles_y > (1ll << 24))
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "more than 2^24 tiles");  // three tile-digit histograms
    if ((int64_t)cp.tiles_x * cp.tiles_y > 65536 && c->set.sort_mode == 0 && c->set.tri_depth == 0)
        return fail(c, UNIMGS_ERR_UNSUPPORTED, "sort_mode 0 supports at most 65536 tiles; use sort_mode 1");
    return UNIMGS_OK;
}

extern "C" int unimgs_preprocess(unimgs_ctx *c, const unimgs_gaussians *g, const unimgs_mesh *m,
                                 const unimgs_camera *cam, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (!c->reserved) return fail(c, UNIMGS_ERR_STATE, "preprocess before reserve");
    CamParams cp;
    int rc = make_cam(c, cam, cp);
    if (rc) return rc;
    GaussInput gi{};
    if (g && g->count > 0) {
        if (g->count > c->max_g) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "gaussian count %lld above reserved %lld",
                                             (long long)g->count, (long long)c->max_g);
        if (!g->means || (!g->cov3d && (!g->quats || !g->scales)) || !g->opacities || !g->sh)
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "gaussian array is NULL");
        if (g->sh_degree < 0 || g->sh_degree > 3) return fail(c, UNIMGS_ERR_UNSUPPORTED, "sh_degree must be 0..3");
        gi = GaussInput{g->count, g->means, g->quats, g->scales, g->opacities, g->sh, g->sh_degree, g->cov3d};
    } else if (g && g->count < 0) {
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "negative gaussian count");
    }
    MeshInput mi{};
    if (m && m->num_triangles > 0) {
        if (m->num_triangles > c->max_t) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "triangle count above reserved");
        if (m->num_vertices < 1 || !m->positions || !m->faces || !m->opacity)
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "mesh array is NULL");
        if (m->texture && (m->tex_width < 1 || m->tex_height < 1))
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "texture size < 1");
        const uint8_t *tex = (m->texture && m->uvs) ? m->texture : nullptr;
        mi = MeshInput{m->num_vertices, m->num_triangles, m->positions, m->uvs, m->colors, m->opacity, m->faces,
                       tex, m->tex_width, m->tex_height};
    } else if (m && (m->num_triangles < 0 || m->num_vertices < 0)) {
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "negative mesh count");
    }
    if (gi.N + mi.F > c->max_prims) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "N + F above reserved");
    cudaStream_t s = (cudaStream_t)stream;
    c->launches += launch_begin_frame(c->buf.st, s);
    c->launches += launch_setup_triangles(mi, cp, c->buf, s);
    c->launches += launch_preprocess_gaussians(gi, mi.F, cp, c->set.dilation, c->buf, s);
    rc = check_launch(c, "preprocess");
    if (rc) return rc;
    c->g = gi;
    c->m = mi;
    c->cam = cp;
    c->P = gi.N + mi.F;
    c->stage = 1;
    return UNIMGS_OK;
}

extern "C" int unimgs_preprocess_multi(unimgs_ctx *const *ctxs, int32_t n, const unimgs_gaussians *g,
                                       const unimgs_mesh *m, const unimgs_camera *cams, void *stream) {
    if (!ctxs || !cams || n < 1) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (n > kMaxMultiViews) return fail(ctxs[0], UNIMGS_ERR_UNSUPPORTED, "preprocess_multi: at most %d views", kMaxMultiViews);
    for (int v = 0; v < n; v++) {
        if (!ctxs[v]) return UNIMGS_ERR_INVALID_ARGUMENT;
        for (int u = 0; u < v; u++)
            if (ctxs[u] == ctxs[v]) return fail(ctxs[v], UNIMGS_ERR_INVALID_ARGUMENT, "preprocess_multi: a context twice");
    }
    // every host check of unimgs_preprocess, per view, before anything is enqueued
    GaussInput gi{};
    MeshInput mi{};
    MultiView mv{};
    mv.n = n;
    for (int v = 0; v < n; v++) {
        unimgs_ctx *c = ctxs[v];
        if (!c->reserved) return fail(c, UNIMGS_ERR_STATE, "preprocess before reserve");
        int rc = make_cam(c, &cams[v], mv.cam[v]);
        if (rc) return rc;
        if (g && g->count > 0) {
            if (g->count > c->max_g)
                return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "gaussian count %lld above reserved %lld",
                            (long long)g->count, (long long)c->max_g);
            if (!g->means || (!g->cov3d && (!g->quats || !g->scales)) || !g->opacities || !g->sh)
                return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "gaussian array is NULL");
            if (g->sh_degree < 0 || g->sh_degree > 3) return fail(c, UNIMGS_ERR_UNSUPPORTED, "sh_degree must be 0..3");
            gi = GaussInput{g->count, g->means, g->quats, g->scales, g->opacities, g->sh, g->sh_degree, g->cov3d};
        } else if (g && g->count < 0) {
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "negative gaussian count");
        }
        if (m && m->num_triangles > 0) {
            if (m->num_triangles > c->max_t) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "triangle count above reserved");
            if (m->num_vertices < 1 || !m->positions || !m->faces || !m->opacity)
                return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "mesh array is NULL");
            if (m->texture && (m->tex_width < 1 || m->tex_height < 1))
                return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "texture size < 1");
            const uint8_t *tex = (m->texture && m->uvs) ? m->texture : nullptr;
            mi = MeshInput{m->num_vertices, m->num_triangles, m->positions, m->uvs, m->colors, m->opacity, m->faces,
                           tex, m->tex_width, m->tex_height};
        } else if (m && (m->num_triangles < 0 || m->num_vertices < 0)) {
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "negative mesh count");
        }
        if (gi.N + mi.F > c->max_prims) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "N + F above reserved");
        if (c->set.dilation != ctxs[0]->set.dilation)
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "preprocess_multi: the contexts' dilations differ");
        mv.buf[v] = c->buf;
    }
    cudaStream_t s = (cudaStream_t)stream;
    for (int v = 0; v < n; v++) {
        unimgs_ctx *c = ctxs[v];
        c->launches += launch_begin_frame(c->buf.st, s);
        c->launches += launch_setup_triangles(mi, mv.cam[v], c->buf, s);
    }
    ctxs[0]->launches += launch_preprocess_gaussians_multi(gi, mi.F, mv, ctxs[0]->set.dilation, s);
    int rc = check_launch(ctxs[0], "preprocess_multi");
    if (rc) return rc;
    for (int v = 0; v < n; v++) {
        unimgs_ctx *c = ctxs[v];
        c->g = gi;
        c->m = mi;
        c->cam = mv.cam[v];
        c->P = gi.N + mi.F;
        c->stage = 1;
    }
    return UNIMGS_OK;
}

extern "C" int unimgs_bin(unimgs_ctx *c, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    // exactly one bin per preprocess: only k_begin_frame (run by preprocess) resets the
    // per-frame counters, histograms and scans the bin consumes in place
    if (c->stage != 1)
        return fail(c, UNIMGS_ERR_STATE, c->stage < 1 ? "bin before preprocess" : "bin twice after one preprocess");
    c->sort_mode_used = c->set.tri_depth ? 1 : c->set.sort_mode;  // per-pair triangle keys need the full sort
    c->launches += launch_bin(c->buf, c->P, c->g.N, c->m.F, c->cam, c->sort_mode_used, c->set.tri_depth,
                              (cudaStream_t)stream, c->sm_count,
                              c->set.sort_ctas_per_sm ? c->set.sort_ctas_per_sm : c->sort_per_sm_auto);
    int rc = check_launch(c, "bin");
    if (rc) return rc;
    c->stage = 2;
    return UNIMGS_OK;
}

extern "C" int unimgs_render(unimgs_ctx *c, float *out, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (c->stage < 2) return fail(c, UNIMGS_ERR_STATE, "render before bin");
    if (!out) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "out is NULL");
    BlendParams bp{c->set.alpha_max, c->set.t_eps, c->set.bg_alpha, {c->set.bg[0], c->set.bg[1], c->set.bg[2]},
                   c->set.blend_mode, c->set.msaa_samples, c->set.tri_depth == 2};
    c->launches += launch_blend(c->buf, c->g, c->m, c->cam, bp, out, (cudaStream_t)stream);
    return check_launch(c, "render");
}

extern "C" int unimgs_render_counted(unimgs_ctx *c, float *out, int64_t *work_host, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (c->stage < 2) return fail(c, UNIMGS_ERR_STATE, "render before bin");
    if (!out || !work_host) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "out/work is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(c, cudaMemsetAsync(c->buf.st->work, 0, sizeof(c->buf.st->work), s));
    BlendParams bp{c->set.alpha_max, c->set.t_eps, c->set.bg_alpha, {c->set.bg[0], c->set.bg[1], c->set.bg[2]},
                   c->set.blend_mode, c->set.msaa_samples, c->set.tri_depth == 2};
    c->launches += launch_blend(c->buf, c->g, c->m, c->cam, bp, out, s, true);
    int rc = check_launch(c, "render_counted");
    if (rc) return rc;
    unsigned long long w[4];
    CUDA_TRY(c, cudaMemcpyAsync(w, c->buf.st->work, sizeof w, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    for (int k = 0; k < 4; k++) work_host[k] = (int64_t)w[k];
    return UNIMGS_OK;
}

extern "C" int unimgs_render_fragments(unimgs_ctx *c, float *out, uint32_t *counts, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (c->stage < 2) return fail(c, UNIMGS_ERR_STATE, "render before bin");
    if (!out || !counts) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "out/counts is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    BlendParams bp{c->set.alpha_max, c->set.t_eps, c->set.bg_alpha, {c->set.bg[0], c->set.bg[1], c->set.bg[2]},
                   c->set.blend_mode, c->set.msaa_samples, c->set.tri_depth == 2};
    c->launches += launch_blend(c->buf, c->g, c->m, c->cam, bp, out, s, true, counts);
    return check_launch(c, "render_fragments");
}

extern "C" int unimgs_deform(const unimgs_gaussians *rest, const unimgs_binding *b, const unimgs_vertex_field *f,
                             float *means_out, float *cov_out, void *stream) {
    if (!rest || !b || !f || !means_out || !cov_out) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (rest->count < 0 || b->count != rest->count) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (rest->count == 0) return UNIMGS_OK;
    if (b->anchors < 1 || b->anchors > 8) return UNIMGS_ERR_UNSUPPORTED;
    if (!rest->means || (!rest->cov3d && (!rest->quats || !rest->scales)) || !b->face || !b->bary || !f->faces ||
        !f->data || f->num_faces < 0 || f->num_vertices < 1)
        return UNIMGS_ERR_INVALID_ARGUMENT;
    if (reinterpret_cast<uintptr_t>(f->data) & 15) return UNIMGS_ERR_INVALID_ARGUMENT;
    DeformInput d{rest->count, rest->means, rest->quats, rest->scales, rest->cov3d, b->anchors, b->face, b->bary,
                  f->num_faces, f->num_vertices, f->faces, reinterpret_cast<const float4 *>(f->data)};
    launch_deform(d, means_out, cov_out, (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? UNIMGS_OK : UNIMGS_ERR_CUDA;
}

extern "C" int unimgs_bind(const unimgs_gaussians *g, const unimgs_mesh *m, const unimgs_camera *cams, int32_t num_cams,
                           const unimgs_bind_settings *s, int32_t *face_out, float *bary_out, double *dist2_out,
                           void *stream) {
    if (!g || !m || !cams || !s || !face_out || !bary_out || num_cams < 1 || g->count < 0 || m->num_triangles < 0 ||
        m->num_vertices < 0)
        return UNIMGS_ERR_INVALID_ARGUMENT;
    if (s->mode != 0 && s->mode != 1) return UNIMGS_ERR_UNSUPPORTED;
    if (s->mode == 1 && !(s->k_sigma > 0.f && std::isfinite(s->k_sigma))) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (g->count > 0 && (!g->means || (s->mode == 1 && (!g->quats || !g->scales)))) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (m->num_triangles > 0 && (!m->positions || !m->faces)) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (m->num_triangles >= (1ll << 31) || g->count * (s->mode ? 8 : 1) >= (1ll << 40)) return UNIMGS_ERR_UNSUPPORTED;
    std::vector<float> ca((size_t)num_cams * 12);
    for (int i = 0; i < num_cams; i++) {
        memcpy(&ca[12 * (size_t)i], cams[i].R, 9 * sizeof(float));
        memcpy(&ca[12 * (size_t)i + 9], cams[i].t, 3 * sizeof(float));
    }
    if (g->count == 0) return UNIMGS_OK;
    BindInput in{g->count, g->means, g->quats, g->scales, s->mode, s->k_sigma, num_cams, ca.data(),
                 m->num_vertices, m->num_triangles, m->positions, m->faces};
    if (launch_bind(in, face_out, bary_out, dist2_out, (cudaStream_t)stream) < 0) return UNIMGS_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? UNIMGS_OK : UNIMGS_ERR_CUDA;
}

extern "C" int unimgs_get_stats(unimgs_ctx *c, unimgs_stats *out, void *stream) {
    if (!c || !out) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (!c->reserved) return fail(c, UNIMGS_ERR_STATE, "stats before reserve");
    cudaStream_t s = (cudaStream_t)stream;
    memset(out, 0, sizeof *out);
    if (c->stage >= 2) {
        c->launches += launch_tile_stats(c->buf, c->cam.tiles_x * c->cam.tiles_y, s);
        int rc = check_launch(c, "tile_stats");
        if (rc) return rc;
    }
    DevState h;
    CUDA_TRY(c, cudaMemcpyAsync(&h, c->buf.st, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    out->num_pairs = h.K;
    out->needed_pairs = (int64_t)h.needed;
    out->visible_gaussians = h.vis_g;
    out->visible_triangles = h.vis_t;
    out->culled_guard_band = h.culled_guard;
    out->overflow = (int32_t)h.overflow;
    out->max_tile_pairs = c->stage >= 2 ? (int32_t)h.max_tile_pairs : 0;
    out->max_tile_id = c->stage >= 2 ? (int32_t)h.max_tile_id : -1;
    out->tiles_x = c->cam.tiles_x;
    out->tiles_y = c->cam.tiles_y;
    if (h.overflow)
        return fail(c, UNIMGS_ERR_CAPACITY, "capacity: %llu pairs needed, %lld reserved (heaviest tile %d)",
                    (unsigned long long)h.needed, (long long)c->max_pairs, out->max_tile_id);
    return UNIMGS_OK;
}

extern "C" int unimgs_get_bins(unimgs_ctx *c, uint64_t *keys, uint32_t *vals, uint32_t *ranges, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (c->stage < 2) return fail(c, UNIMGS_ERR_STATE, "get_bins before bin");
    cudaStream_t s = (cudaStream_t)stream;
    DevState h;
    CUDA_TRY(c, cudaMemcpyAsync(&h, c->buf.st, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (keys) {
        c->launches += launch_full_keys(c->buf, keys, s);
        int rc = check_launch(c, "full_keys");
        if (rc) return rc;
    }
    if (vals && h.K) CUDA_TRY(c, cudaMemcpyAsync(vals, c->buf.sorted_vals, sizeof(uint32_t) * h.K, cudaMemcpyDeviceToDevice, s));
    if (ranges)
        CUDA_TRY(c, cudaMemcpyAsync(ranges, c->buf.ranges, sizeof(uint2) * c->cam.tiles_x * c->cam.tiles_y,
                                    cudaMemcpyDeviceToDevice, s));
    return UNIMGS_OK;
}

extern "C" int unimgs_get_records(unimgs_ctx *c, float *grec, uint32_t *trec, uint32_t *rects, uint32_t *touched,
                                  uint32_t *depth_keys, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (c->stage < 1) return fail(c, UNIMGS_ERR_STATE, "get_records before preprocess");
    cudaStream_t s = (cudaStream_t)stream;
    const Buffers &b = c->buf;
    if (grec && c->g.N) CUDA_TRY(c, cudaMemcpyAsync(grec, b.grec, sizeof(GaussRecord) * c->g.N, cudaMemcpyDeviceToDevice, s));
    if (trec && c->m.F) CUDA_TRY(c, cudaMemcpyAsync(trec, b.trec, sizeof(TriRecord) * c->m.F, cudaMemcpyDeviceToDevice, s));
    if (c->P) {
        if (rects) CUDA_TRY(c, cudaMemcpyAsync(rects, b.rect, sizeof(uint2) * c->P, cudaMemcpyDeviceToDevice, s));
        if (touched) CUDA_TRY(c, cudaMemcpyAsync(touched, b.touched, sizeof(uint32_t) * c->P, cudaMemcpyDeviceToDevice, s));
        if (depth_keys) CUDA_TRY(c, cudaMemcpyAsync(depth_keys, b.dkey, sizeof(uint32_t) * c->P, cudaMemcpyDeviceToDevice, s));
    }
    return UNIMGS_OK;
}

// ---- end-to-end path over host buffers ------------------------------------------
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" int unimgs_render_host_async(unimgs_ctx *c, const unimgs_gaussians *gh, const unimgs_mesh *mh,
                                        const unimgs_camera *cams, int32_t n_views, float *out_host, void *stream) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (!c->reserved) return fail(c, UNIMGS_ERR_STATE, "render_host before reserve");
    if (!cams || n_views < 1 || !out_host) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "render_host: cams/out");
    const int W = cams[0].width, H = cams[0].height;
    for (int v = 1; v < n_views; v++)
        if (cams[v].width != W || cams[v].height != H)
            return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "render_host: all cameras must share one size");
    const int64_t N = gh ? gh->count : 0, F = mh ? mh->num_triangles : 0, V = mh ? mh->num_vertices : 0;
    if (N < 0 || F < 0 || V < 0) return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "negative counts");
    // every host-side check of preprocess, done before anything is enqueued
    if (N > c->max_g || F > c->max_t || N + F > c->max_prims)
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "render_host: counts above reserved");
    if (N && (!gh->means || !gh->opacities || !gh->sh || (!gh->cov3d && (!gh->quats || !gh->scales))))
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "render_host: gaussian array is NULL");
    if (N && (gh->sh_degree < 0 || gh->sh_degree > 3)) return fail(c, UNIMGS_ERR_UNSUPPORTED, "sh_degree must be 0..3");
    if (F && (V < 1 || !mh->positions || !mh->faces || !mh->opacity))
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "render_host: mesh array is NULL");
    if (F && mh->texture && (mh->tex_width < 1 || mh->tex_height < 1))
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "texture size < 1");
    for (int v = 0; v < n_views; v++) {
        CamParams cp;
        int rc = make_cam(c, &cams[v], cp);
        if (rc) return rc;
    }
    const bool cov = N && gh->cov3d;  // given covariances replace quats/scales (N3)
    const int shk = N ? (gh->sh_degree + 1) * (gh->sh_degree + 1) : 0;
    const bool tex = mh && mh->texture && mh->uvs && F;
    const size_t sz[] = {al256(N * 12), al256(cov ? 0 : N * 16), al256(cov ? 0 : N * 12), al256(N * 4),
                         al256(N * shk * 12), al256(V * 12), al256(mh && mh->uvs ? V * 8 : 0),
                         al256(mh && mh->colors ? V * 12 : 0), al256(F * 12), al256(F * 4),
                         al256(tex ? (size_t)mh->tex_width * mh->tex_height * 4 : 0), al256(cov ? N * 24 : 0)};
    size_t total = 0;
    for (size_t x : sz) total += x;
    cudaStream_t s = (cudaStream_t)stream;
    if (!c->copy_stream) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->up_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) {
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_render[i], cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_uploaded[i], cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_stage_free[i], cudaEventDisableTiming));
        }
    }
    const int slot = (int)(c->host_calls & 1);
    if (total > c->stage_bytes[slot]) {  // growth: drain everything that may use the old buffer
        CUDA_TRY(c, cudaDeviceSynchronize());
        if (c->stage_buf[slot]) cudaFree(c->stage_buf[slot]);
        c->stage_buf[slot] = nullptr;
        c->stage_bytes[slot] = 0;
        CUDA_TRY(c, cudaMalloc(&c->stage_buf[slot], total));
        c->stage_bytes[slot] = total;
    }
    const size_t fb = (size_t)W * H * 16;
    for (int l = 0; l < c->lanes; l++) {
        unimgs_ctx *x = l ? c->child[l] : c;
        if (fb > x->frame_bytes) {
            CUDA_TRY(c, cudaDeviceSynchronize());
            for (int i = 0; i < 2; i++) {
                if (x->frames[i]) cudaFree(x->frames[i]);
                x->frames[i] = nullptr;
            }
            x->frame_bytes = 0;
            for (int i = 0; i < 2; i++) CUDA_TRY(c, cudaMalloc(&x->frames[i], fb));
            x->frame_bytes = fb;
        }
        if (l && !x->ev_render[0])
            for (int i = 0; i < 2; i++) {
                CUDA_TRY(c, cudaEventCreateWithFlags(&x->ev_render[i], cudaEventDisableTiming));
                CUDA_TRY(c, cudaEventCreateWithFlags(&x->ev_copy[i], cudaEventDisableTiming));
            }
        if (!x->bin_stream) {
            int lo = 0, hi = 0;
            CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CUDA_TRY(c, cudaStreamCreateWithPriority(&x->bin_stream, cudaStreamNonBlocking, hi));
            CUDA_TRY(c, cudaEventCreateWithFlags(&x->ev_ready, cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&x->ev_binned, cudaEventDisableTiming));
        }
    }
    char *p = (char *)c->stage_buf[slot];
    constexpr int kArrays = 12;
    char *dp[kArrays];
    for (int i = 0; i < kArrays; i++) { dp[i] = p; p += sz[i]; }
    const void *src[] = {N ? gh->means : nullptr, cov ? nullptr : (N ? gh->quats : nullptr),
                         cov ? nullptr : (N ? gh->scales : nullptr), N ? gh->opacities : nullptr,
                         N ? gh->sh : nullptr, F ? mh->positions : nullptr, F ? mh->uvs : nullptr,
                         F ? mh->colors : nullptr, F ? mh->faces : nullptr, F ? mh->opacity : nullptr,
                         tex ? mh->texture : nullptr, cov ? gh->cov3d : nullptr};
    const size_t bytes[] = {(size_t)N * 12, cov ? 0 : (size_t)N * 16, cov ? 0 : (size_t)N * 12, (size_t)N * 4,
                            (size_t)N * shk * 12, (size_t)V * 12, (mh && mh->uvs) ? (size_t)V * 8 : 0,
                            (mh && mh->colors) ? (size_t)V * 12 : 0, (size_t)F * 12, (size_t)F * 4,
                            tex ? (size_t)mh->tex_width * mh->tex_height * 4 : 0, cov ? (size_t)N * 24 : 0};
    // upload on its own stream, once the call two back (same buffer) has rendered
    if (c->host_calls >= 2) {
        CUDA_TRY(c, cudaStreamWaitEvent(c->up_stream, c->ev_stage_free[slot], 0));
        for (int l = 1; l < c->lanes; l++) CUDA_TRY(c, cudaStreamWaitEvent(c->up_stream, c->ev_lane_free[slot][l], 0));
    }
    for (int i = 0; i < kArrays; i++)
        if (src[i] && bytes[i])
            CUDA_TRY(c, cudaMemcpyAsync(dp[i], src[i], bytes[i], cudaMemcpyHostToDevice, c->up_stream));
    CUDA_TRY(c, cudaEventRecord(c->ev_uploaded[slot], c->up_stream));
    CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_uploaded[slot], 0));
    unimgs_gaussians gd{N, (const float *)dp[0], cov ? nullptr : (const float *)dp[1],
                        cov ? nullptr : (const float *)dp[2], (const float *)dp[3], (const float *)dp[4],
                        N ? gh->sh_degree : 0, cov ? (const float *)dp[11] : nullptr};
    unimgs_mesh md{V, F, (const float *)dp[5], (F && mh->uvs) ? (const float *)dp[6] : nullptr,
                   (F && mh->colors) ? (const float *)dp[7] : nullptr, (const int32_t *)dp[8], (const float *)dp[9],
                   tex ? (const uint8_t *)dp[10] : nullptr, tex ? mh->tex_width : 0, tex ? mh->tex_height : 0};
    for (int l = 1; l < c->lanes; l++) CUDA_TRY(c, cudaStreamWaitEvent(c->lane_stream[l], c->ev_uploaded[slot], 0));
    for (int v = 0; v < n_views; v++) {
        const int l = v % c->lanes;
        unimgs_ctx *x = l ? c->child[l] : c;  // lane 0 is this context on the caller's stream
        cudaStream_t ls = l ? c->lane_stream[l] : s;
        const int bi = (v / c->lanes) & 1;
        // preprocess + bin on the lane's high-priority stream after everything before
        // on the lane (the upload, the lane's previous blend), the blend back on ls
        CUDA_TRY(c, cudaEventRecord(x->ev_ready, ls));
        CUDA_TRY(c, cudaStreamWaitEvent(x->bin_stream, x->ev_ready, 0));
        int rc = unimgs_preprocess(x, &gd, &md, &cams[v], x->bin_stream);
        if (!rc) rc = unimgs_bin(x, x->bin_stream);
        if (rc) {  // (host checks all passed above, so this is a CUDA error): drain so the
                   // slot's next upload cannot race with the views already queued
            if (x != c) c->err = x->err;
            cudaDeviceSynchronize();
            return rc;
        }
        CUDA_TRY(c, cudaEventRecord(x->ev_binned, x->bin_stream));
        CUDA_TRY(c, cudaStreamWaitEvent(ls, x->ev_binned, 0));
        CUDA_TRY(c, cudaStreamWaitEvent(ls, x->ev_copy[bi], 0));  // frame buffer drained (no-op if never recorded)
        rc = unimgs_render(x, x->frames[bi], ls);
        if (rc) {
            if (x != c) c->err = x->err;
            cudaDeviceSynchronize();
            return rc;
        }
        CUDA_TRY(c, cudaEventRecord(x->ev_render[bi], ls));
        CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, x->ev_render[bi], 0));
        CUDA_TRY(c, cudaMemcpyAsync(out_host + (size_t)v * W * H * 4, x->frames[bi], fb, cudaMemcpyDeviceToHost,
                                    c->copy_stream));
        CUDA_TRY(c, cudaEventRecord(x->ev_copy[bi], c->copy_stream));
    }
    for (int l = 1; l < c->lanes; l++) {  // the scene slot is free once every lane has rendered
        // (no join onto `stream`: only the upload two calls later waits for these)
        CUDA_TRY(c, cudaEventRecord(c->ev_lane_free[slot][l], c->lane_stream[l]));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_stage_free[slot], s));
    c->host_calls++;
    c->host_stream = s;
    return UNIMGS_OK;
}

extern "C" int unimgs_host_wait(unimgs_ctx *c) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (!c->copy_stream) return UNIMGS_OK;
    CUDA_TRY(c, cudaStreamSynchronize(c->up_stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->copy_stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->host_stream));
    bool overflowed = false;
    unsigned long long needed = 0;
    for (int l = 0; l < c->lanes; l++) {
        unimgs_ctx *x = l ? c->child[l] : c;
        if (l) CUDA_TRY(c, cudaStreamSynchronize(c->lane_stream[l]));
        DevState h;
        CUDA_TRY(c, cudaMemcpy(&h, x->buf.st, sizeof h, cudaMemcpyDeviceToHost));
        if (h.overflow_sticky) {  // any view since the last wait (begin_frame clears only `overflow`)
            CUDA_TRY(c, cudaMemset(&x->buf.st->overflow_sticky, 0, sizeof(unsigned int)));
            overflowed = true;
            needed = std::max(needed, (unsigned long long)h.needed);
        }
    }
    if (overflowed)
        return fail(c, UNIMGS_ERR_CAPACITY,
                    "capacity: at least one view since the last wait overflowed (its frame is not valid); "
                    "the last view needed %llu pairs, %lld reserved", needed, (long long)c->max_pairs);
    return UNIMGS_OK;
}

extern "C" int unimgs_set_host_lanes(unimgs_ctx *c, int32_t lanes) {
    if (!c) return UNIMGS_ERR_INVALID_ARGUMENT;
    if (!c->reserved) return fail(c, UNIMGS_ERR_STATE, "set_host_lanes before reserve");
    if (lanes < 1 || lanes > unimgs_ctx::kMaxLanes)
        return fail(c, UNIMGS_ERR_INVALID_ARGUMENT, "host lanes must be 1..%d", unimgs_ctx::kMaxLanes);
    CUDA_TRY(c, cudaDeviceSynchronize());
    for (int l = 1; l < c->lanes; l++) {  // drop the previous lanes
        unimgs_destroy(c->child[l]);
        cudaStreamDestroy(c->lane_stream[l]);
        for (int i = 0; i < 2; i++) cudaEventDestroy(c->ev_lane_free[i][l]);
        c->child[l] = nullptr;
    }
    c->lanes = 1;
    c->sort_per_sm_auto = lanes > 1 ? 1 : 4;
    for (int l = 1; l < lanes; l++) {
        int rc = unimgs_create(&c->child[l], &c->set);
        if (!rc) rc = unimgs_reserve2(c->child[l], c->max_g, c->max_t, c->max_pairs, c->max_w, c->max_h);
        if (rc) {
            if (c->child[l]) unimgs_destroy(c->child[l]);
            c->child[l] = nullptr;
            return fail(c, rc, "set_host_lanes: lane %d allocation failed", l);
        }
        c->child[l]->sort_per_sm_auto = 1;
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->lane_stream[l], cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_lane_free[i][l], cudaEventDisableTiming));
        c->lanes = l + 1;
    }
    return UNIMGS_OK;
}

extern "C" int unimgs_render_host(unimgs_ctx *c, const unimgs_gaussians *gh, const unimgs_mesh *mh,
                                  const unimgs_camera *cams, int32_t n_views, float *out_host, void *stream) {
    int rc = unimgs_render_host_async(c, gh, mh, cams, n_views, out_host, stream);
    if (rc) return rc;
    return unimgs_host_wait(c);
}

extern "C" int unimgs_debug_check_guards(unimgs_ctx *c, int64_t *bad_bytes) {
    if (!c || !bad_bytes) return UNIMGS_ERR_INVALID_ARGUMENT;
    *bad_bytes = 0;
#ifdef UNIMGS_CHECKED
    CUDA_TRY(c, cudaDeviceSynchronize());
    std::vector<unsigned char> h(kGuardBytes);
    for (int l = 0; l < c->lanes; l++) {
        unimgs_ctx *x = l ? c->child[l] : c;
        for (const auto &g : x->guards) {
            CUDA_TRY(c, cudaMemcpy(h.data(), static_cast<char *>(g.first) + g.second, kGuardBytes,
                                   cudaMemcpyDeviceToHost));
            for (unsigned char v : h) *bad_bytes += v != kGuardByte;
        }
    }
    return UNIMGS_OK;
#else
    return fail(c, UNIMGS_ERR_UNSUPPORTED, "guard bands exist only in the checked build (libunimgs_checked.so)");
#endif
}

extern "C" int64_t unimgs_launch_count(const unimgs_ctx *c) {
    if (!c) return 0;
    int64_t n = c->launches;
    for (int l = 1; l < c->lanes; l++) n += c->child[l]->launches;
    return n;
}

extern "C" const char *unimgs_error_string(const unimgs_ctx *c) {
    if (!c) return "null context";
    return c->err.empty() ? "ok" : c->err.c_str();
}

extern "C" void unimgs_destroy(unimgs_ctx *c) {
    if (!c) return;
    for (int l = 1; l < c->lanes; l++) {
        cudaStreamSynchronize(c->lane_stream[l]);
        unimgs_destroy(c->child[l]);
        cudaStreamDestroy(c->lane_stream[l]);
        for (int i = 0; i < 2; i++) cudaEventDestroy(c->ev_lane_free[i][l]);
    }
    free_buffers(c);
    if (c->copy_stream) cudaDeviceSynchronize();
    for (int i = 0; i < 2; i++) {
        if (c->stage_buf[i]) cudaFree(c->stage_buf[i]);
        if (c->frames[i]) cudaFree(c->frames[i]);
        if (c->ev_render[i]) cudaEventDestroy(c->ev_render[i]);
        if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
        if (c->ev_uploaded[i]) cudaEventDestroy(c->ev_uploaded[i]);
        if (c->ev_stage_free[i]) cudaEventDestroy(c->ev_stage_free[i]);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->up_stream) cudaStreamDestroy(c->up_stream);
    if (c->bin_stream) {
        cudaStreamSynchronize(c->bin_stream);
        cudaStreamDestroy(c->bin_stream);
        cudaEventDestroy(c->ev_ready);
        cudaEventDestroy(c->ev_binned);
    }
    delete c;
}
