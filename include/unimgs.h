/*
 * unimgs.h -- C ABI of libunimgs.so, the B200 (sm_100a) implementation of the
 * UniMGS single-pass anti-aliased mesh + 3DGS tile rasterizer
 * (arXiv 2601.19233, §3.2).
 *
 * The operation: render 3D Gaussians and textured triangle meshes that carry an
 * opacity attribute ("directly assigning an opacity attribute to textured
 * meshes allows for unified rendering through alpha-blending") from a
 * camera in ONE front-to-back alpha-blend.  Gaussian fragments
 * blend by Eq.1-2; depth-adjacent triangle fragments form an
 * entity whose transmittance is tracked per sub-pixel sample (Eq.7),
 * weighted by coverage (Eq.8) and blended by Eq.9; the
 * background is composited per Eq.10-11.  The readings adopted
 * where the paper is ambiguous are listed in DESIGN.md §3 (R1-R24).
 *
 * The pipeline is three calls per view, enqueued on one CUDA stream:
 *   unimgs_preprocess  B1 EWA projection of Gaussians + B2 triangle
 *                      setup with 4-sample coverage (M = 4)
 *   unimgs_bin         per-tile key duplication, stable radix sorts (onesweep
 *                      depth passes, reduce-then-scan tile passes) and tile
 *                      ranges ("incorporate triangle fragments into the
 *                      depth-sorting process")
 *   unimgs_render      B8 unified blend -> out[H][W][4] = (R, G, B, T)
 *
 * Conventions (all calls):
 *   - Every call returns an unimgs_status; no C++ exception crosses the ABI.
 *     On failure the context records a message (unimgs_error_string).
 *   - Array pointers in unimgs_gaussians / unimgs_mesh and the out/debug
 *     buffers are CUDA DEVICE pointers owned by the caller, except where a
 *     call says "host".  They must stay valid until the work enqueued on
 *     `stream` completes.  Host structs are copied at call time.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - Host-validated arguments (null required pointers, negative counts,
 *     counts or sizes above what unimgs_reserve sized, unsupported settings)
 *     return immediately and enqueue nothing.
 *   - Device data is NOT validated: NaN, z <= near, non-PD covariance,
 *     o < 1/255, degenerate or out-of-guard-band triangles are culled as
 *     values (N1-N7) and counted in unimgs_stats.
 *   - Capacity: if the number of (tile, primitive) pairs K exceeds the
 *     reserved max_pairs, nothing is written out of bounds, a device overflow
 *     flag is set, unimgs_render leaves `out` untouched, and the next
 *     unimgs_get_stats returns UNIMGS_ERR_CAPACITY with needed_pairs.
 *   - No call except unimgs_reserve allocates, and no call except
 *     unimgs_reserve / unimgs_get_stats / unimgs_render_host synchronises the
 *     host, so preprocess -> bin -> render is CUDA-graph capturable.
 *   - A context is used by one host thread and one stream at a time.
 */
#ifndef UNIMGS_H
#define UNIMGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UNIMGS_ABI_VERSION 1

#if defined(__GNUC__)
#define UNIMGS_API __attribute__((visibility("default")))
#else
#define UNIMGS_API
#endif

typedef enum {
    UNIMGS_OK = 0,
    UNIMGS_ERR_INVALID_ARGUMENT = 1,
    UNIMGS_ERR_UNSUPPORTED = 2,
    UNIMGS_ERR_CAPACITY = 3,
    UNIMGS_ERR_CUDA = 4,
    UNIMGS_ERR_STATE = 5
} unimgs_status;

typedef struct unimgs_ctx unimgs_ctx;

/* Pinhole camera (R21): pixel (x, y) covers [x, x+1) x [y, y+1), centre at
 * (x + .5, y + .5); u = fx * X / Z + cx.  R, t map world to camera, OpenCV
 * convention (+z forward, y down), R row-major.  near_z default 0.2. */
typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float R[9], t[3];
    float near_z, far_z;
} unimgs_camera;

/* 3D Gaussians (3DGS parameterisation).  means [N][3], quats [N][4]
 * (w, x, y, z; need not be normalised), scales [N][3] linear, opacities [N]
 * post-sigmoid in [0, 1], sh [N][(D+1)^2][3] real SH in the 3DGS basis,
 * D = sh_degree in 0..3.  cov3d [N][6] (xx xy xz yy yz zz), optional: when
 * non-NULL it is Sigma and quats/scales are ignored (may be NULL) -- e.g. the
 * output of unimgs_deform.  count may be 0 (then pointers may be NULL). */
typedef struct {
    int64_t count;
    const float *means, *quats, *scales, *opacities, *sh;
    int32_t sh_degree;
    const float *cov3d;
} unimgs_gaussians;

/* Gaussian-to-mesh binding: K = 1 (ray through the centre,
 * "UniMGS*") or 8 (rays to the BBX corners) anchors per Gaussian; face [N][K]
 * (< 0 = unbound anchor), bary [N][K][3] barycentric (u, v, w) of the anchor. */
typedef struct {
    int64_t count;
    int32_t anchors;
    const int32_t *face;
    const float *bary;
} unimgs_binding;

/* Per-vertex transforms of the manipulated proxy mesh (from ACAP or
 * any mesh deformer), one 48-byte record per vertex: data [V][12] float =
 * delta xyz (V' - V), log_rot xyz (the rotation as an axis-angle vector),
 * shear xx xy xz yy yz zz (symmetric S); 16-byte aligned.  faces [F][3] of the
 * rest mesh. */
typedef struct {
    int64_t num_vertices, num_faces;
    const int32_t *faces;
    const float *data;
} unimgs_vertex_field;

/* Triangle mesh with a per-triangle opacity (reading R13).
 * positions [V][3]; faces [F][3] int32 vertex ids; opacity [F] in [0, 1].
 * Shading source, first that applies: uvs [V][2] + texture [Ht][Wt][4] RGBA8
 * (bilinear, texel centres at (i+.5)/W, clamp-to-edge, row 0 at v = 0, alpha
 * ignored); else colors [V][3]; else white.  num_triangles may be 0. */
typedef struct {
    int64_t num_vertices, num_triangles;
    const float *positions, *uvs, *colors;
    const int32_t *faces;
    const float *opacity;
    const uint8_t *texture;
    int32_t tex_width, tex_height;
} unimgs_mesh;

/* Render settings.  msaa_samples M in {1, 2, 4, 8, 16} (Direct3D
 * standard patterns; the paper uses 4); tile_size = 16 and alpha_min =
 * 1/255 only (else UNIMGS_ERR_UNSUPPORTED).
 * alpha_max clamps Gaussian alpha; t_eps is the blend-then-test
 * termination threshold (R16); dilation is added to the cov2d diagonal
 * (S:194); out = C + T * bg_alpha * bg (Eq.10 under reading R5).
 * sort_mode: 0 = factored sort (32-bit depth sort of the visible primitives,
 * then a stable 2-pass radix sort of the pairs by tile), 1 = one onesweep over
 * 64-bit (tile << 32 | depth) keys.  Both produce the identical order.
 * blend_mode (the paper's ablation, Fig.3 / Fig.4):
 *   0 = exact depth-adjacent entity (the method; exit T = T_e * mean_j t_j, R3)
 *   1 = naive: triangle fragments blended at full coverage (Fig.3a / 4a)
 *   2 = per-pixel MSAA with alpha, geometric coverage (Eq.5-6)
 *   3 = whole-pixel entity across Gaussians (Fig.3b-c / 4c, colour overflow)
 *   4 = exact entity with the paper-literal exit update T *= (1 - O_geo alpha)
 *       per triangle (Eq.6 as "still updated by Eq.(6)")
 * tri_depth: the sort depth of a triangle ("incorporate triangle fragments
 * into the depth-sorting process"):
 *   0 = view z of its centroid, one key per triangle (reading R9, default)
 *   1 = per (tile, triangle) pair: the view z of its plane at the tile centre,
 *       clamped to the triangle's z range (N8) -- interpenetrating
 *       surfaces swap order across tiles.  Per-pair keys need the full 64-bit
 *       sort, so tri_depth 1 always bins as sort_mode 1.
 *   2 = the keys of 1, plus a per-pixel resort window in the blend (SPEC S:235:
 *       triangle fragments ordered by their plane depth at the pixel centre):
 *       each pixel passes its fragments, in list order, through a bounded
 *       priority queue of 4 entries on (bits(depth at the pixel), id) -- the
 *       plane depth at the pixel centre clamped to the triangle's z range (N9)
 *       for a triangle, the view z for a Gaussian -- blending the smallest on
 *       overflow and the rest at the end of the list, so surfaces swap order
 *       at the pixel where they cross.  blend_mode 0 and msaa_samples 4 only.
 * sort_ctas_per_sm: persistent CTAs per SM of the radix-sort passes, 1..4, or
 *   0 = automatic (4 for a context rendering alone; 1 for the contexts of a
 *   unimgs_render_host call with several lanes).  4 gives the lowest latency
 *   for one frame; 1 leaves 3/4 of every SM to the blends of other contexts
 *   rendering concurrently, the higher multi-view throughput.
 *   Scheduling only: the output is identical for every value.              */
typedef struct {
    int32_t msaa_samples, tile_size;
    float alpha_min, alpha_max, t_eps, dilation;
    float bg[3], bg_alpha;
    int32_t sort_mode;
    int32_t blend_mode;
    int32_t tri_depth;
    int32_t sort_ctas_per_sm;
} unimgs_settings;

typedef struct {
    int64_t num_pairs;          /* K written (0 on overflow) */
    int64_t needed_pairs;       /* K required by the last bin */
    int64_t visible_gaussians;
    int64_t visible_triangles;
    int64_t culled_guard_band;  /* triangles culled by near plane / guard band */
    int32_t overflow;           /* 1 if needed_pairs > reserved max_pairs */
    int32_t max_tile_pairs;     /* longest tile list */
    int32_t max_tile_id;        /* its tile index ty * tiles_x + tx */
    int32_t tiles_x, tiles_y;
} unimgs_stats;

/* Fill *s with the defaults (M = 4, 16x16 tiles, alpha in [1/255, 0.99],
 * t_eps 1e-4, dilation 0.3, black opaque background, sort_mode 0, blend_mode 0,
 * tri_depth 0). */
UNIMGS_API void unimgs_default_settings(unimgs_settings *s);

/* Create a context.  s may be NULL (defaults).  No device memory yet. */
UNIMGS_API int unimgs_create(unimgs_ctx **out, const unimgs_settings *s);

/* Replace the settings (validated as in unimgs_create). */
UNIMGS_API int unimgs_set_settings(unimgs_ctx *c, const unimgs_settings *s);

/* Allocate all scratch: records for max_prims = N + F primitives, max_pairs
 * (tile, primitive) pairs, images up to max_w x max_h.  Synchronises the
 * device.  May be called again to grow. */
UNIMGS_API int unimgs_reserve(unimgs_ctx *c, int64_t max_prims, int64_t max_pairs, int32_t max_w, int32_t max_h);

/* As unimgs_reserve with separate Gaussian and triangle capacities
 * (unimgs_reserve(c, P, ...) == unimgs_reserve2(c, P, P, ...)). */
UNIMGS_API int unimgs_reserve2(unimgs_ctx *c, int64_t max_gaussians, int64_t max_triangles, int64_t max_pairs,
                    int32_t max_w, int32_t max_h);

/* B1 + B2: project Gaussians (EWA, N1-N5) and set up
 * triangles (N7).  g or m may be NULL or empty.  Device pointers. */
UNIMGS_API int unimgs_preprocess(unimgs_ctx *c, const unimgs_gaussians *g, const unimgs_mesh *m,
                      const unimgs_camera *cam, void *stream);

/* unimgs_preprocess for n <= 4 views of ONE scene at once, view v into context
 * ctxs[v] (distinct, reserved, equal dilation): every Gaussian's inputs and its
 * Sigma (N3) are read / computed once for all n views, so the scene crosses HBM
 * once per n views instead of once per view (the multi-view batch of BASELINE
 * configs[4]).  Each context's records are bit-identical to a unimgs_preprocess
 * of its view; each is then binned and rendered on its own (after `stream`). */
UNIMGS_API int unimgs_preprocess_multi(unimgs_ctx *const *ctxs, int32_t n, const unimgs_gaussians *g,
                                       const unimgs_mesh *m, const unimgs_camera *cams, void *stream);

/* Duplicate (tile, primitive) pairs, sort them by (tile, depth bits, id) and
 * compute per-tile ranges.  Exactly once per unimgs_preprocess (the
 * per-frame counters it consumes are reset only by preprocess): a second bin
 * without a new preprocess returns UNIMGS_ERR_STATE and enqueues nothing. */
UNIMGS_API int unimgs_bin(unimgs_ctx *c, void *stream);

/* B8: the unified single-pass blend (Eq.1-2, 7-11).  Writes
 * out_rgbt [height][width][4] float32 (R, G, B, final T), device pointer.
 * Must follow unimgs_bin. */
UNIMGS_API int unimgs_render(unimgs_ctx *c, float *out_rgbt, void *stream);

/* Deformation transfer, Eq.12-13, one thread per Gaussian:
 * blend (Delta, log R, S) barycentrically at each bound anchor (Eq.12), then
 * R' = exp(mean log R_i), S' = mean S_i, Sigma' = R'S' Sigma (R'S')^T,
 * mu' = mu + mean Delta_i (Eq.13).  Sigma from rest->cov3d or quats/scales.
 * Device data is culled as values: an anchor whose face is outside [0, F) or
 * has a vertex id outside [0, V) (V = field->num_vertices) is skipped.
 * Writes means_out [N][3] and cov_out [N][6] (device; pass them as means and
 * cov3d of the next unimgs_preprocess).  No context, no allocation, no sync. */
UNIMGS_API int unimgs_deform(const unimgs_gaussians *rest, const unimgs_binding *binding,
                             const unimgs_vertex_field *field, float *means_out, float *cov_out, void *stream);

/* Gaussian-centric ray-cast binding (§3.3.1; B1-B6).
 * For every Gaussian and target -- its centre (mode 0, "UniMGS*") or the 8
 * corners mu + R (+-k s0, +-k s1, +-k s2) of its oriented box at k = k_sigma
 * standard deviations (mode 1, "UniMGS"; corner i takes + on axis a iff bit a
 * of i is set) -- a ray is cast from each camera centre through the target
 * (cameras that see the target at view z <= 0 are skipped).  Per ray the
 * nearest Moller-Trumbore hit (|det| >= 1e-9, t > 1e-6; ties to the lower
 * face id); per target the hit nearest the Gaussian centre over the cameras
 * ("bound to the nearest candidate face"; ties: lower face id, then the
 * earlier camera).  Arithmetic: IEEE double in a fixed order, so the table
 * equals exhaustive search bit for bit.
 *   g: count, means, quats, scales (device; quats/scales only for mode 1)
 *   m: num_vertices, num_triangles, positions, faces (device; faces with an
 *      out-of-range vertex id are ignored)
 *   cams: HOST array of num_cams >= 1 cameras (only R and t are used)
 *   face_out [N][K] int32 (-1 = no camera ray hit the mesh), bary_out
 *   [N][K][3] float (weights of face vertices 0, 1, 2; zeros when unbound),
 *   dist2_out [N][K] double squared hit distance to the centre (-1 unbound) or
 *   NULL; K = 1 or 8.  Layout matches unimgs_binding for unimgs_deform.
 * Builds an LBVH over the mesh in stream-ordered scratch (cudaMallocAsync,
 * freed on the stream); asynchronous; not graph-capturable.  No context. */
typedef struct {
    int32_t mode;   /* 0 = centre, 1 = bbx8 */
    float k_sigma;  /* box half-extent in standard deviations (> 0; 3 by convention) */
} unimgs_bind_settings;

UNIMGS_API int unimgs_bind(const unimgs_gaussians *g, const unimgs_mesh *m, const unimgs_camera *cams,
                           int32_t num_cams, const unimgs_bind_settings *s, int32_t *face_out, float *bary_out,
                           double *dist2_out, void *stream);

/* Measurement variant of unimgs_render: identical output, plus the blend's
 * work counts (host work[4]): Gaussian entries tested, Gaussian fragments
 * blended, triangle entries tested, triangle fragments blended, summed over
 * pixels up to each pixel's termination.  Synchronises `stream`. */
UNIMGS_API int unimgs_render_counted(unimgs_ctx *c, float *out_rgbt, int64_t *work, void *stream);

/* Debug variant of unimgs_render (the counting kernel): identical out_rgbt, plus
 * per pixel counts [height][width][4] uint32 (device): {Gaussian fragments
 * blended, triangle fragments blended, unified id of the last fragment blended
 * (0xFFFFFFFF = none), Gaussian list entries tested}, each up to the pixel's
 * termination (T_eff < t_eps; with t_eps = 0 every fragment of the pixel).  A
 * fragment is a Gaussian with q <= q_max (N6, alpha >= 1/255) or a
 * triangle with a non-zero coverage mask ("fragments overlapping the
 * pixel"), so these counts check fragment membership bit for bit.  Async. */
UNIMGS_API int unimgs_render_fragments(unimgs_ctx *c, float *out_rgbt, uint32_t *counts, void *stream);

/* Synchronise `stream` and report the last frame's counters (host *out). */
UNIMGS_API int unimgs_get_stats(unimgs_ctx *c, unimgs_stats *out, void *stream);

/* Debug copy of the sorted bins into caller device buffers: keys [K] uint64
 * (tile << 32 | bits(depth)), vals [K] uint32 unified primitive ids
 * (triangles 0..F-1, then Gaussians F..F+N-1), ranges [tiles][2] uint32
 * [start, end).  Any pointer may be NULL.  K from unimgs_get_stats. */
UNIMGS_API int unimgs_get_bins(unimgs_ctx *c, uint64_t *keys, uint32_t *vals, uint32_t *ranges, void *stream);

/* Debug copy of the per-primitive records into caller device buffers (any
 * may be NULL):
 *   grec   [N][12] float: u, v, q_max, o, conic a, b, c, cull half-extent y,
 *          r, g, b, cull half-extent x (-1 = never culled; depth is in depth_keys)
 *   trec   [F][24] 32-bit words: X0 Y0 X1 Y1 X2 Y2 (int32, 1/256 px, after
 *          the orientation swap), shading kind, alpha bits, z0 z1 z2 depth,
 *          then 9 attribute floats, then padding
 *   rects  [N+F][2] uint32 packed tile rect: x0 | y0 << 16, x1 | y1 << 16
 *   touched[N+F] uint32 tiles touched (0 = culled), unified id order
 *   depth_keys [N+F] uint32 bits(depth) (0xFFFFFFFF = culled)            */
UNIMGS_API int unimgs_get_records(unimgs_ctx *c, float *grec, uint32_t *trec, uint32_t *rects, uint32_t *touched,
                       uint32_t *depth_keys, void *stream);

/* End-to-end convenience path over HOST buffers: copies the scene (host
 * arrays in g_host / m_host; pinned memory gives async copies) into
 * context-owned device buffers, renders n_views cameras, and copies each
 * frame to out_host [n_views][H][W][4] float32 (all cameras must share one
 * size).  Synchronises before returning.  Allocates the staging buffers on
 * first use or growth (so not graph-capturable). */
UNIMGS_API int unimgs_render_host(unimgs_ctx *c, const unimgs_gaussians *g_host, const unimgs_mesh *m_host,
                       const unimgs_camera *cams, int32_t n_views, float *out_host, void *stream);

/* Pipelined form of unimgs_render_host: enqueues the same work and returns
 * without synchronising.  The context keeps two device copies of the scene,
 * so the host->device upload of this call (on an internal copy stream) runs
 * while the previous call still renders on `stream`, and the frame read-backs
 * run on a third stream.  Each view's preprocess + bin run on an internal
 * highest-priority stream of its lane (joined to `stream` by events), so the
 * latency-bound sort of one lane is scheduled ahead of the queued blend CTAs
 * of another.  The host input arrays and out_host must stay valid
 * and unmodified until unimgs_host_wait returns (or, for the inputs, until
 * the call after next has been issued).  Capacity overflow is reported by
 * unimgs_host_wait.  unimgs_render_host == render_host_async + host_wait. */
UNIMGS_API int unimgs_render_host_async(unimgs_ctx *c, const unimgs_gaussians *g_host, const unimgs_mesh *m_host,
                                        const unimgs_camera *cams, int32_t n_views, float *out_host, void *stream);

/* (render_host_async validates every host pointer, count and camera before it
 * enqueues anything; cov3d, when given, is uploaded in place of quats/scales.)
 *
 * Render lanes of the host path (1..8, default 1): lanes - 1 child contexts,
 * each with the reserved scratch and its own stream, render the views of a
 * unimgs_render_host[_async] call round-robin from the shared uploaded scene
 * (independent views overlap one view's latency-bound binning with another's
 * blend).  Must follow unimgs_reserve (re-call after growing); allocates and
 * synchronises. */
UNIMGS_API int unimgs_set_host_lanes(unimgs_ctx *c, int32_t lanes);

/* Wait for every unimgs_render_host_async call of this context (uploads,
 * renders, read-backs); UNIMGS_ERR_CAPACITY if ANY view rendered since the
 * previous wait overflowed max_pairs (a device flag that only this call
 * clears): the frames of that batch in out_host are then not all valid. */
UNIMGS_API int unimgs_host_wait(unimgs_ctx *c);

/* Checked build only (libunimgs_checked.so, -DUNIMGS_CHECKED: device bounds
 * checks that trap on a violated index, and a 4 KiB guard band after every
 * context scratch buffer): synchronises the device and writes to *bad_bytes
 * (host) the number of guard bytes overwritten, over this context and its host
 * lanes.  The production library returns UNIMGS_ERR_UNSUPPORTED. */
UNIMGS_API int unimgs_debug_check_guards(unimgs_ctx *c, int64_t *bad_bytes);

/* Number of kernel launches enqueued by this context since creation. */
UNIMGS_API int64_t unimgs_launch_count(const unimgs_ctx *c);

/* Last error message of the context (never NULL). */
UNIMGS_API const char *unimgs_error_string(const unimgs_ctx *c);

UNIMGS_API void unimgs_destroy(unimgs_ctx *c);

#ifdef __cplusplus
}
#endif
#endif /* UNIMGS_H */
