// internal.cuh -- device-side data layout and launch interface of libunimgs.
// Shared by the .cu files of the CUDA path only (never by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace unimgs {

// Bounds checks of the checked build (-DUNIMGS_CHECKED, paper_2601_19233_b200/
// libunimgs_checked.so): a violated index trap-kills the kernel with a message, so
// the launch fails loudly.  Compiled out of the production library.
#ifdef UNIMGS_CHECKED
#define UNIMGS_CHECK(c)                                                                                    \
    do {                                                                                                   \
        if (!(c)) {                                                                                        \
            printf("UNIMGS_CHECK failed: %s (%s:%d, block %d thread %d)\n", #c, __FILE__, __LINE__,        \
                   (int)blockIdx.x, (int)threadIdx.x);                                                     \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
#define UNIMGS_CHECK(c) \
    do {                \
    } while (0)
#endif

constexpr int kTile = 16;
// B1's visible counts (Buffers::bcnt) are per run of kGaussRun Gaussians (B2's: per 256 triangles)
constexpr int kGaussRunLog2 = 10, kGaussRun = 1 << kGaussRunLog2;
constexpr int kBlendThreads = 256;
constexpr int kMaxPasses = 8;

// Per-frame device counters.  frame_epoch survives across frames (it tags
// decoupled-look-back entries so the look-back buffers never need clearing) and so
// do overflow_sticky and the capacities; everything from n_vis on is zeroed by
// k_begin_frame.
struct DevState {
    unsigned int frame_epoch;
    unsigned int overflow_sticky;  // set by any frame that overflowed; cleared only by unimgs_host_wait
    // capacities written by unimgs_reserve (read by the UNIMGS_CHECKED bounds checks)
    unsigned int cap_prims, cap_pairs, cap_tiles, cap_rstart;
    unsigned int n_vis;         // visible primitives (compacted) -- first field k_begin_frame zeroes
    unsigned int K;             // pairs written (0 on overflow)
    unsigned long long needed;  // pairs required (saturating at 2^32-1)
    unsigned int overflow;
    unsigned int vis_g, vis_t, culled_guard;
    unsigned int ctr[16];       // dynamic tile counters of the scans / sort passes
    unsigned int hist[kMaxPasses][256];
    unsigned int max_tile_pairs, max_tile_id;
    unsigned long long work[4];  // blend work counters (counting variant only)
};

// Camera + the per-frame constants every stage needs.
struct CamParams {
    int W, H, tiles_x, tiles_y;
    float fx, fy, cx, cy;
    float R[9], t[3];
    float near_z, far_z;
    float campos[3];
    float lx, ly;  // N4 clamp limits 1.3 (W/2) / fx, 1.3 (H/2) / fy (fp32, computed on the host)
};

// Triangle record, 96 B (6 x 16 B), written by B2 and read by B8:
//   q0 int4   {X0, Y0, X1, Y1}          snapped 1/256-px coords after orientation
//   q1 int4   {X2, Y2, kind, alpha bits} kind 1 = textured (uv), 0 = vertex colours, 2 = white
//   q2 float4 {z0, z1, z2, depth}       view z per vertex; sort depth
//   q3 float4 {a0.x, a0.y, a0.z, a1.x}  shading attributes per vertex (uv,0 or rgb)
//   q4 float4 {a1.y, a1.z, a2.x, a2.y}
//   q5 float4 {a2.z, 0, 0, 0}
struct TriRecord {
    int4 q0, q1;
    float4 q2, q3, q4, q5;
};

// Gaussian record, 48 B: {u, v, q_max, o}, {ca, cb, cc, cull_ey}, {r, g, b, cull_ex}
// (cull_e* = half-extents of the blend's exact per-warp culling, -1 = never cull).
struct GaussRecord {
    float4 a, b, c;
};

struct Buffers {
    // per primitive, unified id (triangles 0..F-1, Gaussians F..F+N-1)
    uint2 *rect;          // x0 | y0 << 16, x1 | y1 << 16
    uint32_t *touched;
    uint32_t *dkey;       // bits(depth), 0xFFFFFFFF if culled
    GaussRecord *grec;    // [N]
    TriRecord *trec;      // [F]
    // sort buffers
    uint32_t *pk[2];      // depth keys ping-pong [max_prims]
    uint32_t *pv[2];      // primitive ids ping-pong [max_prims]
    void *tk[2];          // pair keys ping-pong (uint16 tile ids, or uint64 full keys) [max_pairs]
    uint32_t *tv[2];      // pair values ping-pong [max_pairs]
    uint2 *ranges;        // [tiles]
    uint32_t *order;      // [tiles] blend schedule: tiles by decreasing pair count (approx., k_tile_order)
    uint32_t *bcnt;       // per-CTA visible counts of B2 then B1 (256 primitives each), scanned in place
    uint32_t *dcnt;       // per-CTA pair counts of the duplication (2048 primitives each), scanned in place
    uint32_t *rstart;     // [max_pairs / 1024 + 2] first primitive of each expansion range (k_range_starts)
    unsigned long long *lookback;  // [max_lb_tiles][256]
    uint32_t *tcnt;       // [max_lb_tiles][256] per sort tile (2048 pairs) digit counts -> exclusive within group
    uint32_t *gsum;       // [max_lb_tiles / 32 + 2][256] per group of 32 sort tiles -> exclusive; then totals
    DevState *st;
    int64_t max_prims, max_pairs, max_tiles, max_lb_tiles;
    const uint32_t *sorted_vals;   // final per-tile lists (points into tv[*])
    const void *sorted_keys;       // final keys (tk[*])
    int key_bytes;                 // 2 (factored) or 8 (full)
};

struct GaussInput {
    int64_t N;
    const float *means, *quats, *scales, *opac, *sh;
    int sh_degree;
    const float *cov3d;  // optional [N][6]: replaces quats/scales
};

struct DeformInput {
    int64_t N;
    const float *means, *quats, *scales, *cov3d;
    int K;                 // anchors per Gaussian
    const int32_t *face;   // [N][K]
    const float *bary;     // [N][K][3]
    int64_t F, V;
    const int32_t *faces;  // [F][3], vertex ids checked against [0, V)
    const float4 *vdata;   // per vertex 3 x float4: delta xyz + log_rot x | log_rot yz + shear xx xy | shear xz yy yz zz
};

struct MeshInput {
    int64_t V, F;
    const float *pos, *uvs, *cols, *opac;
    const int32_t *faces;
    const uint8_t *tex;
    int tw, th;
};

struct BlendParams {
    float alpha_max, t_eps, bg_alpha;
    float bg[3];
    int mode;   // unimgs_settings::blend_mode
    int msaa;   // M samples
    int resort; // tri_depth 2: the per-pixel resort window (k_blend_resort)
};

struct BindInput {
    int64_t N;
    const float *means, *quats, *scales;  // device
    int mode;                             // 0 = centre, 1 = bbx8
    float k_sigma;
    int ncams;
    const float *cams;                    // HOST [ncams][12]: R row-major, then t
    int64_t V, F;
    const float *pos;                     // device [V][3]
    const int32_t *faces;                 // device [F][3]
};

// Several views of one scene for the multi-view Gaussian preprocess (each view: its
// camera and its context's buffers).
constexpr int kMaxMultiViews = 4;
struct MultiView {
    int n;
    CamParams cam[kMaxMultiViews];
    Buffers buf[kMaxMultiViews];
};

// ---- launchers (return number of kernels enqueued) --------------------------
int launch_begin_frame(DevState *st, cudaStream_t s);
int launch_preprocess_gaussians(const GaussInput &g, int64_t F, const CamParams &cam, float dilation,
                                const Buffers &b, cudaStream_t s);
int launch_setup_triangles(const MeshInput &m, const CamParams &cam, const Buffers &b, cudaStream_t s);
int launch_preprocess_gaussians_multi(const GaussInput &g, int64_t F, const MultiView &mv, float dilation,
                                      cudaStream_t s);
// binning: factored (sort_mode 0) or full 64-bit keys (sort_mode 1)
// Look-back rows the sort passes need (one per sort tile of the largest pass).
int64_t sort_lookback_tiles(int64_t max_pairs, int64_t max_prims);
// sort_per_sm: persistent CTAs per SM of the sort passes (1..4; registers are capped
// at 64 so four fit beside nothing else, one leaves 3/4 of the SM to other streams)
int launch_bin(Buffers &b, int64_t P, int64_t N, int64_t F, const CamParams &cam, int sort_mode, int tri_depth,
               cudaStream_t s, int sm_count, int sort_per_sm);
// count_work: the counting variant (DevState::work); frag_counts (counting variant only,
// may be NULL): per pixel uint4 {Gaussian fragments blended, triangle fragments blended,
// id of the last fragment blended (0xFFFFFFFF: none), Gaussian entries tested}
int launch_blend(const Buffers &b, const GaussInput &g, const MeshInput &m, const CamParams &cam,
                 const BlendParams &bp, float *out, cudaStream_t s, bool count_work = false,
                 uint32_t *frag_counts = nullptr);
int launch_tile_stats(const Buffers &b, int tiles, cudaStream_t s);
int launch_deform(const DeformInput &d, float *mu_out, float *cov_out, cudaStream_t s);
// ray-cast binding (bind.cu): builds an LBVH in stream-ordered scratch; -1 if that allocation fails
int launch_bind(const BindInput &in, int32_t *face_out, float *bary_out, double *dist2_out, cudaStream_t s);
int launch_full_keys(const Buffers &b, uint64_t *keys, cudaStream_t s);
// stable LSD sort of (u32 key, u32 value) pairs in keys[0]/vals[0] (binning.cu's onesweep);
// st zeroed with n_vis = n, lookback zeroed with sort_lookback_tiles(n, n) rows
int launch_sort_u32_pairs(uint32_t *keys[2], uint32_t *vals[2], int64_t n, DevState *st, unsigned long long *lookback,
                          int sm_count, cudaStream_t s);

}  // namespace unimgs
