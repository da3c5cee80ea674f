// blend.cu -- B8: the unified single-pass anti-aliased blend (§3.2).
//
// One warp per 8x4 sub-tile of a 16x16 tile (8 per tile, handed out as work items
// in runs per CTA), one pixel per lane; each warp walks its tile's sorted list
// (unified ids, (tile, depth, id) order) independently:
// records are gathered with 16-byte loads, culled exactly against the warp's
// 8x4 sub-tile, packed into a per-warp shared buffer and blended in list
// order; triangle entries are resolved from their 96-byte setup record
// (broadcast loads: every lane reads the same address).
//
// Per pixel (state machine of DESIGN.md §2 / the oracle):
//   Gaussian fragment  iff q <= q_max (N6, bit-exact with the oracle):
//       close an open entity (T = T_e * mean_j t_j, reading R3),
//       alpha = min(alpha_max, o e^{-q/2}); C += T alpha c; T *= 1 - alpha  (Eq.1-2)
//   triangle fragment  iff its M-sample coverage mask m != 0 (exact int64
//       edge functions, top-left rule, D3D patterns, M = 4 by default; N7, R10-R11):
//       open an entity if none (T_e = T, t_j = 1; Eq.7), O = sum_j m_j t_j / 4
//       (Eq.8), C += T_e O alpha c (Eq.9), t_j *= 1 - m_j alpha (Eq.7)
//   stop once T_eff < t_eps (blend-then-test, R16); a warp exits when all of
//   its pixels have stopped.
//   out = (C + T bg_alpha bg, T) with the exit T of an open entity (R3, R5).
// Triangle colour: perspective-correct barycentrics at the pixel centre in
// fp32 (w_k = E_k z_i z_j), manual fp32 bilinear texture (colour tolerance 1e-3).
#include "internal.cuh"

namespace unimgs {

struct TexView {
    const uchar4 *tex;
    int w, h;
};

__device__ __forceinline__ float4 texel(const TexView &t, int i, int j) {
    i = min(max(i, 0), t.w - 1);
    j = min(max(j, 0), t.h - 1);
    const uchar4 c = __ldg(t.tex + (size_t)j * t.w + i);
    return make_float4(c.x, c.y, c.z, c.w);
}

// Direct3D standard multisample patterns, 1/16 px from the pixel centre (R10);
// M = 4 is the paper's setting.
template <int M>
__device__ __forceinline__ void sample_offset(int j, int &ox, int &oy) {
    if (M == 1) { ox = 0; oy = 0; return; }
    if (M == 2) {
        constexpr int P[2][2] = {{4, 4}, {-4, -4}};
        ox = P[j][0]; oy = P[j][1]; return;
    }
    if (M == 4) {
        constexpr int P[4][2] = {{-2, -6}, {6, -2}, {-6, 2}, {2, 6}};
        ox = P[j][0]; oy = P[j][1]; return;
    }
    if (M == 8) {
        constexpr int P[8][2] = {{1, -3}, {-1, 3}, {5, 1}, {-3, -5}, {-5, 5}, {-7, -1}, {3, 7}, {7, -7}};
        ox = P[j][0]; oy = P[j][1]; return;
    }
    constexpr int P[16][2] = {{1, 1}, {-1, -3}, {-3, 2}, {4, -1}, {-5, -2}, {2, 5}, {5, 3}, {3, -5},
                              {-2, 6}, {0, -7}, {-4, -6}, {-6, 4}, {-8, 0}, {7, -4}, {6, 7}, {-7, -8}};
    ox = P[j][0]; oy = P[j][1];
}

// M-sample coverage mask of a triangle record at pixel (x, y): sample j at
// (256x + 128 + 16 ox_j, 256y + 128 + 16 oy_j) in 1/256 px; exact int64 edge
// functions with the top-left-style rule (N7, R11).  Ec = edge functions at the centre.
template <int M>
__device__ __forceinline__ unsigned coverage(const int X[3], const int Y[3], int x, int y, long long Ec[3]) {
    const int PX = 256 * x + 128, PY = 256 * y + 128;
    unsigned m = (M == 32) ? 0xFFFFFFFFu : ((1u << M) - 1u);
    // int32 path when the pixel centre is within 64 px of every vertex: |dx|, |dy| < 2^15
    // and |P - V| < 2^14, so each edge value is below 2^30 and a sample offset below 2^24
    // -- the same integers as the int64 evaluation below, without its wide multiplies
    const unsigned near = (unsigned)(abs(PX - X[0]) | abs(PX - X[1]) | abs(PX - X[2]) | abs(PY - Y[0]) |
                                     abs(PY - Y[1]) | abs(PY - Y[2]));
    if (near < 16384u) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const int a = (k + 1) % 3, b = (k + 2) % 3;
            const int dx = X[b] - X[a], dy = Y[b] - Y[a];
            const int e = dx * (PY - Y[a]) - dy * (PX - X[a]);
            Ec[k] = e;
            const int thr = (dy > 0 || (dy == 0 && dx < 0)) ? 0 : 1;
            unsigned mk = 0;
#pragma unroll
            for (int j = 0; j < M; j++) {
                int ox, oy;
                sample_offset<M>(j, ox, oy);
                mk |= (e + 16 * (dx * oy - dy * ox) >= thr ? 1u : 0u) << j;
            }
            m &= mk;
        }
        return m;
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const int a = (k + 1) % 3, b = (k + 2) % 3;
        const int dx = X[b] - X[a], dy = Y[b] - Y[a];
        // E_k(P) = dx (PY - Ya) - dy (PX - Xa) at the centre, then per-sample offsets 16 (dx oy - dy ox)
        const long long e = (long long)dx * (PY - Y[a]) - (long long)dy * (PX - X[a]);
        Ec[k] = e;
        const long long thr = (dy > 0 || (dy == 0 && dx < 0)) ? 0 : 1;
        unsigned mk = 0;
#pragma unroll
        for (int j = 0; j < M; j++) {
            int ox, oy;
            sample_offset<M>(j, ox, oy);
            const long long ej = e + 16LL * ((long long)dx * oy - (long long)dy * ox);
            mk |= (ej >= thr ? 1u : 0u) << j;
        }
        m &= mk;
    }
    return m;
}

// Colour of a covered triangle at the pixel centre (R12): perspective-correct,
// unclamped barycentrics from the exact centre edge functions, in fp32 (colour
// only has to meet the 1e-3 tolerance; w_k = E_k z_i z_j has ~6e-8 relative
// error, far below it), bilinear texture in fp32.
// The record's depth/attribute words q2..q5, staged in shared memory by cp.async.
struct TriAttr {
    float4 q2, q3, q4, q5;
};

__device__ __forceinline__ void tri_colour(const TriAttr &r, int kind, const long long Ec[3], const TexView &tv,
                                           float rgb[3]) {
    const float z0 = r.q2.x, z1 = r.q2.y, z2 = r.q2.z;
    // w_k = b_k / z_k  ~  E_k * (product of the other two z)
    const float w0 = (float)Ec[0] * (z1 * z2), w1 = (float)Ec[1] * (z0 * z2), w2 = (float)Ec[2] * (z0 * z1);
    const float sw = w0 + w1 + w2;
    float l0, l1, l2;
    if (sw != 0.0f) {
        const float is = 1.0f / sw;
        l0 = w0 * is; l1 = w1 * is; l2 = w2 * is;
    } else {
        const float iA = 1.0f / (float)(Ec[0] + Ec[1] + Ec[2]);
        l0 = (float)Ec[0] * iA; l1 = (float)Ec[1] * iA; l2 = (float)Ec[2] * iA;
    }
    if (kind == 1) {
        const float uu = l0 * r.q3.x + l1 * r.q3.w + l2 * r.q4.z;
        const float vv = l0 * r.q3.y + l1 * r.q4.x + l2 * r.q4.w;
        const float txd = uu * (float)tv.w - 0.5f, tyd = vv * (float)tv.h - 0.5f;
        const float fi = floorf(txd), fj = floorf(tyd);
        const float ax = txd - fi, ay = tyd - fj;
        // clamp before converting so huge coordinates stay defined
        const int i0 = (int)fminf(fmaxf(fi, -2.0f), (float)tv.w + 1.0f);
        const int j0 = (int)fminf(fmaxf(fj, -2.0f), (float)tv.h + 1.0f);
        const float4 t00 = texel(tv, i0, j0), t10 = texel(tv, i0 + 1, j0);
        const float4 t01 = texel(tv, i0, j0 + 1), t11 = texel(tv, i0 + 1, j0 + 1);
        const float s = 1.0f / 255.0f;
        rgb[0] = ((1.f - ay) * ((1.f - ax) * t00.x + ax * t10.x) + ay * ((1.f - ax) * t01.x + ax * t11.x)) * s;
        rgb[1] = ((1.f - ay) * ((1.f - ax) * t00.y + ax * t10.y) + ay * ((1.f - ax) * t01.y + ax * t11.y)) * s;
        rgb[2] = ((1.f - ay) * ((1.f - ax) * t00.z + ax * t10.z) + ay * ((1.f - ax) * t01.z + ax * t11.z)) * s;
    } else if (kind == 0) {
        const float c0 = l0 * r.q3.x + l1 * r.q3.w + l2 * r.q4.z;
        const float c1 = l0 * r.q3.y + l1 * r.q4.x + l2 * r.q4.w;
        const float c2 = l0 * r.q3.z + l1 * r.q4.y + l2 * r.q5.x;
        rgb[0] = fminf(fmaxf(c0, 0.0f), 1.0f);
        rgb[1] = fminf(fmaxf(c1, 0.0f), 1.0f);
        rgb[2] = fminf(fmaxf(c2, 0.0f), 1.0f);
    } else {
        rgb[0] = rgb[1] = rgb[2] = 1.f;
    }
}

// Exact per-warp culling (never drops a fragment of a live pixel).  Warp w owns
// the 8x4 sub-tile (w & 1, w >> 1) of the 16x16 tile; the culling rectangle is
// the bounding box of the sub-tile's pixels that have not terminated yet (it
// shrinks as pixels finish: a finished pixel consumes no entry), and an entry
// is skipped by the warp only when no pixel of that box can hold the fragment:
//   triangle: its snapped integer bbox misses the box's 1/256-px extent;
//   Gaussian: the box's pixel centres lie outside the bbox of the exact
//   ellipse {d : Q(d) <= q_max (1 + 0.02)} of the fp32 conic Q, padded by
//   1% + 0.01 px (half-extents computed once per Gaussian in B1).  Only for
//   cond(Q) <= ~1000, where the fp32 evaluation of q (10 roundings,
//   cancellation factor <= 2(cond + 1)) errs by < 1.3e-3 q, so a pixel outside
//   that ellipse cannot satisfy the N6 test q <= q_max.  Other conics
//   (needles, NaN) are never skipped.
// The box: pixel-centre extents [cx0, cx1] x [cy0, cy1] (px) and the covered
// 1/256-px extents [X0, X1] x [Y0, Y1] of the live pixels.
struct LiveBox {
    float cx0, cx1, cy0, cy1;
    int X0, X1, Y0, Y1;
};

__device__ __forceinline__ bool gauss_touches(const float4 &a, const float4 &b, const float4 &c, const LiveBox &lb) {
    const float ex = c.w, ey = b.w;  // precomputed in B1; -1 = never cull
    if (!(ex >= 0.f)) return true;
    return a.x + ex >= lb.cx0 && a.x - ex <= lb.cx1 && a.y + ey >= lb.cy0 && a.y - ey <= lb.cy1;
}

__device__ __forceinline__ bool tri_touches(const float4 &a, const float4 &b, const LiveBox &lb) {
    const int X0 = __float_as_int(a.x), Y0 = __float_as_int(a.y), X1 = __float_as_int(a.z), Y1 = __float_as_int(a.w);
    const int X2 = __float_as_int(b.x), Y2 = __float_as_int(b.y);
    const int mnx = min(X0, min(X1, X2)), mxx = max(X0, max(X1, X2));
    const int mny = min(Y0, min(Y1, Y2)), mxy = max(Y0, max(Y1, Y2));
    return mxx >= lb.X0 && mnx <= lb.X1 && mxy >= lb.Y0 && mny <= lb.Y1;
}

__device__ __forceinline__ float lg2_ftz(float x) {  // x = o >= 1/255: never subnormal
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// blend modes (the paper's ablation, Fig.3 / Fig.4)
enum { MODE_EXACT = 0, MODE_NAIVE = 1, MODE_MSAA_PIXEL = 2, MODE_WHOLE_PIXEL = 3, MODE_PAPER_LITERAL = 4 };

// Per-pixel blend state (registers).  G / Tl only exist for the modes that use them.
// While an entity is open, T holds its exit transmittance (R3: refreshed by every
// triangle) and Tlast a copy of it: any Gaussian fragment (alpha >= 1/255) lowers T,
// so "the entity is still open" is exactly T == Tlast and the Gaussian path keeps
// no entity state at all.  (T == 0 would stay "open", which changes nothing: every
// later contribution is then 0 either way.)  The whole-pixel ablation mode, whose
// Gaussians do not close the entity, keeps an explicit flag.  A finished pixel is
// marked by py = NaN: its Gaussian test q <= q_max then fails by itself.
template <int MODE, int M>
struct Px {
    float C0, C1, C2, T, Te;
    float t[M];
    float G, Tl;
    float Tlast;  // T after the last triangle fragment (NaN: none yet)
    float py;     // pixel centre y for the Gaussian test; NaN once done
    bool open;    // MODE_WHOLE_PIXEL only
    __device__ __forceinline__ bool done() const { return py != py; }
    __device__ __forceinline__ void finish() { py = __int_as_float(0x7fc00000); }
    __device__ __forceinline__ float mean_t() const {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < M; j++) a += t[j];
        return a * (1.f / M);
    }
    // transmittance leaving the entity (R3; Eq.6 product for the paper-literal mode)
    __device__ __forceinline__ float exit_T() const {
        if (MODE == MODE_PAPER_LITERAL) return Tl;
        if (MODE == MODE_WHOLE_PIXEL) return Te * mean_t() * G;
        return Te * mean_t();
    }
};

template <int M>
__device__ __forceinline__ float popc_frac(unsigned m) {
    return (float)__popc(m) * (1.f / M);
}

// One triangle fragment candidate at pixel (x, y): coverage, then the mode's update
// (exact: Eq.7-9 in a depth-adjacent entity).
// X, Y, kind and alpha come from the warp's staged entry; the rest of the record
// (depths, attributes) arrives in shared memory by cp.async at packing time.
template <bool COUNT, int MODE, int M>
__device__ __forceinline__ void tri_pixel(Px<MODE, M> &s, const int X[3], const int Y[3], int kind, float al,
                                          const TriAttr &r, int x, int y, const TexView &tv, float t_eps,
                                          unsigned long long &w_tt, unsigned long long &w_tf) {
    long long Ec[3];
    if (COUNT) w_tt++;
    {   // exact pre-test: no sample (centre +- 16 R in 1/256 px) can lie in the triangle's bbox
        constexpr int R16 = 16 * (M == 1 ? 0 : M == 2 ? 4 : M == 4 ? 6 : M == 8 ? 7 : 8);
        const int PX = 256 * x + 128, PY = 256 * y + 128;
        if (PX + R16 < min(X[0], min(X[1], X[2])) || PX - R16 > max(X[0], max(X[1], X[2])) ||
            PY + R16 < min(Y[0], min(Y[1], Y[2])) || PY - R16 > max(Y[0], max(Y[1], Y[2])))
            return;
    }
    const unsigned m = coverage<M>(X, Y, x, y, Ec);
    if (!m) return;
    if (COUNT) w_tf++;
    float rgb[3];
    tri_colour(r, kind, Ec, tv, rgb);
    if (MODE == MODE_NAIVE || MODE == MODE_MSAA_PIXEL) {
        const float O = MODE == MODE_NAIVE ? 1.f : popc_frac<M>(m);  // full / geometric coverage (Eq.5-6)
        const float w = s.T * O * al;
        s.C0 += w * rgb[0]; s.C1 += w * rgb[1]; s.C2 += w * rgb[2];
        s.T -= w;
        if (s.T < t_eps) s.finish();
        return;
    }
    const bool open = MODE == MODE_WHOLE_PIXEL ? s.open : s.T == s.Tlast;
    if (!open) {
        s.open = true;
        s.Te = s.T;
        s.G = 1.f;
        s.Tl = s.T;
#pragma unroll
        for (int j = 0; j < M; j++) s.t[j] = 1.f;
    }
    float O = 0.f;
#pragma unroll
    for (int j = 0; j < M; j++) O += ((m >> j) & 1u) ? s.t[j] : 0.f;
    O *= 1.f / M;  // Eq.8
    const float w = s.Te * O * al;  // Eq.9
    s.C0 += w * rgb[0]; s.C1 += w * rgb[1]; s.C2 += w * rgb[2];
    const float kk = 1.f - al;
#pragma unroll
    for (int j = 0; j < M; j++)
        if ((m >> j) & 1u) s.t[j] *= kk;  // Eq.7
    if (MODE == MODE_PAPER_LITERAL) s.Tl *= 1.f - popc_frac<M>(m) * al;
    s.T = s.exit_T();  // T_eff (and the T a closing Gaussian continues from)
    s.Tlast = s.T;
    if (s.T < t_eps) s.finish();
}

// Packed f32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2, one issue slot for two
// IEEE round-to-nearest fp32 operations -- per element identical to __fadd_rn etc.,
// so N6 stays bit-exact).  The pair lives in one 64-bit register.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 r, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Per-warp packed entry buffer.  Entries 2p and 2p+1 form pair p; a pair's 80 bytes
// are contiguous (one pointer walks the buffer), stored structure-of-arrays so that
// one 16-byte shared load yields f32x2 operands:
//   v[p][0] = {u0, u1, v0, v1}        (triangle: X0, Y0 bits)
//   v[p][1] = {ca0, ca1, cc0, cc1}    (triangle: X1, Y1 bits)
//   v[p][2] = {2cb0, 2cb1, qm0, qm1}  (triangle: X2 bits, q_max = -1; padding: NaN)
//   v[p][3 + j] = col(2p + j) = {r, g, b, log2 o}  (triangle: Y2 bits, kind, alpha, id)
struct WarpBuf {
    float4 v[16][5];
    __device__ __forceinline__ float4 &col(unsigned k) { return v[k >> 1][3 + (k & 1)]; }
};
constexpr int kPairFloats = 20;  // floats per pair in WarpBuf

// 8 independent warps per CTA, one pixel per lane.  A warp's item (tile, w) is the
// 8x4 sub-tile (w & 1, w >> 1); it walks the whole tile list in chunks of 32
// entries (lane l <-> entry 32c + l):
//   1. the chunk's records (48 B per Gaussian, the first 32 B per triangle) were
//      copied by cp.async into the warp's stage while the previous chunk was
//      blended (ids are prefetched one chunk further ahead, in registers);
//   2. each lane culls its entry exactly against the warp's sub-tile, a ballot
//      ranks the survivors, which are packed into the warp's pair buffer;
//   3. the next chunk's records are requested (cp.async, no registers held);
//   4. the packed entries are tested four at a time (two f32x2 pairs) and the
//      hits blended in list order.
// No block-wide barrier: a warp stops as soon as all of its pixels have terminated.
// The (tile, sub-tile) items, in the longest-first tile order (k_tile_order), are
// dealt to CTAs in runs of items_per_cta (several tiles of similar length); inside a
// run each warp takes the next item when it is done with its last (a shared-memory
// counter), so the warps of a CTA end together and an SM slot is not held by one
// slow sub-tile while its other warps idle.
#ifndef UNIMGS_BLEND_CTA_WARPS
#define UNIMGS_BLEND_CTA_WARPS 8  // warps per k_blend CTA (any number: the items are (tile, sub-tile))
#endif
#ifndef UNIMGS_BLEND_MINB
#define UNIMGS_BLEND_MINB (32 / UNIMGS_BLEND_CTA_WARPS)  // 64 registers: 32 warps per SM
#endif
constexpr int kBlendCtaThreads = 32 * UNIMGS_BLEND_CTA_WARPS, kSubTiles = 8;  // 8 x (8x4) per 16x16 tile
template <bool COUNT, int MODE, int M>
__global__ void __launch_bounds__(kBlendCtaThreads, UNIMGS_BLEND_MINB) k_blend(const uint2 *__restrict__ ranges,
                                                                     const uint32_t *__restrict__ order,
                                                                     const uint32_t *__restrict__ vals,
                                                                     const GaussRecord *__restrict__ grec,
                                                                     const TriRecord *__restrict__ trec, TexView tv,
                                                                     unsigned F, int W, int H, int tiles_x,
                                                                     unsigned n_items, int items_per_cta,
                                                                     BlendParams bp, float4 *__restrict__ out,
                                                                     DevState *st, uint4 *__restrict__ frag_counts) {
    if (st->overflow) return;
    constexpr int NW = UNIMGS_BLEND_CTA_WARPS;  // warps per CTA
    __shared__ unsigned s_ids[COUNT ? NW : 1][32];  // COUNT only: packed entry k's id
    __shared__ WarpBuf s_buf[NW];
    __shared__ float4 s_stage[NW][32][3];  // this lane's record of the next chunk (cp.async)
    __shared__ TriAttr s_tri[NW][32];      // a packed triangle entry's q2..q5 (cp.async)
    __shared__ __align__(16) LiveBox s_lb[NW];
    __shared__ int s_next;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    WarpBuf &wb = s_buf[warp];
    float *ef = &wb.v[0][0].x;
    TriAttr *tat = s_tri[warp];
    float4 *stg = s_stage[warp][lane];
    const unsigned stg_s = (unsigned)__cvta_generic_to_shared(stg);
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();

    for (;;) {
    unsigned item = 0xFFFFFFFFu;
    if (lane == 0) {
        const int j = atomicAdd(&s_next, 1);
        if (j < items_per_cta) item = blockIdx.x * (unsigned)items_per_cta + (unsigned)j;
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int sub = (int)(item % kSubTiles);
    // COUNT only: per lane (= per pixel) Gaussian / triangle entries tested and fragments
    // blended, and the unified id of the last fragment blended
    unsigned long long w_gt = 0, w_gf = 0, w_tt = 0, w_tf = 0;
    unsigned last_id = 0xFFFFFFFFu;
    const int tile = (int)__ldg(order + item / kSubTiles);  // longest-first schedule (k_tile_order)
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int sx0 = tx * kTile + (sub & 1) * 8, sy0 = ty * kTile + (sub >> 1) * 4;
    const int x = sx0 + (lane & 7), y = sy0 + (lane >> 3);
    const float px = (float)x + 0.5f;
    const uint2 rg = ranges[tile];
    UNIMGS_CHECK((unsigned)tile < st->cap_tiles && rg.x <= rg.y && rg.y <= st->K);

    Px<MODE, M> s;
    s.C0 = s.C1 = s.C2 = 0.f;
    s.T = s.Te = s.G = s.Tl = 1.f;
#pragma unroll
    for (int j = 0; j < M; j++) s.t[j] = 1.f;
    s.open = false;
    s.Tlast = __int_as_float(0x7fc00000);
    s.py = (float)y + 0.5f;
    if (!(x < W && y < H)) s.finish();

    // cp.async of entry id's record into this lane's stage slot (Gaussian 48 B,
    // triangle q0/q1 32 B); always commits one group
    auto stage_rec = [&](unsigned id) {
        if (id != 0xFFFFFFFFu) {
            const char *src = id >= F ? reinterpret_cast<const char *>(grec + (id - F))
                                      : reinterpret_cast<const char *>(trec + id);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s), "l"(src) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s + 16), "l"(src + 16) : "memory");
            if (id >= F)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s + 32), "l"(src + 32) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    unsigned id0 = rg.x + lane < rg.y ? __ldg(vals + rg.x + lane) : 0xFFFFFFFFu;
    unsigned id1 = rg.x + 32 + lane < rg.y ? __ldg(vals + rg.x + 32 + lane) : 0xFFFFFFFFu;
    stage_rec(id0);
    const float kexp = -0.72134752044448170f;  // -log2(e) / 2

    // Eq.1-2 blend of Gaussian fragment k (membership already decided bit-exactly):
    // alpha = min(alpha_max, o e^{-q/2}) = min(alpha_max, 2^(q kexp + log2 o))
    auto gblend = [&](float q, unsigned k) {
        if (COUNT) {
            w_gf++;
            last_id = s_ids[COUNT ? warp : 0][k];
        }
        const float4 ec = wb.col(k);
        const float al = fminf(bp.alpha_max, ex2_ftz(fmaf(q, kexp, ec.w)));
        if (MODE == MODE_WHOLE_PIXEL && s.open) {
            // Fig.3b/c: the entity spans the whole list; the Gaussian does not
            // attenuate its sub-pixel state (colour overflow)
            const float base = s.Te * s.mean_t();
            const float w = base * s.G * al;
            s.C0 += w * ec.x; s.C1 += w * ec.y; s.C2 += w * ec.z;
            s.G *= 1.f - al;
            if (base * s.G < bp.t_eps) s.finish();
            return;
        }
        // depth adjacency broken: T already holds the entity's exit T (R3),
        // and lowering it closes the entity (T != Tlast)
        const float w = s.T * al;
        s.C0 += w * ec.x; s.C1 += w * ec.y; s.C2 += w * ec.z;
        s.T -= w;
        if (s.T < bp.t_eps) s.finish();
    };
    // N6 for the two entries of pair p at this lane's pixel:
    //   dx = (x + .5) - u; dy = (y + .5) - v; q = fma(ca, dx dx, fma(cc, dy dy, 2cb (dx dy)))
    // (py is NaN once the pixel is done, so its q is NaN and no test passes)
    auto qpair = [&](unsigned p, float &q0, float &q1, float &m0, float &m1) {
        const float4 A = wb.v[p][0], B = wb.v[p][1], Cc = wb.v[p][2];
        const f32x2 dx = sub2(pk2(px, px), pk2(A.x, A.y));
        const f32x2 dy = sub2(pk2(s.py, s.py), pk2(A.z, A.w));
        const f32x2 t = fma2(pk2(B.z, B.w), mul2(dy, dy), mul2(pk2(Cc.x, Cc.y), mul2(dx, dy)));
        upk2(fma2(pk2(B.x, B.y), mul2(dx, dx), t), q0, q1);
        m0 = Cc.z;
        m1 = Cc.w;
    };

    unsigned live_prev = 0;
    for (unsigned base = rg.x; base < rg.y; base += 32) {
        // the live pixels' bounding box (lane = 8 row + column), kept in shared memory
        // and recomputed only when a pixel of the warp has terminated
        const unsigned live = __ballot_sync(0xffffffffu, !s.done());
        if (!live) break;
        if (live != live_prev) {
            live_prev = live;
            const unsigned cols = (live | (live >> 8) | (live >> 16) | (live >> 24)) & 0xFFu;
            const int c0 = __ffs(cols) - 1, c1 = 31 - __clz(cols);
            const int r0 = (__ffs(live) - 1) >> 3, r1 = (31 - __clz(live)) >> 3;
            if (lane == 0) {
                LiveBox &w = s_lb[warp];
                w.cx0 = (float)(sx0 + c0) + 0.5f;
                w.cx1 = (float)(sx0 + c1) + 0.5f;
                w.cy0 = (float)(sy0 + r0) + 0.5f;
                w.cy1 = (float)(sy0 + r1) + 0.5f;
                w.X0 = 256 * (sx0 + c0);
                w.X1 = 256 * (sx0 + c1 + 1) - 1;
                w.Y0 = 256 * (sy0 + r0);
                w.Y1 = 256 * (sy0 + r1 + 1) - 1;
            }
            __syncwarp();
        }
        const LiveBox lb = s_lb[warp];
        const unsigned id = id0;
        id0 = id1;
        id1 = base + 64 + lane < rg.y ? __ldg(vals + base + 64 + lane) : 0xFFFFFFFFu;
        asm volatile("cp.async.wait_all;\n" ::: "memory");  // this chunk's records (own slot only)
        bool rel = false;
        float4 a, b, c;
        if (id != 0xFFFFFFFFu) {
            a = stg[0];
            b = stg[1];
            if (id >= F) {
                c = stg[2];
                rel = gauss_touches(a, b, c, lb);
            } else {
                rel = tri_touches(a, b, lb);
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, rel);
        const bool has_tri = __any_sync(0xffffffffu, rel && id < F);
        const unsigned cnt = __popc(bal);
        const unsigned slot = __popc(bal & lt);
        UNIMGS_CHECK(!rel || (slot < 32u && id < st->cap_prims));
        if (COUNT && rel) s_ids[COUNT ? warp : 0][slot] = id;
        if (rel) {
            float *e = ef + kPairFloats * (slot >> 1) + (slot & 1);
            if (id >= F) {
                e[0] = a.x; e[2] = a.y; e[4] = b.x; e[6] = b.z; e[8] = b.y + b.y; e[10] = a.z;
                wb.col(slot) = make_float4(c.x, c.y, c.z, lg2_ftz(a.w));
            } else {
                // triangle: the staged vertices, kind and alpha; q_max = -1 marks it
                e[0] = a.x; e[2] = a.y; e[4] = a.z; e[6] = a.w; e[8] = b.x; e[10] = -1.f;
                wb.col(slot) = make_float4(b.y, b.z, b.w, __uint_as_float(id));
                const char *src = reinterpret_cast<const char *>(&trec[id].q2);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&tat[slot]);
#pragma unroll
                for (int w = 0; w < 4; w++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * w), "l"(src + 16 * w)
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");  // this chunk's triangle attributes
        // padding up to a multiple of 4 entries: q_max = NaN fails every test, and a
        // zero colour keeps the predicated blend's 0 * colour finite
        const unsigned cnt4 = (cnt + 3) & ~3u;
        if (lane >= cnt && lane < cnt4) {
            ef[kPairFloats * (lane >> 1) + 10 + (lane & 1)] = __int_as_float(0x7fc00000);
            wb.col(lane) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncwarp();  // packing done, the stage slot is free again
        stage_rec(id0);  // next chunk's records land while this one is blended
        if (!has_tri && MODE != MODE_WHOLE_PIXEL) {
            // Gaussian-only chunk: four entries per iteration.  Membership of all four by
            // two f32x2 pairs, their alphas computed unconditionally (independent chains),
            // then Eq.1-2 as a predicated sequence: entry k blends iff it is a fragment
            // and the pixel has not terminated (T >= t_eps) -- blend-then-test, R16.
#pragma unroll 1
            for (unsigned p = 0; 2 * p < cnt; p += 2) {
                float q[4], m[4];
                qpair(p, q[0], q[1], m[0], m[1]);
                qpair(p + 1, q[2], q[3], m[2], m[3]);
                if (COUNT && !s.done()) w_gt += min(4u, cnt - 2 * p);
                float4 ec[4];
                float al[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    ec[k] = wb.col(2 * p + k);
                    al[k] = fminf(bp.alpha_max, ex2_ftz(fmaf(q[k], kexp, ec[k].w)));
                }
                f32x2 c01 = pk2(s.C0, s.C1);  // (R, G) accumulated as one f32x2 FFMA2
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    // (entry 0: a pixel already done has q = NaN, so no T test is needed)
                    const bool h = q[k] <= m[k] && (k == 0 || s.T >= bp.t_eps);
                    float w;
                    if (COUNT || k == 0) {
                        w = h ? s.T * al[k] : 0.f;
                    } else {  // h as one predicate (setp ... .and), one select
                        asm("{\n\t.reg .pred ph, pl;\n\t"
                            "setp.le.f32 ph, %1, %2;\n\t"
                            "setp.ge.and.f32 pl, %3, %4, ph;\n\t"
                            "selp.f32 %0, %5, 0f00000000, pl;\n\t}"
                            : "=f"(w)
                            : "f"(q[k]), "f"(m[k]), "f"(s.T), "f"(bp.t_eps), "f"(s.T * al[k]));
                    }
                    c01 = fma2(pk2(w, w), pk2(ec[k].x, ec[k].y), c01);
                    s.C2 += w * ec[k].z;
                    s.T -= w;  // a fragment closes an open entity: T != Tlast
                    if (COUNT && h) {
                        w_gf++;
                        last_id = s_ids[COUNT ? warp : 0][2 * p + k];
                    }
                }
                upk2(c01, s.C0, s.C1);
                if (s.T < bp.t_eps) s.finish();
            }
        } else if (!has_tri) {
            // (whole-pixel ablation mode: the Gaussian update depends on the open entity)
#pragma unroll 1
            for (unsigned p = 0; 2 * p < cnt; p += 2) {
                float q0, q1, q2, q3, m0, m1, m2, m3;
                qpair(p, q0, q1, m0, m1);
                qpair(p + 1, q2, q3, m2, m3);
                if (COUNT && !s.done()) w_gt += min(4u, cnt - 2 * p);
                const bool h1 = q1 <= m1, h2 = q2 <= m2, h3 = q3 <= m3;
                if (q0 <= m0) gblend(q0, 2 * p);
                if (h1 && !s.done()) gblend(q1, 2 * p + 1);
                if (h2 && !s.done()) gblend(q2, 2 * p + 2);
                if (h3 && !s.done()) gblend(q3, 2 * p + 3);
            }
        } else {
            // a chunk holding a triangle: entries one by one, in list order
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // triangle attributes (not the next records)
            __syncwarp();
            for (unsigned p = 0; 2 * p < cnt; p++) {
                float q[2], m[2];
                qpair(p, q[0], q[1], m[0], m[1]);
#pragma unroll
                for (int j = 0; j < 2; j++) {
                    const unsigned k = 2 * p + j;
                    if (k >= cnt) break;
                    if (m[j] >= 0.f) {  // warp-uniform: entry k is the same for every lane
                        if (COUNT && !s.done()) w_gt++;
                        if (q[j] <= m[j] && !s.done()) gblend(q[j], k);
                        continue;
                    }
                    const float *e = ef + kPairFloats * p + j;
                    const float4 ec = wb.col(k);
                    const int X[3] = {__float_as_int(e[0]), __float_as_int(e[4]), __float_as_int(e[8])};
                    const int Y[3] = {__float_as_int(e[2]), __float_as_int(e[6]), __float_as_int(ec.x)};
                    if (!s.done()) {
                        const unsigned long long f0 = w_tf;
                        tri_pixel<COUNT, MODE, M>(s, X, Y, __float_as_int(ec.y), ec.z, tat[k], x, y, tv, bp.t_eps,
                                                  w_tt, w_tf);
                        if (COUNT && w_tf != f0) last_id = __float_as_uint(ec.w);
                    }
                }
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // no copy may outlive the CTA's shared memory
    if (COUNT && frag_counts && x < W && y < H)
        frag_counts[(size_t)y * W + x] = make_uint4((unsigned)w_gf, (unsigned)w_tf, last_id, (unsigned)w_gt);
    if (COUNT) {
        unsigned long long v[4] = {w_gt, w_gf, w_tt, w_tf};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            unsigned long long xs = v[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
            if (lane == 0 && xs) atomicAdd(&st->work[k], xs);
        }
    }
    if (x < W && y < H) {
        const float T = (MODE == MODE_WHOLE_PIXEL && s.open) ? s.exit_T() : s.T;
        const float sb = T * bp.bg_alpha;
        out[(size_t)y * W + x] = make_float4(s.C0 + sb * bp.bg[0], s.C1 + sb * bp.bg[1], s.C2 + sb * bp.bg[2], T);
    }
    __syncwarp();  // the warp's buffers are reused by its next item
    }
}

// ----------------------------------------------------------------------------
// tri_depth 2: the per-pixel resort window (SPEC S:235/S:280:
// triangle fragments ordered by their plane depth at the pixel centre).  The tile
// lists are keyed like tri_depth 1 (N8); every pixel passes its fragments, in list
// order, through a window of kResortW entries in shared memory -- a bounded priority
// queue on (bits(depth at the pixel), id): N9 (N8's plane depth at the pixel centre,
// IEEE double as in the oracle) for a triangle, the view z for a Gaussian -- and
// blends the smallest entry whenever the window overflows, the rest at the end of
// the list (the oracle's or_window).  Exact-entity mode, M = 4 only; a quality
// variant, not the throughput path.
// ----------------------------------------------------------------------------
constexpr int kResortW = 4;

struct WinE {
    float a, r, g, b;
    unsigned mk;    // triangle: coverage mask | 1 << 31; Gaussian: 0
    unsigned dbits; // bits(depth at the pixel)
    unsigned id;
    unsigned pad;
};

__device__ __forceinline__ bool win_less(unsigned da, unsigned ia, unsigned db, unsigned ib) {
    return da != db ? da < db : ia < ib;
}

// N9: triangle plane depth at the pixel centre from the exact centre edge functions
__device__ __forceinline__ unsigned pixel_plane_depth_bits(const int X[3], const int Y[3], const long long Ec[3],
                                                           const TriAttr &r) {
    const long long A2 = (long long)(X[1] - X[0]) * (Y[2] - Y[0]) - (long long)(X[2] - X[0]) * (Y[1] - Y[0]);
    const double sd = __dadd_rn(__dadd_rn(__ddiv_rn((double)Ec[0], (double)r.q2.x), __ddiv_rn((double)Ec[1], (double)r.q2.y)),
                                __ddiv_rn((double)Ec[2], (double)r.q2.z));
    const float zmin = fminf(fminf(r.q2.x, r.q2.y), r.q2.z), zmax = fmaxf(fmaxf(r.q2.x, r.q2.y), r.q2.z);
    if (!(sd > 0.0)) return __float_as_uint(zmax);
    return __float_as_uint(fminf(fmaxf(__double2float_rn(__ddiv_rn((double)A2, sd)), zmin), zmax));
}

template <bool COUNT>
__global__ void __launch_bounds__(kBlendThreads, 3) k_blend_resort(const uint2 *__restrict__ ranges,
                                                                 const uint32_t *__restrict__ order,
                                                                 const uint32_t *__restrict__ vals,
                                                                 const GaussRecord *__restrict__ grec,
                                                                 const TriRecord *__restrict__ trec,
                                                                 const uint32_t *__restrict__ dkey, TexView tv,
                                                                 unsigned F, int W, int H, int tiles_x, BlendParams bp,
                                                                 float4 *__restrict__ out, DevState *st,
                                                                 uint4 *__restrict__ frag_counts) {
    constexpr int M = 4, MODE = MODE_EXACT;
    if (st->overflow) return;
    constexpr int NW = kBlendThreads / 32;
    unsigned long long w_gt = 0, w_gf = 0, w_tt = 0, w_tf = 0;
    unsigned last_id = 0xFFFFFFFFu;
    __shared__ unsigned s_ids[NW][32];
    __shared__ float s_dep[NW][32];  // a packed Gaussian's view z
    __shared__ WarpBuf s_buf[NW];
    __shared__ float4 s_stage[NW][32][3];
    __shared__ TriAttr s_tri[NW][32];
    extern __shared__ __align__(16) WinE s_win[];  // [kResortW][kBlendThreads]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = (int)__ldg(order + blockIdx.x);
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int sx0 = tx * kTile + (warp & 1) * 8, sy0 = ty * kTile + (warp >> 1) * 4;
    const int x = sx0 + (lane & 7), y = sy0 + (lane >> 3);
    const float px = (float)x + 0.5f;
    const uint2 rg = ranges[tile];
    const unsigned lt = (1u << lane) - 1u;
    WarpBuf &wb = s_buf[warp];
    float *ef = &wb.v[0][0].x;
    TriAttr *tat = s_tri[warp];
    float4 *stg = s_stage[warp][lane];
    const unsigned stg_s = (unsigned)__cvta_generic_to_shared(stg);
    WinE *win = s_win + threadIdx.x;  // entry j at win[j * kBlendThreads]
    int wn = 0;

    Px<MODE, M> s;
    s.C0 = s.C1 = s.C2 = 0.f;
    s.T = s.Te = s.G = s.Tl = 1.f;
#pragma unroll
    for (int j = 0; j < M; j++) s.t[j] = 1.f;
    s.open = false;
    s.Tlast = __int_as_float(0x7fc00000);
    s.py = (float)y + 0.5f;
    if (!(x < W && y < H)) s.finish();

    auto apply = [&](const WinE &e) {  // the state machine, one fragment
        if (COUNT) {
            if (e.mk >> 31) w_tf++;
            else w_gf++;
            last_id = e.id;
        }
        if (!(e.mk >> 31)) {  // Gaussian: Eq.1-2 (T holds an open entity's exit T, R3)
            const float w = s.T * e.a;
            s.C0 += w * e.r; s.C1 += w * e.g; s.C2 += w * e.b;
            s.T -= w;
        } else {  // triangle: Eq.7-9 in a depth-adjacent entity
            const unsigned m = e.mk & 0xFu;
            if (!(s.T == s.Tlast)) {
                s.Te = s.T;
#pragma unroll
                for (int j = 0; j < M; j++) s.t[j] = 1.f;
            }
            float O = 0.f;
#pragma unroll
            for (int j = 0; j < M; j++) O += ((m >> j) & 1u) ? s.t[j] : 0.f;
            O *= 1.f / M;
            const float w = s.Te * O * e.a;
            s.C0 += w * e.r; s.C1 += w * e.g; s.C2 += w * e.b;
            const float kk = 1.f - e.a;
#pragma unroll
            for (int j = 0; j < M; j++)
                if ((m >> j) & 1u) s.t[j] *= kk;
            s.T = s.exit_T();
            s.Tlast = s.T;
        }
        if (s.T < bp.t_eps) s.finish();
    };
    auto push = [&](const WinE &e) {  // into the window; blends the smallest on overflow
        if (wn < kResortW) {
            win[wn * kBlendThreads] = e;
            wn++;
            return;
        }
        int mi = 0;
        WinE best = win[0];
        for (int j = 1; j < kResortW; j++) {
            const WinE c = win[j * kBlendThreads];
            if (win_less(c.dbits, c.id, best.dbits, best.id)) { best = c; mi = j; }
        }
        if (win_less(e.dbits, e.id, best.dbits, best.id)) {
            apply(e);
        } else {
            apply(best);
            win[mi * kBlendThreads] = e;
        }
    };

    auto stage_rec = [&](unsigned id) {
        if (id != 0xFFFFFFFFu) {
            const char *src = id >= F ? reinterpret_cast<const char *>(grec + (id - F))
                                      : reinterpret_cast<const char *>(trec + id);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s), "l"(src) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s + 16), "l"(src + 16) : "memory");
            if (id >= F)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s + 32), "l"(src + 32) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    unsigned id0 = rg.x + lane < rg.y ? __ldg(vals + rg.x + lane) : 0xFFFFFFFFu;
    unsigned id1 = rg.x + 32 + lane < rg.y ? __ldg(vals + rg.x + 32 + lane) : 0xFFFFFFFFu;
    stage_rec(id0);
    const float kexp = -0.72134752044448170f;

    for (unsigned base = rg.x; base < rg.y; base += 32) {
        const unsigned live = __ballot_sync(0xffffffffu, !s.done());
        if (!live) break;
        LiveBox lb;
        {
            const unsigned cols = (live | (live >> 8) | (live >> 16) | (live >> 24)) & 0xFFu;
            const int c0 = __ffs(cols) - 1, c1 = 31 - __clz(cols);
            const int r0 = (__ffs(live) - 1) >> 3, r1 = (31 - __clz(live)) >> 3;
            lb.cx0 = (float)(sx0 + c0) + 0.5f; lb.cx1 = (float)(sx0 + c1) + 0.5f;
            lb.cy0 = (float)(sy0 + r0) + 0.5f; lb.cy1 = (float)(sy0 + r1) + 0.5f;
            lb.X0 = 256 * (sx0 + c0); lb.X1 = 256 * (sx0 + c1 + 1) - 1;
            lb.Y0 = 256 * (sy0 + r0); lb.Y1 = 256 * (sy0 + r1 + 1) - 1;
        }
        const unsigned id = id0;
        id0 = id1;
        id1 = base + 64 + lane < rg.y ? __ldg(vals + base + 64 + lane) : 0xFFFFFFFFu;
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        bool rel = false;
        float4 a, b, c;
        if (id != 0xFFFFFFFFu) {
            a = stg[0];
            b = stg[1];
            if (id >= F) {
                c = stg[2];
                rel = gauss_touches(a, b, c, lb);
            } else {
                rel = tri_touches(a, b, lb);
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, rel);
        const unsigned cnt = __popc(bal);
        const unsigned slot = __popc(bal & lt);
        if (rel) {
            s_ids[warp][slot] = id;
            float *e = ef + kPairFloats * (slot >> 1) + (slot & 1);
            if (id >= F) {
                e[0] = a.x; e[2] = a.y; e[4] = b.x; e[6] = b.z; e[8] = b.y + b.y; e[10] = a.z;
                wb.col(slot) = make_float4(c.x, c.y, c.z, lg2_ftz(a.w));
                s_dep[warp][slot] = __uint_as_float(__ldg(dkey + id));
            } else {
                e[0] = a.x; e[2] = a.y; e[4] = a.z; e[6] = a.w; e[8] = b.x; e[10] = -1.f;
                wb.col(slot) = make_float4(b.y, b.z, b.w, __uint_as_float(id));
                const char *src = reinterpret_cast<const char *>(&trec[id].q2);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&tat[slot]);
#pragma unroll
                for (int w = 0; w < 4; w++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * w), "l"(src + 16 * w)
                                 : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        __syncwarp();
        stage_rec(id0);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
        for (unsigned p = 0; 2 * p < cnt; p++) {
            float q[2], m[2];
            {
                const float4 A = wb.v[p][0], B = wb.v[p][1], Cc = wb.v[p][2];
                const f32x2 dx = sub2(pk2(px, px), pk2(A.x, A.y));
                const f32x2 dy = sub2(pk2(s.py, s.py), pk2(A.z, A.w));
                const f32x2 t = fma2(pk2(B.z, B.w), mul2(dy, dy), mul2(pk2(Cc.x, Cc.y), mul2(dx, dy)));
                upk2(fma2(pk2(B.x, B.y), mul2(dx, dx), t), q[0], q[1]);
                m[0] = Cc.z;
                m[1] = Cc.w;
            }
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const unsigned k = 2 * p + j;
                if (k >= cnt) break;
                if (m[j] >= 0.f) {  // Gaussian entry
                    if (COUNT && !s.done()) w_gt++;
                    if (q[j] <= m[j] && !s.done()) {
                        const float4 ec = wb.col(k);
                        WinE e;
                        e.a = fminf(bp.alpha_max, ex2_ftz(fmaf(q[j], kexp, ec.w)));
                        e.r = ec.x; e.g = ec.y; e.b = ec.z;
                        e.mk = 0;
                        e.dbits = __float_as_uint(s_dep[warp][k]);
                        e.id = s_ids[warp][k];
                        push(e);
                    }
                    continue;
                }
                if (s.done()) continue;
                const float *e = ef + kPairFloats * p + j;
                const float4 ec = wb.col(k);
                const int X[3] = {__float_as_int(e[0]), __float_as_int(e[4]), __float_as_int(e[8])};
                const int Y[3] = {__float_as_int(e[2]), __float_as_int(e[6]), __float_as_int(ec.x)};
                if (COUNT) w_tt++;
                {   // exact pre-test: no sample can lie in the triangle's bbox
                    constexpr int R16 = 16 * 6;
                    const int PX = 256 * x + 128, PY = 256 * y + 128;
                    if (PX + R16 < min(X[0], min(X[1], X[2])) || PX - R16 > max(X[0], max(X[1], X[2])) ||
                        PY + R16 < min(Y[0], min(Y[1], Y[2])) || PY - R16 > max(Y[0], max(Y[1], Y[2])))
                        continue;
                }
                long long Ec[3];
                const unsigned mk = coverage<M>(X, Y, x, y, Ec);
                if (!mk) continue;
                float rgb[3];
                tri_colour(tat[k], __float_as_int(ec.y), Ec, tv, rgb);
                WinE we;
                we.a = ec.z;
                we.r = rgb[0]; we.g = rgb[1]; we.b = rgb[2];
                we.mk = mk | 0x80000000u;
                we.dbits = pixel_plane_depth_bits(X, Y, Ec, tat[k]);
                we.id = __float_as_uint(ec.w);
                push(we);
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    // end of the list: blend the window's rest in (depth, id) order
    while (wn > 0 && !s.done()) {
        int mi = 0;
        WinE best = win[0];
        for (int j = 1; j < wn; j++) {
            const WinE c2 = win[j * kBlendThreads];
            if (win_less(c2.dbits, c2.id, best.dbits, best.id)) { best = c2; mi = j; }
        }
        apply(best);
        win[mi * kBlendThreads] = win[(wn - 1) * kBlendThreads];
        wn--;
    }
    if (COUNT && frag_counts && x < W && y < H)
        frag_counts[(size_t)y * W + x] = make_uint4((unsigned)w_gf, (unsigned)w_tf, last_id, (unsigned)w_gt);
    if (COUNT) {
        unsigned long long v[4] = {w_gt, w_gf, w_tt, w_tf};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            unsigned long long xs = v[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
            if (lane == 0 && xs) atomicAdd(&st->work[k], xs);
        }
    }
    if (x < W && y < H) {
        const float sb = s.T * bp.bg_alpha;
        out[(size_t)y * W + x] = make_float4(s.C0 + sb * bp.bg[0], s.C1 + sb * bp.bg[1], s.C2 + sb * bp.bg[2], s.T);
    }
}

template <bool COUNT>
static void launch_resort(const Buffers &b, const MeshInput &m, const CamParams &cam, const BlendParams &bp, float *out,
                          cudaStream_t s, uint32_t *fc) {
    const size_t smem = sizeof(WinE) * kResortW * kBlendThreads;
    static const bool attr = [smem] {
        cudaFuncSetAttribute(k_blend_resort<COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return true;
    }();
    (void)attr;
    TexView tv{reinterpret_cast<const uchar4 *>(m.tex), m.tw, m.th};
    k_blend_resort<COUNT><<<cam.tiles_x * cam.tiles_y, kBlendThreads, smem, s>>>(
        b.ranges, b.order, b.sorted_vals, b.grec, b.trec, b.dkey, tv, (unsigned)m.F, cam.W, cam.H, cam.tiles_x, bp,
        reinterpret_cast<float4 *>(out), b.st, reinterpret_cast<uint4 *>(fc));
}

// k_blend's per-CTA item budget (UNIMGS_BLEND_ITEMS overrides it for experiments):
// 8 = one tile per CTA, as a plain grid; more lets a CTA's warps balance several tiles.
static int blend_items_per_cta() {
    static const int v = [] {
        const char *e = getenv("UNIMGS_BLEND_ITEMS");
        const int n = e ? atoi(e) : 0;
        return n >= 1 ? n : 2 * UNIMGS_BLEND_CTA_WARPS;
    }();
    return v;
}

template <int MODE, int M>
static void launch_mode(const Buffers &b, const MeshInput &m, const CamParams &cam, const BlendParams &bp, float *out,
                        cudaStream_t s, bool count_work, uint32_t *frag_counts) {
    const int tiles = cam.tiles_x * cam.tiles_y;
    const unsigned n_items = (unsigned)tiles * kSubTiles;
    const int per_cta = blend_items_per_cta();
    const unsigned grid = (n_items + per_cta - 1) / per_cta;
    TexView tv{reinterpret_cast<const uchar4 *>(m.tex), m.tw, m.th};
    if (count_work)
        k_blend<true, MODE, M><<<grid, kBlendCtaThreads, 0, s>>>(b.ranges, b.order, b.sorted_vals, b.grec, b.trec, tv,
                                                               (unsigned)m.F, cam.W, cam.H, cam.tiles_x, n_items,
                                                               per_cta, bp, reinterpret_cast<float4 *>(out), b.st,
                                                               reinterpret_cast<uint4 *>(frag_counts));
    else
        k_blend<false, MODE, M><<<grid, kBlendCtaThreads, 0, s>>>(b.ranges, b.order, b.sorted_vals, b.grec, b.trec, tv,
                                                                (unsigned)m.F, cam.W, cam.H, cam.tiles_x, n_items,
                                                                per_cta, bp, reinterpret_cast<float4 *>(out), b.st,
                                                                nullptr);
}

template <int MODE>
static void launch_m(int M, const Buffers &b, const MeshInput &m, const CamParams &cam, const BlendParams &bp,
                     float *out, cudaStream_t s, bool count_work, uint32_t *fc) {
    switch (M) {
        case 1: launch_mode<MODE, 1>(b, m, cam, bp, out, s, count_work, fc); break;
        case 2: launch_mode<MODE, 2>(b, m, cam, bp, out, s, count_work, fc); break;
        case 8: launch_mode<MODE, 8>(b, m, cam, bp, out, s, count_work, fc); break;
        case 16: launch_mode<MODE, 16>(b, m, cam, bp, out, s, count_work, fc); break;
        default: launch_mode<MODE, 4>(b, m, cam, bp, out, s, count_work, fc); break;
    }
}

int launch_blend(const Buffers &b, const GaussInput &g, const MeshInput &m, const CamParams &cam,
                 const BlendParams &bp, float *out, cudaStream_t s, bool count_work, uint32_t *fc) {
    (void)g;
    if (bp.resort) {  // tri_depth 2 (exact mode, M = 4: validated by the API)
        if (count_work) launch_resort<true>(b, m, cam, bp, out, s, fc);
        else launch_resort<false>(b, m, cam, bp, out, s, nullptr);
        return 1;
    }
    switch (bp.mode) {
        case MODE_NAIVE: launch_m<MODE_NAIVE>(bp.msaa, b, m, cam, bp, out, s, count_work, fc); break;
        case MODE_MSAA_PIXEL: launch_m<MODE_MSAA_PIXEL>(bp.msaa, b, m, cam, bp, out, s, count_work, fc); break;
        case MODE_WHOLE_PIXEL: launch_m<MODE_WHOLE_PIXEL>(bp.msaa, b, m, cam, bp, out, s, count_work, fc); break;
        case MODE_PAPER_LITERAL: launch_m<MODE_PAPER_LITERAL>(bp.msaa, b, m, cam, bp, out, s, count_work, fc); break;
        default: launch_m<MODE_EXACT>(bp.msaa, b, m, cam, bp, out, s, count_work, fc); break;
    }
    return 1;
}

}  // namespace unimgs
