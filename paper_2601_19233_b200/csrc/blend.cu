// blend.cu -- B8: the unified single-pass anti-aliased blend (§3.2).
//
// One CTA per 16x16 tile, one pixel per thread, 8 warps that each walk the
// tile's sorted list (unified ids, (tile, depth, id) order) independently:
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
// fp64 (lambda_k ~ E_k z_i z_j, exact products), manual fp32 bilinear texture.
#include "internal.cuh"

namespace unimgs {

#ifndef UNIMGS_BLEND_PIX
#define UNIMGS_BLEND_PIX 1
#endif

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

// Exact per-warp culling (never drops a fragment).  Warp w owns the 8x4
// sub-tile (w & 1, w >> 1) of the 16x16 tile; an entry is skipped by the warp
// only when no pixel of its sub-tile can hold the fragment:
//   triangle: its snapped integer bbox misses the sub-tile's 1/256-px extent;
//   Gaussian: the sub-tile's pixel centres lie outside the bbox of the exact
//   ellipse {d : Q(d) <= q_max (1 + 0.02)} of the fp32 conic Q, padded by
//   1% + 0.01 px (half-extents computed once per Gaussian in B1).  Only for
//   cond(Q) <= ~1000, where the fp32 evaluation of q (10 roundings,
//   cancellation factor <= 2(cond + 1)) errs by < 1.3e-3 q, so a pixel outside
//   that ellipse cannot satisfy the N6 test q <= q_max.  Other conics
//   (needles, NaN) are never skipped.
__device__ __forceinline__ bool gauss_touches(const float4 &a, const float4 &b, const float4 &c, float rx0, float ry0,
                                              float ry1) {
    const float ex = c.w, ey = b.w;  // precomputed in B1; -1 = never cull
    if (!(ex >= 0.f)) return true;
    return a.x + ex >= rx0 && a.x - ex <= rx0 + 7.f && a.y + ey >= ry0 && a.y - ey <= ry1;
}

__device__ __forceinline__ bool tri_touches(const float4 &a, const float4 &b, int Rx0, int Ry0, int Ry1) {
    const int X0 = __float_as_int(a.x), Y0 = __float_as_int(a.y), X1 = __float_as_int(a.z), Y1 = __float_as_int(a.w);
    const int X2 = __float_as_int(b.x), Y2 = __float_as_int(b.y);
    const int mnx = min(X0, min(X1, X2)), mxx = max(X0, max(X1, X2));
    const int mny = min(Y0, min(Y1, Y2)), mxy = max(Y0, max(Y1, Y2));
    return mxx >= Rx0 && mnx <= Rx0 + 256 * 8 - 1 && mxy >= Ry0 && mny <= Ry1;
}

__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// blend modes (the paper's ablation, Fig.3 / Fig.4)
enum { MODE_EXACT = 0, MODE_NAIVE = 1, MODE_MSAA_PIXEL = 2, MODE_WHOLE_PIXEL = 3, MODE_PAPER_LITERAL = 4 };

// Per-pixel blend state (registers).  G / Tl only exist for the modes that use them.
template <int MODE, int M>
struct Px {
    float C0, C1, C2, T, Te;
    float t[M];
    float G, Tl;
    float Tx;  // cached exit transmittance of the open entity (refreshed by each triangle)
    float py;  // pixel centre y for the Gaussian test; NaN once done (the test then fails by itself)
    bool open, done;
    __device__ __forceinline__ void finish() {
        done = true;
        py = __int_as_float(0x7fc00000);
    }
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
    if (!s.open) {
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
    s.Tx = s.exit_T();
    if (s.Tx < t_eps) s.finish();
}

// One CTA per 16x16 tile, independent warps, PIX pixels per lane (vertically
// 4 rows apart).  Warp w owns an 8 x (4 PIX) sub-tile.  Each warp walks the
// whole tile list in chunks of 32 (lane l holds entry 32c + l; ids are
// prefetched two chunks ahead and records one chunk ahead), keeps the entries
// that touch its sub-tile (ballot), packs them into its own shared buffer and
// blends them in list order with broadcast reads.  No block-wide barrier: a
// warp stops as soon as all of its pixels have terminated.  A packed triangle
// entry carries q_max = -1, so the Gaussian membership test rejects it for
// free and only the (rare) miss path checks for triangles.
#ifndef UNIMGS_BLEND_MINB
#define UNIMGS_BLEND_MINB (4 * PIX)
#endif
template <bool COUNT, int PIX, int MODE, int M>
__global__ void __launch_bounds__(kBlendThreads / PIX, UNIMGS_BLEND_MINB) k_blend(const uint2 *__restrict__ ranges,
                                                                     const uint32_t *__restrict__ order,
                                                                     const uint32_t *__restrict__ vals,
                                                                     const GaussRecord *__restrict__ grec,
                                                                     const TriRecord *__restrict__ trec, TexView tv,
                                                                     unsigned F, int W, int H, int tiles_x,
                                                                     BlendParams bp, float4 *__restrict__ out,
                                                                     DevState *st) {
    if (st->overflow) return;
    constexpr int NW = kBlendThreads / PIX / 32;  // warps per tile
    unsigned long long w_gt = 0, w_gf = 0, w_tt = 0, w_tf = 0;  // COUNT only
    __shared__ float4 s_buf[NW][32][3];  // per-warp packed entries: a (u, v, q_max, o), (ca, 2cb, cc, id), c
    __shared__ TriAttr s_tri[NW][32];    // a packed triangle entry's q2..q5 (cp.async)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = (int)__ldg(order + blockIdx.x);  // longest-first schedule (k_tile_order)
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int sx0 = tx * kTile + (warp & 1) * 8, sy0 = ty * kTile + (warp >> 1) * 4 * PIX;
    const int x = sx0 + (lane & 7), y0 = sy0 + (lane >> 3);
    const float px = (float)x + 0.5f;
    const float rx0 = (float)sx0 + 0.5f, ry0 = (float)sy0 + 0.5f, ry1 = ry0 + (float)(4 * PIX - 1);
    const int Rx0 = 256 * sx0, Ry0 = 256 * sy0, Ry1 = 256 * (sy0 + 4 * PIX) - 1;
    const uint2 rg = ranges[tile];
    const unsigned lt = (1u << lane) - 1u;
    float4(*buf)[3] = s_buf[warp];
    TriAttr *tat = s_tri[warp];

    Px<MODE, M> s[PIX];
#pragma unroll
    for (int p = 0; p < PIX; p++) {
        s[p].C0 = s[p].C1 = s[p].C2 = 0.f;
        s[p].T = s[p].Te = s[p].G = s[p].Tl = s[p].Tx = 1.f;
#pragma unroll
        for (int j = 0; j < M; j++) s[p].t[j] = 1.f;
        s[p].open = false;
        s[p].done = false;
        s[p].py = (float)(y0 + 4 * p) + 0.5f;
        if (!(x < W && y0 + 4 * p < H)) s[p].finish();
    }
    auto all_done = [&]() {
        bool d = true;
#pragma unroll
        for (int p = 0; p < PIX; p++) d = d && s[p].done;
        return d;
    };

    // ids two chunks ahead, records one chunk ahead
    unsigned id1 = rg.x + lane < rg.y ? __ldg(vals + rg.x + lane) : 0xFFFFFFFFu;
    unsigned id2 = rg.x + 32 + lane < rg.y ? __ldg(vals + rg.x + 32 + lane) : 0xFFFFFFFFu;
    float4 na = make_float4(0.f, 0.f, 0.f, 0.f), nb = na, nc = na;
    auto fetch_rec = [&](unsigned id) {
        if (id == 0xFFFFFFFFu) return;
        if (id >= F) {
            const GaussRecord *g = grec + (id - F);
            na = __ldg(&g->a); nb = __ldg(&g->b); nc = __ldg(&g->c);
        } else {
            const int4 *q = reinterpret_cast<const int4 *>(trec + id);
            const int4 q0 = __ldg(q), q1 = __ldg(q + 1);
            na = make_float4(__int_as_float(q0.x), __int_as_float(q0.y), __int_as_float(q0.z), __int_as_float(q0.w));
            nb = make_float4(__int_as_float(q1.x), __int_as_float(q1.y), __int_as_float(q1.z), __int_as_float(q1.w));
        }
    };
    fetch_rec(id1);
    const float kexp = -0.72134752044448170f;  // -log2(e) / 2

    for (unsigned base = rg.x; base < rg.y; base += 32) {
        if (__all_sync(0xffffffffu, all_done())) break;
        const unsigned id = id1;
        const float4 a = na, b = nb, c = nc;
        id1 = id2;
        id2 = base + 64 + lane < rg.y ? __ldg(vals + base + 64 + lane) : 0xFFFFFFFFu;
        fetch_rec(id1);
        bool rel = false;
        if (id != 0xFFFFFFFFu)
            rel = id >= F ? gauss_touches(a, b, c, rx0, ry0, ry1) : tri_touches(a, b, Rx0, Ry0, Ry1);
        const unsigned bal = __ballot_sync(0xffffffffu, rel);
        const bool has_tri = __any_sync(0xffffffffu, rel && id < F);
        if (rel) {
            const unsigned slot = __popc(bal & lt);
            if (id >= F) {
                buf[slot][0] = a;
                buf[slot][1] = make_float4(b.x, b.y + b.y, b.z, __uint_as_float(id));
                buf[slot][2] = c;
            } else {
                // triangle: q_max = -1 (no Gaussian test passes), the prefetched vertices,
                // kind and alpha staged with it: (X0, Y0, -1, Y1), (X2, Y2, X1, id), (kind, alpha)
                buf[slot][0] = make_float4(a.x, a.y, -1.f, a.w);
                buf[slot][1] = make_float4(b.x, b.y, a.z, __uint_as_float(id));
                buf[slot][2] = make_float4(b.z, b.w, 0.f, 0.f);
                const char *src = reinterpret_cast<const char *>(&trec[id].q2);
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&tat[slot]);
#pragma unroll
                for (int w = 0; w < 4; w++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * w), "l"(src + 16 * w)
                                 : "memory");
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            }
        }
        __syncwarp();
        const unsigned cnt = __popc(bal);
        // Gaussian fragment test + blend (Eq.1-2) of packed entry k for each pixel
        auto gauss = [&](const float4 &ea, const float4 &eb, unsigned k) {
            const float dx = __fsub_rn(px, ea.x);
            const float dxx = __fmul_rn(dx, dx);
            bool hit[PIX], any = false;
            float q[PIX];
#pragma unroll
            for (int p = 0; p < PIX; p++) {
                const float dy = __fsub_rn(s[p].py, ea.y);
                q[p] = __fmaf_rn(eb.x, dxx, __fmaf_rn(eb.z, __fmul_rn(dy, dy), __fmul_rn(eb.y, __fmul_rn(dx, dy))));
                hit[p] = q[p] <= ea.z;  // false once done: py is NaN
                if (COUNT && ea.z >= 0.f && !s[p].done) w_gt++;
                any = any || hit[p];
            }
            if (!any) return false;
            const float4 ec = buf[k][2];
#pragma unroll
            for (int p = 0; p < PIX; p++) {
                if (!hit[p]) continue;
                if (COUNT) w_gf++;
                const float al = fminf(bp.alpha_max, ea.w * ex2_ftz(q[p] * kexp));
                if (MODE == MODE_WHOLE_PIXEL && s[p].open) {
                    // Fig.3b/c: the entity spans the whole list; the Gaussian does not
                    // attenuate its sub-pixel state (colour overflow)
                    const float base = s[p].Te * s[p].mean_t();
                    const float w = base * s[p].G * al;
                    s[p].C0 += w * ec.x; s[p].C1 += w * ec.y; s[p].C2 += w * ec.z;
                    s[p].G *= 1.f - al;
                    if (base * s[p].G < bp.t_eps) s[p].finish();
                    continue;
                }
                if (MODE != MODE_NAIVE && MODE != MODE_MSAA_PIXEL && s[p].open) {
                    s[p].T = s[p].Tx;  // depth adjacency broken: exit T (R3)
                    s[p].open = false;
                }
                const float w = s[p].T * al;
                s[p].C0 += w * ec.x; s[p].C1 += w * ec.y; s[p].C2 += w * ec.z;
                s[p].T -= w;
                if (s[p].T < bp.t_eps) s[p].finish();
            }
            return true;
        };
        if (!has_tri) {
            // Gaussian-only chunk: two entries per iteration (independent q chains)
            unsigned k = 0;
            for (; k + 2 <= cnt; k += 2) {
                const float4 ea0 = buf[k][0], eb0 = buf[k][1], ea1 = buf[k + 1][0], eb1 = buf[k + 1][1];
                gauss(ea0, eb0, k);
                gauss(ea1, eb1, k + 1);
            }
            if (k < cnt) gauss(buf[k][0], buf[k][1], k);
        } else {
            bool staged = false;
            for (unsigned k = 0; k < cnt; k++) {
                const float4 ea = buf[k][0];
                const float4 eb = buf[k][1];
                if (ea.z >= 0.f) {  // warp-uniform: entry k is the same for every lane
                    gauss(ea, eb, k);
                } else {
                    if (!staged) {  // the chunk's triangle attributes, waited for once
                        asm volatile("cp.async.wait_all;\n" ::: "memory");
                        __syncwarp();
                        staged = true;
                    }
                    const float4 ec = buf[k][2];
                    const int X[3] = {__float_as_int(ea.x), __float_as_int(eb.z), __float_as_int(eb.x)};
                    const int Y[3] = {__float_as_int(ea.y), __float_as_int(ea.w), __float_as_int(eb.y)};
                    const TriAttr &r = tat[k];
#pragma unroll
                    for (int p = 0; p < PIX; p++)
                        if (!s[p].done)
                            tri_pixel<COUNT, MODE, M>(s[p], X, Y, __float_as_int(ec.x), ec.y, r, x, y0 + 4 * p, tv,
                                                      bp.t_eps, w_tt, w_tf);
                }
            }
        }
        __syncwarp();
    }
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
#pragma unroll
    for (int p = 0; p < PIX; p++) {
        const int y = y0 + 4 * p;
        if (x < W && y < H) {
            float T = s[p].T;
            if (s[p].open) T = s[p].exit_T();
            const float sb = T * bp.bg_alpha;
            out[(size_t)y * W + x] = make_float4(s[p].C0 + sb * bp.bg[0], s[p].C1 + sb * bp.bg[1], s[p].C2 + sb * bp.bg[2], T);
        }
    }
}

template <int MODE, int M>
static void launch_mode(const Buffers &b, const MeshInput &m, const CamParams &cam, const BlendParams &bp, float *out,
                        cudaStream_t s, bool count_work) {
    constexpr int PIX = UNIMGS_BLEND_PIX;
    const int tiles = cam.tiles_x * cam.tiles_y;
    TexView tv{reinterpret_cast<const uchar4 *>(m.tex), m.tw, m.th};
    if (count_work)
        k_blend<true, PIX, MODE, M><<<tiles, kBlendThreads / PIX, 0, s>>>(b.ranges, b.order, b.sorted_vals, b.grec, b.trec, tv,
                                                                        (unsigned)m.F, cam.W, cam.H, cam.tiles_x, bp,
                                                                        reinterpret_cast<float4 *>(out), b.st);
    else
        k_blend<false, PIX, MODE, M><<<tiles, kBlendThreads / PIX, 0, s>>>(b.ranges, b.order, b.sorted_vals, b.grec, b.trec, tv,
                                                                         (unsigned)m.F, cam.W, cam.H, cam.tiles_x, bp,
                                                                         reinterpret_cast<float4 *>(out), b.st);
}

template <int MODE>
static void launch_m(int M, const Buffers &b, const MeshInput &m, const CamParams &cam, const BlendParams &bp,
                     float *out, cudaStream_t s, bool count_work) {
    switch (M) {
        case 1: launch_mode<MODE, 1>(b, m, cam, bp, out, s, count_work); break;
        case 2: launch_mode<MODE, 2>(b, m, cam, bp, out, s, count_work); break;
        case 8: launch_mode<MODE, 8>(b, m, cam, bp, out, s, count_work); break;
        case 16: launch_mode<MODE, 16>(b, m, cam, bp, out, s, count_work); break;
        default: launch_mode<MODE, 4>(b, m, cam, bp, out, s, count_work); break;
    }
}

int launch_blend(const Buffers &b, const GaussInput &g, const MeshInput &m, const CamParams &cam,
                 const BlendParams &bp, float *out, cudaStream_t s, bool count_work) {
    (void)g;
    switch (bp.mode) {
        case MODE_NAIVE: launch_m<MODE_NAIVE>(bp.msaa, b, m, cam, bp, out, s, count_work); break;
        case MODE_MSAA_PIXEL: launch_m<MODE_MSAA_PIXEL>(bp.msaa, b, m, cam, bp, out, s, count_work); break;
        case MODE_WHOLE_PIXEL: launch_m<MODE_WHOLE_PIXEL>(bp.msaa, b, m, cam, bp, out, s, count_work); break;
        case MODE_PAPER_LITERAL: launch_m<MODE_PAPER_LITERAL>(bp.msaa, b, m, cam, bp, out, s, count_work); break;
        default: launch_m<MODE_EXACT>(bp.msaa, b, m, cam, bp, out, s, count_work); break;
    }
    return 1;
}

}  // namespace unimgs
