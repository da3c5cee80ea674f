// preprocess.cu -- B1 Gaussian projection (EWA) and B2 triangle setup
// with 4-sample integer coverage (M = 4).
//
// Everything that decides a key, an order or fragment membership follows
// DESIGN.md "normative fp32 arithmetic" N1-N7 with explicit round-to-nearest
// intrinsics (no FMA contraction), so the keys are bit-identical to the
// independent CPU oracle.  Colour (SH) is ordinary fp32.
#include <cstddef>

#include "internal.cuh"

#ifndef UNIMGS_SH_PREFETCH
#define UNIMGS_SH_PREFETCH 1
#endif
#ifndef UNIMGS_SH_PF_MARGIN
#define UNIMGS_SH_PF_MARGIN 0.25f // prefetch window: the image grown by this fraction on every side
#endif

namespace unimgs {

// explicit IEEE single ops: one rounding each, never contracted
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float dot3(const float *a, const float *b) {
    return fma_(a[0], b[0], fma_(a[1], b[1], mul(a[2], b[2])));
}

// N1: pv[r] = fma(R[r][0],x, fma(R[r][1],y, fma(R[r][2],z, t[r])))
__device__ __forceinline__ void view_point(const CamParams &c, float x, float y, float z, float pv[3]) {
#pragma unroll
    for (int r = 0; r < 3; r++) pv[r] = fma_(c.R[3 * r], x, fma_(c.R[3 * r + 1], y, fma_(c.R[3 * r + 2], z, c.t[r])));
}

__global__ void k_begin_frame(DevState *st) {
    unsigned int *w = reinterpret_cast<unsigned int *>(st);
    const int n = sizeof(DevState) / 4, first = offsetof(DevState, n_vis) / 4;
    if (threadIdx.x == 0) st->frame_epoch += 1;
    for (int i = first + threadIdx.x; i < n; i += blockDim.x) w[i] = 0;
}

int launch_begin_frame(DevState *st, cudaStream_t s) {
    k_begin_frame<<<1, 256, 0, s>>>(st);
    return 1;
}

// Count of `flag` over the CTA (256 threads) written to *out by thread 0 (the
// per-CTA visible counts the compaction scans; no atomics, no look-back).
__device__ __forceinline__ void block_count(bool flag, unsigned *out) {
    __shared__ unsigned s_c[8];
    const unsigned c = __popc(__ballot_sync(0xffffffffu, flag));
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (unsigned w = 0; w < (blockDim.x >> 5); w++) t += s_c[w];
        *out = t;
    }
}

// 3DGS real SH basis, fp32
__device__ __forceinline__ void sh_eval(const float *__restrict__ sh, int deg, float x, float y, float z, float out[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float b[16];
    b[0] = C0;
    int k = 1;
    if (deg > 0) {
        b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
        k = 4;
        if (deg > 1) {
            float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            b[4] = 1.0925484305920792f * xy;
            b[5] = -1.0925484305920792f * yz;
            b[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
            b[7] = -1.0925484305920792f * xz;
            b[8] = 0.5462742152960396f * (xx - yy);
            k = 9;
            if (deg > 2) {
                b[9] = -0.5900435899266435f * y * (3.f * xx - yy);
                b[10] = 2.890611442640554f * xy * z;
                b[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
                b[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
                b[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
                b[14] = 1.445305721320277f * z * (xx - yy);
                b[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
                k = 16;
            }
        }
    }
    float r = 0.f, g = 0.f, bl = 0.f;
    // coefficients of one Gaussian are contiguous: k * 3 floats
    const float4 *v4 = reinterpret_cast<const float4 *>(sh);
    if ((reinterpret_cast<uintptr_t>(sh) & 15) == 0 && k == 16) {
        float c[48];
#pragma unroll
        for (int i = 0; i < 12; i++) {
            float4 q = __ldg(v4 + i);
            c[4 * i] = q.x; c[4 * i + 1] = q.y; c[4 * i + 2] = q.z; c[4 * i + 3] = q.w;
        }
#pragma unroll
        for (int i = 0; i < 16; i++) {
            r += b[i] * c[3 * i]; g += b[i] * c[3 * i + 1]; bl += b[i] * c[3 * i + 2];
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (i < k) {
                r += b[i] * __ldg(sh + 3 * i); g += b[i] * __ldg(sh + 3 * i + 1); bl += b[i] * __ldg(sh + 3 * i + 2);
            }
        }
    }
    out[0] = fmaxf(r + 0.5f, 0.f);
    out[1] = fmaxf(g + 0.5f, 0.f);
    out[2] = fmaxf(bl + 0.5f, 0.f);
}

// The per-view part of B1 for Gaussian g (N1, N2, N4, N5, SH): writes the record,
// rect and depth key of view `cam` into `b` and returns whether g is visible;
// get_sig(Sig) supplies Sigma (N3, or the given cov3d) -- only called once g passed
// the near/far cull, so the multi-view kernel can compute it once for all views.
template <typename GetSig>
__device__ __forceinline__ bool project_gaussian(const GaussInput &gin, int64_t g, int64_t F, const CamParams &cam,
                                                 float dilation, const Buffers &b, float mx, float my, float mz, float o,
                                                 uint32_t &touched, GetSig get_sig) {
    const int64_t p = F + g;
    bool vis = false;
    touched = 0;
    do {
        float pv[3];
        view_point(cam, mx, my, mz, pv);
        if (!(pv[2] > cam.near_z) || pv[2] > cam.far_z) break;
        const float xz = dv(pv[0], pv[2]), yz = dv(pv[1], pv[2]);          // N2
        const float u = fma_(cam.fx, xz, cam.cx), v = fma_(cam.fy, yz, cam.cy);
#if UNIMGS_SH_PREFETCH
        // likely visible: start pulling its SH coefficients into L2 now, so the
        // EWA math below hides the latency of the dependent SH loads
        if (u > -UNIMGS_SH_PF_MARGIN * (float)cam.W && u < (1.f + UNIMGS_SH_PF_MARGIN) * (float)cam.W &&
            v > -UNIMGS_SH_PF_MARGIN * (float)cam.H && v < (1.f + UNIMGS_SH_PF_MARGIN) * (float)cam.H) {
            const char *shp = reinterpret_cast<const char *>(gin.sh + g * (gin.sh_degree + 1) * (gin.sh_degree + 1) * 3);
            const int bytes = (gin.sh_degree + 1) * (gin.sh_degree + 1) * 12;
            for (int off = 0; off < bytes; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(shp + off));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(shp + bytes - 1));
        }
#endif
        float Sig[9];
        get_sig(Sig);
        float A[9], Sv[9];
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const float col[3] = {Sig[c], Sig[3 + c], Sig[6 + c]};
                A[3 * a + c] = dot3(cam.R + 3 * a, col);
            }
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int c = 0; c < 3; c++) Sv[3 * a + c] = dot3(A + 3 * a, cam.R + 3 * c);
        // N4
        const float lx = cam.lx, ly = cam.ly;  // = mul(1.3, dv(mul(0.5, W), fx)) etc., per camera
        const float tx = mul(fminf(fmaxf(xz, -lx), lx), pv[2]);
        const float ty = mul(fminf(fmaxf(yz, -ly), ly), pv[2]);
        const float zz2 = mul(pv[2], pv[2]);
        const float J0[3] = {dv(cam.fx, pv[2]), 0.0f, -dv(mul(cam.fx, tx), zz2)};
        const float J1[3] = {0.0f, dv(cam.fy, pv[2]), -dv(mul(cam.fy, ty), zz2)};
        float B0[3], B1[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const float col[3] = {Sv[c], Sv[3 + c], Sv[6 + c]};
            B0[c] = dot3(J0, col);
            B1[c] = dot3(J1, col);
        }
        const float ca_ = add(dot3(B0, J0), dilation), cb_ = dot3(B0, J1), cc_ = add(dot3(B1, J1), dilation);
        const float det = fma_(ca_, cc_, -mul(cb_, cb_));
        if (!(det > 0.0f)) break;
        const float inv = dv(1.0f, det);
        const float ka = mul(cc_, inv), kb = mul(-cb_, inv), kc = mul(ca_, inv);
        if (!(ka > 0.0f && fma_(ka, kc, -mul(kb, kb)) > 0.0f)) break;
        // N5
        if (!(255.0 * (double)o >= 1.0)) break;
        const float qmax = (float)(2.0 * log(255.0 * (double)o));
        const float ex = fma_(__fsqrt_rn(mul(qmax, ca_)), 1.0009765625f, 0.00390625f);
        const float ey = fma_(__fsqrt_rn(mul(qmax, cc_)), 1.0009765625f, 0.00390625f);
        const float flx = floorf(mul(sub(u, ex), 0.0625f)), fhx = floorf(mul(add(u, ex), 0.0625f));
        const float fly = floorf(mul(sub(v, ey), 0.0625f)), fhy = floorf(mul(add(v, ey), 0.0625f));
        if (!(fhx >= 0.0f && flx <= (float)(cam.tiles_x - 1) && fhy >= 0.0f && fly <= (float)(cam.tiles_y - 1)))
            break;
        const int x0 = (int)fmaxf(flx, 0.0f), x1 = (int)fminf(fhx, (float)(cam.tiles_x - 1));
        const int y0 = (int)fmaxf(fly, 0.0f), y1 = (int)fminf(fhy, (float)(cam.tiles_y - 1));
        touched = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
        // colour: SH at normalize(mu - campos)
        float dxw = mx - cam.campos[0], dyw = my - cam.campos[1], dzw = mz - cam.campos[2];
        const float rn = rsqrtf(dxw * dxw + dyw * dyw + dzw * dzw);
        float rgb[3];
        const int kc3 = (gin.sh_degree + 1) * (gin.sh_degree + 1) * 3;
        sh_eval(gin.sh + g * kc3, gin.sh_degree, dxw * rn, dyw * rn, dzw * rn, rgb);
        // half-extents of the blend's exact per-warp culling (see blend.cu): the bbox of
        // {d : Q(d) <= q_max (1 + 0.02)} of the fp32 conic Q, padded; -1 = never cull
        float cex = -1.f, cey = -1.f;
        {
            const float cdet = ka * kc - kb * kb, csum = ka + kc;
            if (cdet > 0.f && csum * csum <= 1000.f * cdet) {
                const float ex2 = sqrtf(qmax * kc / cdet) * 1.01f + 0.01f;
                const float ey2 = sqrtf(qmax * ka / cdet) * 1.01f + 0.01f;
                if (ex2 < 1e30f && ey2 < 1e30f) { cex = ex2; cey = ey2; }
            }
        }
        GaussRecord rec;
        rec.a = make_float4(u, v, qmax, o);
        rec.b = make_float4(ka, kb, kc, cey);
        rec.c = make_float4(rgb[0], rgb[1], rgb[2], cex);
        b.grec[g] = rec;
        b.rect[p] = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16));
        b.dkey[p] = __float_as_uint(pv[2]);
        vis = true;
    } while (0);
    UNIMGS_CHECK(p < b.st->cap_prims);
    b.touched[p] = touched;
    if (!vis) b.dkey[p] = 0xFFFFFFFFu;
    return vis;
}

// N3: Sigma = R S^2 R^T from the quaternion (w, x, y, z) and the scales
__device__ __forceinline__ void sigma_n3(float qw, float qx, float qy, float qz, float s0, float s1, float s2,
                                         float Sig[9]) {
    float w = qw, x = qx, y = qy, z = qz;
    const float n2 = fma_(w, w, fma_(x, x, fma_(y, y, mul(z, z))));
    const float k = dv(1.0f, __fsqrt_rn(n2));
    w = mul(w, k); x = mul(x, k); y = mul(y, k); z = mul(z, k);
    const float qxx = mul(x, x), qyy = mul(y, y), qzz = mul(z, z), qxy = mul(x, y), qxz = mul(x, z),
                qyz = mul(y, z), qwx = mul(w, x), qwy = mul(w, y), qwz = mul(w, z);
    float r[9];
    r[0] = sub(1.0f, mul(2.0f, add(qyy, qzz))); r[1] = mul(2.0f, sub(qxy, qwz)); r[2] = mul(2.0f, add(qxz, qwy));
    r[3] = mul(2.0f, add(qxy, qwz)); r[4] = sub(1.0f, mul(2.0f, add(qxx, qzz))); r[5] = mul(2.0f, sub(qyz, qwx));
    r[6] = mul(2.0f, sub(qxz, qwy)); r[7] = mul(2.0f, add(qyz, qwx)); r[8] = sub(1.0f, mul(2.0f, add(qxx, qyy)));
    float m[9];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        m[3 * a] = mul(r[3 * a], s0); m[3 * a + 1] = mul(r[3 * a + 1], s1); m[3 * a + 2] = mul(r[3 * a + 2], s2);
    }
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int c = 0; c < 3; c++) Sig[3 * a + c] = dot3(m + 3 * a, m + 3 * c);
}

__device__ __forceinline__ void sigma_given(const float *cv, float Sig[9]) {
    Sig[0] = __ldg(cv); Sig[1] = Sig[3] = __ldg(cv + 1); Sig[2] = Sig[6] = __ldg(cv + 2);
    Sig[4] = __ldg(cv + 3); Sig[5] = Sig[7] = __ldg(cv + 4); Sig[8] = __ldg(cv + 5);
}

// B1: one thread per Gaussian (N1-N5).
#ifndef UNIMGS_PRE_THREADS
#define UNIMGS_PRE_THREADS 64  // small CTAs (a divisor of kGaussRun): a finished CTA's slot is refilled at once
#endif
#ifndef UNIMGS_PRE_MINB
#define UNIMGS_PRE_MINB (5 * 256 / UNIMGS_PRE_THREADS)  // 48 registers
#endif
__global__ void __launch_bounds__(UNIMGS_PRE_THREADS, UNIMGS_PRE_MINB) k_preprocess_gaussians(GaussInput gin, int64_t F, CamParams cam,
                                                                               float dilation, Buffers b) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool vis = false;
    if (g < gin.N) {
        uint32_t touched = 0;
        // all per-Gaussian inputs except SH are loaded up front (one round trip)
        const float mx = __ldg(gin.means + 3 * g), my = __ldg(gin.means + 3 * g + 1), mz = __ldg(gin.means + 3 * g + 2);
        const bool qs = gin.cov3d == nullptr;
        const float qw = qs ? __ldg(gin.quats + 4 * g) : 1.f, qx = qs ? __ldg(gin.quats + 4 * g + 1) : 0.f,
                    qy = qs ? __ldg(gin.quats + 4 * g + 2) : 0.f, qz = qs ? __ldg(gin.quats + 4 * g + 3) : 0.f;
        const float s0 = qs ? __ldg(gin.scales + 3 * g) : 0.f, s1 = qs ? __ldg(gin.scales + 3 * g + 1) : 0.f,
                    s2 = qs ? __ldg(gin.scales + 3 * g + 2) : 0.f;
        const float o = __ldg(gin.opac + g);
        vis = project_gaussian(gin, g, F, cam, dilation, b, mx, my, mz, o, touched, [&](float Sig[9]) {
            if (gin.cov3d) sigma_given(gin.cov3d + 6 * g, Sig);  // given covariance (e.g. deformation transfer)
            else sigma_n3(qw, qx, qy, qz, s0, s1, s2, Sig);
        });
    }
    // per-warp counts into the (zeroed) count of the Gaussian's run of kGaussRun: no
    // CTA barrier, so a CTA retires as soon as its warps are done
    const unsigned cnt = __popc(__ballot_sync(0xffffffffu, vis));
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicAdd(&b.st->vis_g, cnt);
        atomicAdd(b.bcnt + (F + 255) / 256 + (g >> kGaussRunLog2), cnt);
    }
}

// B1 for several views of one scene (unimgs_preprocess_multi): every Gaussian's
// inputs -- and Sigma (N3) -- are read / computed once and projected into each view's
// context; the SH coefficients are re-read per view from L1 / L2.  Per view the
// arithmetic is exactly the single-view kernel's, so the records are bit-identical.
__global__ void __launch_bounds__(256, 4) k_preprocess_gaussians_multi(GaussInput gin, int64_t F,
                                                                                     MultiView mv, float dilation) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = g < gin.N;
    float mx = 0.f, my = 0.f, mz = 0.f, qw = 1.f, qx = 0.f, qy = 0.f, qz = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f, o = 0.f;
    if (in) {
        mx = __ldg(gin.means + 3 * g); my = __ldg(gin.means + 3 * g + 1); mz = __ldg(gin.means + 3 * g + 2);
        if (!gin.cov3d) {
            qw = __ldg(gin.quats + 4 * g); qx = __ldg(gin.quats + 4 * g + 1);
            qy = __ldg(gin.quats + 4 * g + 2); qz = __ldg(gin.quats + 4 * g + 3);
            s0 = __ldg(gin.scales + 3 * g); s1 = __ldg(gin.scales + 3 * g + 1); s2 = __ldg(gin.scales + 3 * g + 2);
        }
        o = __ldg(gin.opac + g);
    }
    // Sigma once for all views (the 6 distinct entries; in registers)
    float Sg[9];
    if (in) {
        if (gin.cov3d) sigma_given(gin.cov3d + 6 * g, Sg);
        else sigma_n3(qw, qx, qy, qz, s0, s1, s2, Sg);
    }
    const float c00 = Sg[0], c01 = Sg[1], c02 = Sg[2], c11 = Sg[4], c12 = Sg[5], c22 = Sg[8];
    for (int v = 0; v < mv.n; v++) {
        bool vis = false;
        if (in) {
            uint32_t touched = 0;
            vis = project_gaussian(gin, g, F, mv.cam[v], dilation, mv.buf[v], mx, my, mz, o, touched,
                                   [&](float S[9]) {
                                       S[0] = c00; S[1] = S[3] = c01; S[2] = S[6] = c02;
                                       S[4] = c11; S[5] = S[7] = c12; S[8] = c22;
                                   });
        }
        const unsigned cnt = __popc(__ballot_sync(0xffffffffu, vis));
        if ((threadIdx.x & 31) == 0 && cnt) {
            atomicAdd(&mv.buf[v].st->vis_g, cnt);
            atomicAdd(mv.buf[v].bcnt + (F + 255) / 256 + (g >> kGaussRunLog2), cnt);
        }
    }
}

int launch_preprocess_gaussians_multi(const GaussInput &g, int64_t F, const MultiView &mv, float dilation,
                                      cudaStream_t s) {
    if (g.N <= 0) return 0;
    for (int v = 0; v < mv.n; v++)
        cudaMemsetAsync(mv.buf[v].bcnt + (F + 255) / 256, 0,
                        sizeof(uint32_t) * (size_t)((g.N + kGaussRun - 1) / kGaussRun), s);
    const unsigned blocks = (unsigned)((g.N + 255) / 256);
    k_preprocess_gaussians_multi<<<blocks, 256, 0, s>>>(g, F, mv, dilation);
    return 1;
}

int launch_preprocess_gaussians(const GaussInput &g, int64_t F, const CamParams &cam, float dilation,
                                const Buffers &b, cudaStream_t s) {
    if (g.N <= 0) return 0;
    cudaMemsetAsync(b.bcnt + (F + 255) / 256, 0, sizeof(uint32_t) * (size_t)((g.N + kGaussRun - 1) / kGaussRun), s);
    const int threads = UNIMGS_PRE_THREADS;
    const unsigned blocks = (unsigned)((g.N + threads - 1) / threads);
    k_preprocess_gaussians<<<blocks, threads, 0, s>>>(g, F, cam, dilation, b);
    return 1;
}

// B2: one thread per triangle (N7).
__global__ void __launch_bounds__(256) k_setup_triangles(MeshInput m, CamParams cam, Buffers b) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool vis = false, guard = false;
    if (f < m.F) {
        uint32_t touched = 0;
        do {
            int id[3];
            int X[3], Y[3];
            float z[3];
            bool ok = true;
#pragma unroll
            for (int k = 0; k < 3; k++) {
                id[k] = __ldg(m.faces + 3 * f + k);
                if (id[k] < 0 || id[k] >= m.V) ok = false;
            }
            if (!ok) break;
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const float *P = m.pos + 3 * (int64_t)id[k];
                float pv[3];
                view_point(cam, __ldg(P), __ldg(P + 1), __ldg(P + 2), pv);
                if (!(pv[2] > cam.near_z) || pv[2] > cam.far_z) ok = false;
                const float u = fma_(cam.fx, dv(pv[0], pv[2]), cam.cx);
                const float v = fma_(cam.fy, dv(pv[1], pv[2]), cam.cy);
                if (!(fabsf(u) < 32768.0f && fabsf(v) < 32768.0f)) ok = false;
                X[k] = __float2int_rn(mul(u, 256.0f));
                Y[k] = __float2int_rn(mul(v, 256.0f));
                z[k] = pv[2];
            }
            if (!ok) { guard = true; break; }
            const float depth = dv(add(add(z[0], z[1]), z[2]), 3.0f);  // original face order
            const long long A2 = (long long)(X[1] - X[0]) * (Y[2] - Y[0]) - (long long)(X[2] - X[0]) * (Y[1] - Y[0]);
            if (A2 == 0) break;
            if (A2 < 0) {  // two-sided: swap vertices 1 and 2 with attributes
                int t;
                float tf;
                t = X[1]; X[1] = X[2]; X[2] = t;
                t = Y[1]; Y[1] = Y[2]; Y[2] = t;
                t = id[1]; id[1] = id[2]; id[2] = t;
                tf = z[1]; z[1] = z[2]; z[2] = tf;
            }
            const int mnx = min(X[0], min(X[1], X[2])), mxx = max(X[0], max(X[1], X[2]));
            const int mny = min(Y[0], min(Y[1], Y[2])), mxy = max(Y[0], max(Y[1], Y[2]));
            int x0 = mnx >> 12, x1 = mxx >> 12, y0 = mny >> 12, y1 = mxy >> 12;  // floor_div(., 4096)
            if (x1 < 0 || x0 > cam.tiles_x - 1 || y1 < 0 || y0 > cam.tiles_y - 1) break;
            x0 = max(x0, 0); y0 = max(y0, 0);
            x1 = min(x1, cam.tiles_x - 1); y1 = min(y1, cam.tiles_y - 1);
            touched = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
            int kind;
            float a[9];
            if (m.tex && m.uvs) {
                kind = 1;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    a[3 * k] = __ldg(m.uvs + 2 * (int64_t)id[k]);
                    a[3 * k + 1] = __ldg(m.uvs + 2 * (int64_t)id[k] + 1);
                    a[3 * k + 2] = 0.f;
                }
            } else if (m.cols) {
                kind = 0;
#pragma unroll
                for (int k = 0; k < 3; k++)
#pragma unroll
                    for (int c = 0; c < 3; c++) a[3 * k + c] = __ldg(m.cols + 3 * (int64_t)id[k] + c);
            } else {
                kind = 2;
#pragma unroll
                for (int k = 0; k < 9; k++) a[k] = 0.f;
            }
            TriRecord rec;
            rec.q0 = make_int4(X[0], Y[0], X[1], Y[1]);
            rec.q1 = make_int4(X[2], Y[2], kind, __float_as_int(__ldg(m.opac + f)));
            rec.q2 = make_float4(z[0], z[1], z[2], depth);
            rec.q3 = make_float4(a[0], a[1], a[2], a[3]);
            rec.q4 = make_float4(a[4], a[5], a[6], a[7]);
            rec.q5 = make_float4(a[8], 0.f, 0.f, 0.f);
            b.trec[f] = rec;
            b.rect[f] = make_uint2((uint32_t)x0 | ((uint32_t)y0 << 16), (uint32_t)x1 | ((uint32_t)y1 << 16));
            b.dkey[f] = __float_as_uint(depth);
            vis = true;
        } while (0);
        UNIMGS_CHECK(f < b.st->cap_prims);
        b.touched[f] = touched;
        if (!vis) b.dkey[f] = 0xFFFFFFFFu;
    }
    const unsigned cv = __popc(__ballot_sync(0xffffffffu, vis));
    const unsigned cg = __popc(__ballot_sync(0xffffffffu, guard));
    if ((threadIdx.x & 31) == 0) {
        if (cv) atomicAdd(&b.st->vis_t, cv);
        if (cg) atomicAdd(&b.st->culled_guard, cg);
    }
    block_count(vis, b.bcnt + blockIdx.x);
}

int launch_setup_triangles(const MeshInput &m, const CamParams &cam, const Buffers &b, cudaStream_t s) {
    if (m.F <= 0) return 0;
    const int threads = 256;
    const unsigned blocks = (unsigned)((m.F + threads - 1) / threads);
    k_setup_triangles<<<blocks, threads, 0, s>>>(m, cam, b);
    return 1;
}

}  // namespace unimgs
