// deform.cu -- deformation transfer (Eq.12-13).
//
// One thread per Gaussian.  For each bound anchor i (K = 1 centre ray or 8 BBX
// corners) on face (v1, v2, v3) with barycentrics (u, v, w):
//   Delta_i = u Delta^1 + v Delta^2 + w Delta^3,  L_i = u log R^1 + v log R^2 + w log R^3,
//   S_i = u S^1 + v S^2 + w S^3                                        (Eq.12)
// then R' = exp(mean L_i) (Rodrigues), S' = mean S_i, A = R' S',
//   Sigma' = A Sigma A^T,  mu' = mu + mean Delta_i                      (Eq.13)
// Anchors with face < 0 are unbound and skipped; a Gaussian without bound
// anchors keeps mu and Sigma.  The per-vertex arrays are gathered through the
// read-only path (a proxy mesh of ~1e4-1e5 vertices stays L2-resident).
// Output: means [N][3], covariances [N][6] (xx xy xz yy yz zz) -- the cov3d
// input of unimgs_preprocess, so no eigen-refactoring is needed to render.
#include "internal.cuh"

namespace unimgs {

__global__ void __launch_bounds__(256) k_deform(DeformInput d, float *__restrict__ mu_out, float *__restrict__ cov_out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= d.N) return;
    float S[6];
    if (d.cov3d) {
#pragma unroll
        for (int a = 0; a < 6; a++) S[a] = __ldg(d.cov3d + 6 * g + a);
    } else {
        float w = __ldg(d.quats + 4 * g), x = __ldg(d.quats + 4 * g + 1), y = __ldg(d.quats + 4 * g + 2),
              z = __ldg(d.quats + 4 * g + 3);
        const float k = rsqrtf(w * w + x * x + y * y + z * z);
        w *= k; x *= k; y *= k; z *= k;
        const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                            2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                            2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
        const float s0 = __ldg(d.scales + 3 * g), s1 = __ldg(d.scales + 3 * g + 1), s2 = __ldg(d.scales + 3 * g + 2);
        const float e[3] = {s0 * s0, s1 * s1, s2 * s2};
        auto sig = [&](int a, int b) { return R[3 * a] * e[0] * R[3 * b] + R[3 * a + 1] * e[1] * R[3 * b + 1] + R[3 * a + 2] * e[2] * R[3 * b + 2]; };
        S[0] = sig(0, 0); S[1] = sig(0, 1); S[2] = sig(0, 2); S[3] = sig(1, 1); S[4] = sig(1, 2); S[5] = sig(2, 2);
    }
    float sd[3] = {0.f, 0.f, 0.f}, sl[3] = {0.f, 0.f, 0.f}, ss[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int n = 0;
    for (int i = 0; i < d.K; i++) {
        const int f = __ldg(d.face + g * d.K + i);
        if (f < 0 || f >= d.F) continue;
        const float *bw = d.bary + 3 * (g * d.K + i);
        const float b3[3] = {__ldg(bw), __ldg(bw + 1), __ldg(bw + 2)};
        const int v3[3] = {__ldg(d.faces + 3 * (int64_t)f), __ldg(d.faces + 3 * (int64_t)f + 1),
                           __ldg(d.faces + 3 * (int64_t)f + 2)};
        // a face with a vertex id outside [0, V) is junk: the anchor is skipped like an unbound one
        if ((unsigned)v3[0] >= (unsigned long long)d.V || (unsigned)v3[1] >= (unsigned long long)d.V ||
            (unsigned)v3[2] >= (unsigned long long)d.V)
            continue;
#pragma unroll
        for (int j = 0; j < 3; j++) {
            const float4 *vp = d.vdata + 3 * (int64_t)v3[j];
            const float4 p0 = __ldg(vp), p1 = __ldg(vp + 1), p2 = __ldg(vp + 2);
            const float wj = b3[j];
            sd[0] += wj * p0.x; sd[1] += wj * p0.y; sd[2] += wj * p0.z;
            sl[0] += wj * p0.w; sl[1] += wj * p1.x; sl[2] += wj * p1.y;
            ss[0] += wj * p1.z; ss[1] += wj * p1.w; ss[2] += wj * p2.x;
            ss[3] += wj * p2.y; ss[4] += wj * p2.z; ss[5] += wj * p2.w;
        }
        n++;
    }
    float *mo = mu_out + 3 * g, *co = cov_out + 6 * g;
    if (n == 0) {
#pragma unroll
        for (int a = 0; a < 3; a++) mo[a] = __ldg(d.means + 3 * g + a);
#pragma unroll
        for (int a = 0; a < 6; a++) co[a] = S[a];
        return;
    }
    const float inv = 1.f / (float)n;
    // R' = exp([L]x) by Rodrigues: I + a K + b K^2
    const float L0 = sl[0] * inv, L1 = sl[1] * inv, L2 = sl[2] * inv;
    const float th2 = L0 * L0 + L1 * L1 + L2 * L2, th = sqrtf(th2);
    float ca, cb;
    if (th < 1e-3f) {
        ca = 1.f - th2 * (1.f / 6.f);
        cb = 0.5f - th2 * (1.f / 24.f);
    } else {
        float sn, cs;
        sincosf(th, &sn, &cs);
        ca = sn / th;
        cb = (1.f - cs) / th2;
    }
    const float Kx[9] = {0.f, -L2, L1, L2, 0.f, -L0, -L1, L0, 0.f};
    float Rm[9];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const float k2 = Kx[3 * r] * Kx[c] + Kx[3 * r + 1] * Kx[3 + c] + Kx[3 * r + 2] * Kx[6 + c];
            Rm[3 * r + c] = (r == c ? 1.f : 0.f) + ca * Kx[3 * r + c] + cb * k2;
        }
    const float Sm[9] = {ss[0] * inv, ss[1] * inv, ss[2] * inv, ss[1] * inv, ss[3] * inv,
                         ss[4] * inv, ss[2] * inv, ss[4] * inv, ss[5] * inv};
    const float Sg[9] = {S[0], S[1], S[2], S[1], S[3], S[4], S[2], S[4], S[5]};
    float A[9], AS[9];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int c = 0; c < 3; c++)
            A[3 * r + c] = Rm[3 * r] * Sm[c] + Rm[3 * r + 1] * Sm[3 + c] + Rm[3 * r + 2] * Sm[6 + c];
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
        for (int c = 0; c < 3; c++)
            AS[3 * r + c] = A[3 * r] * Sg[c] + A[3 * r + 1] * Sg[3 + c] + A[3 * r + 2] * Sg[6 + c];
    auto sp = [&](int r, int c) { return AS[3 * r] * A[3 * c] + AS[3 * r + 1] * A[3 * c + 1] + AS[3 * r + 2] * A[3 * c + 2]; };
    co[0] = sp(0, 0); co[1] = sp(0, 1); co[2] = sp(0, 2); co[3] = sp(1, 1); co[4] = sp(1, 2); co[5] = sp(2, 2);
#pragma unroll
    for (int a = 0; a < 3; a++) mo[a] = __ldg(d.means + 3 * g + a) + sd[a] * inv;
}

int launch_deform(const DeformInput &d, float *mu_out, float *cov_out, cudaStream_t s) {
    if (d.N <= 0) return 0;
    k_deform<<<(unsigned)((d.N + 255) / 256), 256, 0, s>>>(d, mu_out, cov_out);
    return 1;
}

}  // namespace unimgs
