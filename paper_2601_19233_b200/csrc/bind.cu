// bind.cu -- Gaussian-centric ray-cast binding (§3.3.1, P:387-398;
// SURVEY §8(f) row 4): "we cast rays from these cameras toward the center of a
// Gaussian ... The Gaussian is then bound to the nearest candidate face"
// (P:390-392), and with 8 rays per camera "toward the corners of a Gaussian's
// BBX.  For each ray, we retain the face closest to the Gaussian".
// The paper uses OptiX; here an LBVH built on the device and one
// thread per (Gaussian, target) that walks it for every camera.
//
//   k_centroid_bounds  scene box of the face centroids (ordered-int atomics)
//   k_morton           30-bit Morton code per valid face (invalid: 0xFFFFFFFF)
//   onesweep sort      (code, face) pairs, stable LSD (binning.cu's depth-sort kernels)
//                      (not on the per-frame path); invalid faces sort last
//   k_karras           internal nodes of the radix tree (Karras 2012): ranges
//                      and splits from common-prefix lengths, ties by index
//   k_leaf_boxes       padded leaf boxes, then the bottom-up union (the second
//                      child to arrive at a node computes it)
//   k_bind_trace       targets (B1), per camera a nearest-hit traversal (B2-B3),
//                      selection by distance to the centre (B4), output (B5)
//
// Bit-exactness (readings B1-B6): everything that decides a face or
// a barycentric -- targets, ray origin and direction, Moller-Trumbore, the hit
// distance -- is IEEE double with explicit _rn intrinsics in the order
// oracle/bind_oracle.c writes it (no FMA contraction).  The traversal only
// prunes with padded boxes and t_near > best t, and ties go to the lower face
// id, so the result does not depend on the visiting order: it equals the
// exhaustive search.

#include "internal.cuh"

namespace unimgs {

namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double ddot(const double a[3], const double b[3]) {
    return dadd(dadd(dm(a[0], b[0]), dm(a[1], b[1])), dm(a[2], b[2]));
}
__device__ __forceinline__ void dcross(const double a[3], const double b[3], double o[3]) {
    o[0] = dsub(dm(a[1], b[2]), dm(a[2], b[1]));
    o[1] = dsub(dm(a[2], b[0]), dm(a[0], b[2]));
    o[2] = dsub(dm(a[0], b[1]), dm(a[1], b[0]));
}

__device__ __forceinline__ unsigned f2ord(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

struct BvhScratch {
    unsigned *bounds;  // [6] ordered-int min xyz, max xyz; [6] = valid face count
    uint32_t *code[2], *face[2];
    int2 *child;       // [n-1] internal node children (unified numbering)
    int *parent;       // [2n-1]
    unsigned *arrive;  // [n-1]
    float4 *lo, *hi;   // [2n-1] padded boxes
};

__device__ __forceinline__ bool face_ok(const int32_t *faces, int64_t f, int64_t V, int32_t idx[3]) {
    for (int k = 0; k < 3; k++) {
        idx[k] = faces[3 * f + k];
        if (idx[k] < 0 || idx[k] >= V) return false;
    }
    return true;
}

__global__ void k_centroid_bounds(int64_t F, int64_t V, const float *__restrict__ pos, const int32_t *__restrict__ faces,
                                  unsigned *bounds) {
    unsigned mn[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, mx[3] = {0u, 0u, 0u};
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x) {
        int32_t id[3];
        if (!face_ok(faces, f, V, id)) continue;
        for (int a = 0; a < 3; a++) {
            const float c = (pos[3 * (int64_t)id[0] + a] + pos[3 * (int64_t)id[1] + a] + pos[3 * (int64_t)id[2] + a]) *
                            (1.f / 3.f);
            mn[a] = min(mn[a], f2ord(c));
            mx[a] = max(mx[a], f2ord(c));
        }
    }
    for (int a = 0; a < 3; a++) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    }
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; a++) {
            atomicMin(bounds + a, mn[a]);
            atomicMax(bounds + 3 + a, mx[a]);
        }
}

__device__ __forceinline__ unsigned spread10(unsigned v) {  // 10 bits -> every third bit
    v = (v * 0x00010001u) & 0xFF0000FFu;
    v = (v * 0x00000101u) & 0x0F00F00Fu;
    v = (v * 0x00000011u) & 0xC30C30C3u;
    v = (v * 0x00000005u) & 0x49249249u;
    return v;
}

__global__ void k_morton(int64_t F, int64_t V, const float *__restrict__ pos, const int32_t *__restrict__ faces,
                         unsigned *bounds, uint32_t *code, uint32_t *face) {
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    int32_t id[3];
    uint32_t c = 0xFFFFFFFFu;
    if (face_ok(faces, f, V, id)) {
        unsigned q[3];
        for (int a = 0; a < 3; a++) {
            const float lo = ord2f(bounds[a]), hi = ord2f(bounds[3 + a]);
            const float v = (pos[3 * (int64_t)id[0] + a] + pos[3 * (int64_t)id[1] + a] + pos[3 * (int64_t)id[2] + a]) *
                            (1.f / 3.f);
            const float x = hi > lo ? (v - lo) / (hi - lo) : 0.5f;
            q[a] = (unsigned)fminf(fmaxf(x * 1024.f, 0.f), 1023.f);
        }
        c = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
        atomicAdd(bounds + 6, 1u);
    }
    code[f] = c;
    face[f] = (uint32_t)f;
}

// common-prefix length of sorted codes i and j (ties broken by index), -1 outside [0, n)
__device__ __forceinline__ int delta(const uint32_t *code, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const uint32_t a = code[i], b = code[j];
    if (a != b) return __clz(a ^ b);
    return 32 + __clz((unsigned)i ^ (unsigned)j);
}

__global__ void k_karras(const unsigned *bounds, const uint32_t *__restrict__ code, int2 *child, int *parent) {
    const int n = (int)bounds[6];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = delta(code, n, i, i + 1) - delta(code, n, i, i - 1) >= 0 ? 1 : -1;
    const int dmin = delta(code, n, i, i - d);
    int lmax = 2;
    while (delta(code, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(code, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = delta(code, n, i, j);
    int s = 0;
    for (int t = (l + 1) >> 1;; t = (t + 1) >> 1) {
        if (delta(code, n, i, i + (s + t) * d) > dnode) s += t;
        if (t == 1) break;
    }
    const int gamma = i + s * d + min(d, 0);
    const int lo = min(i, j), hi = max(i, j);
    const int left = lo == gamma ? (n - 1) + gamma : gamma;             // leaf or internal
    const int right = hi == gamma + 1 ? (n - 1) + gamma + 1 : gamma + 1;
    child[i] = make_int2(left, right);
    parent[left] = i;
    parent[right] = i;
}

__global__ void k_leaf_boxes(const unsigned *bounds, int64_t V, const float *__restrict__ pos,
                             const int32_t *__restrict__ faces, const uint32_t *__restrict__ sface, const int2 *child,
                             const int *parent, unsigned *arrive, float4 *lo, float4 *hi) {
    const int n = (int)bounds[6];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t f = sface[i];
    float l[3], h[3];
    for (int a = 0; a < 3; a++) {
        float mn = pos[3 * (int64_t)faces[3 * f] + a], mx = mn;
        for (int k = 1; k < 3; k++) {
            const float v = pos[3 * (int64_t)faces[3 * f + k] + a];
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
        // pad by 1e-6 (|v| + 1): rounding can only move the padded bound outwards,
        // and the pad dwarfs the double error of any accepted hit point
        l[a] = mn - 1e-6f * (fabsf(mn) + 1.f);
        h[a] = mx + 1e-6f * (fabsf(mx) + 1.f);
    }
    int node = (n - 1) + i;
    lo[node] = make_float4(l[0], l[1], l[2], 0.f);
    hi[node] = make_float4(h[0], h[1], h[2], 0.f);
    if (n == 1) return;
    __threadfence();
    node = parent[node];
    while (true) {
        if (atomicAdd(arrive + node, 1u) == 0) return;  // the sibling finishes this node
        __threadfence();
        const int2 c = child[node];
        const float4 la = __ldcg(lo + c.x), lb = __ldcg(lo + c.y), ha = __ldcg(hi + c.x), hb = __ldcg(hi + c.y);
        lo[node] = make_float4(fminf(la.x, lb.x), fminf(la.y, lb.y), fminf(la.z, lb.z), 0.f);
        hi[node] = make_float4(fmaxf(ha.x, hb.x), fmaxf(ha.y, hb.y), fmaxf(ha.z, hb.z), 0.f);
        if (node == 0) return;
        __threadfence();
        node = parent[node];
    }
}

// B3: Moller-Trumbore in the oracle's operation order
__device__ __forceinline__ bool mt(const double o[3], const double d[3], const double v0[3], const double v1[3],
                                   const double v2[3], double &t, double &u, double &v) {
    double e1[3], e2[3], p[3], s[3], q[3];
    for (int a = 0; a < 3; a++) {
        e1[a] = dsub(v1[a], v0[a]);
        e2[a] = dsub(v2[a], v0[a]);
    }
    dcross(d, e2, p);
    const double det = ddot(e1, p);
    if (fabs(det) < 1e-9) return false;
    const double inv = __ddiv_rn(1.0, det);
    for (int a = 0; a < 3; a++) s[a] = dsub(o[a], v0[a]);
    const double uu = dm(ddot(s, p), inv);
    if (uu < 0.0 || uu > 1.0) return false;
    dcross(s, e1, q);
    const double vv = dm(ddot(d, q), inv);
    if (vv < 0.0 || dadd(uu, vv) > 1.0) return false;
    const double tt = dm(ddot(e2, q), inv);
    if (!(tt > 1e-6)) return false;
    t = tt;
    u = uu;
    v = vv;
    return true;
}

struct TraceArgs {
    int64_t N;
    const float *means, *quats, *scales;
    int mode;
    float k_sigma;
    int ncams;
    const float *cams;  // [C][12] R then t
    int64_t V;
    const float *pos;
    const int32_t *faces;
    const unsigned *bounds;
    const int2 *child;
    const float4 *lo, *hi;
    const uint32_t *sface;
    int32_t *face_out;
    float *bary_out;
    double *dist2_out;
};

constexpr int kStack = 64;

__global__ void __launch_bounds__(128) k_bind_trace(TraceArgs A) {
    const int K = A.mode == 0 ? 1 : 8;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= A.N * K) return;
    const int64_t g = gid / K;
    const int k = (int)(gid % K);
    const int n = (int)A.bounds[6];
    const double mu[3] = {A.means[3 * g], A.means[3 * g + 1], A.means[3 * g + 2]};
    double P[3];
    if (A.mode == 0) {
        for (int a = 0; a < 3; a++) P[a] = mu[a];
    } else {  // B1: corner k of the oriented box mu + R (+-k s)
        double w = A.quats[4 * g], x = A.quats[4 * g + 1], y = A.quats[4 * g + 2], z = A.quats[4 * g + 3];
        const double nq = __dsqrt_rn(dadd(dadd(dadd(dm(w, w), dm(x, x)), dm(y, y)), dm(z, z)));
        w = __ddiv_rn(w, nq); x = __ddiv_rn(x, nq); y = __ddiv_rn(y, nq); z = __ddiv_rn(z, nq);
        const double R[9] = {dsub(1.0, dm(2.0, dadd(dm(y, y), dm(z, z)))), dm(2.0, dsub(dm(x, y), dm(w, z))),
                             dm(2.0, dadd(dm(x, z), dm(w, y))),          dm(2.0, dadd(dm(x, y), dm(w, z))),
                             dsub(1.0, dm(2.0, dadd(dm(x, x), dm(z, z)))), dm(2.0, dsub(dm(y, z), dm(w, x))),
                             dm(2.0, dsub(dm(x, z), dm(w, y))),          dm(2.0, dadd(dm(y, z), dm(w, x))),
                             dsub(1.0, dm(2.0, dadd(dm(x, x), dm(y, y))))};
        const double kk = (double)A.k_sigma;
        const double l[3] = {dm((k & 1) ? kk : -kk, (double)A.scales[3 * g]),
                             dm((k & 2) ? kk : -kk, (double)A.scales[3 * g + 1]),
                             dm((k & 4) ? kk : -kk, (double)A.scales[3 * g + 2])};
        for (int a = 0; a < 3; a++)
            P[a] = dadd(mu[a], dadd(dadd(dm(R[3 * a], l[0]), dm(R[3 * a + 1], l[1])), dm(R[3 * a + 2], l[2])));
    }
    int64_t bf = -1;
    double bd = 0.0, bu = 0.0, bv = 0.0;
    int stack[kStack];
    for (int ci = 0; ci < A.ncams; ci++) {
        const float *Rf = A.cams + 12 * ci, *tf = Rf + 9;
        double c[3];
        for (int a = 0; a < 3; a++)
            c[a] = -dadd(dadd(dm((double)Rf[a], (double)tf[0]), dm((double)Rf[3 + a], (double)tf[1])),
                         dm((double)Rf[6 + a], (double)tf[2]));
        const double vz = dadd(dadd(dadd(dm((double)Rf[6], P[0]), dm((double)Rf[7], P[1])), dm((double)Rf[8], P[2])),
                               (double)tf[2]);
        if (!(vz > 0.0)) continue;  // B2: target behind this camera
        double d[3] = {dsub(P[0], c[0]), dsub(P[1], c[1]), dsub(P[2], c[2])};
        const double len = __dsqrt_rn(ddot(d, d));
        if (!(len > 0.0)) continue;
        for (int a = 0; a < 3; a++) d[a] = __ddiv_rn(d[a], len);
        double inv[3];
        for (int a = 0; a < 3; a++) inv[a] = d[a] != 0.0 ? 1.0 / d[a] : 0.0;
        // nearest hit along the ray (B3), ties to the lower face id
        int64_t hf = -1;
        double ht = 0.0, hu = 0.0, hv = 0.0;
        auto box_tnear = [&](int node, double &tn) {
            const float4 l4 = __ldg(A.lo + node), h4 = __ldg(A.hi + node);
            const double lo[3] = {l4.x, l4.y, l4.z}, hi[3] = {h4.x, h4.y, h4.z};
            double tmin = 0.0, tmax = 1e300;
            for (int a = 0; a < 3; a++) {
                if (d[a] != 0.0) {
                    const double t1 = (lo[a] - c[a]) * inv[a], t2 = (hi[a] - c[a]) * inv[a];
                    tmin = fmax(tmin, fmin(t1, t2));
                    tmax = fmin(tmax, fmax(t1, t2));
                } else if (c[a] < lo[a] || c[a] > hi[a]) {
                    return false;
                }
            }
            tn = tmin;
            return tmin <= tmax && (hf < 0 || tmin <= ht);
        };
        int sp = 0;
        double tn0;
        if (n > 0 && box_tnear(0, tn0)) stack[sp++] = 0;
        while (sp > 0) {
            const int node = stack[--sp];
            if (node >= n - 1) {  // leaf
                const int64_t f = A.sface[node - (n - 1)];
                double v0[3], v1[3], v2[3];
                const int32_t *fc = A.faces + 3 * f;
                for (int a = 0; a < 3; a++) {
                    v0[a] = A.pos[3 * (int64_t)fc[0] + a];
                    v1[a] = A.pos[3 * (int64_t)fc[1] + a];
                    v2[a] = A.pos[3 * (int64_t)fc[2] + a];
                }
                double t, u, v;
                if (mt(c, d, v0, v1, v2, t, u, v) && (hf < 0 || t < ht || (t == ht && f < hf))) {
                    hf = f;
                    ht = t; hu = u; hv = v;
                }
                continue;
            }
            const int2 ch = __ldg(A.child + node);
            double ta, tb;
            const bool ha = box_tnear(ch.x, ta), hb = box_tnear(ch.y, tb);
            if (ha && hb) {  // nearer child on top
                if (sp + 2 > kStack) { sp = -1; break; }
                if (ta <= tb) { stack[sp++] = ch.y; stack[sp++] = ch.x; }
                else { stack[sp++] = ch.x; stack[sp++] = ch.y; }
            } else if (ha || hb) {
                if (sp + 1 > kStack) { sp = -1; break; }
                stack[sp++] = ha ? ch.x : ch.y;
            }
        }
        if (sp < 0) {  // stack overflow (pathological tree): exhaustive fallback over the leaves
            hf = -1;
            for (int i = 0; i < n; i++) {
                const int64_t f = A.sface[i];
                double v0[3], v1[3], v2[3];
                const int32_t *fc = A.faces + 3 * f;
                for (int a = 0; a < 3; a++) {
                    v0[a] = A.pos[3 * (int64_t)fc[0] + a];
                    v1[a] = A.pos[3 * (int64_t)fc[1] + a];
                    v2[a] = A.pos[3 * (int64_t)fc[2] + a];
                }
                double t, u, v;
                if (mt(c, d, v0, v1, v2, t, u, v) && (hf < 0 || t < ht || (t == ht && f < hf))) {
                    hf = f;
                    ht = t; hu = u; hv = v;
                }
            }
        }
        if (hf < 0) continue;
        // B4: the hit nearest the Gaussian centre over the cameras
        double e[3];
        for (int a = 0; a < 3; a++) e[a] = dsub(dadd(c[a], dm(ht, d[a])), mu[a]);
        const double d2 = ddot(e, e);
        if (bf < 0 || d2 < bd || (d2 == bd && hf < bf)) {
            bf = hf;
            bd = d2; bu = hu; bv = hv;
        }
    }
    A.face_out[gid] = (int32_t)bf;
    float *b = A.bary_out + 3 * gid;
    if (bf >= 0) {
        b[0] = __double2float_rn(dsub(dsub(1.0, bu), bv));
        b[1] = __double2float_rn(bu);
        b[2] = __double2float_rn(bv);
    } else {
        b[0] = b[1] = b[2] = 0.f;
    }
    if (A.dist2_out) A.dist2_out[gid] = bf >= 0 ? bd : -1.0;
}

}  // namespace

int launch_bind(const BindInput &in, int32_t *face_out, float *bary_out, double *dist2_out, cudaStream_t s) {
    const int64_t F = in.F;
    const int64_t Fa = F > 0 ? F : 1;
    int launches = 0;
    BvhScratch b{};
    // the sort's scratch: a DevState (n_vis = F) and the look-back rows, both zeroed
    const int64_t lb_rows = sort_lookback_tiles(Fa, Fa);
    const size_t sort_bytes = sizeof(DevState) + 256 + (size_t)lb_rows * 256 * sizeof(unsigned long long);
    // one stream-ordered scratch block
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t nb = 2 * (size_t)Fa;
    const size_t sz[] = {al(8 * sizeof(unsigned)),  al(Fa * 4), al(Fa * 4), al(Fa * 4), al(Fa * 4),
                         al(Fa * sizeof(int2)),     al(nb * 4), al(Fa * 4), al(nb * 16), al(nb * 16),
                         al((size_t)in.ncams * 48), al(sort_bytes)};
    size_t total = 0;
    for (size_t x : sz) total += x;
    char *base = nullptr;
    if (cudaMallocAsync(&base, total, s) != cudaSuccess) return -1;
    char *p = base;
    auto take = [&](size_t i) { char *r = p; p += sz[i]; return r; };
    b.bounds = (unsigned *)take(0);
    b.code[0] = (uint32_t *)take(1); b.code[1] = (uint32_t *)take(2);
    b.face[0] = (uint32_t *)take(3); b.face[1] = (uint32_t *)take(4);
    b.child = (int2 *)take(5);
    b.parent = (int *)take(6);
    b.arrive = (unsigned *)take(7);
    b.lo = (float4 *)take(8);
    b.hi = (float4 *)take(9);
    float *cams = (float *)take(10);
    void *sort_tmp = take(11);
    const unsigned init[8] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u, 0u, 0u};
    cudaMemcpyAsync(b.bounds, init, sizeof init, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(cams, in.cams, (size_t)in.ncams * 48, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(b.arrive, 0, Fa * 4, s);
    if (F > 0) {
        const int blocks = (int)std::min<int64_t>((F + 255) / 256, 148 * 8);
        k_centroid_bounds<<<blocks, 256, 0, s>>>(F, in.V, in.pos, in.faces, b.bounds);
        k_morton<<<(unsigned)((F + 255) / 256), 256, 0, s>>>(F, in.V, in.pos, in.faces, b.bounds, b.code[0],
                                                             b.face[0]);
        {   // stable sort of (code, face); invalid faces (code 0xFFFFFFFF) last
            DevState *st = reinterpret_cast<DevState *>(sort_tmp);
            unsigned long long *lb = reinterpret_cast<unsigned long long *>(static_cast<char *>(sort_tmp) +
                                                                           al(sizeof(DevState)));
            cudaMemsetAsync(sort_tmp, 0, sort_bytes, s);
            const unsigned n32 = (unsigned)F;
            cudaMemcpyAsync(&st->n_vis, &n32, sizeof n32, cudaMemcpyHostToDevice, s);
            int dev = 0, sms = 148;
            if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            launches += launch_sort_u32_pairs(b.code, b.face, F, st, lb, sms, s);  // result in code[0] / face[0]
        }
        k_karras<<<(unsigned)((F + 255) / 256), 256, 0, s>>>(b.bounds, b.code[0], b.child, b.parent);
        k_leaf_boxes<<<(unsigned)((F + 255) / 256), 256, 0, s>>>(b.bounds, in.V, in.pos, in.faces, b.face[0], b.child,
                                                                 b.parent, b.arrive, b.lo, b.hi);
        launches += 4;
    }
    const int K = in.mode == 0 ? 1 : 8;
    const int64_t threads = in.N * K;
    if (threads > 0) {
        TraceArgs A{in.N,  in.means, in.quats, in.scales, in.mode,  in.k_sigma, in.ncams,  cams,      in.V,
                    in.pos, in.faces, b.bounds, b.child,   b.lo,     b.hi,       b.face[0], face_out, bary_out,
                    dist2_out};
        k_bind_trace<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(A);
        launches++;
    }
    cudaFreeAsync(base, s);
    return launches;
}

}  // namespace unimgs
