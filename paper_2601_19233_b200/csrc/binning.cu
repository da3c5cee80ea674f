// binning.cu -- per-tile key duplication, onesweep radix sort and tile ranges.
//
// "incorporate triangle fragments into the depth-sorting process" of
// the 3DGS tile rasterizer: every (tile, primitive) pair is ordered by
// (tile, bits(depth), unified id) -- the lexicographic order of the 64-bit key
// tile << 32 | bits(depth) with ties by id (readings R8, R9, R23).
//
// Pipeline (both sort modes produce the identical order):
//   k_scan_counts + k_compact   visible primitives in id order, reduce-then-
//                    scan over the per-CTA counts written by B1/B2 (no chains);
//   k_hist_depth     depth-digit histograms of the compacted keys.
//   sort_mode 0 (factored, default):
//     k_onesweep<u32> x4   stable LSD on the 32-bit depth key of the visible
//                          primitives (id ties stay in id order);
//     k_dup_count + k_scan_counts + k_range_starts + k_expand<false>
//                          tiles_touched scan in depth order (reduce-then-scan,
//                          sets K and the capacity flag) and load-balanced
//                          emission of (u16 tile, u32 id) pairs: fixed ranges of
//                          output slots per CTA, staged so every store is
//                          coalesced, with the tile-digit histograms of the
//                          radix passes;
//     k_onesweep<u16> x2   stable LSD on the tile id: pairs emitted in
//                          (depth, id) order come out in (tile, depth, id)
//                          order -- ~4x fewer bytes than sorting K 64-bit keys;
//     k_ranges16           tile ranges from the sorted tile ids.
//   sort_mode 1 (full, the literal form):
//     k_expand<true>       (tile << 32 | depth, id) pairs in id order;
//     k_onesweep<u64> x(4 + ceil(tile_bits/8)) over bits [0, 32 + tile_bits);
//     k_ranges64.
//
// Scans and sort passes are single-pass decoupled look-back over tiles claimed
// from an atomic counter (forward progress).  Look-back entries are 64-bit
// {epoch tag << 2 | flag, value}; the tag changes every pass of every frame, so
// nothing is cleared between frames and the whole frame is graph-capturable.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"

#ifndef UNIMGS_EXPAND_PER_SM
#define UNIMGS_EXPAND_PER_SM 4  // k_expand CTAs per SM (persistent over slot ranges)
#endif
#ifndef UNIMGS_SORT_ITEMS
#define UNIMGS_SORT_ITEMS 8
#endif

namespace unimgs {

constexpr unsigned kFlagAgg = 1, kFlagInc = 2;
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr int kSortThreads = 256, kSortItems = UNIMGS_SORT_ITEMS, kSortTile = kSortThreads * kSortItems;
#ifndef UNIMGS_LOOKWIN
#define UNIMGS_LOOKWIN 4
#endif
constexpr int kLookWin = UNIMGS_LOOKWIN;  // predecessors inspected per look-back round trip

// scan/pass slots (select the dynamic tile counter and the epoch tag)
enum { SLOT_COMPACT = 0, SLOT_DUP = 1, SLOT_PASS0 = 2, SLOT_RTS0 = 12 };  // ctr[16]
// histogram rows: 0..3 depth digits, 4..5 tile digits (weighted by pairs in mode 1)
enum { HIST_DEPTH0 = 0, HIST_TILE0 = 4 };

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long pack(unsigned tag, unsigned flag, unsigned v) {
    return ((unsigned long long)((tag << 2) | flag) << 32) | v;
}
__device__ __forceinline__ unsigned sat_add(unsigned a, unsigned b) {
    unsigned s = a + b;
    return s < a ? 0xFFFFFFFFu : s;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ unsigned epoch_tag(const DevState *st, int slot) {
    return (st->frame_epoch * 16u + (unsigned)slot) & 0x3FFFFFFFu;
}

// Claim the next tile of a dynamically scheduled pass (uniform across the block).
__device__ __forceinline__ unsigned claim_tile(unsigned *ctr, unsigned *s_tile) {
    __syncthreads();
    if (threadIdx.x == 0) *s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    return *s_tile;
}

// ----------------------------------------------------------------------------
// Reduce-then-scan (no look-back chains):
//   B2 / B1 write one visible count per run of 256 triangles / kGaussRun Gaussians (bcnt);
//   k_scan_counts scans a count array in place in one CTA;
//   k_compact writes every visible primitive at its CTA offset + local rank;
//   k_dup_count / k_scan_counts / k_expand do the same for the pairs.
// ----------------------------------------------------------------------------
// mode 0: total -> st->n_vis; mode 1: total -> needed / overflow / K (cap check)
__global__ void __launch_bounds__(1024) k_scan_counts(uint32_t *cnt, int64_t n, int mode, int64_t cap, DevState *st) {
    __shared__ unsigned s_w[32];
    __shared__ unsigned s_carry;
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < n; c0 += 4 * 1024) {
        unsigned v[4], tsum = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t i = c0 + 4 * (int64_t)threadIdx.x + j;
            v[j] = i < n ? cnt[i] : 0u;
            tsum = sat_add(tsum, v[j]);
        }
        unsigned x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x = sat_add(x, y);
        }
        const unsigned xe = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 31) s_w[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned w = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= (unsigned)o) w = sat_add(w, y);
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const unsigned carry = s_carry;
        unsigned run = sat_add(carry, sat_add(wid ? s_w[wid - 1] : 0u, lane ? xe : 0u));
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t i = c0 + 4 * (int64_t)threadIdx.x + j;
            if (i < n) cnt[i] = run;
            run = sat_add(run, v[j]);
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry = sat_add(carry, s_w[31]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const unsigned total = s_carry;
        if (mode == 0) {
            st->n_vis = total;
        } else {
            st->needed = total;
            const bool over = (int64_t)total > cap;
            st->overflow = over ? 1u : 0u;
            if (over) st->overflow_sticky = 1u;  // survives k_begin_frame of later views (unimgs_host_wait)
            st->K = over ? 0u : total;
        }
    }
}

// One CTA (256 threads) per count run, triangles first: a run of 256 triangles
// (B2's counts) or of kGaussRun Gaussians (B1's counts, walked 256 at a time); each
// visible primitive goes to its run's offset + its rank in the run.
__global__ void __launch_bounds__(256) k_compact(int64_t F, int64_t N, int nbt, const uint32_t *__restrict__ touched,
                                                 const uint32_t *__restrict__ dkey, const uint32_t *__restrict__ boff,
                                                 uint32_t *ok, uint32_t *ov, const DevState *st) {
    __shared__ unsigned s_c[2][8];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int blk = blockIdx.x;
    const bool tri = blk < nbt;
    unsigned base = boff[blk];
    const int nsub = tri ? 1 : kGaussRun / 256;
    for (int sub = 0; sub < nsub; sub++) {
        int64_t p;
        bool in;
        if (tri) {
            p = (int64_t)blk * 256 + threadIdx.x;
            in = p < F;
        } else {
            const int64_t g = (int64_t)(blk - nbt) * kGaussRun + sub * 256 + threadIdx.x;
            in = g < N;
            p = F + g;
        }
        const bool v = in && touched[p] > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, v);
        if (lane == 0) s_c[sub & 1][wid] = __popc(bal);
        __syncthreads();  // (double-buffered s_c: one barrier per sub-block)
        unsigned before = 0, total = 0;
#pragma unroll
        for (unsigned w = 0; w < 8; w++) {
            const unsigned c = s_c[sub & 1][w];
            before += w < wid ? c : 0u;
            total += c;
        }
        if (v) {
            const unsigned pos = base + before + __popc(bal & ((1u << lane) - 1u));
            UNIMGS_CHECK(pos < st->cap_prims);
            ok[pos] = dkey[p];
            ov[pos] = (uint32_t)p;
        }
        base += total;
    }
}

// Block-wide exclusive scan of warp-striped items (item i of lane l of warp w is
// element w * 32 * ITEMS + i * 32 + l), saturating u32.
template <int ITEMS>
__device__ __forceinline__ void block_scan_striped(const unsigned (&val)[ITEMS], unsigned (&excl)[ITEMS],
                                                   unsigned *s_w) {
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned carry = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        unsigned x = val[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x = sat_add(x, y);
        }
        const unsigned e = __shfl_up_sync(0xffffffffu, x, 1);
        excl[i] = sat_add(carry, lane ? e : 0u);
        carry = sat_add(carry, __shfl_sync(0xffffffffu, x, 31));
    }
    if (lane == 0) s_w[wid] = carry;
    __syncthreads();
    unsigned pre = 0;
    for (unsigned w = 0; w < wid; w++) pre = sat_add(pre, s_w[w]);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) excl[i] = sat_add(pre, excl[i]);
}

// Pair counts of CTA-sized runs (kScanTile) of the (sorted) visible primitives.
__global__ void __launch_bounds__(kScanThreads) k_dup_count(const uint32_t *__restrict__ ids,
                                                            const uint32_t *__restrict__ touched, uint32_t *dcnt,
                                                            uint32_t *prel, const DevState *st) {
    __shared__ unsigned s_w[8];
    const unsigned n = st->n_vis;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (base >= n) {
        if (threadIdx.x == 0) dcnt[blockIdx.x] = 0;
        return;
    }
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int e0 = (int)wid * 32 * kScanItems + (int)lane;  // warp-striped element index
    unsigned v[kScanItems], ex[kScanItems];
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        const int64_t j = base + e0 + 32 * i;
        v[i] = j < n ? touched[ids[j]] : 0u;
    }
    block_scan_striped<kScanItems>(v, ex, s_w);
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {  // in-chunk exclusive prefix of each sorted position
        const int64_t j = base + e0 + 32 * i;
        UNIMGS_CHECK(j >= n || j < st->cap_prims);
        if (j < n) prel[j] = ex[i];
    }
    if (threadIdx.x == kScanThreads - 1) dcnt[blockIdx.x] = sat_add(ex[kScanItems - 1], v[kScanItems - 1]);
}

// Depth-digit histograms (4 x 256 bins) of the compacted depth keys, for the
// four depth passes.  Persistent CTAs, CTA-shared histograms for the three low
// digits and warp-private ones for the top digit (few distinct exponent bytes:
// the contended one), one flush per CTA.
__global__ void __launch_bounds__(256) k_hist_depth(const uint32_t *__restrict__ keys, DevState *st) {
    __shared__ unsigned s_h[3 * 256];
    __shared__ unsigned s_top[8][256];
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) s_h[i] = 0;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&s_top[0][0])[i] = 0;
    __syncthreads();
    const unsigned n = st->n_vis, wid = threadIdx.x >> 5;
    auto add = [&](uint32_t k) {
        atomicAdd(&s_h[k & 255u], 1u);
        atomicAdd(&s_h[256 + ((k >> 8) & 255u)], 1u);
        atomicAdd(&s_h[512 + ((k >> 16) & 255u)], 1u);
        atomicAdd(&s_top[wid][k >> 24], 1u);
    };
    // 2 x 16-byte loads in flight per thread and iteration (keys is 16-byte aligned)
    const unsigned n8 = n / 8;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(keys);
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
        const uint4 a = __ldg(k4 + 2 * i), c = __ldg(k4 + 2 * i + 1);
        add(a.x); add(a.y); add(a.z); add(a.w);
        add(c.x); add(c.y); add(c.z); add(c.w);
    }
    for (unsigned i = 8 * n8 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) add(keys[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x)
        if (s_h[i]) atomicAdd(&st->hist[HIST_DEPTH0 + i / 256][i % 256], s_h[i]);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        unsigned t = 0;
        for (int w = 0; w < 8; w++) t += s_top[w][i];
        if (t) atomicAdd(&st->hist[HIST_DEPTH0 + 3][i], t);
    }
}


// Pair key type: u16 tile id (sort_mode 0) or u64 (tile << 32 | depth bits).
template <bool FULL>
struct DupCfg {
    using Key = typename std::conditional<FULL, unsigned long long, uint16_t>::type;
};

// N8: bits of triangle f's sort depth in tile
// (tx, ty) -- the view z of its plane at the tile centre, clamped to its z range.
// 1/z is affine in screen space: 1/z(P) = sum_k (E_k(P) / A2) / z_k with the
// exact integer edge functions of N7.  Normative order, in double:
// w_k = E_k / z_k; s = (w_0 + w_1) + w_2; z = (float)(A2 / s); s <= 0 -> max z.
__device__ __forceinline__ uint32_t tile_plane_depth_bits(const int4 q0, const int4 q1, const float4 q2, unsigned tx,
                                                          unsigned ty) {
    const long long PX = 4096ll * tx + 2048, PY = 4096ll * ty + 2048;
    const long long X0 = q0.x, Y0 = q0.y, X1 = q0.z, Y1 = q0.w, X2 = q1.x, Y2 = q1.y;
    const long long E0 = (X2 - X1) * (PY - Y1) - (Y2 - Y1) * (PX - X1);
    const long long E1 = (X0 - X2) * (PY - Y2) - (Y0 - Y2) * (PX - X2);
    const long long E2 = (X1 - X0) * (PY - Y0) - (Y1 - Y0) * (PX - X0);
    const long long A2 = (X1 - X0) * (Y2 - Y0) - (X2 - X0) * (Y1 - Y0);
    const double s = __dadd_rn(__dadd_rn(__ddiv_rn((double)E0, (double)q2.x), __ddiv_rn((double)E1, (double)q2.y)),
                               __ddiv_rn((double)E2, (double)q2.z));
    const float zmin = fminf(fminf(q2.x, q2.y), q2.z), zmax = fmaxf(fmaxf(q2.x, q2.y), q2.z);
    if (!(s > 0.0)) return __float_as_uint(zmax);
    return __float_as_uint(fminf(fmaxf(__double2float_rn(__ddiv_rn((double)A2, s)), zmin), zmax));
}

// ----------------------------------------------------------------------------
// k_range_starts + k_expand: the (tile, primitive) pairs, load-balanced over
// the OUTPUT.  The K pair slots are cut into ranges of ExpandCfg::SLOTS; the
// global offset of sorted primitive i is dcnt[i / kScanTile] + prel[i] (the
// chunk scan plus k_dup_count's in-chunk prefix), and k_range_starts records the
// primitive holding the first slot of every range.  One CTA per range (grid-
// stride) stages that range's primitives (<= SLOTS + 1: each has >= 1 pair) in
// shared memory; each thread expands 8 consecutive slots after one binary search
// (then walks forward), the keys and ids are staged and written out coalesced.
// Slot order = (primitive order, tile row-major).
// ----------------------------------------------------------------------------
template <bool FULL>
struct ExpandCfg {
    static constexpr int SLOTS = FULL ? 1024 : 2048;
    static constexpr int PER = SLOTS / kScanThreads;  // slots per thread
};

__global__ void k_range_starts(const uint32_t *__restrict__ dcnt, const uint32_t *__restrict__ prel, int slots,
                               uint32_t *rstart, const DevState *st) {
    const unsigned n = st->n_vis, K = st->K;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned off = dcnt[i / kScanTile] + prel[i];
        const unsigned nxt = i + 1 < n ? dcnt[(i + 1) / kScanTile] + prel[i + 1] : K;
        for (unsigned r = (off + slots - 1) / slots; (unsigned long long)r * slots < nxt && r * slots < K; r++) {
            UNIMGS_CHECK(r < st->cap_rstart);
            rstart[r] = i;
        }
    }
}

template <bool FULL>
__global__ void __launch_bounds__(kScanThreads) k_expand(const uint32_t *__restrict__ ids,
                                                         const uint2 *__restrict__ rect,
                                                         const uint32_t *__restrict__ dkey,
                                                         const uint32_t *__restrict__ dcnt,
                                                         const uint32_t *__restrict__ prel,
                                                         const uint32_t *__restrict__ rstart, int tiles_x,
                                                         const TriRecord *__restrict__ trec, unsigned F, int tri_depth,
                                                         int lo_bits, void *tk_, uint32_t *tv, uint32_t *tcnt,
                                                         DevState *st) {
    using Key = typename DupCfg<FULL>::Key;
    constexpr int SLOTS = ExpandCfg<FULL>::SLOTS, PER = ExpandCfg<FULL>::PER, MP = SLOTS + 2;
    __shared__ int s_off[MP];          // primitive start slot relative to the range (first may be < 0)
    __shared__ uint32_t s_id[MP];
    __shared__ uint2 s_rect[MP];
    __shared__ uint32_t s_dk[FULL ? MP : 1];
    __shared__ __align__(16) Key s_k[SLOTS];
    __shared__ __align__(16) uint32_t s_v[SLOTS];
    __shared__ unsigned s_hl[256], s_hh[256];
    __shared__ unsigned s_h3[FULL ? 256 : 1];  // mode 1: third tile digit (tile ids >= 65536)
    __shared__ unsigned s_hd[FULL ? 4 * 256 : 1];
    // s_mark[t]: the last primitive whose first slot lies in (t - 1) PER .. t PER (-1: none);
    // a prefix max over t gives each thread the primitive holding its first slot
    __shared__ int s_mark[kScanThreads];
    __shared__ int s_wm[kScanThreads / 32];
    Key *tk = reinterpret_cast<Key *>(tk_);
    if (st->overflow) return;
    const unsigned K = st->K, n = st->n_vis;
    const unsigned nranges = (K + SLOTS - 1) / SLOTS;
    if (blockIdx.x >= nranges) return;
    s_mark[threadIdx.x] = -1;
    for (int i = threadIdx.x; i < 256; i += kScanThreads) {
        s_hl[i] = s_hh[i] = 0;
        if (FULL) s_h3[FULL ? i : 0] = 0;
    }
    if (FULL)
        for (int i = threadIdx.x; i < 4 * 256; i += kScanThreads) s_hd[FULL ? i : 0] = 0;
    unsigned n_h3_zero = 0;
    for (unsigned r = blockIdx.x; r < nranges; r += gridDim.x) {
        const unsigned S = r * SLOTS, E = min(K, S + SLOTS), ns = E - S;
        const unsigned p0 = rstart[r];
        const unsigned p1 = r + 1 < nranges ? rstart[r + 1] : n - 1;  // holds slot E (or E - 1)
        const int m = (int)(p1 - p0) + 1;
        UNIMGS_CHECK(m >= 1 && m + 1 <= MP && p1 < n);
        __syncthreads();  // previous range's staging consumed
        if (!FULL)  // sort_mode 0: the range is one sort tile; its low-digit counts, per range
            for (int i = threadIdx.x; i < 256; i += kScanThreads) s_hl[i] = 0;
        for (int j = threadIdx.x; j < m; j += kScanThreads) {
            const unsigned i = p0 + j;
            const uint32_t id = ids[i];
            const int o = (int)(dcnt[i / kScanTile] + prel[i]) - (int)S;
            s_off[j] = o;
            s_id[j] = id;
            s_rect[j] = rect[id];
            if (FULL) s_dk[FULL ? j : 0] = dkey[id];
            const int b = o <= 0 ? 0 : (o + PER - 1) / PER;  // first thread whose first slot is >= o
            if (b < kScanThreads) atomicMax(&s_mark[b], j);
        }
        if (threadIdx.x == 0) s_off[m] = 0x7FFFFFFF;  // sentinel for the forward walk
        __syncthreads();
        // e = the largest j < m with s_off[j] <= k0: a block-wide prefix max of the marks
        int e;
        {
            const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            int v = s_mark[threadIdx.x];
            s_mark[threadIdx.x] = -1;  // reset for the next range (staged after its first barrier)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= (unsigned)o) v = max(v, y);
            }
            if (lane == 31) s_wm[w] = v;
            __syncthreads();
            for (unsigned q = 0; q < w; q++) v = max(v, s_wm[q]);
            e = v;
        }
        // thread t expands slots [t * PER, t * PER + PER) of the range
        const int k0 = (int)threadIdx.x * PER;
        if (k0 < (int)ns) {
            UNIMGS_CHECK(e >= 0 && e < m && s_off[e] <= k0 && s_off[e + 1] > k0);
            // the first slot's tile by one division, the rest by walking the rectangle
            // row-major (a primitive change lands on its first slot: local 0)
            unsigned x0, x1, tx, ty;
            uint32_t pid;
            {
                const uint2 rr = s_rect[e];
                x0 = rr.x & 0xFFFF, x1 = rr.y & 0xFFFF;
                const unsigned w = x1 - x0 + 1, local = (unsigned)(k0 - s_off[e]);
                const unsigned qq = local / w;
                tx = x0 + (local - qq * w), ty = (rr.x >> 16) + qq;
                pid = s_id[e];
            }
            for (int q = 0; q < PER; q++) {
                const int k = k0 + q;
                if (k >= (int)ns) break;
                if (q > 0) {
                    if (s_off[e + 1] <= k) {
                        while (s_off[e + 1] <= k) e++;
                        const uint2 rr = s_rect[e];
                        x0 = tx = rr.x & 0xFFFF, x1 = rr.y & 0xFFFF, ty = rr.x >> 16;
                        pid = s_id[e];
                    } else if (++tx > x1) {
                        tx = x0;
                        ty++;
                    }
                }
                const unsigned t = ty * (unsigned)tiles_x + tx;
                UNIMGS_CHECK(e < m && t < st->cap_tiles && S + (unsigned)k < st->cap_pairs &&
                             (unsigned)(k - s_off[e]) == (ty - (s_rect[e].x >> 16)) * (x1 - x0 + 1) + (tx - x0));
                if (FULL) {
                    uint32_t d = s_dk[FULL ? e : 0];
                    if (tri_depth && pid < F) {  // N8 per-tile triangle depth
                        const int4 *qp = reinterpret_cast<const int4 *>(trec + pid);
                        d = tile_plane_depth_bits(__ldg(qp), __ldg(qp + 1),
                                                  __ldg(reinterpret_cast<const float4 *>(qp + 2)), tx, ty);
                    }
                    s_k[k] = (Key)(((unsigned long long)t << 32) | d);
#pragma unroll
                    for (int dd = 0; dd < 4; dd++) atomicAdd(&s_hd[FULL ? dd * 256 + ((d >> (8 * dd)) & 255u) : 0], 1u);
                } else {
                    s_k[k] = (Key)t;
                }
                s_v[k] = pid;
                // sort_mode 0 splits the tile id into lo_bits + the rest (balanced digits)
                atomicAdd(&s_hl[FULL ? t & 255u : t & ((1u << lo_bits) - 1u)], 1u);
                if (FULL) atomicAdd(&s_hh[FULL ? (t >> 8) & 255u : 0], 1u);
                if (FULL) {
                    if (t >= 65536u) atomicAdd(&s_h3[FULL ? (t >> 16) & 255u : 0], 1u);
                    else n_h3_zero++;  // third tile digit 0, added once per thread below
                }
            }
        }
        __syncthreads();
        if (ns == (unsigned)SLOTS) {  // a full range: 16-byte copies (S is a multiple of SLOTS)
            const uint4 *sk4 = reinterpret_cast<const uint4 *>(s_k), *sv4 = reinterpret_cast<const uint4 *>(s_v);
            uint4 *tk4 = reinterpret_cast<uint4 *>(tk + S), *tv4 = reinterpret_cast<uint4 *>(tv + S);
            constexpr int NK4 = SLOTS * (int)sizeof(Key) / 16, NV4 = SLOTS * 4 / 16;
            for (int i = threadIdx.x; i < NK4; i += kScanThreads) tk4[i] = sk4[i];
            for (int i = threadIdx.x; i < NV4; i += kScanThreads) tv4[i] = sv4[i];
        } else {
            for (unsigned k = threadIdx.x; k < ns; k += kScanThreads) {
                tk[S + k] = s_k[k];
                tv[S + k] = s_v[k];
            }
        }
        if (!FULL)
            for (int i = threadIdx.x; i < 256; i += kScanThreads) tcnt[(size_t)r * 256 + i] = s_hl[i];
    }
    if (FULL && n_h3_zero) atomicAdd(&s_h3[0], n_h3_zero);
    if (!FULL) return;  // sort_mode 0: the reduce-then-scan tile sort needs no global histograms
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += kScanThreads) {
        if (s_hl[i]) atomicAdd(&st->hist[FULL ? 4 : HIST_TILE0][i], s_hl[i]);
        if (s_hh[i]) atomicAdd(&st->hist[FULL ? 5 : HIST_TILE0 + 1][i], s_hh[i]);
        // digit 0 of the third tile byte is every pair with a tile id < 65536
        if (FULL) {
            unsigned c3 = s_h3[FULL ? i : 0];
            if (c3) atomicAdd(&st->hist[6][i], c3);
        }
    }
    if (FULL)
        for (int i = threadIdx.x; i < 4 * 256; i += kScanThreads)
            if (s_hd[FULL ? i : 0]) atomicAdd(&st->hist[i / 256][i % 256], s_hd[FULL ? i : 0]);
}


// The lanes of the warp whose digit equals this lane's (the stable multisplit's peer
// mask; invalid lanes form a group of their own): one ballot per digit bit (4
// instructions per bit), or one MATCH.ANY -- whose cost grows with the number of
// distinct digits in the warp, so it is used only for the passes whose digits are
// nearly uniform across a warp (the depth key's top byte, the tile id's high digit).
template <int NB, bool MATCH>
__device__ __forceinline__ unsigned digit_peers(unsigned d, bool valid) {
    if constexpr (MATCH) {
        return __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu);
    } else {
        unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int bt = 0; bt < NB; bt++)  // peers &= bit ? ballot : ~ballot
            asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
                "and.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
                "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
                "@!p not.b32 t, t;\n\tand.b32 %0, %0, t;\n\t}"
                : "+r"(peers)
                : "r"(d), "r"(1u << bt));
        return peers;
    }
}

// ----------------------------------------------------------------------------
// One stable onesweep LSD pass on `bits` bits at `shift` (Adinets & Merrill).
// Tiles of 256 x ITEMS keys, warp-striped; warp-level multisplit ranking from
// one ballot per digit bit; keys are moved into shared memory at their block-sorted
// position BEFORE the per-digit decoupled look-back (so no key register is live
// across it); then a coalesced-by-digit scatter to global memory.
// ----------------------------------------------------------------------------
#ifndef UNIMGS_SORT_MINB
#define UNIMGS_SORT_MINB 4  // 64 registers: a sort CTA holds a quarter of the SM's register file
#endif
template <typename KT, int ITEMS, int NB, bool MATCH = false>
__global__ void __launch_bounds__(kSortThreads, (ITEMS <= 4 ? 4 : UNIMGS_SORT_MINB)) k_onesweep(const KT *__restrict__ kin,
                                                              const uint32_t *__restrict__ vin, KT *__restrict__ kout,
                                                              uint32_t *__restrict__ vout, const unsigned *n_ptr,
                                                              int shift, const unsigned *hist, int slot,
                                                              unsigned long long *lb, DevState *st) {
    static_assert(NB >= 1 && NB <= 8, "digit width");
    constexpr int TILE_ = kSortThreads * ITEMS;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned *s_wh = reinterpret_cast<unsigned *>(smem);           // [8][256]
    unsigned *s_doff = s_wh + 8 * 256;                              // [256] block-local digit offsets
    int *s_glob = reinterpret_cast<int *>(s_doff + 256);            // [256] global base - local offset
    unsigned *s_hex = reinterpret_cast<unsigned *>(s_glob + 256);   // [256] global exclusive histogram
    unsigned *s_misc = s_hex + 256;                                 // [16]
    KT *s_k = reinterpret_cast<KT *>(s_misc + 16);
    uint32_t *s_v = reinterpret_cast<uint32_t *>(s_k + TILE_);

    const unsigned n = *n_ptr;
    const unsigned tag = epoch_tag(st, slot);
    constexpr unsigned mask = (1u << NB) - 1u;
    const unsigned t = threadIdx.x, lane = t & 31, wid = t >> 5;

    // global exclusive digit offsets (block scan of the histogram, 1 digit per thread)
    {
        const unsigned h = hist[t];
        unsigned x = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) s_misc[8 + wid] = x;
        __syncthreads();
        unsigned add = 0;
        for (unsigned w = 0; w < wid; w++) add += s_misc[8 + w];
        s_hex[t] = x - h + add;
    }

    while (true) {
        const unsigned tile = claim_tile(&st->ctr[slot], &s_misc[1]);
        if ((unsigned long long)tile * TILE_ >= n) break;
        const unsigned base = tile * (unsigned)TILE_;
        for (int i = t; i < 8 * 256; i += kSortThreads) s_wh[i] = 0;
        __syncthreads();

        KT key[ITEMS];
        uint32_t val[ITEMS];
        unsigned rank[ITEMS];
        const unsigned wbase = base + wid * 32u * ITEMS + lane;
        const unsigned lt = lanemask_lt();
        unsigned *wh = s_wh + wid * 256;
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const unsigned idx = wbase + 32u * i;
            const bool valid = idx < n;
            key[i] = valid ? kin[idx] : (KT)0;
            val[i] = valid ? vin[idx] : 0u;
        }
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            // stable warp multisplit: the lanes holding the same digit
            const bool valid = wbase + 32u * i < n;
            const unsigned d = valid ? (unsigned)((key[i] >> shift) & mask) : 0u;
            const unsigned peers = digit_peers<NB, MATCH>(d, valid);
            const unsigned before = valid ? wh[d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0) wh[d] = before + __popc(peers);
            __syncwarp();
            rank[i] = before + __popc(peers & lt);
        }
        __syncthreads();
        // per digit: exclusive over warps, block count, publish the aggregate
        unsigned cnt = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const unsigned c = s_wh[w * 256 + t];
            s_wh[w * 256 + t] = cnt;
            cnt += c;
        }
        unsigned long long *my = lb + (size_t)tile * 256 + t;
        st_relaxed(my, pack(tag, tile == 0 ? kFlagInc : kFlagAgg, cnt));
        {  // block-exclusive scan of cnt over digits
            unsigned x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            if (lane == 31) s_misc[8 + wid] = x;
            __syncthreads();
            unsigned add = 0;
            for (unsigned w = 0; w < wid; w++) add += s_misc[8 + w];
            s_doff[t] = x - cnt + add;
        }
        __syncthreads();
        // keys into shared memory at their block-sorted position
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            if (wbase + 32u * i < n) {
                const unsigned d = (unsigned)((key[i] >> shift) & mask);
                const unsigned pos = s_doff[d] + wh[d] + rank[i];
                UNIMGS_CHECK(pos < (unsigned)TILE_);
                s_k[pos] = key[i];
                s_v[pos] = val[i];
            }
        }
        // look-back for digit t, kLookWin predecessors per round trip
        unsigned excl = 0;
        if (tile > 0) {
            int j = (int)tile - 1;
            while (true) {
                unsigned long long e[kLookWin];
#pragma unroll
                for (int k = 0; k < kLookWin; k++)
                    e[k] = (j - k >= 0) ? ld_relaxed(lb + (size_t)(j - k) * 256 + t) : pack(tag, kFlagInc, 0u);
                unsigned acc = 0;
                int k = 0;
                bool found = false;
                for (; k < kLookWin; k++) {
                    const unsigned hi = (unsigned)(e[k] >> 32);
                    const unsigned flag = ((hi >> 2) == tag) ? (hi & 3u) : 0u;
                    if (flag == 0) break;
                    acc += (unsigned)e[k];
                    if (flag == kFlagInc) { found = true; break; }
                }
                excl += acc;
                if (found) break;
                j -= k;  // retry from the first entry that was not ready
            }
            st_relaxed(my, pack(tag, kFlagInc, excl + cnt));
        }
        s_glob[t] = (int)(s_hex[t] + excl) - (int)s_doff[t];
        __syncthreads();
        const unsigned nt = min((unsigned)TILE_, n - base);
        for (unsigned k = t; k < nt; k += kSortThreads) {
            const KT kk = s_k[k];
            const unsigned d = (unsigned)((kk >> shift) & mask);
            const unsigned o = (unsigned)(s_glob[d] + (int)k);
            UNIMGS_CHECK(o < n);
            kout[o] = kk;
            vout[o] = s_v[k];
        }
    }
}

// ----------------------------------------------------------------------------
// Reduce-then-scan LSD pass over the u16 tile keys (sort_mode 0): no decoupled
// look-back, so no sort tile waits on another (the onesweep chain's spinning was
// ~40% of a tile pass's instructions).  Per pass:
//   counts   per sort tile (kSortTile keys) and digit: tcnt[tile][d] -- written by
//            k_expand for the first pass, by k_tile_count for the second;
//   scan     per group of kRtsGroup sort tiles: tcnt := exclusive prefix within the
//            group, gsum[group][d] := the group's total; the last CTA to finish
//            then makes gsum the exclusive prefix over groups and writes the digit
//            totals into gsum row `ngroups_max` (the histogram the downsweep scans);
//   down     per sort tile: the onesweep ranking (stable warp multisplit), then
//            global position = exclusive(totals)[d] + gsum[group][d] + tcnt[tile][d]
//            + the key's rank within the tile.
// ----------------------------------------------------------------------------
constexpr int kRtsGroup = 32;

template <typename KT, int NB>
__global__ void __launch_bounds__(256) k_tile_count(const KT *__restrict__ keys, const unsigned *n_ptr, int shift,
                                                    uint32_t *tcnt, const DevState *st) {
    __shared__ unsigned h[256];
    if (st->overflow) return;
    const unsigned n = *n_ptr;
    for (unsigned tile = blockIdx.x; (unsigned long long)tile * kSortTile < n; tile += gridDim.x) {
    const unsigned base = tile * (unsigned)kSortTile;
    __syncthreads();
    h[threadIdx.x] = 0;
    __syncthreads();
    constexpr unsigned mask = (1u << NB) - 1u;
    const unsigned i0 = base + 8 * threadIdx.x;  // 8 keys per thread, 16-byte loads
    if (i0 + 8 <= n) {
        if (sizeof(KT) == 2) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(keys + i0));
            const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                atomicAdd(&h[((w[j] & 0xFFFFu) >> shift) & mask], 1u);
                atomicAdd(&h[((w[j] >> 16) >> shift) & mask], 1u);
            }
        } else {
            const uint4 q0 = __ldg(reinterpret_cast<const uint4 *>(keys + i0));
            const uint4 q1 = __ldg(reinterpret_cast<const uint4 *>(keys + i0) + 1);
            const unsigned w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
            for (int j = 0; j < 8; j++) atomicAdd(&h[(w[j] >> shift) & mask], 1u);
        }
    } else {
        for (unsigned i = i0; i < n && i < i0 + 8; i++) atomicAdd(&h[((unsigned)keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    tcnt[(size_t)tile * 256 + threadIdx.x] = h[threadIdx.x];
    }
}

// Scan A, and -- in the last CTA to finish (threadfence + counter in DevState::ctr[slot])
// -- scan B over the group sums, so one launch scans a pass's counts.
__global__ void __launch_bounds__(256) k_rts_scan(uint32_t *tcnt, uint32_t *gsum, const unsigned *n_ptr, int totals_row,
                                                  int slot, DevState *st) {
    __shared__ bool s_last;
    if (st->overflow) return;
    const unsigned ntiles = (*n_ptr + kSortTile - 1) / kSortTile;
    const unsigned ng = (ntiles + kRtsGroup - 1) / kRtsGroup;
    const unsigned t0 = blockIdx.x * kRtsGroup;
    if (t0 >= ntiles) return;
    const unsigned t1 = min(ntiles, t0 + kRtsGroup), d = threadIdx.x;
    unsigned c[kRtsGroup];
#pragma unroll
    for (int i = 0; i < kRtsGroup; i++) c[i] = t0 + i < t1 ? tcnt[(size_t)(t0 + i) * 256 + d] : 0u;
    unsigned run = 0;
#pragma unroll
    for (int i = 0; i < kRtsGroup; i++) {
        if (t0 + i < t1) tcnt[(size_t)(t0 + i) * 256 + d] = run;
        run += c[i];
    }
    gsum[(size_t)blockIdx.x * 256 + d] = run;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&st->ctr[slot], 1u) == ng - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // scan B: exclusive prefix over the groups per digit, the digit totals in row totals_row
    unsigned acc = 0;
    for (unsigned g = 0; g < ng; g += 8) {
        unsigned v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = g + j < ng ? __ldcg(gsum + (size_t)(g + j) * 256 + d) : 0u;
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (g + j < ng) {
                gsum[(size_t)(g + j) * 256 + d] = acc;
                acc += v[j];
            }
    }
    gsum[(size_t)totals_row * 256 + d] = acc;
}

template <typename KT, int ITEMS, int NB, bool MATCH = false>
__global__ void __launch_bounds__(kSortThreads, UNIMGS_SORT_MINB) k_downsweep(const KT *__restrict__ kin,
                                                                           const uint32_t *__restrict__ vin,
                                                                           KT *__restrict__ kout,
                                                                           uint32_t *__restrict__ vout,
                                                                           const unsigned *n_ptr, int shift,
                                                                           const uint32_t *__restrict__ tcnt,
                                                                           const uint32_t *__restrict__ gsum,
                                                                           int totals_row, const DevState *st) {
    constexpr int TILE_ = kSortThreads * ITEMS;
    static_assert(TILE_ == kSortTile, "one count row per sort tile");
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned *s_wh = reinterpret_cast<unsigned *>(smem);           // [8][256]
    unsigned *s_doff = s_wh + 8 * 256;                              // [256] block-local digit offsets
    int *s_glob = reinterpret_cast<int *>(s_doff + 256);            // [256] global base - local offset
    unsigned *s_hex = reinterpret_cast<unsigned *>(s_glob + 256);   // [256] global exclusive digit offsets
    unsigned *s_misc = s_hex + 256;                                 // [16]
    KT *s_k = reinterpret_cast<KT *>(s_misc + 16);
    uint32_t *s_v = reinterpret_cast<uint32_t *>(s_k + TILE_);
    if (st->overflow) return;
    const unsigned n = *n_ptr;
    constexpr unsigned mask = (1u << NB) - 1u;
    const unsigned t = threadIdx.x, lane = t & 31, wid = t >> 5;
    unsigned hex;
    {   // exclusive scan of the digit totals, 1 digit per thread
        const unsigned h = gsum[(size_t)totals_row * 256 + t];
        unsigned x = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) s_misc[8 + wid] = x;
        __syncthreads();
        unsigned add = 0;
        for (unsigned w = 0; w < wid; w++) add += s_misc[8 + w];
        hex = x - h + add;
    }
    // persistent: sort tiles are independent (no look-back), so a fixed stride suffices
    for (unsigned tile = blockIdx.x; (unsigned long long)tile * TILE_ < n; tile += gridDim.x) {
    const unsigned base = tile * (unsigned)TILE_;
    __syncthreads();  // the previous tile's shared state consumed
    for (int i = t; i < 8 * 256; i += kSortThreads) s_wh[i] = 0;
    s_hex[t] = hex + gsum[(size_t)(tile / kRtsGroup) * 256 + t] + tcnt[(size_t)tile * 256 + t];
    __syncthreads();
    KT key[ITEMS];
    uint32_t val[ITEMS];
    unsigned rank[ITEMS];
    const unsigned wbase = base + wid * 32u * ITEMS + lane;
    const unsigned lt = lanemask_lt();
    unsigned *wh = s_wh + wid * 256;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const unsigned idx = wbase + 32u * i;
        const bool valid = idx < n;
        key[i] = valid ? kin[idx] : (KT)0;
        val[i] = valid ? vin[idx] : 0u;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const bool valid = wbase + 32u * i < n;
        const unsigned d = valid ? (unsigned)((key[i] >> shift) & mask) : 0u;
        const unsigned peers = digit_peers<NB, MATCH>(d, valid);
        const unsigned before = valid ? wh[d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0) wh[d] = before + __popc(peers);
        __syncwarp();
        rank[i] = before + __popc(peers & lt);
    }
    __syncthreads();
    unsigned cnt = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const unsigned c = s_wh[w * 256 + t];
        s_wh[w * 256 + t] = cnt;
        cnt += c;
    }
    {   // block-exclusive scan of cnt over digits
        unsigned x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) s_misc[8 + wid] = x;
        __syncthreads();
        unsigned add = 0;
        for (unsigned w = 0; w < wid; w++) add += s_misc[8 + w];
        s_doff[t] = x - cnt + add;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        if (wbase + 32u * i < n) {
            const unsigned d = (unsigned)((key[i] >> shift) & mask);
            const unsigned pos = s_doff[d] + wh[d] + rank[i];
            UNIMGS_CHECK(pos < (unsigned)TILE_);
            s_k[pos] = key[i];
            s_v[pos] = val[i];
        }
    }
    s_glob[t] = (int)s_hex[t] - (int)s_doff[t];
    __syncthreads();
    const unsigned nt = min((unsigned)TILE_, n - base);
    for (unsigned k = t; k < nt; k += kSortThreads) {
        const KT kk = s_k[k];
        const unsigned d = (unsigned)((kk >> shift) & mask);
        const unsigned o = (unsigned)(s_glob[d] + (int)k);
        UNIMGS_CHECK(o < n);
        kout[o] = kk;
        vout[o] = s_v[k];
    }
    }
}

// ranges[tile] = [first, last + 1) over the sorted u16 tile keys; 8 keys per
// thread through one 16-byte load (the buffer base is 256-byte aligned).
__global__ void __launch_bounds__(256) k_ranges16(const uint16_t *__restrict__ keys, const unsigned *n_ptr,
                                                  uint2 *ranges, const DevState *st) {
    if (st->overflow) return;
    const unsigned n = *n_ptr;
    const unsigned chunks = (n + 7) / 8;
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < chunks; c += gridDim.x * blockDim.x) {
        const unsigned i0 = c * 8;
        uint16_t k[8];
        if (i0 + 8 <= n) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(keys) + c);
            const uint16_t *p = reinterpret_cast<const uint16_t *>(&q);
#pragma unroll
            for (int j = 0; j < 8; j++) k[j] = p[j];
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) k[j] = i0 + j < n ? keys[i0 + j] : 0;
        }
        const unsigned prev = i0 > 0 ? keys[i0 - 1] : 0xFFFFFFFFu;
        const unsigned next = i0 + 8 < n ? keys[i0 + 8] : 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (i0 + j >= n) break;
            const unsigned cur = k[j];
            UNIMGS_CHECK(cur < st->cap_tiles);
            const unsigned pv = j ? (unsigned)k[j - 1] : prev;
            const unsigned nx = (j < 7 && i0 + j + 1 < n) ? (unsigned)k[j + 1] : (i0 + j + 1 < n ? next : 0xFFFFFFFFu);
            if (cur != pv) ranges[cur].x = i0 + j;
            if (cur != nx) ranges[cur].y = i0 + j + 1;
        }
    }
}

__global__ void k_ranges64(const unsigned long long *__restrict__ keys, const unsigned *n_ptr, uint2 *ranges,
                           const DevState *st) {
    if (st->overflow) return;
    const unsigned n = *n_ptr;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned tl = (unsigned)(keys[i] >> 32);
        UNIMGS_CHECK(tl < st->cap_tiles);
        const unsigned prev = i > 0 ? (unsigned)(keys[i - 1] >> 32) : 0xFFFFFFFFu;
        const unsigned next = i + 1 < n ? (unsigned)(keys[i + 1] >> 32) : 0xFFFFFFFFu;
        if (tl != prev) ranges[tl].x = i;
        if (tl != next) ranges[tl].y = i + 1;
    }
}

template <typename KT, int ITEMS>
static size_t onesweep_smem() {
    return (8 * 256 + 256 * 3 + 16) * sizeof(unsigned) + kSortThreads * ITEMS * (sizeof(KT) + sizeof(uint32_t));
}
#ifndef UNIMGS_DEPTH_ITEMS
#define UNIMGS_DEPTH_ITEMS 8
#endif
constexpr int kDepthItems = UNIMGS_DEPTH_ITEMS;  // small depth sort: short tiles, latency-bound


int64_t sort_lookback_tiles(int64_t max_pairs, int64_t max_prims) {
    const int64_t pair_tiles = (max_pairs + kSortTile - 1) / kSortTile;
    const int64_t prim_tiles = (max_prims + kSortThreads * kDepthItems - 1) / (kSortThreads * kDepthItems);
    return std::max<int64_t>(pair_tiles, prim_tiles) + 2;
}

static int bits_for(int64_t tiles) {
    int b = 0;
    while (((int64_t)1 << b) < tiles) b++;
    return b;
}

template <typename KT, int ITEMS, int NB, bool MATCH = false>
static void onesweep_launch(DevState *st, unsigned long long *lookback, const KT *kin, const uint32_t *vin, KT *kout,
                            uint32_t *vout, const unsigned *n_ptr, int shift, int hist_row, int slot, int grid,
                            cudaStream_t s) {
    static const bool attr = [] {  // dynamic shared memory above 48 KB, once per instantiation (thread-safe)
        cudaFuncSetAttribute(k_onesweep<KT, ITEMS, NB, MATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)onesweep_smem<KT, ITEMS>());
        return true;
    }();
    (void)attr;
    k_onesweep<KT, ITEMS, NB, MATCH><<<grid, kSortThreads, onesweep_smem<KT, ITEMS>(), s>>>(
        kin, vin, kout, vout, n_ptr, shift, &st->hist[hist_row][0], slot, lookback, st);
}

template <typename KT, int ITEMS = kSortItems>
static void onesweep_pass(Buffers &b, const KT *kin, const uint32_t *vin, KT *kout, uint32_t *vout,
                          const unsigned *n_ptr, int shift, int bits, int hist_row, int slot, int grid,
                          cudaStream_t s) {
#define UNIMGS_OS(NB) \
    onesweep_launch<KT, ITEMS, NB>(b.st, b.lookback, kin, vin, kout, vout, n_ptr, shift, hist_row, slot, grid, s)
    switch (bits) {
        case 1: UNIMGS_OS(1); break;
        case 2: UNIMGS_OS(2); break;
        case 3: UNIMGS_OS(3); break;
        case 4: UNIMGS_OS(4); break;
        case 5: UNIMGS_OS(5); break;
        case 6: UNIMGS_OS(6); break;
        case 7: UNIMGS_OS(7); break;
        default: UNIMGS_OS(8); break;
    }
#undef UNIMGS_OS
}

static int sort_grid(int64_t max_items, int sm_count, int per_sm, int tile = kSortTile) {
    const int64_t tiles = (max_items + tile - 1) / tile;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count * per_sm));
}

// Blend schedule (longest first): the hardware hands out CTAs in blockIdx order,
// so listing the tiles by decreasing pair count lets the few heavy tiles start in
// the first wave instead of forming the tail.  Counting sort on an 8-bit
// log-scale bucket (fp32 exponent + 3 mantissa bits of the count); the order
// within a bucket is arbitrary (each tile's pixels do not depend on it).
__global__ void __launch_bounds__(1024) k_tile_order(const uint2 *__restrict__ ranges, int tiles, uint32_t *order,
                                                     const DevState *st) {
    __shared__ unsigned s_h[256];
    if (st->overflow) return;
    auto bucket = [](const uint2 r) {
        const unsigned len = r.y - r.x;
        if (!len) return 0u;
        return min(255u, (__float_as_uint((float)len) >> 20) - 1015u);  // 1..201 for len < 2^24
    };
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < tiles; i += blockDim.x) atomicAdd(&s_h[bucket(ranges[i])], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan from the heaviest bucket down
        unsigned carry = 0;
        for (int c = 7; c >= 0; c--) {
            const int k = c * 32 + (31 - (int)threadIdx.x);  // lane 0 = highest bucket of the chunk
            const unsigned v = s_h[k];
            unsigned x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
                if ((int)threadIdx.x >= o) x += y;
            }
            s_h[k] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < tiles; i += blockDim.x) order[atomicAdd(&s_h[bucket(ranges[i])], 1u)] = (uint32_t)i;
}

// Per-kernel device times of one launch_bin call (UNIMGS_BIN_EVENTS=1: events after
// every launch on the bin stream, printed to stderr; a diagnostic that synchronises).
struct BinMarks {
    bool on = false;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[48];
    const char *name[48];
    int n = 0;
    explicit BinMarks(cudaStream_t st) : s(st) {
        static const bool en = getenv("UNIMGS_BIN_EVENTS") != nullptr;
        on = en;
        if (on) mark("start");
    }
    void mark(const char *nm) {
        if (!on || n >= 48) return;
        cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], s);
        name[n++] = nm;
    }
    ~BinMarks() {
        if (!on) return;
        cudaEventSynchronize(ev[n - 1]);
        for (int i = 1; i < n; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, "bin_event %s %.4f\n", name[i], ms);
        }
        for (int i = 0; i < n; i++) cudaEventDestroy(ev[i]);
    }
};

int launch_bin(Buffers &b, int64_t P, int64_t N, int64_t F, const CamParams &cam, int sort_mode, int tri_depth,
               cudaStream_t s, int sm_count, int sort_per_sm) {
    (void)N;
    int launches = 0;
    BinMarks mk(s);
    const int64_t tiles = (int64_t)cam.tiles_x * cam.tiles_y;
    const int tb = bits_for(tiles);
    const bool full = sort_mode == 1;
    cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * (size_t)tiles, s);
    // compaction of the visible primitives (B2 then B1 CTA counts)
    const int nbt = (int)((F + 255) / 256), nbg = (int)((N + kGaussRun - 1) / kGaussRun);
    if (P > 0) {
        k_scan_counts<<<1, 1024, 0, s>>>(b.bcnt, nbt + nbg, 0, 0, b.st);
        k_compact<<<nbt + nbg, 256, 0, s>>>(F, N, nbt, b.touched, b.dkey, b.bcnt, b.pk[0], b.pv[0], b.st);
        launches += 2;
        mk.mark("scan+compact");
    }
    int slot = SLOT_PASS0;
    const int dgrid = (int)std::max<int64_t>(1, (P + kScanTile - 1) / kScanTile);
    int tc = 0;
    const uint32_t *dup_ids;
    if (!full) {
        // depth sort of the visible primitives: 4 onesweep passes (1.5 M keys, L2-resident:
        // the decoupled look-back's single launch per pass beats reduce-then-scan's four
        // there -- measured: bench +0.5%, but single-stream bin +3% mip360, +13% nerf)
        k_hist_depth<<<sm_count * 2, 256, 0, s>>>(b.pk[0], b.st);
        launches++;
        mk.mark("hist_depth");
        const int g1 = sort_grid(P, sm_count, sort_per_sm, kSortThreads * kDepthItems);
        int cur = 0;
        for (int pass = 0; pass < 4; pass++, slot++) {
            if (pass == 3)  // the exponent byte: few distinct digits per warp
                onesweep_launch<uint32_t, kDepthItems, 8, true>(b.st, b.lookback, b.pk[cur], b.pv[cur], b.pk[cur ^ 1],
                                                                b.pv[cur ^ 1], &b.st->n_vis, 24, HIST_DEPTH0 + 3, slot,
                                                                g1, s);
            else
                onesweep_pass<uint32_t, kDepthItems>(b, b.pk[cur], b.pv[cur], b.pk[cur ^ 1], b.pv[cur ^ 1],
                                                     &b.st->n_vis, 8 * pass, 8, HIST_DEPTH0 + pass, slot, g1, s);
            cur ^= 1;
            launches++;
            mk.mark("depth_onesweep");
        }
        dup_ids = b.pv[cur];
    } else {
        dup_ids = b.pv[0];
    }
    // pair counts per run of kScanTile primitives -> scan (K, capacity) -> emission
    uint32_t *prel = b.pk[1];  // free after the depth sort (its result is in pk[0] / pv[0])
    k_dup_count<<<dgrid, kScanThreads, 0, s>>>(dup_ids, b.touched, b.dcnt, prel, b.st);
    k_scan_counts<<<1, 1024, 0, s>>>(b.dcnt, dgrid, 1, b.max_pairs, b.st);
    launches += 2;
    mk.mark("dup_count+scan");
    {
        const int slots = full ? ExpandCfg<true>::SLOTS : ExpandCfg<false>::SLOTS;
        k_range_starts<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((P + 255) / 256, sm_count * 16)), 256, 0,
                         s>>>(b.dcnt, prel, slots, b.rstart, b.st);
        launches++;
        mk.mark("range_starts");
    }
    const int egrid = (int)std::max<int64_t>(1, std::min<int64_t>((b.max_pairs + 1023) / 1024, sm_count * UNIMGS_EXPAND_PER_SM));
    const int g2 = sort_grid(b.max_pairs, sm_count, sort_per_sm);
    if (!full) {
        // balanced digits (13 tile bits at 1080p: 7 + 6, not 8 + 5): fewer buckets per
        // 2048-key sort tile, so longer runs in each pass's scatter
        const int npass = (tb + 7) / 8, lo_bits = npass > 1 ? (tb + npass - 1) / npass : std::max(tb, 1);
        k_expand<false><<<egrid, kScanThreads, 0, s>>>(dup_ids, b.rect, b.dkey, b.dcnt, prel, b.rstart, cam.tiles_x,
                                                        b.trec, (unsigned)F, 0, lo_bits, b.tk[0], b.tv[0], b.tcnt,
                                                        b.st);
        launches++;
        mk.mark("expand");
        // reduce-then-scan passes (k_expand wrote the first pass's per-tile counts)
        const int ntile_max = (int)((b.max_pairs + kSortTile - 1) / kSortTile);
        const int ngroup_max = (ntile_max + kRtsGroup - 1) / kRtsGroup;
        for (int pass = 0, sh = 0; sh < tb; pass++, slot++) {
            const int nb = pass == 0 ? lo_bits : tb - sh;
            const uint16_t *kin = (const uint16_t *)b.tk[tc];
#define UNIMGS_NB_SWITCH(CALL)  \
    switch (nb) {               \
        case 1: CALL(1); break; \
        case 2: CALL(2); break; \
        case 3: CALL(3); break; \
        case 4: CALL(4); break; \
        case 5: CALL(5); break; \
        case 6: CALL(6); break; \
        case 7: CALL(7); break; \
        default: CALL(8); break; \
    }
            if (pass > 0) {
#define UNIMGS_TC(NB) \
    k_tile_count<uint16_t, NB><<<std::min(ntile_max, sm_count * 8), 256, 0, s>>>(kin, &b.st->K, sh, b.tcnt, b.st)
                UNIMGS_NB_SWITCH(UNIMGS_TC)
#undef UNIMGS_TC
                launches++;
                mk.mark("tile_count");
            }
            k_rts_scan<<<ngroup_max, 256, 0, s>>>(b.tcnt, b.gsum, &b.st->K, ngroup_max, SLOT_RTS0 + pass, b.st);
            mk.mark("rts_scan");
            const size_t smem = onesweep_smem<uint16_t, kSortItems>();
            // the high tile digit (tile rows) is nearly uniform across a warp: MATCH.ANY
#define UNIMGS_DS(NB)                                                                                             \
    do {                                                                                                          \
        if (pass > 0)                                                                                             \
            k_downsweep<uint16_t, kSortItems, NB, true><<<g2, kSortThreads, smem, s>>>(                           \
                kin, b.tv[tc], (uint16_t *)b.tk[tc ^ 1], b.tv[tc ^ 1], &b.st->K, sh, b.tcnt, b.gsum, ngroup_max,   \
                b.st);                                                                                            \
        else                                                                                                      \
            k_downsweep<uint16_t, kSortItems, NB><<<g2, kSortThreads, smem, s>>>(                                 \
                kin, b.tv[tc], (uint16_t *)b.tk[tc ^ 1], b.tv[tc ^ 1], &b.st->K, sh, b.tcnt, b.gsum, ngroup_max,   \
                b.st);                                                                                            \
    } while (0)
            UNIMGS_NB_SWITCH(UNIMGS_DS)
#undef UNIMGS_DS
#undef UNIMGS_NB_SWITCH
            launches += 2;
            mk.mark("downsweep");
            sh += nb;
            tc ^= 1;
        }
        b.key_bytes = 2;
        k_ranges16<<<sm_count * 4, 256, 0, s>>>((const uint16_t *)b.tk[tc], &b.st->K, b.ranges, b.st);
        launches++;
        mk.mark("ranges16");
    } else {
        k_expand<true><<<egrid, kScanThreads, 0, s>>>(dup_ids, b.rect, b.dkey, b.dcnt, prel, b.rstart, cam.tiles_x,
                                                       b.trec, (unsigned)F, tri_depth, 8, b.tk[0], b.tv[0], nullptr,
                                                       b.st);
        launches++;
        const int total_bits = 32 + tb;
        for (int pass = 0, sh = 0; sh < total_bits; pass++, sh += 8, slot++) {
            onesweep_pass<unsigned long long>(b, (const unsigned long long *)b.tk[tc], b.tv[tc],
                                              (unsigned long long *)b.tk[tc ^ 1], b.tv[tc ^ 1], &b.st->K, sh,
                                              std::min(8, total_bits - sh), pass, slot, g2, s);
            tc ^= 1;
            launches++;
        }
        b.key_bytes = 8;
        k_ranges64<<<sm_count * 4, 256, 0, s>>>((const unsigned long long *)b.tk[tc], &b.st->K, b.ranges, b.st);
        launches++;
    }
    b.sorted_keys = b.tk[tc];
    b.sorted_vals = b.tv[tc];
    k_tile_order<<<1, 1024, 0, s>>>(b.ranges, (int)tiles, b.order, b.st);
    launches++;
    mk.mark("tile_order");
    return launches;  // kernels only (the ranges memset is not counted)
}

// Stable LSD sort of n (u32 key, u32 value) pairs, 4 x 8-bit onesweep passes with the
// depth-sort kernels (the ray-cast binding's Morton codes, bind.cu): keys[0]/vals[0] in,
// result back in keys[0]/vals[0] (keys[1]/vals[1] scratch).  st: a zeroed DevState whose
// n_vis holds n; lookback: zeroed [sort_lookback_tiles(n, n)][256].
int launch_sort_u32_pairs(uint32_t *keys[2], uint32_t *vals[2], int64_t n, DevState *st, unsigned long long *lookback,
                          int sm_count, cudaStream_t s) {
    if (n <= 0) return 0;
    k_hist_depth<<<sm_count * 2, 256, 0, s>>>(keys[0], st);
    const int grid = sort_grid(n, sm_count, 4, kSortThreads * kDepthItems);
    for (int pass = 0; pass < 4; pass++)
        onesweep_launch<uint32_t, kDepthItems, 8>(st, lookback, keys[pass & 1], vals[pass & 1], keys[(pass & 1) ^ 1],
                                                  vals[(pass & 1) ^ 1], &st->n_vis, 8 * pass, HIST_DEPTH0 + pass,
                                                  SLOT_PASS0 + pass, grid, s);
    return 5;
}

// ---- debug / stats ------------------------------------------------------------
__global__ void k_full_keys(const void *skeys, int key_bytes, const uint32_t *vals, const uint32_t *dkey,
                            const DevState *st, uint64_t *out) {
    const unsigned n = st->K;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (key_bytes == 8) out[i] = reinterpret_cast<const unsigned long long *>(skeys)[i];
        else out[i] = ((uint64_t)reinterpret_cast<const uint16_t *>(skeys)[i] << 32) | dkey[vals[i]];
    }
}

int launch_full_keys(const Buffers &b, uint64_t *keys, cudaStream_t s) {
    k_full_keys<<<256, 256, 0, s>>>(b.sorted_keys, b.key_bytes, b.sorted_vals, b.dkey, b.st, keys);
    return 1;
}

__global__ void k_tile_stats(const uint2 *ranges, int tiles, DevState *st) {
    __shared__ unsigned long long s_best[256];
    unsigned long long best = 0;
    for (int i = threadIdx.x; i < tiles; i += blockDim.x) {
        const uint2 r = ranges[i];
        const unsigned len = r.y - r.x;
        // larger length wins; on ties the smaller tile id
        const unsigned long long key = ((unsigned long long)len << 32) | (0xFFFFFFFFu - (unsigned)i);
        if (key > best) best = key;
    }
    s_best[threadIdx.x] = best;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o && s_best[threadIdx.x + o] > s_best[threadIdx.x]) s_best[threadIdx.x] = s_best[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        st->max_tile_pairs = (unsigned)(s_best[0] >> 32);
        st->max_tile_id = 0xFFFFFFFFu - (unsigned)(s_best[0] & 0xFFFFFFFFu);
    }
}

int launch_tile_stats(const Buffers &b, int tiles, cudaStream_t s) {
    k_tile_stats<<<1, 256, 0, s>>>(b.ranges, tiles, b.st);
    return 1;
}

}  // namespace unimgs
