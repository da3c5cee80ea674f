// binning.cu -- per-tile key duplication, onesweep radix sort and tile ranges.
//
// "incorporate triangle fragments into the depth-sorting process" of
// the 3DGS tile rasterizer: every (tile, primitive) pair is ordered by
// (tile, bits(depth), unified id) -- the lexicographic order of the 64-bit key
// tile << 32 | bits(depth) with ties by id (readings R8, R9, R23).
//
// Pipeline (both sort modes produce the identical order):
//   k_compact        visible primitives in id order (decoupled look-back scan)
//                    and every digit histogram the radix passes need: depth
//                    digits per primitive, tile digits of all pairs computed
//                    per rect row (no per-pair atomics);
//   k_tile_lo_hist   low tile digit histogram from its difference array.
//   sort_mode 0 (factored, default):
//     k_onesweep<u32> x4   stable LSD on the 32-bit depth key of the visible
//                          primitives (id ties stay in id order);
//     k_duplicate<false>   scan of tiles_touched in depth order fused with the
//                          emission of (u16 tile, u32 id) pairs, staged through
//                          shared memory so every store is coalesced;
//     k_onesweep<u16> x2   stable LSD on the tile id: pairs emitted in
//                          (depth, id) order come out in (tile, depth, id)
//                          order -- ~4x fewer bytes than sorting K 64-bit keys;
//     k_ranges16           tile ranges from the sorted tile ids.
//   sort_mode 1 (full, the literal form):
//     k_duplicate<true>    (tile << 32 | depth, id) pairs in id order;
//     k_onesweep<u64> x(4 + ceil(tile_bits/8)) over bits [0, 32 + tile_bits);
//     k_ranges64.
//
// Scans and sort passes are single-pass decoupled look-back over tiles claimed
// from an atomic counter (forward progress).  Look-back entries are 64-bit
// {epoch tag << 2 | flag, value}; the tag changes every pass of every frame, so
// nothing is cleared between frames and the whole frame is graph-capturable.
#include <algorithm>
#include <type_traits>

#include "internal.cuh"

#ifndef UNIMGS_SORT_ITEMS
#define UNIMGS_SORT_ITEMS 16
#endif

namespace unimgs {

constexpr unsigned kFlagAgg = 1, kFlagInc = 2;
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr int kSortThreads = 256, kSortItems = UNIMGS_SORT_ITEMS, kSortTile = kSortThreads * kSortItems;
#ifndef UNIMGS_LOOKWIN
#define UNIMGS_LOOKWIN 16
#endif
constexpr int kLookWin = UNIMGS_LOOKWIN;  // predecessors inspected per look-back round trip

// scan/pass slots (select the dynamic tile counter and the epoch tag)
enum { SLOT_COMPACT = 0, SLOT_DUP = 1, SLOT_PASS0 = 2 };
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
// Block-wide exclusive scan of ITEMS saturating u32 values per thread plus the
// decoupled look-back across tiles (warp 0 inspects 32 predecessors at once).
// s_w needs 10 entries.  Returns the inclusive grand total through `total`.
// ----------------------------------------------------------------------------
template <int ITEMS>
__device__ __forceinline__ void scan_lookback(const unsigned (&val)[ITEMS], unsigned (&excl)[ITEMS], unsigned tile,
                                              unsigned long long *lb, unsigned tag, unsigned *s_w, unsigned &total) {
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned tsum = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) tsum = sat_add(tsum, val[i]);
    unsigned x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x = sat_add(x, y);
    }
    const unsigned wexcl = __shfl_up_sync(0xffffffffu, x, 1);
    const unsigned my_wexcl = lane ? wexcl : 0u;
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const unsigned nw = blockDim.x >> 5;
        const unsigned wv = lane < nw ? s_w[lane] : 0u;
        unsigned wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (unsigned)o) wi = sat_add(wi, y);
        }
        const unsigned agg = __shfl_sync(0xffffffffu, wi, 31);
        const unsigned wex = __shfl_up_sync(0xffffffffu, wi, 1);
        unsigned prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed(lb, pack(tag, kFlagInc, agg));
        } else {
            if (lane == 0) st_relaxed(lb + tile, pack(tag, kFlagAgg, agg));
            int j = (int)tile - 1;
            while (true) {
                const int idx = j - (int)lane;
                unsigned flag = kFlagInc, v = 0;
                if (idx >= 0) {
                    const unsigned long long e = ld_relaxed(lb + idx);
                    const unsigned hi = (unsigned)(e >> 32);
                    flag = ((hi >> 2) == tag) ? (hi & 3u) : 0u;
                    v = (unsigned)e;
                }
                if (__any_sync(0xffffffffu, flag == 0)) continue;
                const unsigned incm = __ballot_sync(0xffffffffu, flag == kFlagInc);
                const int first = __ffs(incm) - 1;
                unsigned c = (first < 0 || (int)lane <= first) ? v : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c = sat_add(c, __shfl_xor_sync(0xffffffffu, c, o));
                prefix = sat_add(prefix, c);
                if (incm) break;
                j -= 32;
            }
            if (lane == 0) st_relaxed(lb + tile, pack(tag, kFlagInc, sat_add(prefix, agg)));
        }
        if (lane < nw) s_w[lane] = sat_add(prefix, lane ? wex : 0u);
        if (lane == 0) s_w[8] = sat_add(prefix, agg);
    }
    __syncthreads();
    unsigned run = sat_add(s_w[wid], my_wexcl);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        excl[i] = run;
        run = sat_add(run, val[i]);
    }
    total = s_w[8];
}

// Same scan for a warp-striped arrangement: item i of lane l of warp w is element
// base + w * 32 * ITEMS + i * 32 + l (coalesced loads); offsets follow index order.
template <int ITEMS>
__device__ __forceinline__ void scan_lookback_striped(const unsigned (&val)[ITEMS], unsigned (&excl)[ITEMS],
                                                      unsigned tile, unsigned long long *lb, unsigned tag,
                                                      unsigned *s_w, unsigned &total) {
    const unsigned lane = threadIdx.x & 31;
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
    // reuse the blocked scan for the warp totals: lane 0 contributes its warp's total
    unsigned wv[1] = {lane == 0 ? carry : 0u}, wx[1];
    scan_lookback<1>(wv, wx, tile, lb, tag, s_w, total);
    const unsigned wbase = __shfl_sync(0xffffffffu, wx[0], 0);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) excl[i] = sat_add(wbase, excl[i]);
}

// Tile-digit histograms of a primitive's pairs, per rect row: the low digit
// (t & 255) of a run of consecutive tile ids is a cyclic range of bins
// (difference array d_lo[257] + full cycles), the high digit (t >> 8) takes
// one or two values.  Exact pair counts with O(rows) shared atomics.
__device__ __forceinline__ void tile_digit_hist(uint2 r, int tiles_x, unsigned *d_lo, unsigned *h_hi,
                                                unsigned *all_lo) {
    const unsigned x0 = r.x & 0xFFFF, y0 = r.x >> 16, x1 = r.y & 0xFFFF, y1 = r.y >> 16;
    for (unsigned ty = y0; ty <= y1; ty++) {
        const unsigned a = ty * (unsigned)tiles_x + x0, b = ty * (unsigned)tiles_x + x1;
        const unsigned len = b - a + 1, full = len >> 8, rem = len & 255u;
        if (full) atomicAdd(all_lo, full);
        if (rem) {
            const unsigned lo = a & 255u, e = lo + rem;
            if (e <= 256u) {
                atomicAdd(d_lo + lo, 1u);
                atomicAdd(d_lo + e, 0xFFFFFFFFu);
            } else {
                atomicAdd(d_lo + lo, 1u);
                atomicAdd(d_lo + 256, 0xFFFFFFFFu);
                atomicAdd(d_lo + 0, 1u);
                atomicAdd(d_lo + (e - 256u), 0xFFFFFFFFu);
            }
        }
        for (unsigned h = a >> 8; h <= (b >> 8); h++) {
            const unsigned s0 = max(a, h << 8), s1 = min(b, (h << 8) + 255u);
            atomicAdd(h_hi + (h & 255u), s1 - s0 + 1);
        }
    }
}

// ----------------------------------------------------------------------------
// k_compact: visible primitives (touched > 0) in id order -> (depth key, id),
// warp-striped (coalesced) with a ballot scan.  Histograms for the radix
// passes: depth digits of the primitive keys (factored) or of the pair keys
// (FULL: weighted by tiles_touched), and the two tile digits of all pairs.
// ----------------------------------------------------------------------------
template <bool FULL>
__global__ void __launch_bounds__(kScanThreads) k_compact(int64_t P, const uint32_t *__restrict__ touched,
                                                          const uint32_t *__restrict__ dkey,
                                                          const uint2 *__restrict__ rect, int tiles_x, int tile_bits,
                                                          uint32_t *ok, uint32_t *ov, unsigned long long *lb,
                                                          DevState *st) {
    __shared__ unsigned s_w[10], s_tile;
    __shared__ unsigned s_h[4 * 256];
    __shared__ unsigned s_dlo[257], s_hhi[256], s_all;
    const unsigned tag = epoch_tag(st, SLOT_COMPACT);
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    while (true) {
        const unsigned tile = claim_tile(&st->ctr[SLOT_COMPACT], &s_tile);
        const int64_t base = (int64_t)tile * kScanTile;
        if (base >= P) break;
        for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) s_h[i] = 0;
        for (int i = threadIdx.x; i < 257; i += blockDim.x) s_dlo[i] = 0;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) s_hhi[i] = 0;
        if (threadIdx.x == 0) s_all = 0;
        unsigned v[kScanItems], ex[kScanItems], tt[kScanItems];
        const int64_t b0 = base + (int64_t)wid * 32 * kScanItems + lane;  // warp-striped
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            tt[i] = b0 + 32 * i < P ? touched[b0 + 32 * i] : 0u;
            v[i] = tt[i] > 0 ? 1u : 0u;
        }
        unsigned total;
        scan_lookback_striped<kScanItems>(v, ex, tile, lb, tag, s_w, total);
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            if (v[i]) {
                const int64_t p = b0 + 32 * i;
                const uint32_t k = dkey[p];
                ok[ex[i]] = k;
                ov[ex[i]] = (uint32_t)p;
                const unsigned w = FULL ? tt[i] : 1u;
#pragma unroll
                for (int d = 0; d < 4; d++) atomicAdd(&s_h[d * 256 + ((k >> (8 * d)) & 255u)], w);
                tile_digit_hist(rect[p], tiles_x, s_dlo, s_hhi, &s_all);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
            const unsigned h = s_h[i];
            if (h) atomicAdd(&st->hist[HIST_DEPTH0][0] + i, h);
        }
        for (int i = threadIdx.x; i < 257; i += blockDim.x) {
            const unsigned h = s_dlo[i];
            if (h) atomicAdd(&st->tdlo[i], h);
        }
        if (tile_bits > 8)
            for (int i = threadIdx.x; i < 256; i += blockDim.x) {
                const unsigned h = s_hhi[i];
                if (h) atomicAdd(&st->hist[HIST_TILE0 + 1][i], h);
            }
        if (threadIdx.x == 0 && s_all) atomicAdd(&st->tdlo_all, s_all);
        if (base + kScanTile >= P && threadIdx.x == 0) st->n_vis = total;
    }
}

// Tile low-digit histogram from its difference array (one CTA of 256 threads).
__global__ void k_tile_lo_hist(DevState *st) {
    __shared__ unsigned s_ws[8];
    const unsigned t = threadIdx.x, lane = t & 31, wid = t >> 5;
    unsigned x = st->tdlo[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) s_ws[wid] = x;
    __syncthreads();
    unsigned add = 0;
    for (unsigned w = 0; w < wid; w++) add += s_ws[w];
    st->hist[HIST_TILE0][t] = x + add + st->tdlo_all;
}

// ----------------------------------------------------------------------------
// k_duplicate: tiles_touched scan over the (depth-sorted or id-ordered) visible
// primitives fused with the pair emission.  Each CTA's pairs form one
// contiguous range; they are written into shared memory in windows of CAP pairs
// by the owning threads, then copied out with coalesced stores.
// ----------------------------------------------------------------------------
template <bool FULL>
struct DupCfg {
    static constexpr int CAP = FULL ? 4096 : 8192;
    using Key = typename std::conditional<FULL, unsigned long long, uint16_t>::type;
};

template <bool FULL>
__global__ void __launch_bounds__(kScanThreads) k_duplicate(const uint32_t *__restrict__ ids,
                                                            const uint32_t *__restrict__ touched,
                                                            const uint2 *__restrict__ rect,
                                                            const uint32_t *__restrict__ dkey, int tiles_x,
                                                            int64_t cap, void *tk_, uint32_t *tv,
                                                            unsigned long long *lb, DevState *st) {
    using Key = typename DupCfg<FULL>::Key;
    constexpr int CAP = DupCfg<FULL>::CAP;
    extern __shared__ __align__(16) unsigned char smem[];
    Key *s_k = reinterpret_cast<Key *>(smem);
    uint32_t *s_v = reinterpret_cast<uint32_t *>(s_k + CAP);
    __shared__ unsigned s_w[10], s_tile, s_base;
    Key *tk = reinterpret_cast<Key *>(tk_);
    const unsigned tag = epoch_tag(st, SLOT_DUP);
    const int64_t n = (int64_t)st->n_vis;
    const unsigned capu = (unsigned)(cap < 0xFFFFFFFFll ? cap : 0xFFFFFFFFll);
    while (true) {
        const unsigned tile = claim_tile(&st->ctr[SLOT_DUP], &s_tile);
        const int64_t base = (int64_t)tile * kScanTile;
        if (base >= n) break;
        unsigned v[kScanItems], ex[kScanItems];
        uint32_t id[kScanItems];
        const int64_t b0 = base + (int64_t)(threadIdx.x >> 5) * 32 * kScanItems + (threadIdx.x & 31);  // warp-striped
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            const bool in = b0 + 32 * i < n;
            id[i] = in ? ids[b0 + 32 * i] : 0u;
            v[i] = in ? touched[id[i]] : 0u;
        }
        unsigned total;
        scan_lookback_striped<kScanItems>(v, ex, tile, lb, tag, s_w, total);
        if (threadIdx.x == 0) s_base = ex[0];
        uint2 r[kScanItems];
        uint32_t dk[kScanItems];
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            r[i] = v[i] ? rect[id[i]] : make_uint2(0u, 0u);
            dk[i] = (FULL && v[i]) ? dkey[id[i]] : 0u;
        }
        __syncthreads();
        const unsigned pbase = s_base, pend = min(total, capu);
        for (unsigned wb = pbase; wb < pend; wb += CAP) {
            const unsigned we = min(pend, wb + CAP);
#pragma unroll
            for (int i = 0; i < kScanItems; i++) {
                if (!v[i]) continue;
                const unsigned lo = max(ex[i], wb), hi = min(ex[i] + v[i], we);
                if (lo >= hi) continue;
                const unsigned x0 = r[i].x & 0xFFFF, y0 = r[i].x >> 16, x1 = r[i].y & 0xFFFF;
                const unsigned wdt = x1 - x0 + 1, l0 = lo - ex[i];
                unsigned tx = x0 + l0 % wdt, ty = y0 + l0 / wdt;
                for (unsigned g = lo; g < hi; g++) {
                    const unsigned t = ty * (unsigned)tiles_x + tx;
                    if (FULL) s_k[g - wb] = (Key)(((unsigned long long)t << 32) | dk[i]);
                    else s_k[g - wb] = (Key)t;
                    s_v[g - wb] = id[i];
                    if (++tx > x1) { tx = x0; ty++; }
                }
            }
            __syncthreads();
            for (unsigned k = threadIdx.x; k < we - wb; k += kScanThreads) {
                tk[wb + k] = s_k[k];
                tv[wb + k] = s_v[k];
            }
            __syncthreads();
        }
        if (base + kScanTile >= n && threadIdx.x == 0) {
            st->needed = total;
            const bool over = (int64_t)total > cap;
            st->overflow = over ? 1u : 0u;
            st->K = over ? 0u : total;
        }
    }
}

// ----------------------------------------------------------------------------
// One stable onesweep LSD pass on `bits` bits at `shift` (Adinets & Merrill).
// Tiles of 256 x ITEMS keys, warp-striped; warp-level multisplit ranking with
// __match_any_sync; keys are moved into shared memory at their block-sorted
// position BEFORE the per-digit decoupled look-back (so no key register is live
// across it); then a coalesced-by-digit scatter to global memory.
// ----------------------------------------------------------------------------
template <typename KT>
#ifndef UNIMGS_RANK_MATCH
#define UNIMGS_RANK_MATCH 0
#endif
#ifndef UNIMGS_RANK_ATOMS
#define UNIMGS_RANK_ATOMS 0
#endif
#ifndef UNIMGS_SORT_MINB
#define UNIMGS_SORT_MINB 2
#endif
__global__ void __launch_bounds__(kSortThreads, UNIMGS_SORT_MINB) k_onesweep(const KT *__restrict__ kin,
                                                              const uint32_t *__restrict__ vin, KT *__restrict__ kout,
                                                              uint32_t *__restrict__ vout, const unsigned *n_ptr,
                                                              int shift, int bits, const unsigned *hist, int slot,
                                                              unsigned long long *lb, DevState *st) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned *s_wh = reinterpret_cast<unsigned *>(smem);           // [8][256]
    unsigned *s_doff = s_wh + 8 * 256;                              // [256] block-local digit offsets
    int *s_glob = reinterpret_cast<int *>(s_doff + 256);            // [256] global base - local offset
    unsigned *s_hex = reinterpret_cast<unsigned *>(s_glob + 256);   // [256] global exclusive histogram
    unsigned *s_misc = s_hex + 256;                                 // [16]
    KT *s_k = reinterpret_cast<KT *>(s_misc + 16);
    uint32_t *s_v = reinterpret_cast<uint32_t *>(s_k + kSortTile);

    const unsigned n = *n_ptr;
    const unsigned tag = epoch_tag(st, slot);
    const unsigned mask = (1u << bits) - 1u;
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
        if ((unsigned long long)tile * kSortTile >= n) break;
        const unsigned base = tile * (unsigned)kSortTile;
        for (int i = t; i < 8 * 256; i += kSortThreads) s_wh[i] = 0;
        __syncthreads();

        KT key[kSortItems];
        uint32_t val[kSortItems];
        unsigned rank[kSortItems];
        const unsigned wbase = base + wid * 32u * kSortItems + lane;
        const unsigned lt = lanemask_lt();
        unsigned *wh = s_wh + wid * 256;
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const unsigned idx = wbase + 32u * i;
            const bool valid = idx < n;
            key[i] = valid ? kin[idx] : (KT)0;
            val[i] = valid ? vin[idx] : 0u;
        }
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            // stable warp multisplit: the lanes holding the same digit
            const bool valid = wbase + 32u * i < n;
            const unsigned d = valid ? (unsigned)((key[i] >> shift) & mask) : 0u;
#if UNIMGS_RANK_MATCH
            const unsigned peers = __match_any_sync(0xffffffffu, valid ? d : 256u) & __ballot_sync(0xffffffffu, valid);
#else
            // all `bits` ballots first (independent), then combine
            unsigned bb[8];
#pragma unroll
            for (int bt = 0; bt < 8; bt++)
                if (bt < bits) bb[bt] = __ballot_sync(0xffffffffu, (d >> bt) & 1u);
            unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int bt = 0; bt < 8; bt++)
                if (bt < bits) peers &= ((d >> bt) & 1u) ? bb[bt] : ~bb[bt];
#endif
#if UNIMGS_RANK_ATOMS
            // the group's leader reserves its slots with one shared atomic; in-order per warp,
            // so earlier items of the same digit are counted first (stable)
            const int leader = __ffs(peers) - 1;
            unsigned before = 0;
            if (valid && lane == (unsigned)leader) before = atomicAdd(&wh[d], (unsigned)__popc(peers));
            before = __shfl_sync(0xffffffffu, before, valid ? leader : (int)lane);
#else
            const unsigned before = valid ? wh[d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0) wh[d] = before + __popc(peers);
            __syncwarp();
#endif
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
        for (int i = 0; i < kSortItems; i++) {
            if (wbase + 32u * i < n) {
                const unsigned d = (unsigned)((key[i] >> shift) & mask);
                const unsigned pos = s_doff[d] + wh[d] + rank[i];
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
        const unsigned nt = min((unsigned)kSortTile, n - base);
        for (unsigned k = t; k < nt; k += kSortThreads) {
            const KT kk = s_k[k];
            const unsigned d = (unsigned)((kk >> shift) & mask);
            const unsigned o = (unsigned)(s_glob[d] + (int)k);
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
        const unsigned prev = i > 0 ? (unsigned)(keys[i - 1] >> 32) : 0xFFFFFFFFu;
        const unsigned next = i + 1 < n ? (unsigned)(keys[i + 1] >> 32) : 0xFFFFFFFFu;
        if (tl != prev) ranges[tl].x = i;
        if (tl != next) ranges[tl].y = i + 1;
    }
}

template <typename KT>
static size_t onesweep_smem() {
    return (8 * 256 + 256 * 3 + 16) * sizeof(unsigned) + kSortTile * (sizeof(KT) + sizeof(uint32_t));
}

template <bool FULL>
static size_t dup_smem() {
    return DupCfg<FULL>::CAP * (sizeof(typename DupCfg<FULL>::Key) + sizeof(uint32_t));
}

static int bits_for(int64_t tiles) {
    int b = 0;
    while (((int64_t)1 << b) < tiles) b++;
    return b;
}

template <typename KT>
static void onesweep_pass(Buffers &b, const KT *kin, const uint32_t *vin, KT *kout, uint32_t *vout,
                          const unsigned *n_ptr, int shift, int bits, int hist_row, int slot, int grid,
                          cudaStream_t s) {
    k_onesweep<KT><<<grid, kSortThreads, onesweep_smem<KT>(), s>>>(kin, vin, kout, vout, n_ptr, shift, bits,
                                                                  &b.st->hist[hist_row][0], slot, b.lookback, b.st);
}

static int sort_grid(int64_t max_items, int sm_count, int per_sm) {
    const int64_t tiles = (max_items + kSortTile - 1) / kSortTile;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count * per_sm));
}

static void set_attrs() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_onesweep<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)onesweep_smem<uint16_t>());
    cudaFuncSetAttribute(k_onesweep<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)onesweep_smem<uint32_t>());
    cudaFuncSetAttribute(k_onesweep<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)onesweep_smem<unsigned long long>());
    cudaFuncSetAttribute(k_duplicate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dup_smem<false>());
    cudaFuncSetAttribute(k_duplicate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dup_smem<true>());
    done = true;
}

int launch_bin(Buffers &b, int64_t P, int64_t N, int64_t F, const CamParams &cam, int sort_mode, cudaStream_t s,
               int sm_count) {
    (void)N; (void)F;
    set_attrs();
    int launches = 0;
    const int64_t tiles = (int64_t)cam.tiles_x * cam.tiles_y;
    const int tb = bits_for(tiles);
    const bool full = sort_mode == 1;
    cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * (size_t)tiles, s);
    const int scan_grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((P + kScanTile - 1) / kScanTile, (int64_t)sm_count * 8));
    if (P > 0) {
        if (full)
            k_compact<true><<<scan_grid, kScanThreads, 0, s>>>(P, b.touched, b.dkey, b.rect, cam.tiles_x, tb, b.pk[0],
                                                               b.pv[0], b.lookback, b.st);
        else
            k_compact<false><<<scan_grid, kScanThreads, 0, s>>>(P, b.touched, b.dkey, b.rect, cam.tiles_x, tb, b.pk[0],
                                                                b.pv[0], b.lookback, b.st);
        launches++;
    }
    k_tile_lo_hist<<<1, 256, 0, s>>>(b.st);
    launches++;
    int slot = SLOT_PASS0;
    const int dgrid =
        (int)std::max<int64_t>(1, std::min<int64_t>((P + kScanTile - 1) / kScanTile, (int64_t)sm_count * 4));
    const int g2 = sort_grid(b.max_pairs, sm_count, 2);
    int tc = 0;
    if (!full) {
        // depth sort of the visible primitives
        const int g1 = sort_grid(P, sm_count, 2);
        int cur = 0;
        for (int pass = 0; pass < 4; pass++, slot++) {
            onesweep_pass<uint32_t>(b, b.pk[cur], b.pv[cur], b.pk[cur ^ 1], b.pv[cur ^ 1], &b.st->n_vis, 8 * pass, 8,
                                    HIST_DEPTH0 + pass, slot, g1, s);
            cur ^= 1;
            launches++;
        }
        k_duplicate<false><<<dgrid, kScanThreads, dup_smem<false>(), s>>>(b.pv[cur], b.touched, b.rect, b.dkey,
                                                                          cam.tiles_x, b.max_pairs, b.tk[0], b.tv[0],
                                                                          b.lookback, b.st);
        launches++;
        for (int pass = 0, sh = 0; sh < tb; pass++, sh += 8, slot++) {
            onesweep_pass<uint16_t>(b, (const uint16_t *)b.tk[tc], b.tv[tc], (uint16_t *)b.tk[tc ^ 1], b.tv[tc ^ 1],
                                    &b.st->K, sh, std::min(8, tb - sh), HIST_TILE0 + pass, slot, g2, s);
            tc ^= 1;
            launches++;
        }
        b.key_bytes = 2;
        k_ranges16<<<sm_count * 4, 256, 0, s>>>((const uint16_t *)b.tk[tc], &b.st->K, b.ranges, b.st);
        launches++;
    } else {
        k_duplicate<true><<<dgrid, kScanThreads, dup_smem<true>(), s>>>(b.pv[0], b.touched, b.rect, b.dkey, cam.tiles_x,
                                                                        b.max_pairs, b.tk[0], b.tv[0], b.lookback, b.st);
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
    return launches;  // kernels only (the ranges memset is not counted)
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
