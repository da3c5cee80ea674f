// binning.cu -- per-tile key duplication, onesweep radix sort and tile ranges.
//
// "incorporate triangle fragments into the depth-sorting process" of
// the 3DGS tile rasterizer: every (tile, primitive) pair is ordered by
// (tile, bits(depth), unified id) -- the lexicographic order of the 64-bit key
// tile << 32 | bits(depth) with ties by id (readings R8, R9, R23).
//
// Two schedules produce the identical order:
//   sort_mode 0 (factored, default):
//     compact visible primitives (id order) -> 4 stable 8-bit onesweep passes
//     on the 32-bit depth key -> scan of tiles_touched in depth order fused
//     with the pair duplication (u16 tile id + u32 primitive id) -> stable
//     onesweep passes on the tile id only (2 for <= 2^16 tiles) -> ranges.
//     Stable LSD by tile over pairs emitted in (depth, id) order IS the
//     (tile, depth, id) order; it moves ~4x fewer bytes than sorting K
//     64-bit keys over 32 + tile_bits bits.
//   sort_mode 1 (full): scan of tiles_touched in id order fused with the
//     duplication of 64-bit keys -> onesweep over bits [0, 32 + tile_bits).
//
// All scans are single-pass decoupled look-back (tile index claimed from an
// atomic counter for forward progress).  Look-back entries are 64-bit
// {epoch tag << 2 | flag, value}: the tag changes every pass of every frame,
// so the buffers are never cleared and the pipeline stays graph-capturable.
#include <algorithm>

#include "internal.cuh"

namespace unimgs {

constexpr unsigned kFlagAgg = 1, kFlagInc = 2;
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr int kSortThreads = 256, kSortItems = 16, kSortTile = kSortThreads * kSortItems;

// scan/pass slots (select the dynamic tile counter and the epoch tag)
enum { SLOT_COMPACT = 0, SLOT_DEPTH0 = 1, SLOT_DUP = 5, SLOT_TILE0 = 6, SLOT_FULLDUP = 0, SLOT_FULL0 = 1 };
// histogram rows: factored: 0..3 depth digits, 4..5 tile digits; full: 0..3 depth, 4..5 tile
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

__device__ __forceinline__ void flush_hist(unsigned *s_h, unsigned *g_h, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned v = s_h[i];
        if (v) atomicAdd(g_h + i, v);
    }
}

// ----------------------------------------------------------------------------
// sort_mode 0, step 1: compact visible primitives in id order; depth-digit
// histograms for the 4 depth passes.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_compact(int64_t P, const uint32_t *__restrict__ touched,
                                                          const uint32_t *__restrict__ dkey, uint32_t *ok,
                                                          uint32_t *ov, unsigned long long *lb, DevState *st) {
    __shared__ unsigned s_w[10], s_tile;
    __shared__ unsigned s_h[4 * 256];
    const unsigned tag = epoch_tag(st, SLOT_COMPACT);
    while (true) {
        const unsigned tile = claim_tile(&st->ctr[SLOT_COMPACT], &s_tile);
        const int64_t base = (int64_t)tile * kScanTile;
        if (base >= P) break;
        for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) s_h[i] = 0;
        unsigned v[kScanItems], ex[kScanItems];
        const int64_t b0 = base + (int64_t)threadIdx.x * kScanItems;  // blocked arrangement
#pragma unroll
        for (int i = 0; i < kScanItems; i++) v[i] = (b0 + i < P && touched[b0 + i] > 0) ? 1u : 0u;
        unsigned total;
        scan_lookback<kScanItems>(v, ex, tile, lb, tag, s_w, total);
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            if (v[i]) {
                const uint32_t k = dkey[b0 + i];
                ok[ex[i]] = k;
                ov[ex[i]] = (uint32_t)(b0 + i);
#pragma unroll
                for (int d = 0; d < 4; d++) atomicAdd(&s_h[d * 256 + ((k >> (8 * d)) & 255u)], 1u);
            }
        }
        __syncthreads();
        flush_hist(s_h, &st->hist[HIST_DEPTH0][0], 4 * 256);
        if (base + kScanTile >= P && threadIdx.x == 0) st->n_vis = total;
    }
}

// ----------------------------------------------------------------------------
// Duplication fused into the tiles_touched scan.  FULL = false: items are the
// depth-sorted visible primitives, pairs are (u16 tile, id).  FULL = true:
// items are all primitives in id order, pairs are (tile << 32 | depth, id).
// ----------------------------------------------------------------------------
template <bool FULL>
__global__ void __launch_bounds__(kScanThreads) k_duplicate(int64_t P_all, const uint32_t *__restrict__ ids,
                                                            const uint32_t *__restrict__ touched,
                                                            const uint2 *__restrict__ rect,
                                                            const uint32_t *__restrict__ dkey, int tiles_x,
                                                            int tile_bits, int64_t cap, void *tk_, uint32_t *tv,
                                                            unsigned long long *lb, DevState *st) {
    __shared__ unsigned s_w[10], s_tile;
    __shared__ unsigned s_h[6 * 256];
    const int slot = FULL ? SLOT_FULLDUP : SLOT_DUP;
    const unsigned tag = epoch_tag(st, slot);
    const int64_t n = FULL ? P_all : (int64_t)st->n_vis;
    const int nh = FULL ? 6 : 2;
    while (true) {
        const unsigned tile = claim_tile(&st->ctr[slot], &s_tile);
        const int64_t base = (int64_t)tile * kScanTile;
        if (base >= n) break;
        for (int i = threadIdx.x; i < nh * 256; i += blockDim.x) s_h[i] = 0;
        unsigned v[kScanItems], ex[kScanItems];
        uint32_t id[kScanItems];
        const int64_t b0 = base + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
        for (int i = 0; i < kScanItems; i++) {
            const bool in = b0 + i < n;
            id[i] = in ? (FULL ? (uint32_t)(b0 + i) : ids[b0 + i]) : 0u;
            v[i] = in ? touched[id[i]] : 0u;
        }
        unsigned total;
        scan_lookback<kScanItems>(v, ex, tile, lb, epoch_tag(st, slot), s_w, total);
        for (int i = 0; i < kScanItems; i++) {
            if (!v[i]) continue;
            const uint2 r = rect[id[i]];
            const int x0 = r.x & 0xFFFF, y0 = r.x >> 16, x1 = r.y & 0xFFFF, y1 = r.y >> 16;
            const uint32_t dk = FULL ? dkey[id[i]] : 0u;
            int64_t pos = ex[i];
            for (int ty = y0; ty <= y1; ty++)
                for (int tx = x0; tx <= x1; tx++, pos++) {
                    const unsigned t = (unsigned)(ty * tiles_x + tx);
                    if (pos < cap) {
                        if (FULL) reinterpret_cast<unsigned long long *>(tk_)[pos] = ((unsigned long long)t << 32) | dk;
                        else reinterpret_cast<uint16_t *>(tk_)[pos] = (uint16_t)t;
                        tv[pos] = id[i];
                    }
                    if (FULL) {
#pragma unroll
                        for (int d = 0; d < 4; d++) atomicAdd(&s_h[d * 256 + ((dk >> (8 * d)) & 255u)], 1u);
                    }
                    atomicAdd(&s_h[(FULL ? 4 : 0) * 256 + (t & 255u)], 1u);
                    if (tile_bits > 8) atomicAdd(&s_h[(FULL ? 5 : 1) * 256 + ((t >> 8) & 255u)], 1u);
                }
        }
        __syncthreads();
        flush_hist(s_h, &st->hist[FULL ? 0 : HIST_TILE0][0], nh * 256);
        if (base + kScanTile >= n && threadIdx.x == 0) {
            st->needed = total;
            const bool over = (int64_t)total > cap;
            st->overflow = over ? 1u : 0u;
            st->K = over ? 0u : total;
        }
    }
    (void)tag;
}

// ----------------------------------------------------------------------------
// One stable onesweep LSD pass on `bits` bits at `shift` (Adinets & Merrill).
// Tiles of 4096 keys, warp-striped; warp-level multisplit ranking with
// __match_any_sync; per-digit decoupled look-back; scatter through smem.
// ----------------------------------------------------------------------------
template <typename KT>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(const KT *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                           KT *__restrict__ kout, uint32_t *__restrict__ vout,
                                                           const unsigned *n_ptr, int shift, int bits,
                                                           const unsigned *hist, int slot,
                                                           unsigned long long *lb, DevState *st) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned *s_wh = reinterpret_cast<unsigned *>(smem);           // [8][256]
    unsigned *s_doff = s_wh + 8 * 256;                              // [256] block-local digit offsets
    int *s_glob = reinterpret_cast<int *>(s_doff + 256);            // [256] global base - local offset
    unsigned *s_hex = reinterpret_cast<unsigned *>(s_glob + 256);   // [256] global exclusive histogram
    unsigned *s_misc = s_hex + 256;                                 // [4]
    KT *s_k = reinterpret_cast<KT *>(s_misc + 4);
    uint32_t *s_v = reinterpret_cast<uint32_t *>(s_k + kSortTile);

    const unsigned n = *n_ptr;
    if (st->overflow && n_ptr == &st->K) return;
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
        if (lane == 31) s_misc[0] = 0;  // placeholder to keep s_misc initialised
        __shared__ unsigned s_ws[8];
        if (lane == 31) s_ws[wid] = x;
        __syncthreads();
        unsigned add = 0;
        for (unsigned w = 0; w < wid; w++) add += s_ws[w];
        s_hex[t] = x - h + add;
    }

    while (true) {
        const unsigned tile = claim_tile(&st->ctr[slot], &s_misc[1]);
        const unsigned base = tile * (unsigned)kSortTile;
        if ((unsigned long long)tile * kSortTile >= n) break;
        for (int i = t; i < 8 * 256; i += kSortThreads) s_wh[i] = 0;
        __syncthreads();

        KT key[kSortItems];
        uint32_t val[kSortItems];
        unsigned rank[kSortItems];
        unsigned dig[kSortItems];
        const unsigned wbase = base + wid * 32u * kSortItems + lane;
        const unsigned lt = lanemask_lt();
        unsigned *wh = s_wh + wid * 256;
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const unsigned idx = wbase + 32u * i;
            const bool valid = idx < n;
            key[i] = valid ? kin[idx] : (KT)0;
            val[i] = valid ? vin[idx] : 0u;
            dig[i] = valid ? (unsigned)((key[i] >> shift) & mask) : 256u;
        }
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const unsigned d = dig[i];
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const unsigned before = d < 256u ? wh[d] : 0u;
            rank[i] = before + __popc(peers & lt);
            __syncwarp();
            if (d < 256u && (peers & lt) == 0) wh[d] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // per digit: exclusive over warps, block count
        unsigned cnt = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) {
            const unsigned c = s_wh[w * 256 + t];
            s_wh[w * 256 + t] = cnt;
            cnt += c;
        }
        unsigned long long *my = lb + (size_t)tile * 256 + t;
        if (tile == 0) st_relaxed(my, pack(tag, kFlagInc, cnt));
        else st_relaxed(my, pack(tag, kFlagAgg, cnt));
        // block-exclusive scan of cnt over digits
        {
            unsigned x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (unsigned)o) x += y;
            }
            __shared__ unsigned s_ws2[8];
            if (lane == 31) s_ws2[wid] = x;
            __syncthreads();
            unsigned add = 0;
            for (unsigned w = 0; w < wid; w++) add += s_ws2[w];
            s_doff[t] = x - cnt + add;
        }
        // look-back for digit t
        unsigned excl = 0;
        if (tile > 0) {
            int j = (int)tile - 1;
            while (j >= 0) {
                const unsigned long long e = ld_relaxed(lb + (size_t)j * 256 + t);
                const unsigned hi = (unsigned)(e >> 32);
                const unsigned flag = ((hi >> 2) == tag) ? (hi & 3u) : 0u;
                if (flag == 0) continue;
                excl += (unsigned)e;
                if (flag == kFlagInc) break;
                j--;
            }
            st_relaxed(my, pack(tag, kFlagInc, excl + cnt));
        }
        s_glob[t] = (int)(s_hex[t] + excl) - (int)s_doff[t];
        __syncthreads();
        // scatter into smem in block-sorted order
#pragma unroll
        for (int i = 0; i < kSortItems; i++) {
            const unsigned d = dig[i];
            if (d < 256u) {
                const unsigned pos = s_doff[d] + wh[d] + rank[i];
                s_k[pos] = key[i];
                s_v[pos] = val[i];
            }
        }
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

template <typename KT>
static size_t onesweep_smem() {
    return (8 * 256 + 256 * 3 + 4) * sizeof(unsigned) + kSortTile * (sizeof(KT) + sizeof(uint32_t));
}

// ranges[tile] = [first, last + 1) over the sorted keys
template <typename KT>
__global__ void k_ranges(const KT *__restrict__ keys, const unsigned *n_ptr, int shift, uint2 *ranges,
                         const DevState *st) {
    if (st->overflow) return;
    const unsigned n = *n_ptr;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned tl = (unsigned)(keys[i] >> shift);
        const unsigned prev = i > 0 ? (unsigned)(keys[i - 1] >> shift) : 0xFFFFFFFFu;
        const unsigned next = i + 1 < n ? (unsigned)(keys[i + 1] >> shift) : 0xFFFFFFFFu;
        if (tl != prev) ranges[tl].x = i;
        if (tl != next) ranges[tl].y = i + 1;
    }
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
    const size_t sm = onesweep_smem<KT>();
    k_onesweep<KT><<<grid, kSortThreads, sm, s>>>(kin, vin, kout, vout, n_ptr, shift, bits,
                                                  &b.st->hist[hist_row][0], slot, b.lookback, b.st);
}

static int sort_grid(int64_t max_items, int sm_count, int per_sm) {
    const int64_t tiles = (max_items + kSortTile - 1) / kSortTile;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count * per_sm));
}

int launch_bin(Buffers &b, int64_t P, int64_t N, int64_t F, const CamParams &cam, int sort_mode, cudaStream_t s,
               int sm_count) {
    (void)N; (void)F;
    int launches = 0;
    const int64_t tiles = (int64_t)cam.tiles_x * cam.tiles_y;
    const int tb = bits_for(tiles);
    static bool attr_done = false;
    if (!attr_done) {
        cudaFuncSetAttribute(k_onesweep<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)onesweep_smem<uint16_t>());
        cudaFuncSetAttribute(k_onesweep<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)onesweep_smem<uint32_t>());
        cudaFuncSetAttribute(k_onesweep<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)onesweep_smem<unsigned long long>());
        attr_done = true;
    }
    cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * tiles, s);
    const int scan_grid = (int)std::max<int64_t>(1, std::min<int64_t>((P + kScanTile - 1) / kScanTile, (int64_t)sm_count * 8));
    if (sort_mode == 0) {
        // 1. compact visible primitives + depth histograms
        if (P > 0) {
            k_compact<<<scan_grid, kScanThreads, 0, s>>>(P, b.touched, b.dkey, b.pk[0], b.pv[0], b.lookback, b.st);
            launches++;
        }
        // 2. four stable 8-bit passes on the depth key
        const int g1 = sort_grid(P, sm_count, 3);
        int cur = 0;
        for (int pass = 0; pass < 4; pass++) {
            onesweep_pass<uint32_t>(b, b.pk[cur], b.pv[cur], b.pk[cur ^ 1], b.pv[cur ^ 1], &b.st->n_vis, 8 * pass, 8,
                                    HIST_DEPTH0 + pass, SLOT_DEPTH0 + pass, g1, s);
            cur ^= 1;
            launches++;
        }
        // 3. scan tiles_touched in depth order + duplicate (u16 tile, id)
        k_duplicate<false><<<scan_grid, kScanThreads, 0, s>>>(P, b.pv[cur], b.touched, b.rect, b.dkey, cam.tiles_x,
                                                              tb, b.max_pairs, b.tk[0], b.tv[0], b.lookback, b.st);
        launches++;
        // 4. stable passes on the tile id
        const int g2 = sort_grid(b.max_pairs, sm_count, 4);
        int tc = 0;
        for (int pass = 0, sh = 0; sh < tb; pass++, sh += 8) {
            onesweep_pass<uint16_t>(b, (const uint16_t *)b.tk[tc], b.tv[tc], (uint16_t *)b.tk[tc ^ 1], b.tv[tc ^ 1],
                                    &b.st->K, sh, std::min(8, tb - sh), HIST_TILE0 + pass, SLOT_TILE0 + pass, g2, s);
            tc ^= 1;
            launches++;
        }
        b.sorted_keys = b.tk[tc];
        b.sorted_vals = b.tv[tc];
        b.key_bytes = 2;
        k_ranges<uint16_t><<<sm_count * 4, 256, 0, s>>>((const uint16_t *)b.tk[tc], &b.st->K, 0, b.ranges, b.st);
        launches++;
    } else {
        // 1. scan tiles_touched in id order + duplicate 64-bit keys (all 6 digit histograms)
        if (P > 0) {
            k_duplicate<true><<<scan_grid, kScanThreads, 0, s>>>(P, nullptr, b.touched, b.rect, b.dkey, cam.tiles_x, tb,
                                                                 b.max_pairs, b.tk[0], b.tv[0], b.lookback, b.st);
            launches++;
        }
        const int g2 = sort_grid(b.max_pairs, sm_count, 3);
        int tc = 0;
        const int total_bits = 32 + tb;
        for (int pass = 0, sh = 0; sh < total_bits; pass++, sh += 8) {
            onesweep_pass<unsigned long long>(b, (const unsigned long long *)b.tk[tc], b.tv[tc],
                                              (unsigned long long *)b.tk[tc ^ 1], b.tv[tc ^ 1], &b.st->K, sh,
                                              std::min(8, total_bits - sh), pass, SLOT_FULL0 + pass, g2, s);
            tc ^= 1;
            launches++;
        }
        b.sorted_keys = b.tk[tc];
        b.sorted_vals = b.tv[tc];
        b.key_bytes = 8;
        k_ranges<unsigned long long><<<sm_count * 4, 256, 0, s>>>((const unsigned long long *)b.tk[tc], &b.st->K, 32,
                                                                  b.ranges, b.st);
        launches++;
    }
    return launches + 1;  // + the ranges memset
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
