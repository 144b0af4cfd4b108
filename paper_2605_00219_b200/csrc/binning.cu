// binning.cu — "Index Offset", "Generate Keys", "Sorting" and
// "Tile Ranges"; DESIGN.md §4.2 and §6.
//
// Result (identical to a stable sort of the (tile << 32 | f32bits(depth)) keys generated at
// slots offsets[i] + k, rows outer / columns inner): the Gaussian ids of every tile list in
// ascending (depth bits, id) order, plus CSR tile ranges.  B200 design — "depth-major" binning:
// every key of a Gaussian shares its depth bits, so the 32 depth bits are sorted over the N
// Gaussians (16 B/Gaussian per pass) instead of over the M ~ 4.4 N keys, and only the tile bits
// are sorted over the keys:
//
//  1. scan (id order)    reduce-then-scan of tiles_touched -> offsets, M, V; the reduce step also
//                         writes each visible Gaussian's tile rect as a 64-bit code (4 x u16) at
//                         its id, the down-sweep compacts the V visible ones, in id order, into
//                         (depth bits, id).
//  2. radix pass x1-4     LSD passes over the V (depth bits - min, id) pairs, <= 8-bit digits, as
//                         many as the visible depth-bit range needs (bicycle: 27 bits, 4 x 7).
//  3. scan (depth order) reduce-then-scan of the rect tile counts; the reduce gathers the rect
//                         codes into depth order -> first key slot of each Gaussian, and
//                         first[c] = the Gaussian holding key slot 512 c (one per warp chunk).
//  4. rect_diff_kernel    2-D difference array of the rects (4 shared-memory updates per Gaussian)
//     tile_count_kernel   2-D prefix -> per-tile list lengths -> CSR tile_offsets.
//  5. key pass            the first tile-bit pass straight from the rect codes, never storing the
//                         unsorted keys: keys_count_kernel histograms the digit of each 4096-slot
//                         key block from whole rect rows (a row is a run of consecutive tile ids);
//                         keys_scatter_kernel expands the block's keys (tile, id) into shared memory
//                         and ranks / stores them like any radix pass.
//  6. radix pass x0-2     the remaining stable LSD tile-bit passes (<= 8 bits each) over the M
//                         pairs; the last one writes the ids (and, on request, the u64 keys).
// Every radix pass is reduce-then-scan: digit counts per 4096-key block, one exclusive scan of
// the (digit-major) count matrix, then a scatter kernel (TMA bulk copy of the block into shared
// memory, warp-level ballot multi-split ranking, in-place reorder, digit-contiguous stores).  No block
// ever waits on another (a single-pass decoupled look-back over 256 digits walked hundreds of
// in-flight blocks back on this workload).
// The TU is compiled with -fmad=false (the tile-rect computation must equal projection's).
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "vks_common.cuh"

namespace vks {
namespace {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
#ifndef VKS_CNT_SCAN_ITEMS
#define VKS_CNT_SCAN_ITEMS 16
#endif
constexpr int kCntItems = VKS_CNT_SCAN_ITEMS;             // scan_u32 (the digit-count matrices):
constexpr int kCntTile = kScanThreads * kCntItems;         // elements per block
constexpr int kDownThreads = 512;  // the down-sweeps: same 4096-element tiles, 8 items per thread
constexpr int kDownItems = kScanTile / kDownThreads;

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef VKS_SORT_ITEMS
#define VKS_SORT_ITEMS 16
#endif
constexpr int kSortItems = VKS_SORT_ITEMS;  // keys per thread of a radix block
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per block
constexpr int kKeyChunk = 32 * kSortItems;             // key slots one warp expands (512)
constexpr int kChunksPerTile = kSortTile / kKeyChunk;  // 8
constexpr int kDepthPasses = 4;  // at most (32 significant depth bits in digits of <= 9 bits)
constexpr int kMaxRadix = 512;    // digits of <= 9 bits
constexpr int kMaxTilePasses = 3;

constexpr u64 kScanFlagAgg = 1ull << 62;
constexpr u64 kScanFlagInc = 2ull << 62;
constexpr u64 kScanMask = (1ull << 62) - 1;

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct TilePlan {
    int passes;  // 0..3
    int dbits;   // bits per tile pass (<= 8)
};

TilePlan tile_plan(int32_t n_tiles) {
    int tb = 0;
    while ((1ll << tb) < (int64_t)n_tiles) tb++;
    TilePlan p{0, 0};
    if (tb == 0) return p;
    p.passes = (tb + 7) / 8;
    p.dbits = (tb + p.passes - 1) / p.passes;
    return p;
}

constexpr int kPasses = kDepthPasses + kMaxTilePasses;

struct Workspace {
    u32 *dk[2], *dv[2];  // depth sort ping-pong [n]
    u32* doff;           // depth-order slot offsets [n]
    u32 *tk[2], *tv[2];  // tile sort ping-pong [capacity]
    u32* counts;         // [256 * sort tiles] digit counts of the current pass (digit-major)
    u32* offs;           // its exclusive scan
    u64* rcs;            // [n] tile-rect codes in depth order
    u64* rc_by_id;       // [n] tile-rect codes at the Gaussian id (visible rows)
    u32* first;          // [key chunks + 2] depth-order Gaussian holding slot 512 c
    u32* part_sum;       // [scan blocks] block sums of the 1-D scans
    u32* part_vis;       // [scan blocks] visible counts
    // region A (zeroed before the scan)
    u64* cnt_lb[kPasses];  // look-back of each pass's counts scan
    u32* ctr;            // [16] scan tile counters
    u64* totals;         // [3]: M, V, depth-bit range of the visible (2 x u32)
    int* diff;           // [(TY+1)*(TX+1)]
    size_t zeroA_bytes;
    char* zeroA;
    size_t bytes;
};

Workspace carve(void* base, int64_t n, int64_t capacity, int TX, int TY) {
    Workspace w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += align_up(bytes); return p; };
    const size_t nn = (size_t)(n > 0 ? n : 1), cap = (size_t)(capacity > 0 ? capacity : 1);
    const size_t scan_tiles = (nn + kScanTile - 1) / kScanTile;
    const size_t sort_tiles = (std::max(nn, cap) + kSortTile - 1) / kSortTile;
    const size_t cnt_scan_tiles = (kMaxRadix * sort_tiles + kCntTile - 1) / kCntTile;
    for (int i = 0; i < 2; i++) {
        w.dk[i] = reinterpret_cast<u32*>(take(4 * nn));
        w.dv[i] = reinterpret_cast<u32*>(take(4 * nn));
    }
    w.doff = reinterpret_cast<u32*>(take(4 * nn));
    for (int i = 0; i < 2; i++) {
        w.tk[i] = reinterpret_cast<u32*>(take(4 * cap));
        w.tv[i] = reinterpret_cast<u32*>(take(4 * cap));
    }
    w.counts = reinterpret_cast<u32*>(take(4 * kMaxRadix * sort_tiles));
    w.offs = reinterpret_cast<u32*>(take(4 * kMaxRadix * sort_tiles));
    w.rcs = reinterpret_cast<u64*>(take(8 * nn));
    w.rc_by_id = reinterpret_cast<u64*>(take(8 * nn));
    w.first = reinterpret_cast<u32*>(take(4 * ((cap + kKeyChunk - 1) / kKeyChunk + 2)));
    w.part_sum = reinterpret_cast<u32*>(take(4 * scan_tiles));
    w.part_vis = reinterpret_cast<u32*>(take(4 * scan_tiles));
    const size_t a0 = off;
    w.zeroA = b ? b + off : nullptr;
    for (int p = 0; p < kPasses; p++) w.cnt_lb[p] = reinterpret_cast<u64*>(take(8 * cnt_scan_tiles));
    w.ctr = reinterpret_cast<u32*>(take(4 * 16));
    w.totals = reinterpret_cast<u64*>(take(8 * 3));  // M, V, (u32 max ~depth bits, u32 max depth bits)
    w.diff = reinterpret_cast<int*>(take(4 * (size_t)(TX + 1) * (TY + 1)));
    w.zeroA_bytes = off - a0;
    w.bytes = off;
    return w;
}

// counter slots in w.ctr
enum { kCtrPass = 0 };  // kCtrPass + p: counts scan of pass p
static_assert(kPasses <= 16, "scan tile counters");

// ------------------------------------------------------------------------------------------
// tile rect codes: x0 | y0 << 16 | x1 << 32 | y1 << 48 (16 bits each), 0 for culled Gaussians

// tile rect recomputed exactly as projection step 11
__device__ __forceinline__ void rect_of(const float2 m, const int2 r, int TX, int TY, int& x0, int& x1, int& y0,
                                        int& y1) {
    const float rx = (float)r.x, ry = (float)r.y;
    x0 = (int)fminf(fmaxf(floorf((m.x - rx) * 0.0625f), 0.0f), (float)TX);
    x1 = (int)fminf(fmaxf(ceilf((m.x + rx) * 0.0625f), 0.0f), (float)TX);
    y0 = (int)fminf(fmaxf(floorf((m.y - ry) * 0.0625f), 0.0f), (float)TY);
    y1 = (int)fminf(fmaxf(ceilf((m.y + ry) * 0.0625f), 0.0f), (float)TY);
}
__device__ __forceinline__ u64 pack_rect(int x0, int x1, int y0, int y1) {
    return (u64)(u32)x0 | ((u64)(u32)y0 << 16) | ((u64)(u32)x1 << 32) | ((u64)(u32)y1 << 48);
}
__device__ __forceinline__ void unpack_rect(u64 c, int& x0, int& x1, int& y0, int& y1) {
    x0 = (int)(c & 0xFFFF); y0 = (int)((c >> 16) & 0xFFFF); x1 = (int)((c >> 32) & 0xFFFF); y1 = (int)(c >> 48);
}
__device__ __forceinline__ int rect_tiles(u64 c) {
    int x0, x1, y0, y1;
    unpack_rect(c, x0, x1, y0, y1);
    return (x1 - x0) * (y1 - y0);
}

// ------------------------------------------------------------------------------------------
// 1./3. exclusive scans of tiles_touched, reduce-then-scan (no block waits on another):
//   scan_reduce_kernel   per 4096-element block: sum (and number of visible Gaussians)
//   scan_down_kernel     per block: the block prefix (sum of the predecessors' block sums, read
//                        by every block itself), rescan -> output; the last block writes totals
// MODE 0: element i = tiles_touched[i];  MODE 1: element r = tiles of the depth-sorted rect code r.
// Warp-striped layout: warp w of a block owns the 512 consecutive elements starting at
// blockIdx.x * kScanTile + 512 w; lane l holds elements 32 j + l (j < 16), so every load and store
// instruction of a warp touches 32 consecutive elements.
template <int ITEMS = kScanItems>
__device__ __forceinline__ u64 warp_base(int warp) { return (u64)blockIdx.x * kScanTile + (u64)warp * 32 * ITEMS; }

template <int MODE, int ITEMS = kScanItems>
__device__ __forceinline__ void load_scan_items(const int* __restrict__ tiles, const u64* __restrict__ rc, u64 count,
                                                u64 wbase, int lane, int v[ITEMS]) {
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        const u64 i = wbase + 32 * j + lane;
        if (MODE == 0) v[j] = i < count ? max(__ldg(tiles + i), 0) : 0;
        else v[j] = i < count ? rect_tiles(__ldg(rc + i)) : 0;
    }
}

// Extra inputs / outputs of the scans.  MODE 0 (id order): the reduce step writes every visible
// Gaussian's tile-rect code at its id (rc_by_id); the down-sweep compacts the visible Gaussians,
// in id order, into (depth bits, id) pairs at their visible index (the input of the depth sort)
// and reduces the depth-bit range.
struct CompactOut {
    const u32* vis_prefix;   // [blocks] the reduce step's block visible counts
    const u32* depth_bits;   // [n]
    const float2* means2d;   // [n]
    const int2* radii;       // [n]
    int TX, TY;
    u32* vkeys;              // [V] depth bits, id order
    u32* vids;               // [V] ids
    u64* rc_by_id;           // [n] rect codes (visible rows only)
    u32* dminmax;            // [2] max(~depth bits), max(depth bits) over the visible (zeroed)
    // MODE 1 (depth order): the reduce step gathers the rect codes of the depth-sorted ids into
    // rc_out (coalesced), the down-sweep writes first[c] = the Gaussian holding key slot 512 c
    const u32* sid;
    u64* rc_out;
    u32* first;
};

// dcount (nullable, vks_bin_sort_async): the element count on the device; `count` is then the
// host-side bound the grid was sized for
__device__ __forceinline__ u64 eff_count(u64 bound, const u64* __restrict__ dcount) {
    return dcount ? min(bound, *dcount) : bound;
}

template <int MODE>
__global__ void __launch_bounds__(kDownThreads) scan_reduce_kernel(const int* __restrict__ tiles,
                                                                  const u64* __restrict__ rc_in, u64 count,
                                                                  u32* __restrict__ part_sum,
                                                                  u32* __restrict__ part_vis, const CompactOut co,
                                                                  const u64* __restrict__ dcount) {
    pdl_wait();
    constexpr int ITEMS = kDownItems;
    count = eff_count(count, dcount);
    __shared__ u32 s_sum[kDownThreads / 32], s_vis[kDownThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int v[ITEMS];
    const u64 wbase = warp_base<ITEMS>(warp);
    if (MODE == 1) {  // gather the rect codes into depth order (one random 8-byte read each)
        u32 g[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            const u64 i = wbase + 32 * j + lane;
            g[j] = i < count ? __ldg(co.sid + i) : 0u;
        }
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            const u64 i = wbase + 32 * j + lane;
            v[j] = 0;
            if (i < count) {
                const u64 c = __ldg(co.rc_by_id + g[j]);
                co.rc_out[i] = c;
                v[j] = rect_tiles(c);
            }
        }
    } else {
        load_scan_items<MODE, ITEMS>(tiles, rc_in, count, wbase, lane, v);
        // tile rect code of every visible Gaussian at its id (0 for the others: whole sectors are
        // written), computed exactly as projection step 11 (this TU is compiled -fmad=false).
        // means2d / radii are loaded for every row in range (the projection writes culled rows as
        // zeros), not only where tiles > 0: one DRAM round trip instead of two dependent ones
        const float2* __restrict__ means2d = co.means2d;
        const int2* __restrict__ radii = co.radii;
#pragma unroll
        for (int h = 0; h < ITEMS; h += 8) {
            float2 m[8];
            int2 r[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const u64 i = wbase + 32 * (h + q) + lane;
                if (i < count) {
                    m[q] = __ldg(means2d + i);
                    r[q] = __ldg(radii + i);
                }
            }
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const u64 i = wbase + 32 * (h + q) + lane;
                if (i >= count) continue;
                u64 code = 0;
                if (v[h + q] > 0) {
                    int x0, x1, y0, y1;
                    rect_of(m[q], r[q], co.TX, co.TY, x0, x1, y0, y1);
                    code = pack_rect(x0, x1, y0, y1);
                }
                co.rc_by_id[i] = code;
            }
        }
    }
    u32 sum = 0, vis = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        sum += (u32)v[j];
        vis += v[j] > 0;
    }
    sum = __reduce_add_sync(VKS_FULL_MASK, sum);
    vis = __reduce_add_sync(VKS_FULL_MASK, vis);
    if (lane == 0) { s_sum[warp] = sum; s_vis[warp] = vis; }
    __syncthreads();
    if (tid == 0) {
        u32 a = 0, b = 0;
#pragma unroll
        for (int w = 0; w < kDownThreads / 32; w++) { a += s_sum[w]; b += s_vis[w]; }
        part_sum[blockIdx.x] = a;
        if (part_vis) part_vis[blockIdx.x] = b;
    }
}

// inclusive scan across the warp
__device__ __forceinline__ u32 warp_incl_scan(u32 x, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(VKS_FULL_MASK, x, d);
        if (lane >= d) x += t;
    }
    return x;
}

// exclusive scan of the striped items of one warp: out[j] = warp-local exclusive prefix of v[j]
template <int ITEMS = kScanItems>
__device__ __forceinline__ u32 warp_striped_excl(const int v[ITEMS], u32 out[ITEMS], int lane) {
    u32 carry = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        const u32 incl = warp_incl_scan((u32)v[j], lane);
        out[j] = carry + incl - (u32)v[j];
        carry += __shfl_sync(VKS_FULL_MASK, incl, 31);
    }
    return carry;  // warp total
}

// The block's prefix is the sum of the block sums before it (part_sum / part_vis hold the reduce
// step's raw block sums): every block sums its predecessors' sums itself (<= a few thousand u32
// from L2), which replaces a single-block scan kernel and its launch between the two passes; the
// last block writes the totals (M and the visible count) for the host.
template <int MODE>
__global__ void __launch_bounds__(kDownThreads) scan_down_kernel(const int* __restrict__ tiles, const u64* __restrict__ rc,
                                                                u64 count, const u32* __restrict__ part_sum,
                                                                u32* __restrict__ out, const CompactOut co,
                                                                u64* __restrict__ totals, const u64* __restrict__ dcount) {
    pdl_wait();
    constexpr int ITEMS = kDownItems;
    count = eff_count(count, dcount);
    __shared__ u32 s_w[kDownThreads / 32], s_v[kDownThreads / 32];
    __shared__ u32 s_pre[kDownThreads / 32], s_vpre[kDownThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // the tile's items first (the DRAM round trip), the predecessors' block sums (L2) while they
    // are in flight
    const u64 wbase = warp_base<ITEMS>(warp);
    int v[ITEMS];
    u32 ex[ITEMS];
    u32 dbits_pre[ITEMS];  // MODE 0: depth bits loaded with the tile counts (one DRAM round trip)
#pragma unroll
    for (int q = 0; q < ITEMS; q++) {
        const u64 i = wbase + 32 * q + lane;
        dbits_pre[q] = (MODE == 0 && i < count) ? __ldg(co.depth_bits + i) : 0u;
    }
    load_scan_items<MODE, ITEMS>(tiles, rc, count, wbase, lane, v);
    {
        u32 ps = 0, pv = 0;
        for (u32 i = tid; i < blockIdx.x; i += kDownThreads) {
            ps += __ldg(part_sum + i);
            if (MODE == 0) pv += __ldg(co.vis_prefix + i);
        }
        ps = __reduce_add_sync(VKS_FULL_MASK, ps);
        pv = __reduce_add_sync(VKS_FULL_MASK, pv);
        if (lane == 0) { s_pre[warp] = ps; s_vpre[warp] = pv; }
    }
    const u32 wtot = warp_striped_excl<ITEMS>(v, ex, lane);
    u32 wvis = 0;
    if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < ITEMS; j++) wvis += __popc(__ballot_sync(VKS_FULL_MASK, v[j] > 0));
    }
    if (lane == 0) { s_w[warp] = wtot; s_v[warp] = wvis; }
    __syncthreads();
    u32 pre = 0, vpre = 0, btot = 0, bvis = 0;
#pragma unroll
    for (int w = 0; w < kDownThreads / 32; w++) {
        pre += s_pre[w];
        vpre += s_vpre[w];
    }
    const u32 pre_blk = pre, vpre_blk = vpre;
#pragma unroll
    for (int w = 0; w < kDownThreads / 32; w++) {
        if (w < warp) { pre += s_w[w]; vpre += s_v[w]; }
        btot += s_w[w];
        bvis += s_v[w];
    }
    if (blockIdx.x == gridDim.x - 1 && tid == 0) {
        totals[0] = (u64)pre_blk + btot;
        if (MODE == 0) totals[1] = (u64)vpre_blk + bvis;
    }
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
        const u64 i = wbase + 32 * j + lane;
        if (i < count) {
            out[i] = pre + ex[j];
            if (MODE == 1) {  // key blocks whose first slot lies in this Gaussian's range
                const u32 a = pre + ex[j], e = a + (u32)v[j];
                for (u32 b = (a + kKeyChunk - 1) / kKeyChunk; b * (u32)kKeyChunk < e; b++) co.first[b] = (u32)i;
                if (i == count - 1) co.first[(e + kKeyChunk - 1) / kKeyChunk] = (u32)i;  // sentinel: last one
            }
        }
    }
    if (MODE == 0) {
        const u32 ltmask = lanemask_lt();
        u32 nmin = 0, dmax = 0;  // max of ~bits (= ~min) and of bits over this thread's visible
        u32 db[ITEMS];
#pragma unroll
        for (int q = 0; q < ITEMS; q++) db[q] = dbits_pre[q];
#pragma unroll
        for (int q = 0; q < ITEMS; q++) {
            const u64 i = wbase + 32 * q + lane;
            const bool vis = v[q] > 0;
            const u32 bal = __ballot_sync(VKS_FULL_MASK, vis);
            if (vis) {
                const u32 slot = vpre + __popc(bal & ltmask);
                co.vkeys[slot] = db[q];
                co.vids[slot] = (u32)i;
                nmin = max(nmin, ~db[q]);
                dmax = max(dmax, db[q]);
            }
            vpre += __popc(bal);
        }
        // block-wide max first: one pair of global atomics per block (per-warp atomics on the same
        // two addresses serialised in L2: 45K of them made this kernel 55 us instead of ~30)
        nmin = __reduce_max_sync(VKS_FULL_MASK, nmin);
        dmax = __reduce_max_sync(VKS_FULL_MASK, dmax);
        __shared__ u32 s_mm[2];
        if (tid == 0) { s_mm[0] = 0; s_mm[1] = 0; }
        __syncthreads();
        if (lane == 0 && (nmin | dmax)) {
            atomicMax(&s_mm[0], nmin);
            atomicMax(&s_mm[1], dmax);
        }
        __syncthreads();
        if (tid == 0 && (s_mm[0] | s_mm[1])) {
            atomicMax(co.dminmax, s_mm[0]);
            atomicMax(co.dminmax + 1, s_mm[1]);
        }
    }
}

// ------------------------------------------------------------------------------------------
// 4a. tile-rect difference array (per-tile key counts without touching the keys): persistent
// blocks, 4 shared-memory updates per visible Gaussian, one flush per block.
constexpr int kDiffThreads = 512;
constexpr int kDiffSmemMax = 160 * 1024 / 4;  // cells
constexpr size_t kTileCountSmemMax = 200 * 1024;  // bytes

template <bool SMEM_DIFF>
__global__ void __launch_bounds__(kDiffThreads) rect_diff_kernel(int TX, int TY, u32 count, const u64* __restrict__ rc,
                                                                int* __restrict__ diff, const u64* __restrict__ dcount) {
    pdl_wait();
    extern __shared__ int s_diff[];
    count = (u32)eff_count(count, dcount);
    const int tid = threadIdx.x;
    const int W1 = TX + 1;
    const int cells = W1 * (TY + 1);
    if (SMEM_DIFF) {
        for (int j = tid; j < cells; j += kDiffThreads) s_diff[j] = 0;
        __syncthreads();
    }
    int* dd = SMEM_DIFF ? s_diff : diff;
    constexpr int U = 8;  // rect codes in flight per thread (the loop is load-latency bound; 4 in flight: 14.9 us, 8: 13.7)
    const u32 stride = gridDim.x * kDiffThreads;
    for (u32 r0 = blockIdx.x * kDiffThreads + tid; r0 < count; r0 += U * stride) {
        u64 c[U];
#pragma unroll
        for (int q = 0; q < U; q++) c[q] = r0 + q * stride < count ? __ldg(rc + r0 + q * stride) : 0ull;
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (r0 + q * stride >= count) break;
            int x0, x1, y0, y1;
            unpack_rect(c[q], x0, x1, y0, y1);
            VKS_DCHECK(x0 <= x1 && x1 <= TX && y0 <= y1 && y1 <= TY);
            atomicAdd(dd + y0 * W1 + x0, 1);
            atomicAdd(dd + y0 * W1 + x1, -1);
            atomicAdd(dd + y1 * W1 + x0, -1);
            atomicAdd(dd + y1 * W1 + x1, 1);
        }
    }
    if (SMEM_DIFF) {
        __syncthreads();
        for (int j = tid; j < cells; j += kDiffThreads) {
            const int v = s_diff[j];
            if (v) atomicAdd(diff + j, v);
        }
    }
}

// 4b. debug only (keys_unsorted / vals_unsorted): the u64 keys in id order exactly as "Generate
// Keys" defines them, written at offsets[i] + k, rows outer.  One warp expands 32 rects.
constexpr int kKeysThreads = 256;
constexpr int kKeysWarps = kKeysThreads / 32;

__global__ void __launch_bounds__(kKeysThreads) keys_debug_kernel(vks_camera cam, int64_t count,
                                                                 const int* __restrict__ tiles,
                                                                 const float2* __restrict__ means2d,
                                                                 const int2* __restrict__ radii,
                                                                 const float* __restrict__ depths,
                                                                 const u32* __restrict__ slot0,
                                                                 u32* __restrict__ tvals, u64* __restrict__ keys64) {
    __shared__ int s_incl[kKeysWarps][32];
    __shared__ int s_x0[kKeysWarps][32], s_y0[kKeysWarps][32], s_w[kKeysWarps][32];
    __shared__ u32 s_db[kKeysWarps][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int64_t stride = (int64_t)gridDim.x * kKeysWarps * 32;
    for (int64_t r0 = ((int64_t)blockIdx.x * kKeysWarps + warp) * 32; r0 < count; r0 += stride) {
        const int64_t r = r0 + lane;
        int cnt = 0, x0 = 0, y0 = 0, w = 1;
        u32 db = 0;
        if (r < count && __ldg(tiles + r) > 0) {
            int x1, y1;
            rect_of(__ldg(means2d + r), __ldg(radii + r), TX, TY, x0, x1, y0, y1);
            w = x1 - x0;
            cnt = w * (y1 - y0);
            db = __float_as_uint(__ldg(depths + r));
            if (cnt <= 0) { cnt = 0; w = 1; }
        }
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
            if (lane >= d) incl += t;
        }
        const int total = __shfl_sync(VKS_FULL_MASK, incl, 31);
        if (total == 0) continue;
        __syncwarp();
        s_incl[warp][lane] = incl;
        s_x0[warp][lane] = x0;
        s_y0[warp][lane] = y0;
        s_w[warp][lane] = w;
        s_db[warp][lane] = db;
        __syncwarp();
        const u64 base = (u64)__ldg(slot0 + r0);  // slot of the group's first Gaussian (even if empty)
        for (int e = lane; e < total; e += 32) {
            int pos = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
                if (s_incl[warp][pos + step - 1] <= e) pos += step;
            const int k = e - (pos ? s_incl[warp][pos - 1] : 0);  // index within the rect, rows outer
            const int ww = s_w[warp][pos];
            const int ry = k / ww;
            const int tx = s_x0[warp][pos] + (k - ry * ww);
            const int ty = s_y0[warp][pos] + ry;
            const u32 t = (u32)(ty * TX + tx);
            if (keys64) keys64[base + e] = ((u64)t << 32) | (u64)s_db[warp][pos];
            if (tvals) tvals[base + e] = (u32)(r0 + pos);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------
// 5. per-tile counts -> CSR tile_offsets
__global__ void iota_kernel(u32* __restrict__ out, u32 n) {
    pdl_wait();
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

// Scheduling hint for the rasterizer: tile ids by decreasing list length, bucketed into 64
// log-spaced length classes (4 per octave); order within a class is arbitrary.
__device__ __forceinline__ int length_class(u32 len) {
    if (len == 0) return 0;
    const int e = 31 - __clz(len);                                   // octave
    const int f = e >= 2 ? (int)((len >> (e - 2)) & 3u) : (int)((len << (2 - e)) & 3u);
    return min(63, 4 * e + f + 1);
}

// The (TX+1) x (TY+1) difference array is staged in shared memory when it fits (SMEM) so the
// serial column walk is not a chain of global-memory round trips.
template <bool SMEM>
__global__ void __launch_bounds__(1024) tile_count_kernel(int TX, int TY, int* __restrict__ diff,
                                                         u32* __restrict__ tile_offsets, u32* __restrict__ order) {
    pdl_wait();
    extern __shared__ int s_cells[];
    __shared__ u32 s_wsum[32];
    __shared__ u32 s_carry;
    __shared__ u32 s_cls[64];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W1 = TX + 1;
    const int cells = W1 * (TY + 1);
    int* a = SMEM ? s_cells : diff;
    if (SMEM) {
        for (int j = tid; j < cells; j += 1024) s_cells[j] = diff[j];
        __syncthreads();
    }
    // prefix along x: one warp per row, 32 cells per step
    for (int y = warp; y < TY; y += 32) {
        int carry = 0;
        for (int x0 = 0; x0 < TX; x0 += 32) {
            const int x = x0 + lane;
            const int v = x < TX ? a[y * W1 + x] : 0;
            const int incl = (int)warp_incl_scan((u32)v, lane) + carry;
            if (x < TX) a[y * W1 + x] = incl;
            carry = __shfl_sync(VKS_FULL_MASK, incl, 31);
        }
    }
    __syncthreads();
    // prefix along y: one thread per column
    for (int x = tid; x < TX; x += 1024) {
        int acc = 0;
        for (int y = 0; y < TY; y++) { acc += a[y * W1 + x]; a[y * W1 + x] = acc; }
    }
    __syncthreads();
    // exclusive scan of the per-tile counts in tile order (+ the length-class histogram) in one
    // pass: thread t owns the `per` consecutive tiles [t per, t per + per), sums them, a block-wide
    // scan of the 1024 thread sums gives each thread its base, and the thread writes its tiles'
    // offsets (round 1 scanned 1024 tiles per round with four barriers and a 32-step walk per
    // round: 15.1 -> 11.8 us on bicycle's 4,056 tiles)
    const int n_tiles = TX * TY;
    const int per = (n_tiles + 1023) / 1024;
    if (tid < 64) s_cls[tid] = 0;
    const int t0 = min(tid * per, n_tiles), t1 = min(t0 + per, n_tiles);
    u32 mine = 0;
    for (int t = t0; t < t1; t++) mine += (u32)a[(t / TX) * W1 + (t % TX)];
    const u32 incl = warp_incl_scan(mine, lane);
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const u32 wv = s_wsum[lane];
        const u32 wi = warp_incl_scan(wv, lane);
        s_wsum[lane] = wi - wv;  // exclusive prefix of the warp totals
        if (lane == 31) s_carry = wi;
    }
    __syncthreads();
    u32 run = s_wsum[warp] + incl - mine;
    for (int t = t0; t < t1; t++) {
        const u32 c = (u32)a[(t / TX) * W1 + (t % TX)];
        tile_offsets[t] = run;
        run += c;
        if (order) atomicAdd(&s_cls[63 - length_class(c)], 1u);
    }
    if (tid == 0) tile_offsets[n_tiles] = s_carry;
    if (!order) return;
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 64 class counts (longest class first)
        const u32 ca = s_cls[tid], cb = s_cls[tid + 32];
        const u32 ia = warp_incl_scan(ca, tid);
        const u32 tot_a = __shfl_sync(VKS_FULL_MASK, ia, 31);
        const u32 ib = warp_incl_scan(cb, tid);
        s_cls[tid] = ia - ca;
        s_cls[tid + 32] = tot_a + ib - cb;
    }
    __syncthreads();
    for (int t = tid; t < n_tiles; t += 1024) {
        const u32 c = (u32)a[(t / TX) * W1 + (t % TX)];
        order[atomicAdd(&s_cls[63 - length_class(c)], 1u)] = (u32)t;
    }
}

// ------------------------------------------------------------------------------------------
// LSD radix pass over DBITS bits starting at `shift` of u32 keys with u32 values, as
// reduce-then-scan (no inter-block waiting):
//   digit_count_kernel   per 4096-key tile: digit histogram (warp ballot multi-split aggregation)
//                        -> counts[d * T + tile]
//   scan_u32_kernel      exclusive scan of counts in digit-major order = global start of
//                        (digit d, tile t) for every tile and digit
//   scatter_kernel       per tile: TMA bulk copy of keys/values into shared memory (mbarrier),
//                        stable warp-level ranking (ballot multi-split), in-place shared-memory
//                        reorder by digit, digit-contiguous coalesced stores.
enum { kPassPlain = 0, kPassTileLast = 2 };


// lanes of the warp holding the same DBITS-bit digit (and the same `valid`): DBITS ballots
// instead of __match_any_sync, whose cost grows with the number of distinct values
// Each bit: the predicate straight from d & (1 << b) (one LOP3), the ballot, and the lanes with
// the same bit as this lane — the ballot, inverted under the predicate's complement — ANDed in:
// 4 instructions per bit (the C++ form compiled to 6: shift, and, compare, select, vote, merge).
template <int DBITS>
__device__ __forceinline__ u32 digit_peers(u32 d, bool valid = true) {
    u32 peers = __ballot_sync(VKS_FULL_MASK, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < DBITS; b++) {
        u32 same;
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "@!p not.b32 %0, %0;\n\t}"
            : "=r"(same)
            : "r"(d), "r"(1u << b));
        peers &= same;
    }
    return peers;
}

template <int DBITS>
__global__ void __launch_bounds__(kSortThreads) digit_count_kernel(const u32* __restrict__ kin, u32 n, int shift,
                                                                  u32 kbias, u32 T, u32* __restrict__ counts,
                                                                  const u64* __restrict__ dcount) {
    pdl_wait();
    n = (u32)eff_count(n, dcount);
    constexpr int RADIX = 1 << DBITS;
    constexpr u32 DMASK = RADIX - 1;
    __shared__ u32 whist[kSortWarps][RADIX];  // per-warp histograms: contention only within a warp
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int j = tid; j < kSortWarps * RADIX; j += kSortThreads) (&whist[0][0])[j] = 0;
    __syncthreads();
    const u64 base = (u64)blockIdx.x * kSortTile;
    u32 key[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {  // all loads in flight before any use
        const u64 idx = base + (u64)i * kSortThreads + tid;
        key[i] = idx < n ? __ldg(kin + idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        if (base + (u64)i * kSortThreads + tid < n) atomicAdd(&whist[warp][((key[i] - kbias) >> shift) & DMASK], 1u);
    }
    __syncthreads();
    for (int d = tid; d < RADIX; d += kSortThreads) {
        u32 c = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) c += whist[w][d];
        counts[(u64)d * T + blockIdx.x] = c;
    }
}

// Exclusive scan of a u32 array (the digit-count matrices of the radix passes, <= a few hundred
// tiles): single pass over 4096-element tiles (warp-striped loads and stores) with a decoupled
// look-back done by a whole warp, 32 predecessors' aggregates per step.  (For millions of
// elements — 1,000+ tiles all in flight at once — the look-back walks get long; the 1-D scans of
// the tile counts use reduce-then-scan instead, measured: 39 us vs 30 us on 4.15M elements.)
__global__ void __launch_bounds__(kScanThreads) scan_u32_kernel(const u32* __restrict__ in, u32* __restrict__ out,
                                                               u64 count, u64* __restrict__ lb, u32* __restrict__ ctr) {
    pdl_wait();
    __shared__ u32 s_tile;
    __shared__ u32 s_warp[kScanThreads / 32];
    __shared__ u64 s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    const u64 wbase = tile * kCntTile + (u64)warp * 32 * kCntItems;
    int v[kCntItems];
    u32 ex[kCntItems];
#pragma unroll
    for (int j = 0; j < kCntItems; j++) {
        const u64 i = wbase + 32 * j + lane;
        v[j] = i < count ? (int)__ldg(in + i) : 0;
    }
    const u32 wtot = warp_striped_excl<kCntItems>(v, ex, lane);
    if (lane == 0) s_warp[warp] = wtot;
    __syncthreads();
    u64 wpre = 0, btotal = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; w++) {
        if (w < warp) wpre += s_warp[w];
        btotal += s_warp[w];
    }
    if (warp == 0) {
        u64 excl = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile_u64(reinterpret_cast<unsigned long long*>(lb), kScanFlagInc | btotal);
        } else {
            if (lane == 0) st_volatile_u64(reinterpret_cast<unsigned long long*>(lb + tile), kScanFlagAgg | btotal);
            int64_t j = (int64_t)tile - 1;
            while (true) {
                const int64_t q = j - lane;
                const u64 st = q >= 0 ? ld_volatile_u64(reinterpret_cast<const unsigned long long*>(lb + q))
                                      : kScanFlagInc;  // before tile 0: inclusive prefix 0
                const u64 f = st & ~kScanMask;
                const unsigned inc = __ballot_sync(VKS_FULL_MASK, f == kScanFlagInc);
                const unsigned pend = __ballot_sync(VKS_FULL_MASK, f == 0);
                const int first_inc = inc ? __ffs(inc) - 1 : 32;
                const int first_pend = pend ? __ffs(pend) - 1 : 32;
                const int take = first_pend < first_inc ? first_pend : min(first_inc + 1, 32);
                u64 add = lane < take ? (st & kScanMask) : 0;
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) add += __shfl_xor_sync(VKS_FULL_MASK, add, o);
                excl += add;
                if (first_inc < first_pend) break;  // reached an inclusive prefix
                j -= take;                          // take may be 0: spin on a pending predecessor
            }
            if (lane == 0) st_volatile_u64(reinterpret_cast<unsigned long long*>(lb + tile), kScanFlagInc | (excl + btotal));
        }
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    const u32 pre = (u32)(s_prefix + wpre);
#pragma unroll
    for (int j = 0; j < kCntItems; j++) {
        const u64 i = wbase + 32 * j + lane;
        if (i < count) out[i] = pre + ex[j];
    }
}

#ifndef VKS_SCATTER_MINB
#define VKS_SCATTER_MINB 5  // resident blocks per SM of the scatter kernels (48 registers; 4: 64 registers,
#endif                      // 756 vs 757.5 views/s; 6: 40 registers with spills, 713)
template <int RADIX>
struct SortSmem {
    alignas(128) u32 keys[kSortTile];  // input staging (bulk copy), then the reordered tile
    alignas(128) u32 vals[kSortTile];
    u32 whist[kSortWarps][RADIX];
    u32 gbase[RADIX];
    u32 wsum[kSortWarps];
    alignas(8) unsigned long long mbar;
};

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

// Rank the block's kSortTile staged (key, value) pairs stably by digit, reorder them in shared
// memory and store them digit-contiguously at their global positions.  On entry: S.keys/S.vals
// hold the tile (pads: key 0xFFFFFFFF, which rank last and land at dest >= n), S.whist is zero,
// S.gbase[d] holds the global start of (digit d, this block), and the block is synchronised.
// kPassTileLast: writes only the values (the caller's vals) and, if keys64, the u64 keys.
template <int DBITS, int MODE>
__device__ __forceinline__ void rank_and_store(SortSmem<1 << DBITS>& S, u32 n, int shift, u32 kbias,
                                               u32* __restrict__ kout, u32* __restrict__ vout,
                                               const float* __restrict__ depths, u64* __restrict__ keys64) {
    constexpr int RADIX = 1 << DBITS;
    constexpr u32 DMASK = RADIX - 1;
    constexpr int DPT = (RADIX + kSortThreads - 1) / kSortThreads;  // digits per thread (1 or 2)
    static_assert(RADIX <= 2 * kSortThreads, "radix");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u32 rank[kSortItems];
    const u32 ltmask = lanemask_lt();
    const int seg = warp * 32 * kSortItems;
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        const u32 d = ((S.keys[seg + i * 32 + lane] - kbias) >> shift) & DMASK;
        const u32 peers = digit_peers<DBITS>(d);  // (match.any measured 17% slower for the whole sort)
        const u32 below = __popc(peers & ltmask);
        const u32 before = S.whist[warp][d];
        rank[i] = before + below;
        __syncwarp();
        if (below == 0) S.whist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // thread t owns digits [t DPT, t DPT + DPT): exclusive prefix over warps per digit, then a
    // block-wide exclusive scan of the digit totals in digit order
    u32 dtot[DPT];
    u32 total = 0;
#pragma unroll
    for (int q = 0; q < DPT; q++) {
        const int d = tid * DPT + q;
        u32 run = 0;
        if (d < RADIX) {
#pragma unroll
            for (int w = 0; w < kSortWarps; w++) {
                const u32 c = S.whist[w][d];
                S.whist[w][d] = run;
                run += c;
            }
        }
        dtot[q] = run;
        total += run;
    }
    u32 incl = total;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    {   // the digit's block start folded into its per-warp offsets: one shared-memory read per key
        u32 start = incl - total;
        for (int w = 0; w < warp; w++) start += S.wsum[w];
#pragma unroll
        for (int q = 0; q < DPT; q++) {
            const int d = tid * DPT + q;
            if (d < RADIX) {
#pragma unroll
                for (int w = 0; w < kSortWarps; w++) S.whist[w][d] += start;
                S.gbase[d] -= start;
            }
            start += dtot[q];
        }
    }
    __syncthreads();
    u32 kk[kSortItems], vv[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        const int slot = seg + i * 32 + lane;
        kk[i] = S.keys[slot];
        vv[i] = S.vals[slot];
        rank[i] += S.whist[warp][((kk[i] - kbias) >> shift) & DMASK];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        S.keys[rank[i]] = kk[i];
        S.vals[rank[i]] = vv[i];
    }
    __syncthreads();
#pragma unroll 4
    for (int j = tid; j < kSortTile; j += kSortThreads) {
        const u32 key = S.keys[j];
        const u32 dest = S.gbase[((key - kbias) >> shift) & DMASK] + (u32)j;
        VKS_DCHECK(dest < n || key - kbias == 0xFFFFFFFFu);  // only the last block's pads (key kbias - 1) fall past n
        if (dest < n) {
            const u32 val = S.vals[j];
            if (MODE != kPassTileLast) kout[dest] = key;
            vout[dest] = val;
            if (MODE == kPassTileLast && keys64)
                keys64[dest] = ((u64)key << 32) | (u64)__float_as_uint(__ldg(depths + val));
        }
    }
}

template <int DBITS, int MODE>
__global__ void __launch_bounds__(kSortThreads, VKS_SCATTER_MINB) scatter_kernel(const u32* __restrict__ kin, const u32* __restrict__ vin,
                                                             u32* __restrict__ kout, u32* __restrict__ vout, u32 n,
                                                             int shift, u32 kbias, u32 T, const u32* __restrict__ offs,
                                                             const float* __restrict__ depths,
                                                             u64* __restrict__ keys64, const u64* __restrict__ dcount) {
    pdl_wait();
    constexpr int RADIX = 1 << DBITS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SortSmem<RADIX>& S = *reinterpret_cast<SortSmem<RADIX>*>(smem_raw);
    const int tid = threadIdx.x;
    const u32 bar = smem_u32(&S.mbar);
    const u32 tile = blockIdx.x;
    const u64 base = (u64)tile * kSortTile;
    n = (u32)eff_count(n, dcount);
    if (base >= n) return;  // (async: the grid was sized for the bound; the whole block leaves)
    const u32 count = (u32)min((u64)kSortTile, (u64)n - base);
    const u32 nbulk = count & ~3u;  // 16-byte multiples
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nbulk) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nbulk * 8u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(S.keys)), "l"(kin + base), "r"(nbulk * 4u), "r"(bar) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(S.vals)), "l"(vin + base), "r"(nbulk * 4u), "r"(bar) : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
        }
    }
    for (int j = tid; j < kSortWarps * RADIX; j += kSortThreads) (&S.whist[0][0])[j] = 0;
    // the block's digit starts: global start of (digit, tile) from the scanned counts
    for (int d = tid; d < RADIX; d += kSortThreads) S.gbase[d] = __ldg(offs + (u64)d * T + tile);
    for (u32 j = nbulk + tid; j < (u32)kSortTile; j += kSortThreads) {
        const bool ok = j < count;
        S.keys[j] = ok ? kin[base + j] : kbias - 1u;  // pads: the largest digit, rank last (dest >= n)
        S.vals[j] = ok ? vin[base + j] : 0u;
    }
    __syncthreads();  // barrier init visible before anyone waits on it
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT%=;\n\t}" ::"r"(bar) : "memory");
    __syncthreads();
    rank_and_store<DBITS, MODE>(S, n, shift, kbias, kout, vout, depths, keys64);
}

// ------------------------------------------------------------------------------------------
// 4. key generation fused with the first tile pass.  Block b owns the key slots
// [4096 b, 4096 b + 4096) of the depth-ordered key sequence (slot0[r] + k, rows outer) and expands
// exactly those keys from the rect codes: the Gaussians covering the range are r0 = first[8 b] ..
// the one holding slot 4096 (b + 1) (first[c] = the Gaussian holding slot 512 c, written by the
// depth-order scan); each warp expands the 512 slots it later ranks, starting at first[c0 / 512]
// (expand_chunk).  keys_count_kernel only histograms the first tile digit;
// keys_scatter_kernel re-expands the block (cheaper than writing and re-reading M keys) and ranks
// and stores it like any radix pass.
struct ExpandSrc {
    const u64* rc;      // [V] rect codes, depth order
    const u32* slot0;   // [V] first slot of each Gaussian's keys
    const u32* sid;     // [V] Gaussian ids, depth order
    const u32* first;   // [chunks + 1] Gaussian holding slot 512 c (chunks = ceil(M / 512))
    u32 V, M;
    int TX;
    const u64* dtot;    // nullable (vks_bin_sort_async): device totals [M, V]; V / M are then bounds
    __device__ __forceinline__ ExpandSrc resolved() const {
        ExpandSrc e = *this;
        if (dtot) {
            e.M = (u32)min((u64)M, dtot[0]);
            e.V = (u32)min((u64)V, dtot[1]);
        }
        return e;
    }
};

// floor(k / w) for 0 <= k < 2^20, 1 <= w < 2^16: (k + 0.5) / w lies at least 0.5 / w from an
// integer, while x * rcp.approx(w) errs by < 2^-21 (k + 0.5) / w < 0.5 / w
__device__ __forceinline__ float rcp_width(int w) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)w));  // w >= 1: no range special cases
    return r;
}
__device__ __forceinline__ int div_floor_r(int k, float r) { return (int)(((float)k + 0.5f) * r); }
__device__ __forceinline__ int div_floor(int k, int w) { return div_floor_r(k, rcp_width(w)); }

// f(slot, tile, id) for every key slot in [c0, c1) (c1 - c0 <= 512, all inside block b), one
// slot per lane per round of 32.  The Gaussian owning slot s is the last one with slot0 <= s; the
// owner of c0 (a multiple of 512) is first[c0 / 512]; from there the warp takes the chunk's Gaussians in groups
// of 32 (lane j = one Gaussian, its record loaded one group ahead).  Within a group the keys are
// contiguous slots; per round the lanes whose first key falls in the 32-slot window set one bit
// each of an OR-reduced word, and a lane's owner is the last owner before the window plus the
// number of starts at or before its slot.
template <class F>
__device__ __forceinline__ void expand_chunk(const ExpandSrc& src, u32 b, u32 c0, u32 c1, F&& f) {
    const int lane = threadIdx.x & 31;
    // owner of c0 (a multiple of 512): written by the depth-order scan, no search
    (void)b;
    const u32 lo = __ldg(src.first + c0 / kKeyChunk);
    const u32 ltle = 0xFFFFFFFFu >> (31 - lane);  // bits 0..lane
    u32 g = lo;  // first Gaussian of the current group
    u32 a_n = 0xFFFFFFFFu, id_n = 0;
    u64 rc_n = 0;
    if (g + lane < src.V) {
        a_n = __ldg(src.slot0 + g + lane);
        rc_n = __ldg(src.rc + g + lane);
        id_n = __ldg(src.sid + g + lane);
    }
    u32 W = c0;  // next slot to produce
    while (W < c1) {
        const u32 a = a_n, id = id_n;  // lane j: Gaussian g + j (a = its first slot; ~0: none)
        const u64 rc = rc_n;
        // per Gaussian, once per group: slot k of the rect (rows outer) is tile
        // base + k + floor(k / w) (TX - w), base = y0 TX + x0; floor via 1 / w
        int gx0, gx1, gy0, gy1;
        unpack_rect(rc, gx0, gx1, gy0, gy1);
        const int gw = max(gx1 - gx0, 1);
        const u32 gbase = (u32)(gy0 * src.TX + gx0);
        const int gstep = src.TX - gw;
        const float grw = rcp_width(gw);
        const u32 gn = g + 32;
        a_n = 0xFFFFFFFFu;  // the next group's records, in flight while this group expands
        if (gn + lane < src.V) {
            a_n = __ldg(src.slot0 + gn + lane);
            rc_n = __ldg(src.rc + gn + lane);
            id_n = __ldg(src.sid + gn + lane);
        }
        // the group covers slots [W, gend): up to the end of its last Gaussian's keys (= the next
        // group's first slot; known without waiting for the next group's loads), or c1
        const u32 end = a == 0xFFFFFFFFu ? 0xFFFFFFFFu : a + (u32)rect_tiles(rc);
        const u32 gend = min(c1, __shfl_sync(VKS_FULL_MASK, end, 31));
        // owner lane of slot W - 1: lane 0 if its Gaussian started before W (only the chunk's
        // first group), else none (-1: lane 0's start at W is counted in the first window)
        int base = __shfl_sync(VKS_FULL_MASK, a, 0) < W ? 0 : -1;
        for (; W < gend; W += 32) {
            const u32 d = a - W;  // a lane's first key lies in the window when a >= W and d < 32
            const u32 starts = __reduce_or_sync(VKS_FULL_MASK, (a >= W && d < 32u) ? (1u << d) : 0u);
            const int own = base + __popc(starts & ltle);
            const int srcl = own < 0 ? 0 : own;
            const u32 a_o = __shfl_sync(VKS_FULL_MASK, a, srcl);
            const u32 base_o = __shfl_sync(VKS_FULL_MASK, gbase, srcl);
            const int step_o = __shfl_sync(VKS_FULL_MASK, gstep, srcl);
            const float rw_o = __shfl_sync(VKS_FULL_MASK, grw, srcl);
            const u32 id_o = __shfl_sync(VKS_FULL_MASK, id, srcl);
            const u32 slot = W + (u32)lane;
            if (slot < gend) {
                const int k = (int)(slot - a_o);  // index within the rect, rows outer
                const int ry = div_floor_r(k, rw_o);
                f(slot, base_o + (u32)k + (u32)(ry * step_o), id_o);
            }
            base += __popc(starts);
        }
        W = gend;  // the next group starts at its first Gaussian's first slot
        g = gn;
    }
}

// Digit histogram of each 4096-slot key block without enumerating the keys: a Gaussian's keys
// within one rect row are consecutive tile ids, so a row of length L adds floor(L / R) to every
// digit and 1 to a cyclic run of L mod R digits (a difference array over the R digits).  (Counting
// through the key expansion of keys_scatter_kernel issued 1.7x the instructions.)
template <int DBITS>
__global__ void __launch_bounds__(kSortThreads) keys_count_kernel(const ExpandSrc src_in, int shift, u32 T,
                                                                 u32* __restrict__ counts) {
    pdl_wait();
    constexpr int RADIX = 1 << DBITS;
    constexpr int DMASK = RADIX - 1;
    const ExpandSrc src = src_in.resolved();
    if ((u64)blockIdx.x * kSortTile >= src.M) {  // (async: past the keys; first[] is not written there)
        for (int d = threadIdx.x; d < RADIX; d += kSortThreads) counts[(u64)d * T + blockIdx.x] = 0u;
        return;
    }
    __shared__ int wdiff[kSortWarps][RADIX + 1];  // per warp: contention only within a warp
    __shared__ int s_all[kSortWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    (void)shift;  // the key pass sorts the lowest tile bits (shift 0)
    for (int j = tid; j < kSortWarps * (RADIX + 1); j += kSortThreads) (&wdiff[0][0])[j] = 0;
    __syncthreads();
    int* sdiff = wdiff[warp];
    const u32 b = blockIdx.x;
    const u32 S = b * (u32)kSortTile;
    const u32 E = min(S + (u32)kSortTile, src.M);
    // the Gaussians holding the block's first slot and slot E (its chunk, or the sentinel)
    const u32 r0 = __ldg(src.first + b * kChunksPerTile);
    const u32 r1 = __ldg(src.first + (E - 1) / kKeyChunk + 1);
    int all = 0;
    for (u32 r = r0 + tid; r <= r1; r += kSortThreads) {
        int x0, x1, y0, y1;
        unpack_rect(__ldg(src.rc + r), x0, x1, y0, y1);
        const int w = x1 - x0;
        const u32 a = __ldg(src.slot0 + r);
        const u32 c = (u32)(w * (y1 - y0));
        const u32 l = max(a, S), h = min(a + c, E);
        if (h <= l) continue;
        const int k0 = (int)(l - a), k1 = (int)(h - a) - 1;  // key indices within the rect
        const int ry0 = div_floor(k0, w), ry1 = div_floor(k1, w);
        for (int ry = ry0; ry <= ry1; ry++) {
            const int xs = ry == ry0 ? k0 - ry * w : 0;
            const int xe = ry == ry1 ? k1 - ry * w + 1 : w;
            const int len = xe - xs;
            const int t0 = (y0 + ry) * src.TX + x0 + xs;
            all += len >> DBITS;
            const int rem = len & DMASK, b0 = t0 & DMASK;
            if (rem) {
                atomicAdd(&sdiff[b0], 1);
                if (b0 + rem <= RADIX) {
                    atomicAdd(&sdiff[b0 + rem], -1);
                } else {
                    atomicAdd(&sdiff[0], 1);
                    atomicAdd(&sdiff[b0 + rem - RADIX], -1);
                }
            }
        }
    }
    all = __reduce_add_sync(VKS_FULL_MASK, all);
    if (lane == 0) s_all[warp] = all;
    __syncthreads();
    if (tid < 32) {  // prefix of the difference array; RADIX <= 256 = 8 chunks of 32
        int tot = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) tot += s_all[w];
        int carry = 0;
        for (int d0 = 0; d0 < RADIX; d0 += 32) {
            const int d = d0 + lane;
            int v = 0;
            if (d < RADIX) {
#pragma unroll
                for (int w = 0; w < kSortWarps; w++) v += wdiff[w][d];
            }
            const int incl = (int)warp_incl_scan((u32)v, lane) + carry;
            if (d < RADIX) counts[(u64)d * T + b] = (u32)(incl + tot);
            carry = __shfl_sync(VKS_FULL_MASK, incl, 31);
        }
    }
}

template <int DBITS, int MODE>
__global__ void __launch_bounds__(kSortThreads, VKS_SCATTER_MINB) keys_scatter_kernel(const ExpandSrc src_in, int shift, u32 T,
                                                                   const u32* __restrict__ offs, u32* __restrict__ kout,
                                                                   u32* __restrict__ vout, const float* __restrict__ depths,
                                                                   u64* __restrict__ keys64) {
    pdl_wait();
    constexpr int RADIX = 1 << DBITS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SortSmem<RADIX>& S = *reinterpret_cast<SortSmem<RADIX>*>(smem_raw);
    const ExpandSrc src = src_in.resolved();
    const int tid = threadIdx.x, warp = tid >> 5;
    const u32 b = blockIdx.x;
    if ((u64)b * kSortTile >= src.M) return;
    const u32 count = min((u32)kSortTile, src.M - b * (u32)kSortTile);
    for (int j = tid; j < kSortWarps * RADIX; j += kSortThreads) (&S.whist[0][0])[j] = 0;
    for (int d = tid; d < RADIX; d += kSortThreads) S.gbase[d] = __ldg(offs + (u64)d * T + b);
    for (u32 j = count + tid; j < (u32)kSortTile; j += kSortThreads) {
        S.keys[j] = 0xFFFFFFFFu;  // pads rank last
        S.vals[j] = 0u;
    }
    const u32 S0 = b * (u32)kSortTile;
    const u32 c0 = S0 + (u32)warp * 32 * kSortItems;  // the warp expands the slots it ranks
    const u32 c1 = min(c0 + 32u * kSortItems, src.M);
    if (c0 < c1)
        expand_chunk(src, b, c0, c1, [&](u32 slot, u32 tile, u32 id) {
            VKS_DCHECK(slot >= S0 && slot - S0 < (u32)kSortTile && tile < (u32)(1 << 24));
            S.keys[slot - S0] = tile;
            S.vals[slot - S0] = id;
        });
    __syncthreads();
    rank_and_store<DBITS, MODE>(S, src.M, shift, 0u, kout, vout, depths, keys64);
}

struct PassBufs {
    u32* counts;  // [radix * T]
    u32* offs;    // [radix * T]
    u64* lb;      // scan look-back of the counts
    u32* ctr;     // scan tile counter (zeroed)
};

template <int DBITS, int MODE>
int launch_pass(const u32* kin, const u32* vin, u32* kout, u32* vout, u32 n, int shift, u32 kbias, const PassBufs& pb,
                const float* depths, u64* keys64, cudaStream_t s, const u64* dcount = nullptr) {
    constexpr size_t sm = sizeof(SortSmem<1 << DBITS>);
    // set on every call: the attribute belongs to the current device (a process may drive several)
    if (cudaError_t e = cudaFuncSetAttribute(scatter_kernel<DBITS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm))
        return cuda_fail(e, "scatter smem attribute");
    const u32 T = (u32)((n + kSortTile - 1) / kSortTile);
    if (!T) return VKS_OK;
    launch_k(digit_count_kernel<DBITS>, T, kSortThreads, 0, s, kin, n, shift, kbias, T, pb.counts, dcount);
    const u64 cnt = (u64)(1u << DBITS) * T;
    launch_k(scan_u32_kernel, (unsigned)((cnt + kCntTile - 1) / kCntTile), kScanThreads, 0, s, pb.counts, pb.offs, cnt, pb.lb, pb.ctr);
    launch_k(scatter_kernel<DBITS, MODE>, T, kSortThreads, sm, s, kin, vin, kout, vout, n, shift, kbias, T, pb.offs, depths,
                                                            keys64, dcount);
    return check_launch(__func__);
}

// runtime digit width (1..9 bits) -> instantiation
template <int MODE>
int launch_pass_bits(int dbits, const u32* kin, const u32* vin, u32* kout, u32* vout, u32 n, int shift, u32 kbias,
                     const PassBufs& pb, const float* depths, u64* keys64, cudaStream_t s,
                     const u64* dcount = nullptr) {
#define VKS_PASS(B) return launch_pass<B, MODE>(kin, vin, kout, vout, n, shift, kbias, pb, depths, keys64, s, dcount)
    switch (dbits) {
        case 1: VKS_PASS(1);
        case 2: VKS_PASS(2);
        case 3: VKS_PASS(3);
        case 4: VKS_PASS(4);
        case 5: VKS_PASS(5);
        case 6: VKS_PASS(6);
        case 7: VKS_PASS(7);
        case 8: VKS_PASS(8);
        default: VKS_PASS(9);
    }
#undef VKS_PASS
}

constexpr int kMaxDevices = 64;

// SM count of the CURRENT device, cached per device id (relaxed atomics: every writer stores the
// same value, so concurrent first calls are benign)
int sm_count() {
    static std::atomic<int> cache[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = (dev >= 0 && dev < kMaxDevices) ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (sms <= 0) {
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
            cudaGetLastError();
            sms = 148;
        }
        if (dev >= 0 && dev < kMaxDevices) cache[dev].store(sms, std::memory_order_relaxed);
    }
    return sms;
}

// first tile pass straight from the rect codes: count, scan, expand + scatter
template <int DBITS, int MODE>
int launch_keys_pass(const ExpandSrc& src, u32* kout, u32* vout, const PassBufs& pb, const float* depths, u64* keys64,
                     cudaStream_t s) {
    constexpr size_t sm = sizeof(SortSmem<1 << DBITS>);
    if (cudaError_t e = cudaFuncSetAttribute(keys_scatter_kernel<DBITS, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))
        return cuda_fail(e, "keys_scatter smem attribute");
    const u32 T = (src.M + kSortTile - 1) / kSortTile;
    if (!T) return VKS_OK;
    launch_k(keys_count_kernel<DBITS>, T, kSortThreads, 0, s, src, 0, T, pb.counts);
    const u64 cnt = (u64)(1u << DBITS) * T;
    launch_k(scan_u32_kernel, (unsigned)((cnt + kCntTile - 1) / kCntTile), kScanThreads, 0, s, pb.counts, pb.offs, cnt,
                                                                                     pb.lb, pb.ctr);
    launch_k(keys_scatter_kernel<DBITS, MODE>, T, kSortThreads, sm, s, src, 0, T, pb.offs, kout, vout, depths, keys64);
    return check_launch(__func__);
}

template <int MODE>
int launch_keys_pass_bits(int dbits, const ExpandSrc& src, u32* kout, u32* vout, const PassBufs& pb,
                          const float* depths, u64* keys64, cudaStream_t s) {
    switch (dbits) {
        case 1: return launch_keys_pass<1, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 2: return launch_keys_pass<2, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 3: return launch_keys_pass<3, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 4: return launch_keys_pass<4, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 5: return launch_keys_pass<5, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 6: return launch_keys_pass<6, MODE>(src, kout, vout, pb, depths, keys64, s);
        case 7: return launch_keys_pass<7, MODE>(src, kout, vout, pb, depths, keys64, s);
        default: return launch_keys_pass<8, MODE>(src, kout, vout, pb, depths, keys64, s);
    }
}

int launch_rect_diff(int TX, int TY, u32 count, const u64* rc, int* diff, cudaStream_t s,
                     const u64* dcount = nullptr) {
    const int cells = (TX + 1) * (TY + 1);
    const u32 want = (count + kDiffThreads - 1) / kDiffThreads;
    if (want == 0) return VKS_OK;
    if (cells <= kDiffSmemMax) {
        const size_t sm = sizeof(int) * (size_t)cells;
        if (sm > 48 * 1024) {
            if (cudaError_t e = cudaFuncSetAttribute(rect_diff_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)(sizeof(int) * kDiffSmemMax)))
                return cuda_fail(e, "rect_diff smem attribute");
        }
        const unsigned blocks = std::min<u32>(want, (u32)sm_count() * 2);
        launch_k(rect_diff_kernel<true>, blocks, kDiffThreads, sm, s, TX, TY, count, rc, diff, dcount);
    } else {
        const unsigned blocks = std::min<u32>(want, (u32)sm_count() * 4);
        launch_k(rect_diff_kernel<false>, blocks, kDiffThreads, 0, s, TX, TY, count, rc, diff, dcount);
    }
    return check_launch(__func__);
}

int launch_tile_count(int TX, int TY, int* diff, u32* tile_offsets, u32* order, cudaStream_t s) {
    const size_t cells_bytes = sizeof(int) * (size_t)(TX + 1) * (TY + 1);
    if (cells_bytes <= kTileCountSmemMax) {
        if (cells_bytes > 48 * 1024) {
            if (cudaError_t e = cudaFuncSetAttribute(tile_count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)kTileCountSmemMax))
                return cuda_fail(e, "tile_count smem attribute");
        }
        launch_k(tile_count_kernel<true>, 1, 1024, cells_bytes, s, TX, TY, diff, tile_offsets, order);
    } else {
        launch_k(tile_count_kernel<false>, 1, 1024, 0, s, TX, TY, diff, tile_offsets, order);
    }
    return check_launch(__func__);
}

int launch_keys_debug(const vks_camera& cam, int64_t n, const int* tiles, const float* means2d, const int32_t* radii,
                      const float* depths, const u32* offsets, u32* vals, u64* keys64, cudaStream_t s) {
    const int64_t want = (n + kKeysThreads - 1) / kKeysThreads;
    if (want == 0) return VKS_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)sm_count() * 8);
    keys_debug_kernel<<<blocks, kKeysThreads, 0, s>>>(cam, n, tiles, reinterpret_cast<const float2*>(means2d),
                                                      reinterpret_cast<const int2*>(radii), depths, offsets, vals, keys64);
    return check_launch(__func__);
}

// reduce-then-scan of the tile counts (MODE 0: id order from tiles_touched; MODE 1: depth order
// from the sorted rect codes); totals[0] = sum (and, MODE 0, totals[1] = #visible)
template <int MODE>
int run_scan(const int* tiles, const u64* rc_in, u64 count, u32* part_sum, u32* part_vis, u32* out, u64* totals,
             CompactOut co, cudaStream_t s, const u64* dcount = nullptr) {
    const u32 P = (u32)((count + kScanTile - 1) / kScanTile);
    if (!P) return VKS_OK;
    launch_k(scan_reduce_kernel<MODE>, P, kDownThreads, 0, s, tiles, rc_in, count, part_sum, MODE == 0 ? part_vis : nullptr,
                                                       co, dcount);
    co.vis_prefix = part_vis;  // raw block visible counts; the down-sweep sums its predecessors'
    launch_k(scan_down_kernel<MODE>, P, kDownThreads, 0, s, tiles, rc_in, count, part_sum, out, co, totals, dcount);
    return check_launch(__func__);
}

// vks_bin_sort_async's last step: M and the status to the caller's device words; on overflow
// (M > capacity, or M >= 2^30) every tile list is emptied so a rasterizer launched behind it reads
// nothing past the capacity
__global__ void bin_sort_status_kernel(const u64* __restrict__ totals, int64_t capacity, int n_tiles,
                                       u32* __restrict__ tile_offsets, int64_t* __restrict__ num_isects,
                                       int32_t* __restrict__ status) {
    pdl_wait();
    const u64 M = totals[0];
    const int st = M >= (1ull << 30) ? VKS_ERR_UNSUPPORTED : ((int64_t)M > capacity ? VKS_ERR_CAPACITY : VKS_OK);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *num_isects = (int64_t)M;
        *status = st;
    }
    if (st != VKS_OK)
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles; t += gridDim.x * blockDim.x) tile_offsets[t] = 0u;
}

}  // namespace

size_t bin_sort_workspace_bytes(int64_t n, int64_t capacity, int32_t n_tiles) {
    // worst-case grid shape for the difference array: (TX+1)(TY+1) <= 2 n_tiles + 2
    Workspace w = carve(nullptr, n, capacity, n_tiles > 0 ? n_tiles : 1, 1);
    return w.bytes + 1024;
}

int run_bin_sort(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii,
                 const float* depths, const int32_t* tiles_touched, uint32_t* offsets,
                 int64_t capacity, uint64_t* keys, uint32_t* vals, uint64_t* keys_unsorted,
                 uint32_t* vals_unsorted, uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects,
                 void* workspace, size_t workspace_bytes, cudaStream_t s) {
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int32_t n_tiles = TX * TY;
    // rect codes hold 16-bit tile coordinates; the key expansion's exact float division needs
    // rect areas < 2^20 tiles
    if (TX > 65535 || TY > 65535 || (int64_t)TX * TY >= (1 << 20)) return VKS_ERR_INVALID_ARG;
    if (workspace_bytes < bin_sort_workspace_bytes(n, capacity, n_tiles)) return VKS_ERR_WORKSPACE;
    // the scatters bulk-copy (cp.async.bulk) from workspace arrays: 256-byte aligned base required
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return VKS_ERR_WORKSPACE;
    Workspace w = carve(workspace, n, capacity, TX, TY);
    if (cudaError_t e_ = cudaMemsetAsync(w.zeroA, 0, w.zeroA_bytes, s)) return cuda_fail(e_, "memset workspace");
    auto pass_bufs = [&](int p) { return PassBufs{w.counts, w.offs, w.cnt_lb[p], w.ctr + kCtrPass + p}; };
    // 1. index offsets in id order, M, V, rect codes, depth-bit range
    u64 tot[3] = {0, 0, 0};
    if (n > 0) {
        const CompactOut co{nullptr, reinterpret_cast<const u32*>(depths), reinterpret_cast<const float2*>(means2d),
                            reinterpret_cast<const int2*>(radii), TX, TY, w.dk[1], w.dv[1], w.rc_by_id,
                            reinterpret_cast<u32*>(w.totals + 2)};
        int st = run_scan<0>(tiles_touched, nullptr, (u64)n, w.part_sum, w.part_vis, offsets, w.totals, co, s);
        if (st) return st;
        if (cudaError_t e_ = cudaMemcpyAsync(tot, w.totals, sizeof(tot), cudaMemcpyDeviceToHost, s)) return cuda_fail(e_, "read M");
        if (cudaError_t e_ = cudaStreamSynchronize(s)) return cuda_fail(e_, "bin_sort sync");
    }
    const u64 M = tot[0], V = tot[1];
    *num_isects = (int64_t)M;
    // the look-back counters hold 30-bit counts: no capacity makes M >= 2^30 sortable, so that is
    // a hard limit (not a regrow request)
    if (M >= (1ull << 30)) return VKS_ERR_UNSUPPORTED;
    if ((int64_t)M > capacity) return VKS_ERR_CAPACITY;
    if (M == 0) {
        if (cudaMemsetAsync(tile_offsets, 0, sizeof(u32) * (n_tiles + 1), s) != cudaSuccess) return VKS_ERR_CUDA;
        if (tile_order) {  // every list is empty: identity schedule
            launch_k(iota_kernel, (n_tiles + 255) / 256, 256, 0, s, tile_order, (u32)n_tiles);
            if (int e_ = check_launch("tile_order")) return e_;
        }
        return VKS_OK;
    }
    u64* keys64 = reinterpret_cast<u64*>(keys);
    // debug: the pre-sort keys in id order, exactly as "Generate Keys" defines them
    if (keys_unsorted || vals_unsorted) {
        int st = launch_keys_debug(cam, n, tiles_touched, means2d, radii, depths, offsets, vals_unsorted,
                                   reinterpret_cast<u64*>(keys_unsorted), s);
        if (st) return st;
    }
    // 2. depth sort of the V visible Gaussians (compacted in id order into dk[1]/dv[1] by the scan)
    //    over the significant bits of (depth bits - min depth bits): digits of <= 8 bits, as few
    //    passes as the range needs (at least one)
    const u32 dmin = ~(u32)(tot[2] & 0xFFFFFFFFu), dmax = (u32)(tot[2] >> 32);
    const u32 range = V ? dmax - dmin : 0u;
    const int sig = range ? 32 - __builtin_clz(range) : 0;
    const int dpasses = std::max(1, (sig + 7) / 8);
    const int dbits = std::max(1, (sig + dpasses - 1) / dpasses);
    int st = VKS_OK;
    for (int p = 0; p < dpasses; p++) {
        const u32* ki = w.dk[(p + 1) & 1];
        const u32* vi = w.dv[(p + 1) & 1];
        st = launch_pass_bits<kPassPlain>(dbits, ki, vi, w.dk[p & 1], w.dv[p & 1], (u32)V, dbits * p, dmin,
                                          pass_bufs(p), nullptr, nullptr, s);
        if (st) return st;
    }
    const u32* sid = w.dv[(dpasses - 1) & 1];  // visible ids in (depth, id) order
    // 3. slots in depth order (from the depth-ordered rect codes) + the first Gaussian of every
    //    4096-slot key block
    {
        CompactOut co{};
        co.rc_by_id = w.rc_by_id;
        co.sid = sid;
        co.rc_out = w.rcs;
        co.first = w.first;
        if ((st = run_scan<1>(nullptr, w.rcs, V, w.part_sum, nullptr, w.doff, w.totals + 0, co, s))) return st;
    }
    // 4. tile ranges from the 2-D difference array of the rects
    if ((st = launch_rect_diff(TX, TY, (u32)V, w.rcs, w.diff, s))) return st;
    if ((st = launch_tile_count(TX, TY, w.diff, tile_offsets, tile_order, s))) return st;
    // 5. stable tile passes over the M (tile, id) pairs; the first expands the keys from the rect
    //    codes itself, the last writes the caller's vals (+ u64 keys on request)
    const ExpandSrc src{w.rcs, w.doff, sid, w.first, (u32)V, (u32)M, TX};
    TilePlan plan = tile_plan(n_tiles);
    if (plan.passes == 0) plan = TilePlan{1, 1};  // one tile: a trivial 1-bit pass keeps the path uniform
    if (plan.passes == 1)
        return launch_keys_pass_bits<kPassTileLast>(plan.dbits, src, nullptr, vals, pass_bufs(kDepthPasses), depths,
                                                    keys64, s);
    st = launch_keys_pass_bits<kPassPlain>(plan.dbits, src, w.tk[0], w.tv[0], pass_bufs(kDepthPasses), nullptr, nullptr,
                                           s);
    if (st) return st;
    for (int p = 1; p < plan.passes; p++) {
        const u32* kin = w.tk[(p - 1) & 1];
        const u32* vin = w.tv[(p - 1) & 1];
        const bool last = p == plan.passes - 1;
        u32* ko = w.tk[p & 1];
        u32* vo = last ? vals : w.tv[p & 1];
        st = last ? launch_pass_bits<kPassTileLast>(plan.dbits, kin, vin, ko, vo, (u32)M, plan.dbits * p, 0u,
                                                    pass_bufs(kDepthPasses + p), depths, keys64, s)
                  : launch_pass_bits<kPassPlain>(plan.dbits, kin, vin, ko, vo, (u32)M, plan.dbits * p, 0u,
                                                 pass_bufs(kDepthPasses + p), nullptr, nullptr, s);
        if (st) return st;
    }
    return VKS_OK;
}

// Stream-ordered, host-sync-free variant (include/vks.h vks_bin_sort_async): every launch is sized
// from host-side bounds (n visible Gaussians at most, `capacity` keys at most) and the kernels read
// the actual V and M from the device totals, blocks past them leaving at once; the depth sort runs
// four 8-bit passes over all 32 depth bits (no host-read depth range: the same stable order), the
// key-pass grid covers the capacity.  M and a status word are written to device memory.  The
// launch sequence depends only on (n, capacity, tile grid), so a step built on it can be captured
// in a CUDA graph.
int run_bin_sort_async(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const int32_t* tiles_touched, uint32_t* offsets, int64_t capacity,
                       uint32_t* vals, uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects,
                       int32_t* status, void* workspace, size_t workspace_bytes, cudaStream_t s) {
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int32_t n_tiles = TX * TY;
    if (TX > 65535 || TY > 65535 || (int64_t)TX * TY >= (1 << 20)) return VKS_ERR_INVALID_ARG;
    if (workspace_bytes < bin_sort_workspace_bytes(n, capacity, n_tiles)) return VKS_ERR_WORKSPACE;
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return VKS_ERR_WORKSPACE;
    if (capacity >= (1ll << 30)) return VKS_ERR_UNSUPPORTED;  // the look-back counts hold 30 bits
    Workspace w = carve(workspace, n, capacity, TX, TY);
    if (cudaError_t e_ = cudaMemsetAsync(w.zeroA, 0, w.zeroA_bytes, s)) return cuda_fail(e_, "memset workspace");
    auto pass_bufs = [&](int p) { return PassBufs{w.counts, w.offs, w.cnt_lb[p], w.ctr + kCtrPass + p}; };
    const u64* dM = w.totals + 0;
    const u64* dV = w.totals + 1;
    int st = VKS_OK;
    if (n > 0) {
        // 1. index offsets in id order, M, V, rect codes (totals on the device only)
        const CompactOut co{nullptr, reinterpret_cast<const u32*>(depths), reinterpret_cast<const float2*>(means2d),
                            reinterpret_cast<const int2*>(radii), TX, TY, w.dk[1], w.dv[1], w.rc_by_id,
                            reinterpret_cast<u32*>(w.totals + 2)};
        if ((st = run_scan<0>(tiles_touched, nullptr, (u64)n, w.part_sum, w.part_vis, offsets, w.totals, co, s)))
            return st;
        // 2. depth sort of the V visible: four 8-bit passes over all 32 depth bits
        for (int p = 0; p < kDepthPasses; p++) {
            st = launch_pass_bits<kPassPlain>(8, w.dk[(p + 1) & 1], w.dv[(p + 1) & 1], w.dk[p & 1], w.dv[p & 1], (u32)n,
                                              8 * p, 0u, pass_bufs(p), nullptr, nullptr, s, dV);
            if (st) return st;
        }
        const u32* sid = w.dv[(kDepthPasses - 1) & 1];
        // 3. slots in depth order + first[]
        {
            CompactOut co1{};
            co1.rc_by_id = w.rc_by_id;
            co1.sid = sid;
            co1.rc_out = w.rcs;
            co1.first = w.first;
            if ((st = run_scan<1>(nullptr, w.rcs, (u64)n, w.part_sum, nullptr, w.doff, w.totals + 0, co1, s, dV)))
                return st;
        }
        // 4. tile ranges
        if ((st = launch_rect_diff(TX, TY, (u32)n, w.rcs, w.diff, s, dV))) return st;
        if ((st = launch_tile_count(TX, TY, w.diff, tile_offsets, tile_order, s))) return st;
        // 5. tile passes over min(M, capacity) keys (grids sized for the capacity)
        if (capacity > 0) {
            ExpandSrc src{w.rcs, w.doff, sid, w.first, (u32)n, (u32)capacity, TX, w.totals};
            TilePlan plan = tile_plan(n_tiles);
            if (plan.passes == 0) plan = TilePlan{1, 1};
            if (plan.passes == 1) {
                st = launch_keys_pass_bits<kPassTileLast>(plan.dbits, src, nullptr, vals, pass_bufs(kDepthPasses),
                                                          depths, nullptr, s);
            } else {
                st = launch_keys_pass_bits<kPassPlain>(plan.dbits, src, w.tk[0], w.tv[0], pass_bufs(kDepthPasses),
                                                       nullptr, nullptr, s);
                for (int p = 1; !st && p < plan.passes; p++) {
                    const bool last = p == plan.passes - 1;
                    st = last ? launch_pass_bits<kPassTileLast>(plan.dbits, w.tk[(p - 1) & 1], w.tv[(p - 1) & 1],
                                                                w.tk[p & 1], vals, (u32)capacity, plan.dbits * p, 0u,
                                                                pass_bufs(kDepthPasses + p), depths, nullptr, s, dM)
                              : launch_pass_bits<kPassPlain>(plan.dbits, w.tk[(p - 1) & 1], w.tv[(p - 1) & 1],
                                                             w.tk[p & 1], w.tv[p & 1], (u32)capacity, plan.dbits * p,
                                                             0u, pass_bufs(kDepthPasses + p), nullptr, nullptr, s, dM);
                }
            }
            if (st) return st;
        }
    } else {
        if ((st = launch_tile_count(TX, TY, w.diff, tile_offsets, tile_order, s))) return st;  // empty lists
    }
    launch_k(bin_sort_status_kernel, (n_tiles + 1 + 1023) / 1024, 1024, 0, s, w.totals, capacity, n_tiles, tile_offsets,
                                                                        num_isects, status);
    return check_launch("bin_sort_status");
}

}  // namespace vks
