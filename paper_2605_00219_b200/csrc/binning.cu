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
//  1. scan (id order)    reduce-then-scan of tiles_touched -> offsets, M, V.
//  2. radix pass x4       8-bit LSD passes over (depth key, id) of all N Gaussians (culled ones
//                         take the key 0xFFFFFFFF and sort last); pass 0 derives the keys from
//                         tiles_touched / depths on the fly.
//  3. scan (depth order) reduce-then-scan of the tile counts of the depth-ordered rect codes
//                         (the last depth pass gathers each visible Gaussian's rect once and lays it
//                         out as a 64-bit code, 4 x u16) -> slot of each Gaussian's first key.
//  4. keys_kernel         warp-cooperative expansion of the rect codes in depth order into
//                         (tile, id) pairs with coalesced stores; 2-D difference array of the
//                         rects accumulated per block in shared memory.
//  5. tile_count_kernel   2-D prefix of the difference array -> per-tile list lengths -> CSR
//                         tile_offsets.
//  6. radix pass x1-3     stable LSD passes over the tile bits (<= 8 bits each) of the M pairs;
//                         the last one writes the ids (and, on request, the u64 keys).
// Every radix pass is reduce-then-scan: digit counts per 4096-key block, one exclusive scan of
// the (digit-major) count matrix, then a scatter kernel (TMA bulk copy of the block into shared
// memory, warp-level ballot multi-split ranking, in-place reorder, digit-contiguous stores).  No block
// ever waits on another (a single-pass decoupled look-back over 256 digits walked hundreds of
// in-flight blocks back on this workload).
// The TU is compiled with -fmad=false (the tile-rect recomputation must equal projection's).
#include <stdlib.h>

#include <algorithm>

#include "vks_common.cuh"

namespace vks {
namespace {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per block
constexpr int kDepthPasses = 4;
constexpr int kMaxTilePasses = 3;
constexpr int kLookbackChunk = 8;

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
    u32* part_sum;       // [scan blocks] block sums of the 1-D scans
    u32* part_vis;       // [scan blocks] visible counts
    // region A (zeroed before the scan)
    u64* cnt_lb[kPasses];  // look-back of each pass's counts scan
    u32* ctr;            // [16] scan tile counters
    u64* totals;         // [2]: M, V
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
    const size_t cnt_scan_tiles = (256 * sort_tiles + kScanTile - 1) / kScanTile;
    for (int i = 0; i < 2; i++) {
        w.dk[i] = reinterpret_cast<u32*>(take(4 * nn));
        w.dv[i] = reinterpret_cast<u32*>(take(4 * nn));
    }
    w.doff = reinterpret_cast<u32*>(take(4 * nn));
    for (int i = 0; i < 2; i++) {
        w.tk[i] = reinterpret_cast<u32*>(take(4 * cap));
        w.tv[i] = reinterpret_cast<u32*>(take(4 * cap));
    }
    w.counts = reinterpret_cast<u32*>(take(4 * 256 * sort_tiles));
    w.offs = reinterpret_cast<u32*>(take(4 * 256 * sort_tiles));
    w.rcs = reinterpret_cast<u64*>(take(8 * nn));
    w.part_sum = reinterpret_cast<u32*>(take(4 * scan_tiles));
    w.part_vis = reinterpret_cast<u32*>(take(4 * scan_tiles));
    const size_t a0 = off;
    w.zeroA = b ? b + off : nullptr;
    for (int p = 0; p < kPasses; p++) w.cnt_lb[p] = reinterpret_cast<u64*>(take(8 * cnt_scan_tiles));
    w.ctr = reinterpret_cast<u32*>(take(4 * 16));
    w.totals = reinterpret_cast<u64*>(take(8 * 2));
    w.diff = reinterpret_cast<int*>(take(4 * (size_t)(TX + 1) * (TY + 1)));
    w.zeroA_bytes = off - a0;
    w.bytes = off;
    return w;
}

// counter slots in w.ctr
enum { kCtrPass = 0 };  // kCtrPass + p: counts scan of pass p

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
//   scan_partials_kernel one block: exclusive scan of the block sums, totals
//   scan_down_kernel     per block: rescan + block prefix -> output
// MODE 0: element i = tiles_touched[i];  MODE 1: element r = tiles of the depth-sorted rect code r.
template <int MODE>
__device__ __forceinline__ void load_scan_items(const int* __restrict__ tiles, const u64* __restrict__ rc, u64 count,
                                                u64 base, int v[kScanItems]) {
    if (MODE == 0) {
        if (base + kScanItems <= count && ((reinterpret_cast<uintptr_t>(tiles + base) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < kScanItems; j += 4) {
                const int4 q = __ldg(reinterpret_cast<const int4*>(tiles + base + j));
                v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kScanItems; j++) v[j] = base + j < count ? __ldg(tiles + base + j) : 0;
        }
#pragma unroll
        for (int j = 0; j < kScanItems; j++) v[j] = v[j] > 0 ? v[j] : 0;
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; j++) v[j] = base + j < count ? rect_tiles(__ldg(rc + base + j)) : 0;
    }
}

template <int MODE>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(vks_camera cam, const int* __restrict__ tiles,
                                                                  const float2* __restrict__ means2d,
                                                                  const int2* __restrict__ radii,
                                                                  const u64* __restrict__ rc_in, u64* __restrict__ rc_out,
                                                                  u64 count, u32* __restrict__ part_sum,
                                                                  u32* __restrict__ part_vis) {
    __shared__ u32 s_sum[kScanThreads / 32], s_vis[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u64 base = (u64)blockIdx.x * kScanTile + (u64)tid * kScanItems;
    int v[kScanItems];
    load_scan_items<MODE>(tiles, rc_in, count, base, v);
    u32 sum = 0, vis = 0;
    (void)cam; (void)means2d; (void)radii; (void)rc_out;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
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
        for (int w = 0; w < kScanThreads / 32; w++) { a += s_sum[w]; b += s_vis[w]; }
        part_sum[blockIdx.x] = a;
        if (part_vis) part_vis[blockIdx.x] = b;
    }
}

// exclusive scan of the P block sums in place; totals[0] = sum, totals[1] = sum of part_vis
__global__ void __launch_bounds__(1024) scan_partials_kernel(u32* __restrict__ part_sum, const u32* __restrict__ part_vis,
                                                            u32 P, u64* __restrict__ totals) {
    __shared__ u32 s_w[32];
    __shared__ u64 s_carry;
    __shared__ u64 s_vis;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { s_carry = 0; s_vis = 0; }
    __syncthreads();
    u64 vis_acc = 0;
    for (u32 base = 0; base < P; base += 1024) {
        const u32 i = base + tid;
        const u32 c = i < P ? part_sum[i] : 0u;
        if (i < P && part_vis) vis_acc += part_vis[i];
        u32 incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        u32 wpre = 0, btot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wpre += s_w[w];
            btot += s_w[w];
        }
        const u64 carry = s_carry;
        if (i < P) part_sum[i] = (u32)(carry + wpre + incl - c);
        __syncthreads();
        if (tid == 0) s_carry = carry + btot;
        __syncthreads();
    }
    vis_acc = __reduce_add_sync(VKS_FULL_MASK, (u32)vis_acc);
    if (lane == 0 && vis_acc) atomicAdd(reinterpret_cast<unsigned long long*>(&s_vis), (unsigned long long)vis_acc);
    __syncthreads();
    if (tid == 0) {
        totals[0] = s_carry;
        if (part_vis) totals[1] = s_vis;
    }
}

template <int MODE>
__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const int* __restrict__ tiles, const u64* __restrict__ rc,
                                                                u64 count, const u32* __restrict__ part_prefix,
                                                                u32* __restrict__ out) {
    __shared__ u32 s_w[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u64 base = (u64)blockIdx.x * kScanTile + (u64)tid * kScanItems;
    int v[kScanItems];
    load_scan_items<MODE>(tiles, rc, count, base, v);
    u32 tsum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) tsum += (u32)v[j];
    u32 incl = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    u32 wpre = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; w++)
        if (w < warp) wpre += s_w[w];
    u32 run = part_prefix[blockIdx.x] + wpre + incl - tsum;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < count) out[base + j] = run;
        run += (u32)v[j];
    }
}

// ------------------------------------------------------------------------------------------
// 4. key generation (+ tile-rect difference array)
constexpr int kKeysThreads = 512;
constexpr int kKeysWarps = kKeysThreads / 32;
constexpr int kKeysSmemDiffMax = 160 * 1024 / 4;  // cells

// MODE 0: depth order: element r = Gaussian sid[r] with rect code rc[r] -> (tile, id) pairs at
//         slot0[r] + k, plus the difference array of the rects.
// MODE 1: id order (debug keys_unsorted / vals_unsorted): rect of Gaussian i -> u64 keys at slot0[i] + k.
template <bool SMEM_DIFF, int MODE>
__global__ void __launch_bounds__(kKeysThreads) keys_kernel(vks_camera cam, int64_t count, const u32* __restrict__ sid,
                                                           const u64* __restrict__ rc, const int* __restrict__ tiles,
                                                           const float2* __restrict__ means2d,
                                                           const int2* __restrict__ radii, const float* __restrict__ depths,
                                                           const u32* __restrict__ slot0, u32* __restrict__ tkeys,
                                                           u32* __restrict__ tvals, u64* __restrict__ keys64,
                                                           int* __restrict__ diff) {
    extern __shared__ int s_diff[];
    __shared__ int s_incl[kKeysWarps][32];
    __shared__ int s_x0[kKeysWarps][32], s_y0[kKeysWarps][32], s_w[kKeysWarps][32];
    __shared__ u32 s_id[kKeysWarps][32];
    __shared__ u32 s_db[kKeysWarps][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int W1 = TX + 1;
    const int cells = W1 * (TY + 1);
    if (SMEM_DIFF) {
        for (int j = tid; j < cells; j += kKeysThreads) s_diff[j] = 0;
        __syncthreads();
    }
    int* dd = SMEM_DIFF ? s_diff : diff;
    const int64_t stride = (int64_t)gridDim.x * kKeysWarps * 32;
    for (int64_t r0 = ((int64_t)blockIdx.x * kKeysWarps + warp) * 32; r0 < count; r0 += stride) {
        const int64_t r = r0 + lane;
        int cnt = 0, x0 = 0, y0 = 0, w = 1;
        u32 g = 0, db = 0;
        if (r < count) {
            g = MODE == 0 ? __ldg(sid + r) : (u32)r;
            int x1, y1;
            if (MODE == 0) {
                unpack_rect(__ldg(rc + r), x0, x1, y0, y1);
            } else if (__ldg(tiles + r) > 0) {
                rect_of(__ldg(means2d + r), __ldg(radii + r), TX, TY, x0, x1, y0, y1);
            } else {
                x0 = x1 = y0 = y1 = 0;
            }
            w = x1 - x0;
            cnt = w * (y1 - y0);
            if (cnt > 0) {
                if (MODE == 0) {
                    atomicAdd(dd + y0 * W1 + x0, 1);
                    atomicAdd(dd + y0 * W1 + x1, -1);
                    atomicAdd(dd + y1 * W1 + x0, -1);
                    atomicAdd(dd + y1 * W1 + x1, 1);
                } else {
                    db = __float_as_uint(__ldg(depths + g));
                }
            } else {
                w = 1;
            }
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
        s_id[warp][lane] = g;
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
            if (MODE == 0) tkeys[base + e] = t;
            else keys64[base + e] = ((u64)t << 32) | (u64)s_db[warp][pos];
            tvals[base + e] = s_id[warp][pos];
        }
    }
    if (SMEM_DIFF) {
        __syncthreads();
        for (int j = tid; j < cells; j += kKeysThreads) {
            const int v = s_diff[j];
            if (v) atomicAdd(diff + j, v);
        }
    }
}

// ------------------------------------------------------------------------------------------
// 5. per-tile counts -> CSR tile_offsets
__global__ void __launch_bounds__(1024) tile_count_kernel(int TX, int TY, int* __restrict__ diff,
                                                         u32* __restrict__ tile_offsets) {
    __shared__ u32 s_wsum[32];
    __shared__ u32 s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W1 = TX + 1;
    for (int y = tid; y < TY; y += 1024) {
        int acc = 0;
        for (int x = 0; x < TX; x++) { acc += diff[y * W1 + x]; diff[y * W1 + x] = acc; }
    }
    __syncthreads();
    for (int x = tid; x < TX; x += 1024) {
        int acc = 0;
        for (int y = 0; y < TY; y++) { acc += diff[y * W1 + x]; diff[y * W1 + x] = acc; }
    }
    __syncthreads();
    const int n_tiles = TX * TY;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n_tiles; base += 1024) {
        const int t = base + tid;
        const u32 c = t < n_tiles ? (u32)diff[(t / TX) * W1 + (t % TX)] : 0u;
        u32 incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            u32 v = __shfl_up_sync(VKS_FULL_MASK, incl, d);
            if (lane >= d) incl += v;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        u32 wpre = 0, btot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wpre += s_wsum[w];
            btot += s_wsum[w];
        }
        const u32 carry = s_carry;
        if (t < n_tiles) tile_offsets[t] = carry + wpre + incl - c;
        __syncthreads();
        if (tid == 0) s_carry = carry + btot;
        __syncthreads();
    }
    if (tid == 0) tile_offsets[n_tiles] = s_carry;
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
enum { kPassPlain = 0, kPassDepthFirst = 1, kPassTileLast = 2, kPassDepthLast = 3 };

// key of element j of the depth-first pass: visible ? f32bits(depth) : 0xFFFFFFFF (sorts last)
__device__ __forceinline__ u32 depth_key(int tiles, u32 depth_bits) { return tiles > 0 ? depth_bits : 0xFFFFFFFFu; }

// lanes of the warp holding the same DBITS-bit digit (and the same `valid`): DBITS ballots
// instead of __match_any_sync, whose cost grows with the number of distinct values
template <int DBITS>
__device__ __forceinline__ u32 digit_peers(u32 d, bool valid = true) {
    u32 peers = __ballot_sync(VKS_FULL_MASK, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < DBITS; b++) {
        const bool bit = (d >> b) & 1u;
        const u32 bal = __ballot_sync(VKS_FULL_MASK, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

template <int DBITS, int MODE, bool ATOMIC>
__global__ void __launch_bounds__(kSortThreads) digit_count_kernel(const u32* __restrict__ kin, const u32* __restrict__ vin,
                                                                  u32 n, int shift, u32 T, u32* __restrict__ counts) {
    constexpr int RADIX = 1 << DBITS;
    constexpr u32 DMASK = RADIX - 1;
    __shared__ u32 whist[kSortWarps][RADIX];
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int j = tid; j < kSortWarps * RADIX; j += kSortThreads) (&whist[0][0])[j] = 0;
    __syncthreads();
    const u64 base = (u64)blockIdx.x * kSortTile;
    const u32 ltmask = lanemask_lt();
    u32 key[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {  // all loads in flight before any use
        const u64 idx = base + (u64)i * kSortThreads + tid;
        key[i] = 0;
        if (idx < n)
            key[i] = MODE == kPassDepthFirst ? depth_key((int)__ldg(kin + idx), __ldg(vin + idx)) : __ldg(kin + idx);
    }
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        const bool valid = base + (u64)i * kSortThreads + tid < n;
        const u32 d = (key[i] >> shift) & DMASK;
        if (ATOMIC) {  // per-warp histograms: contention only among a warp's lanes
            if (valid) atomicAdd(&whist[warp][d], 1u);
        } else {
            const u32 peers = digit_peers<DBITS>(d, valid);
            if (valid && (peers & ltmask) == 0) whist[warp][d] += __popc(peers);
        }
    }
    __syncthreads();
    for (int d = tid; d < RADIX; d += kSortThreads) {
        u32 c = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) c += whist[w][d];
        counts[(u64)d * T + blockIdx.x] = c;
    }
}

// exclusive scan of a u32 array (decoupled look-back over 4096-element tiles)
__global__ void __launch_bounds__(kScanThreads) scan_u32_kernel(const u32* __restrict__ in, u32* __restrict__ out,
                                                               u64 count, u64* __restrict__ lb, u32* __restrict__ ctr) {
    __shared__ u32 s_tile;
    __shared__ u64 s_warp[kScanThreads / 32];
    __shared__ u64 s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    const u64 base = tile * kScanTile + (u64)tid * kScanItems;
    u32 v[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; j++) v[j] = base + j < count ? __ldg(in + base + j) : 0u;
    u64 tsum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) tsum += v[j];
    u64 incl = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u64 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    u64 wpre = 0, btotal = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; w++) {
        if (w < warp) wpre += s_warp[w];
        btotal += s_warp[w];
    }
    if (tid == 0) {
        u64 excl = 0;
        if (tile == 0) {
            st_volatile_u64(reinterpret_cast<unsigned long long*>(lb), kScanFlagInc | btotal);
        } else {
            st_volatile_u64(reinterpret_cast<unsigned long long*>(lb + tile), kScanFlagAgg | btotal);
            int64_t j = (int64_t)tile - 1;
            bool found = false;
            while (!found) {
                u64 st[kLookbackChunk];
#pragma unroll
                for (int q = 0; q < kLookbackChunk; q++)
                    st[q] = (j - q >= 0) ? ld_volatile_u64(reinterpret_cast<const unsigned long long*>(lb + j - q)) : 0;
                int consumed = 0;
#pragma unroll
                for (int q = 0; q < kLookbackChunk; q++) {
                    if (found || consumed < q) break;
                    const u64 f = st[q] & ~kScanMask;
                    if (f == 0) break;
                    excl += st[q] & kScanMask;
                    consumed = q + 1;
                    if (f == kScanFlagInc) found = true;
                }
                j -= consumed;
            }
            st_volatile_u64(reinterpret_cast<unsigned long long*>(lb + tile), kScanFlagInc | (excl + btotal));
        }
        s_prefix = excl;
    }
    __syncthreads();
    u64 run = s_prefix + wpre + (incl - tsum);
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < count) out[base + j] = (u32)run;
        run += v[j];
    }
}

struct RectSrc {  // kPassDepthLast: where the tile rects come from
    const float2* means2d;
    const int2* radii;
    int TX, TY;
    u32 visible;   // the first `visible` sorted entries are the visible Gaussians
};

struct SortSmem {
    alignas(128) u32 keys[kSortTile];  // input staging (bulk copy), then the reordered tile
    alignas(128) u32 vals[kSortTile];
    u32 whist[kSortWarps][256];
    u32 binstart[256];
    u32 gbase[256];
    u32 wsum[kSortWarps];
    alignas(8) unsigned long long mbar;
};

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

// kPassDepthFirst: kin = tiles_touched, vin = depths; key = depth_key(), value = id.
// kPassTileLast: writes only the values (the caller's vals) and, if keys64, the u64 keys.
// kPassDepthLast: also writes the rect codes in the sorted order (gathered by id).
template <int DBITS, int MODE>
__global__ void __launch_bounds__(kSortThreads) scatter_kernel(const u32* __restrict__ kin, const u32* __restrict__ vin,
                                                             u32* __restrict__ kout, u32* __restrict__ vout, u32 n,
                                                             int shift, u32 T, const u32* __restrict__ offs,
                                                             const float* __restrict__ depths,
                                                             u64* __restrict__ keys64, RectSrc rsrc,
                                                             u64* __restrict__ rc_out) {
    constexpr int RADIX = 1 << DBITS;
    constexpr u32 DMASK = RADIX - 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 bar = smem_u32(&S.mbar);
    const u32 tile = blockIdx.x;
    const u64 base = (u64)tile * kSortTile;
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
    for (int j = tid; j < kSortWarps * 256; j += kSortThreads) (&S.whist[0][0])[j] = 0;
    // the block's digit starts: global start of (digit, tile) from the scanned counts
    for (int d = tid; d < RADIX; d += kSortThreads) S.gbase[d] = __ldg(offs + (u64)d * T + tile);
    for (u32 j = nbulk + tid; j < (u32)kSortTile; j += kSortThreads) {
        const bool ok = j < count;
        S.keys[j] = ok ? kin[base + j] : (MODE == kPassDepthFirst ? 0u : 0xFFFFFFFFu);  // pads rank last
        S.vals[j] = ok ? vin[base + j] : 0u;
    }
    __syncthreads();  // barrier init visible before anyone waits on it
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT%=;\n\t}" ::"r"(bar) : "memory");
    if (MODE == kPassDepthFirst) {
        __syncthreads();
        for (int j = tid; j < kSortTile; j += kSortThreads) {
            S.keys[j] = depth_key((int)S.keys[j], S.vals[j]);  // pads (tiles = 0) become ~0 too
            S.vals[j] = (u32)(base + j);
        }
    }
    __syncthreads();
    u32 rank[kSortItems];
    const u32 ltmask = lanemask_lt();
    const int seg = warp * 32 * kSortItems;
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        const u32 d = (S.keys[seg + i * 32 + lane] >> shift) & DMASK;
        const u32 peers = digit_peers<DBITS>(d);
        const u32 below = __popc(peers & ltmask);
        const u32 before = S.whist[warp][d];
        rank[i] = before + below;
        __syncwarp();
        if (below == 0) S.whist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    u32 total = 0;
    if (tid < RADIX) {
#pragma unroll
        for (int w = 0; w < kSortWarps; w++) {
            const u32 c = S.whist[w][tid];
            S.whist[w][tid] = total;
            total += c;
        }
    }
    u32 incl = total;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    if (tid < RADIX) {
        u32 wpre = 0;
        for (int w = 0; w < warp; w++) wpre += S.wsum[w];
        const u32 binstart = wpre + incl - total;
        S.binstart[tid] = binstart;
        S.gbase[tid] -= binstart;
    }
    __syncthreads();
    u32 kk[kSortItems], vv[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; i++) {
        const int slot = seg + i * 32 + lane;
        kk[i] = S.keys[slot];
        vv[i] = S.vals[slot];
        const u32 d = (kk[i] >> shift) & DMASK;
        rank[i] += S.binstart[d] + S.whist[warp][d];
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
        const u32 dest = S.gbase[(key >> shift) & DMASK] + (u32)j;
        if (dest < n) {
            const u32 val = S.vals[j];
            if (MODE != kPassTileLast) kout[dest] = key;
            vout[dest] = val;
            if (MODE == kPassTileLast && keys64)
                keys64[dest] = ((u64)key << 32) | (u64)__float_as_uint(__ldg(depths + val));
            if (MODE == kPassDepthLast) {  // rect code in depth order
                u64 code = 0;
                if (dest < rsrc.visible) {
                    int x0, x1, y0, y1;
                    rect_of(__ldg(rsrc.means2d + val), __ldg(rsrc.radii + val), rsrc.TX, rsrc.TY, x0, x1, y0, y1);
                    code = pack_rect(x0, x1, y0, y1);
                }
                rc_out[dest] = code;
            }
        }
    }
}

struct PassBufs {
    u32* counts;  // [256 * T]
    u32* offs;    // [256 * T]
    u64* lb;      // scan look-back of the counts
    u32* ctr;     // scan tile counter (zeroed)
};

template <int DBITS, int MODE>
int launch_pass(const u32* kin, const u32* vin, u32* kout, u32* vout, u32 n, int shift, const PassBufs& pb,
                const float* depths, u64* keys64, cudaStream_t s, RectSrc rsrc = RectSrc{}, u64* rc_out = nullptr) {
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(scatter_kernel<DBITS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(SortSmem)) != cudaSuccess)
            return VKS_ERR_CUDA;
        attr = true;
    }
    const u32 T = (u32)((n + kSortTile - 1) / kSortTile);
    if (!T) return VKS_OK;
    static const bool atomic_count = !getenv("VKS_COUNT_BALLOT");
    if (atomic_count) digit_count_kernel<DBITS, MODE, true><<<T, kSortThreads, 0, s>>>(kin, vin, n, shift, T, pb.counts);
    else digit_count_kernel<DBITS, MODE, false><<<T, kSortThreads, 0, s>>>(kin, vin, n, shift, T, pb.counts);
    const u64 cnt = (u64)(1u << DBITS) * T;
    scan_u32_kernel<<<(unsigned)((cnt + kScanTile - 1) / kScanTile), kScanThreads, 0, s>>>(pb.counts, pb.offs, cnt,
                                                                                           pb.lb, pb.ctr);
    scatter_kernel<DBITS, MODE><<<T, kSortThreads, sizeof(SortSmem), s>>>(kin, vin, kout, vout, n, shift, T, pb.offs,
                                                                         depths, keys64, rsrc, rc_out);
    return check_launch(__func__);
}

template <int MODE>
int launch_tile_pass(int dbits, const u32* kin, const u32* vin, u32* kout, u32* vout, u32 n, int shift,
                     const PassBufs& pb, const float* depths, u64* keys64, cudaStream_t s) {
    switch (dbits) {
        case 1: return launch_pass<1, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 2: return launch_pass<2, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 3: return launch_pass<3, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 4: return launch_pass<4, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 5: return launch_pass<5, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 6: return launch_pass<6, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        case 7: return launch_pass<7, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
        default: return launch_pass<8, MODE>(kin, vin, kout, vout, n, shift, pb, depths, keys64, s);
    }
}

// Single-tile grid: the depth order is the final order; u64 keys = (0 << 32) | depth bits.
__global__ void keys64_tile0_kernel(const u32* __restrict__ vals, const float* __restrict__ depths, u64* __restrict__ keys,
                                    u32 m) {
    const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) keys[i] = (u64)__float_as_uint(__ldg(depths + vals[i]));
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int MODE>
int launch_keys(const vks_camera& cam, int64_t count, const u32* sid, const u64* rc, const int* tiles,
                const float* means2d, const int32_t* radii, const float* depths, const u32* slot0, u32* tkeys,
                u32* tvals, u64* keys64, int* diff, cudaStream_t s) {
    const float2* m2 = reinterpret_cast<const float2*>(means2d);
    const int2* r2 = reinterpret_cast<const int2*>(radii);
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int cells = (TX + 1) * (TY + 1);
    const int64_t want = (count + kKeysThreads - 1) / kKeysThreads;
    if (want == 0) return VKS_OK;
    if (MODE == 0 && cells <= kKeysSmemDiffMax) {
        const size_t sm = sizeof(int) * (size_t)cells;
        if (sm > 32 * 1024 &&
            cudaFuncSetAttribute(keys_kernel<true, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
            return VKS_ERR_CUDA;
        const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)sm_count() * 2);
        keys_kernel<true, MODE><<<blocks, kKeysThreads, sm, s>>>(cam, count, sid, rc, tiles, m2, r2, depths, slot0,
                                                                 tkeys, tvals, keys64, diff);
    } else {
        const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)sm_count() * 4);
        keys_kernel<false, MODE><<<blocks, kKeysThreads, 0, s>>>(cam, count, sid, rc, tiles, m2, r2, depths, slot0,
                                                                 tkeys, tvals, keys64, diff);
    }
    return check_launch(__func__);
}

// reduce-then-scan of the tiles counts (MODE 0: id order from tiles_touched, writes rect codes;
// MODE 1: depth order from the sorted rect codes); totals[0] = sum (and totals[1] = #visible)
template <int MODE>
int run_scan(const vks_camera& cam, const int* tiles, const float* means2d, const int32_t* radii, const u64* rc_in,
             u64* rc_out, u64 count, u32* part_sum, u32* part_vis, u32* out, u64* totals, cudaStream_t s) {
    const u32 P = (u32)((count + kScanTile - 1) / kScanTile);
    if (!P) return VKS_OK;
    scan_reduce_kernel<MODE><<<P, kScanThreads, 0, s>>>(cam, tiles, reinterpret_cast<const float2*>(means2d),
                                                       reinterpret_cast<const int2*>(radii), rc_in, rc_out, count,
                                                       part_sum, part_vis);
    scan_partials_kernel<<<1, 1024, 0, s>>>(part_sum, MODE == 0 ? part_vis : nullptr, P, totals);
    scan_down_kernel<MODE><<<P, kScanThreads, 0, s>>>(tiles, rc_in, count, part_sum, out);
    return check_launch(__func__);
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
                 uint32_t* vals_unsorted, uint32_t* tile_offsets, int64_t* num_isects,
                 void* workspace, size_t workspace_bytes, cudaStream_t s) {
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int32_t n_tiles = TX * TY;
    if (workspace_bytes < bin_sort_workspace_bytes(n, capacity, n_tiles)) return VKS_ERR_WORKSPACE;
    Workspace w = carve(workspace, n, capacity, TX, TY);
    if (cudaError_t e_ = cudaMemsetAsync(w.zeroA, 0, w.zeroA_bytes, s)) return cuda_fail(e_, "memset workspace");
    auto pass_bufs = [&](int p) { return PassBufs{w.counts, w.offs, w.cnt_lb[p], w.ctr + kCtrPass + p}; };
    // 1. index offsets in id order, M, V, rect codes
    u64 tot[2] = {0, 0};
    if (n > 0) {
        int st = run_scan<0>(cam, tiles_touched, means2d, radii, nullptr, nullptr, (u64)n, w.part_sum, w.part_vis,
                             offsets, w.totals, s);
        if (st) return st;
        if (cudaError_t e_ = cudaMemcpyAsync(tot, w.totals, sizeof(tot), cudaMemcpyDeviceToHost, s)) return cuda_fail(e_, "read M");
        if (cudaError_t e_ = cudaStreamSynchronize(s)) return cuda_fail(e_, "bin_sort sync");
    }
    const u64 M = tot[0], V = tot[1];
    *num_isects = (int64_t)M;
    if ((int64_t)M > capacity || M >= (1ull << 30)) return VKS_ERR_CAPACITY;
    if (M == 0) {
        if (cudaMemsetAsync(tile_offsets, 0, sizeof(u32) * (n_tiles + 1), s) != cudaSuccess) return VKS_ERR_CUDA;
        return VKS_OK;
    }
    u64* keys64 = reinterpret_cast<u64*>(keys);
    // debug: the pre-sort keys in id order, exactly as "Generate Keys" defines them
    if (keys_unsorted || vals_unsorted) {
        u32* vtmp = vals_unsorted ? vals_unsorted : w.tv[1];
        u64* ktmp = keys_unsorted ? reinterpret_cast<u64*>(keys_unsorted) : reinterpret_cast<u64*>(w.tk[0]);
        int st = launch_keys<1>(cam, n, nullptr, nullptr, tiles_touched, means2d, radii, depths, offsets, nullptr, vtmp,
                                ktmp, w.diff, s);
        if (st) return st;
    }
    // 2. depth sort of all n (culled Gaussians key 0xFFFFFFFF, last); pass 0 reads (tiles, depths),
    //    the last pass also lays out the rect codes in depth order
    int st = launch_pass<8, kPassDepthFirst>(reinterpret_cast<const u32*>(tiles_touched),
                                             reinterpret_cast<const u32*>(depths), w.dk[0], w.dv[0], (u32)n, 0,
                                             pass_bufs(0), nullptr, nullptr, s);
    if (st) return st;
    for (int p = 1; p < kDepthPasses; p++) {
        const u32* ki = w.dk[(p + 1) & 1];
        const u32* vi = w.dv[(p + 1) & 1];
        if (p == kDepthPasses - 1)
            st = launch_pass<8, kPassDepthLast>(ki, vi, w.dk[p & 1], w.dv[p & 1], (u32)n, 8 * p, pass_bufs(p), nullptr,
                                                nullptr, s,
                                                RectSrc{reinterpret_cast<const float2*>(means2d),
                                                        reinterpret_cast<const int2*>(radii), TX, TY, (u32)V},
                                                w.rcs);
        else
            st = launch_pass<8, kPassPlain>(ki, vi, w.dk[p & 1], w.dv[p & 1], (u32)n, 8 * p, pass_bufs(p), nullptr,
                                            nullptr, s);
        if (st) return st;
    }
    const u32* sid = w.dv[(kDepthPasses - 1) & 1];  // ids in (depth, id) order; the first V are visible
    // 3. slots in depth order (from the depth-ordered rect codes)
    st = run_scan<1>(cam, nullptr, nullptr, nullptr, w.rcs, nullptr, V, w.part_sum, nullptr, w.doff, w.totals + 0, s);
    if (st) return st;
    // 4. (tile, id) pairs in depth order + tile-rect difference array
    const TilePlan plan = tile_plan(n_tiles);
    u32* pv0 = plan.passes == 0 ? vals : w.tv[0];
    st = launch_keys<0>(cam, (int64_t)V, sid, w.rcs, tiles_touched, means2d, radii, depths, w.doff, w.tk[0], pv0,
                        nullptr, w.diff, s);
    if (st) return st;
    // 5. tile counts -> tile ranges
    tile_count_kernel<<<1, 1024, 0, s>>>(TX, TY, w.diff, tile_offsets);
    if (int e_ = check_launch(__func__)) return e_;
    // 6. stable tile passes; the last writes the caller's vals (+ u64 keys on request)
    if (plan.passes == 0) {
        if (keys64) {
            keys64_tile0_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(vals, depths, keys64, (u32)M);
            if (int e_ = check_launch(__func__)) return e_;
        }
        return VKS_OK;
    }
    for (int p = 0; p < plan.passes; p++) {
        const u32* kin = w.tk[p & 1];
        const u32* vin = w.tv[p & 1];
        const bool last = p == plan.passes - 1;
        u32* ko = w.tk[(p + 1) & 1];
        u32* vo = last ? vals : w.tv[(p + 1) & 1];
        st = last ? launch_tile_pass<kPassTileLast>(plan.dbits, kin, vin, ko, vo, (u32)M, plan.dbits * p,
                                                    pass_bufs(kDepthPasses + p), depths, keys64, s)
                  : launch_tile_pass<kPassPlain>(plan.dbits, kin, vin, ko, vo, (u32)M, plan.dbits * p,
                                                 pass_bufs(kDepthPasses + p), nullptr, nullptr, s);
        if (st) return st;
    }
    return VKS_OK;
}

}  // namespace vks
