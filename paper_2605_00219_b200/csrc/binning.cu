// binning.cu — "Index Offset", "Generate Keys", "Sorting" and
// "Tile Ranges"; DESIGN.md §4.3 and §6.
//
//  1. scan_kernel     single-pass exclusive prefix sum of tiles_touched with decoupled look-back
//                     (dynamic tile ids for forward progress); writes offsets and M.
//  2. keys_kernel     warp-cooperative key generation: each warp expands the tile rects of its 32
//                     Gaussians into contiguous slots with coalesced 8+4-byte stores.  It also
//                     builds (a) the radix histograms of the 4 depth-bit digits, weighted by
//                     tiles_touched (every key of a Gaussian shares its depth bits), and (b) a 2-D
//                     difference array of the tile rects.
//  3. tile_count_kernel  one block: 2-D prefix of the difference array = per-tile list lengths ->
//                     CSR tile_offsets (exclusive scan; identical to boundary detection on the
//                     sorted keys because the sort is tile-major) and the tile-digit histograms;
//                     exclusive scans of all digit histograms.
//  4. onesweep_pass   LSD radix sort, 8-bit digits, P = ceil((32 + ceil(log2 n_tiles)) / 8)
//                     passes.  Per 4096-key tile: warp-level __match_any_sync ranking (stable),
//                     decoupled look-back across dynamically numbered tiles per digit, local
//                     reordering in shared memory so global stores are digit-contiguous runs.
// The binning TU is compiled with -fmad=false (the rect recomputation must equal projection's).
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
constexpr int kSortMinItems = 8;                              // smallest tile (workspace sizing)
constexpr int kSortMinTile = kSortThreads * kSortMinItems;  // 2048 keys
constexpr int kMaxPasses = 8;
constexpr int kDepthPasses = 4;
constexpr int kLookbackChunk = 8;

constexpr u64 kScanFlagAgg = 1ull << 62;
constexpr u64 kScanFlagInc = 2ull << 62;
constexpr u64 kScanMask = (1ull << 62) - 1;
constexpr u32 kLbAgg = 1u << 30;
constexpr u32 kLbInc = 2u << 30;
constexpr u32 kLbMask = (1u << 30) - 1;

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct Workspace {
    u64* keys_x;
    u32* vals_x;
    // zeroed every call (region A)
    u64* scan_lb;
    u32* scan_ctr;
    u64* total;
    u32* hist;     // [kMaxPasses][256]
    int* diff;     // [(TY+1)*(TX+1)]
    // zeroed once M is known (region B)
    u32* sort_ctr; // [kMaxPasses]
    u32* sort_lb;  // [kMaxPasses][sort tiles][256]
    u32* gstart;   // [kMaxPasses][256]
    size_t zeroA_bytes;
    char* zeroA;
    char* zeroB;
    size_t bytes;
};

Workspace carve(void* base, int64_t n, int64_t capacity, int32_t n_tiles, int TX, int TY) {
    Workspace w{};
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += align_up(bytes); return p; };
    const int64_t scan_tiles = (n + kScanTile - 1) / kScanTile;
    const int64_t sort_tiles = (capacity + kSortMinTile - 1) / kSortMinTile;
    w.keys_x = reinterpret_cast<u64*>(take(sizeof(u64) * (size_t)capacity));
    w.vals_x = reinterpret_cast<u32*>(take(sizeof(u32) * (size_t)capacity));
    w.gstart = reinterpret_cast<u32*>(take(sizeof(u32) * kMaxPasses * 256));
    const size_t a0 = off;
    w.zeroA = b ? b + off : nullptr;
    w.scan_lb = reinterpret_cast<u64*>(take(sizeof(u64) * (size_t)(scan_tiles > 0 ? scan_tiles : 1)));
    w.scan_ctr = reinterpret_cast<u32*>(take(sizeof(u32) * 4));
    w.total = reinterpret_cast<u64*>(take(sizeof(u64)));
    w.hist = reinterpret_cast<u32*>(take(sizeof(u32) * kMaxPasses * 256));
    w.diff = reinterpret_cast<int*>(take(sizeof(int) * (size_t)(TX + 1) * (TY + 1)));
    w.zeroA_bytes = off - a0;
    w.zeroB = b ? b + off : nullptr;
    w.sort_ctr = reinterpret_cast<u32*>(take(sizeof(u32) * kMaxPasses));
    w.sort_lb = reinterpret_cast<u32*>(take(sizeof(u32) * (size_t)kMaxPasses * 256 * (size_t)(sort_tiles > 0 ? sort_tiles : 1)));
    w.bytes = off;
    (void)n_tiles;
    return w;
}

// ------------------------------------------------------------------------------------------
// 1. exclusive scan (decoupled look-back)
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const int* __restrict__ in, u32* __restrict__ out,
                                                           int64_t n, u64* __restrict__ lb, u32* __restrict__ ctr,
                                                           u64* __restrict__ total) {
    __shared__ u32 s_tile;
    __shared__ u64 s_warp[kScanThreads / 32];
    __shared__ u64 s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile + (int64_t)tid * kScanItems;
    int v[kScanItems];
    if (base + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < kScanItems; j += 4) {
            int4 q = __ldg(reinterpret_cast<const int4*>(in + base + j));
            v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; j++) v[j] = (base + j < n) ? __ldg(in + base + j) : 0;
    }
    u64 tsum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) tsum += (u32)v[j];
    // block scan of thread sums
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
            int64_t j = tile - 1;
            while (true) {
                u64 s = ld_volatile_u64(reinterpret_cast<const unsigned long long*>(lb + j));
                const u64 f = s & ~kScanMask;
                if (f == 0) continue;
                excl += s & kScanMask;
                if (f == kScanFlagInc) break;
                j--;
            }
            st_volatile_u64(reinterpret_cast<unsigned long long*>(lb + tile), kScanFlagInc | (excl + btotal));
        }
        s_prefix = excl;
        if ((tile + 1) * kScanTile >= n) *total = excl + btotal;
    }
    __syncthreads();
    u64 run = s_prefix + wpre + (incl - tsum);
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        if (base + j < n) out[base + j] = (u32)run;
        run += (u32)v[j];
    }
}

// ------------------------------------------------------------------------------------------
// 2. key generation (+ depth-digit histograms, tile-rect difference array)
// Persistent grid (a few blocks per SM); each warp takes 32 consecutive Gaussians at a time.  The
// 2-D difference array of the tile rects is accumulated per block in shared memory and flushed
// once per block (non-zero cells only), so hot tiles near the image centre see ~#blocks global
// atomics instead of ~#Gaussians.  Grids too large for shared memory use global atomics.
constexpr int kKeysThreads = 512;
constexpr int kKeysWarps = kKeysThreads / 32;
constexpr int kKeysSmemDiffMax = 160 * 1024 / 4;  // cells

template <bool SMEM_DIFF>
__global__ void __launch_bounds__(kKeysThreads) keys_kernel(vks_camera cam, int64_t n, const float2* __restrict__ means2d,
                                                           const int2* __restrict__ radii, const float* __restrict__ depths,
                                                           const int* __restrict__ tiles, const u32* __restrict__ offsets,
                                                           u64* __restrict__ keys, u32* __restrict__ vals,
                                                           u32* __restrict__ hist, int* __restrict__ diff) {
    extern __shared__ int s_diff[];
    __shared__ u32 s_hist[kDepthPasses][256];
    __shared__ int s_incl[kKeysWarps][32];
    __shared__ int s_x0[kKeysWarps][32], s_y0[kKeysWarps][32], s_w[kKeysWarps][32];
    __shared__ u32 s_db[kKeysWarps][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int W1 = TX + 1;
    const int cells = W1 * (TY + 1);
    for (int j = tid; j < kDepthPasses * 256; j += kKeysThreads) (&s_hist[0][0])[j] = 0;
    if (SMEM_DIFF)
        for (int j = tid; j < cells; j += kKeysThreads) s_diff[j] = 0;
    __syncthreads();
    int* dd = SMEM_DIFF ? s_diff : diff;
    const int64_t stride = (int64_t)gridDim.x * kKeysWarps * 32;
    for (int64_t g0 = ((int64_t)blockIdx.x * kKeysWarps + warp) * 32; g0 < n; g0 += stride) {
        const int64_t g = g0 + lane;
        int cnt = 0, x0 = 0, y0 = 0, w = 1;
        u32 db = 0;
        if (g < n) {
            cnt = __ldg(tiles + g);
            if (cnt > 0) {
                const float2 m = __ldg(means2d + g);
                const int2 r = __ldg(radii + g);
                const float rx = (float)r.x, ry = (float)r.y;
                x0 = (int)fminf(fmaxf(floorf((m.x - rx) * 0.0625f), 0.0f), (float)TX);
                const int x1 = (int)fminf(fmaxf(ceilf((m.x + rx) * 0.0625f), 0.0f), (float)TX);
                y0 = (int)fminf(fmaxf(floorf((m.y - ry) * 0.0625f), 0.0f), (float)TY);
                const int y1 = (int)fminf(fmaxf(ceilf((m.y + ry) * 0.0625f), 0.0f), (float)TY);
                w = x1 - x0;
                db = __float_as_uint(__ldg(depths + g));
#pragma unroll
                for (int p = 0; p < kDepthPasses; p++) atomicAdd(&s_hist[p][(db >> (8 * p)) & 255u], (u32)cnt);
                atomicAdd(dd + y0 * W1 + x0, 1);
                atomicAdd(dd + y0 * W1 + x1, -1);
                atomicAdd(dd + y1 * W1 + x0, -1);
                atomicAdd(dd + y1 * W1 + x1, 1);
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
        s_db[warp][lane] = db;
        __syncwarp();
        const u64 base = (u64)__ldg(offsets + g0);
        for (int e = lane; e < total; e += 32) {
            int pos = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
                if (s_incl[warp][pos + step - 1] <= e) pos += step;
            const int k = e - (pos ? s_incl[warp][pos - 1] : 0);  // index within Gaussian pos's rect
            const int ww = s_w[warp][pos];
            const int ry = k / ww;
            const int tx = s_x0[warp][pos] + (k - ry * ww);
            const int ty = s_y0[warp][pos] + ry;
            const u64 tile = (u64)(ty * TX + tx);
            keys[base + e] = (tile << 32) | (u64)s_db[warp][pos];
            vals[base + e] = (u32)(g0 + pos);
        }
    }
    __syncthreads();
    for (int j = tid; j < kDepthPasses * 256; j += kKeysThreads) {
        const u32 c = (&s_hist[0][0])[j];
        if (c) atomicAdd(hist + j, c);
    }
    if (SMEM_DIFF) {
        for (int j = tid; j < cells; j += kKeysThreads) {
            const int v = s_diff[j];
            if (v) atomicAdd(diff + j, v);
        }
    }
}

// ------------------------------------------------------------------------------------------
// 3. per-tile counts -> CSR tile_offsets + tile-digit histograms + digit start offsets
__global__ void __launch_bounds__(1024) tile_count_kernel(int TX, int TY, int passes, int* __restrict__ diff,
                                                         u32* __restrict__ hist, u32* __restrict__ gstart,
                                                         u32* __restrict__ tile_offsets) {
    __shared__ u32 s_hist[kMaxPasses - kDepthPasses][256];
    __shared__ u32 s_wsum[32];
    __shared__ u32 s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W1 = TX + 1;
    for (int j = tid; j < (kMaxPasses - kDepthPasses) * 256; j += 1024) (&s_hist[0][0])[j] = 0;
    // row prefix (along x), then column prefix (along y): count[ty][tx] = sum diff[<=ty][<=tx]
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
    // exclusive scan of counts in tile-id order + tile-digit histograms
    const int n_tiles = TX * TY;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n_tiles; base += 1024) {
        const int t = base + tid;
        u32 c = 0;
        if (t < n_tiles) {
            c = (u32)diff[(t / TX) * W1 + (t % TX)];
            for (int p = kDepthPasses; p < passes; p++) {
                const u32 d = ((u32)t >> (8 * (p - kDepthPasses))) & 255u;
                if (c) atomicAdd(&s_hist[p - kDepthPasses][d], c);
            }
        }
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
    // digit start offsets for every pass
    for (int p = 0; p < passes; p++) {
        u32 c = 0;
        if (tid < 256) c = (p < kDepthPasses) ? hist[p * 256 + tid] : s_hist[p - kDepthPasses][tid];
        u32 incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            u32 v = __shfl_up_sync(VKS_FULL_MASK, incl, d);
            if (lane >= d) incl += v;
        }
        if (tid < 256 && lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        if (tid < 256) {
            u32 wpre = 0;
            for (int w = 0; w < warp; w++) wpre += s_wsum[w];
            gstart[p * 256 + tid] = wpre + incl - c;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// 4. one onesweep pass over 8 bits starting at `shift`
template <int ITEMS>
struct SortSmem {
    static constexpr int kTile = kSortThreads * ITEMS;
    alignas(128) u64 keys[kTile];  // input staging (bulk copy), then the digit-reordered tile
    alignas(128) u32 vals[kTile];
    u32 whist[kSortWarps][256];
    u32 binstart[256];
    u32 gbase[256];
    u32 wsum[kSortWarps];
    u32 tile;
    alignas(8) unsigned long long mbar;
};

__device__ __forceinline__ u32 digit_of(u64 k, int shift) { return (u32)(k >> shift) & 255u; }

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

// One onesweep pass over 8 bits starting at `shift`.  The tile's keys/values arrive through two
// TMA bulk copies (cp.async.bulk, completion on an mbarrier) while the block clears its
// histograms, so no registers are tied up waiting for DRAM; ranks are computed from shared memory
// with __match_any_sync (stable: warp-striped slot order), per-digit totals are published for the
// decoupled look-back (chunked), and the tile is reordered in place so the stores are
// digit-contiguous runs.
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads) onesweep_pass(const u64* __restrict__ kin, const u32* __restrict__ vin,
                                                            u64* __restrict__ kout, u32* __restrict__ vout, u32 M,
                                                            int shift, const u32* __restrict__ gstart,
                                                            u32* __restrict__ lookback, u32* __restrict__ tile_ctr) {
    using Smem = SortSmem<ITEMS>;
    constexpr int kTile = Smem::kTile;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u32 bar = smem_u32(&S.mbar);
    if (tid == 0) {
        S.tile = atomicAdd(tile_ctr, 1u);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const u32 tile = S.tile;
    const u64 base = (u64)tile * kTile;
    const u32 count = (u32)min((u64)kTile, (u64)M - base);
    const u32 nbulk = count & ~3u;  // 32-byte multiples of keys, 16-byte multiples of values
    if (tid == 0) {
        if (nbulk) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nbulk * 12u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(S.keys)), "l"(kin + base), "r"(nbulk * 8u), "r"(bar) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(S.vals)), "l"(vin + base), "r"(nbulk * 4u), "r"(bar) : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
        }
    }
    for (int j = tid; j < kSortWarps * 256; j += kSortThreads) (&S.whist[0][0])[j] = 0;
    // tail (< 4 keys) and padding: pads (~0) rank last in digit 255 and land at dest >= M
    for (u32 j = nbulk + tid; j < (u32)kTile; j += kSortThreads) {
        const bool ok = j < count;
        S.keys[j] = ok ? kin[base + j] : ~0ull;
        S.vals[j] = ok ? vin[base + j] : 0u;
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT%=;\n\t}" ::"r"(bar) : "memory");
    __syncthreads();
    // stable warp-level ranking with match.any
    u32 rank[ITEMS];
    const u32 ltmask = lanemask_lt();
    const int seg = warp * 32 * ITEMS;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const u32 d = digit_of(S.keys[seg + i * 32 + lane], shift);
        const u32 peers = __match_any_sync(VKS_FULL_MASK, d);
        const u32 below = __popc(peers & ltmask);
        const u32 before = S.whist[warp][d];
        rank[i] = before + below;
        __syncwarp();
        if (below == 0) S.whist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per-digit totals, warp exclusive offsets, block exclusive digit starts
    u32 total = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; w++) {
        const u32 c = S.whist[w][tid];
        S.whist[w][tid] = total;
        total += c;
    }
    st_volatile_u32(lookback + (u64)tile * 256 + tid, (tile == 0 ? kLbInc : kLbAgg) | total);
    u32 incl = total;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    {
        u32 wpre = 0;
        for (int w = 0; w < warp; w++) wpre += S.wsum[w];
        const u32 binstart = wpre + incl - total;
        S.binstart[tid] = binstart;
        // decoupled look-back for digit `tid`, kLookbackChunk predecessors per round trip
        // Digits absent from this tile need no prefix: they keep their aggregate (0) and
        // successors walk past them.
        u32 excl = 0;
        if (tile > 0 && total > 0) {
            int64_t j = (int64_t)tile - 1;
            bool found = false;
            while (!found) {
                u32 st[kLookbackChunk];
#pragma unroll
                for (int q = 0; q < kLookbackChunk; q++)
                    st[q] = (j - q >= 0) ? ld_volatile_u32(lookback + (u64)(j - q) * 256 + tid) : 0u;
                int consumed = 0;
#pragma unroll
                for (int q = 0; q < kLookbackChunk; q++) {
                    if (found || consumed < q) break;  // stop at the first unpublished entry
                    const u32 f = st[q] & ~kLbMask;
                    if (f == 0) break;
                    excl += st[q] & kLbMask;
                    consumed = q + 1;
                    if (f == kLbInc) found = true;
                }
                j -= consumed;
            }
            st_volatile_u32(lookback + (u64)tile * 256 + tid, kLbInc | (excl + total));
        }
        S.gbase[tid] = gstart[tid] + excl - binstart;
    }
    __syncthreads();
    // reorder the tile in shared memory (read everything first, then write: in place)
    u64 kk[ITEMS];
    u32 vv[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const int slot = seg + i * 32 + lane;
        kk[i] = S.keys[slot];
        vv[i] = S.vals[slot];
        rank[i] += S.binstart[digit_of(kk[i], shift)] + S.whist[warp][digit_of(kk[i], shift)];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        S.keys[rank[i]] = kk[i];
        S.vals[rank[i]] = vv[i];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ITEMS; r++) {
        const int j = r * kSortThreads + tid;
        const u64 key = S.keys[j];
        const u32 dest = S.gbase[digit_of(key, shift)] + (u32)j;
        if (dest < M) {
            kout[dest] = key;
            vout[dest] = S.vals[j];
        }
    }
}

int end_bits(int32_t n_tiles) {
    int tb = 0;
    while ((1ll << tb) < (int64_t)n_tiles) tb++;
    return 32 + tb;
}

}  // namespace

size_t bin_sort_workspace_bytes(int64_t n, int64_t capacity, int32_t n_tiles) {
    // worst-case tile grid for the difference array: n_tiles x 1 or the square root; use n_tiles + 2*sqrt + slack
    const int side = (int)(n_tiles > 0 ? n_tiles : 1);
    Workspace w = carve(nullptr, n, capacity, n_tiles, side, 1);
    // diff array sized (TX+1)(TY+1) <= 2*n_tiles + TX + TY + 1 <= 3*n_tiles + 2 for any TX*TY = n_tiles
    return w.bytes + align_up(sizeof(int) * (size_t)(2 * side + 2));
}

int run_bin_sort(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii,
                 const float* depths, const int32_t* tiles_touched, uint32_t* offsets,
                 int64_t capacity, uint64_t* keys, uint32_t* vals, uint64_t* keys_unsorted,
                 uint32_t* vals_unsorted, uint32_t* tile_offsets, int64_t* num_isects,
                 void* workspace, size_t workspace_bytes, cudaStream_t s) {
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    const int32_t n_tiles = TX * TY;
    if (workspace_bytes < bin_sort_workspace_bytes(n, capacity, n_tiles)) return VKS_ERR_WORKSPACE;
    Workspace w = carve(workspace, n, capacity, n_tiles, TX, TY);
    if (cudaMemsetAsync(w.zeroA, 0, w.zeroA_bytes, s) != cudaSuccess) return VKS_ERR_CUDA;
    // 1. index offsets
    u64 M = 0;
    if (n > 0) {
        const unsigned blocks = (unsigned)((n + kScanTile - 1) / kScanTile);
        scan_kernel<<<blocks, kScanThreads, 0, s>>>(tiles_touched, offsets, n, w.scan_lb, w.scan_ctr, w.total);
        if (cudaGetLastError() != cudaSuccess) return VKS_ERR_CUDA;
        if (cudaMemcpyAsync(&M, w.total, sizeof(u64), cudaMemcpyDeviceToHost, s) != cudaSuccess) return VKS_ERR_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return VKS_ERR_CUDA;
    }
    *num_isects = (int64_t)M;
    if ((int64_t)M > capacity || M >= (1ull << 30)) return VKS_ERR_CAPACITY;
    if (M == 0) {
        if (cudaMemsetAsync(tile_offsets, 0, sizeof(u32) * (n_tiles + 1), s) != cudaSuccess) return VKS_ERR_CUDA;
        return VKS_OK;
    }
    const int passes = (end_bits(n_tiles) + 7) / 8;
    // ping-pong so that the last pass lands in the caller's keys/vals
    u64* ukeys = reinterpret_cast<u64*>(keys);
    u64* kA = (passes % 2 == 0) ? ukeys : w.keys_x;
    u32* vA = (passes % 2 == 0) ? vals : w.vals_x;
    u64* kB = (passes % 2 == 0) ? w.keys_x : ukeys;
    u32* vB = (passes % 2 == 0) ? w.vals_x : vals;
    // 2. keys (+ histograms)
    {
        const int cells = (TX + 1) * (TY + 1);
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
        const int64_t want = (n + kKeysThreads - 1) / kKeysThreads;
        if (cells <= kKeysSmemDiffMax) {
            const size_t sm = sizeof(int) * (size_t)cells;
            if (sm > 32 * 1024 &&
                cudaFuncSetAttribute(keys_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
                return VKS_ERR_CUDA;
            const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)sms * 2);
            keys_kernel<true><<<blocks, kKeysThreads, sm, s>>>(cam, n, reinterpret_cast<const float2*>(means2d),
                                                               reinterpret_cast<const int2*>(radii), depths,
                                                               tiles_touched, offsets, kA, vA, w.hist, w.diff);
        } else {
            const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)sms * 4);
            keys_kernel<false><<<blocks, kKeysThreads, 0, s>>>(cam, n, reinterpret_cast<const float2*>(means2d),
                                                               reinterpret_cast<const int2*>(radii), depths,
                                                               tiles_touched, offsets, kA, vA, w.hist, w.diff);
        }
        if (cudaGetLastError() != cudaSuccess) return VKS_ERR_CUDA;
    }
    if (keys_unsorted && cudaMemcpyAsync(keys_unsorted, kA, sizeof(u64) * M, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return VKS_ERR_CUDA;
    if (vals_unsorted && cudaMemcpyAsync(vals_unsorted, vA, sizeof(u32) * M, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return VKS_ERR_CUDA;
    // 3. tile counts -> tile ranges, digit starts
    static int items = 0;
    if (!items) {
        const char* e = getenv("VKS_SORT_ITEMS");
        items = e ? atoi(e) : 16;
        if (items != 8 && items != 12 && items != 16) items = 16;
    }
    const int tile_keys = kSortThreads * items;
    const u64 sort_tiles = (M + tile_keys - 1) / tile_keys;
    const size_t zb = align_up(sizeof(u32) * kMaxPasses) + sizeof(u32) * (size_t)passes * 256 * sort_tiles;
    if (cudaMemsetAsync(w.zeroB, 0, zb, s) != cudaSuccess) return VKS_ERR_CUDA;
    tile_count_kernel<<<1, 1024, 0, s>>>(TX, TY, passes, w.diff, w.hist, w.gstart, tile_offsets);
    if (cudaGetLastError() != cudaSuccess) return VKS_ERR_CUDA;
    // 4. radix passes
    auto launch = [&](auto kernel, size_t sm) -> int {
        if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
            return VKS_ERR_CUDA;
        for (int p = 0; p < passes; p++) {
            const u64* kin = (p % 2 == 0) ? kA : kB;
            const u32* vin = (p % 2 == 0) ? vA : vB;
            u64* ko = (p % 2 == 0) ? kB : kA;
            u32* vo = (p % 2 == 0) ? vB : vA;
            kernel<<<(unsigned)sort_tiles, kSortThreads, sm, s>>>(kin, vin, ko, vo, (u32)M, 8 * p, w.gstart + 256 * p,
                                                                 w.sort_lb + (size_t)p * 256 * sort_tiles,
                                                                 w.sort_ctr + p);
            if (cudaGetLastError() != cudaSuccess) return VKS_ERR_CUDA;
        }
        return VKS_OK;
    };
    int st = VKS_OK;
    if (items == 16) st = launch(onesweep_pass<16>, sizeof(SortSmem<16>));
    else if (items == 12) st = launch(onesweep_pass<12>, sizeof(SortSmem<12>));
    else st = launch(onesweep_pass<8>, sizeof(SortSmem<8>));
    if (st != VKS_OK) return st;
    return VKS_OK;
}

}  // namespace vks
