// raster.cu — "Rasterization Forward" and "Rasterization Backward";
// DESIGN.md §4.3-4.4 and §6.2.
//
// One block per 16x16 tile; each warp owns an 8 x 4*PPT pixel patch (PPT = 2 by default: 8x8,
// two pixels per thread) and walks the tile's sorted list on its own in batches of 32 staged
// into its shared-memory slice (software-pipelined: ids two batches ahead, entries one batch
// ahead) — with the projection's packed records (the default) by cp.async.ca straight into a
// double-buffered stage, else gathered from the separate arrays into registers and stored — so
// there are no block barriers and a warp stops as soon as its own pixels are saturated.  With
// two pixels per thread the per-pixel math runs on paired fp32 instructions (FFMA2 / FMUL2 /
// FADD2, eval_alpha2).  Before a batch is visited each lane tests its entry against the
// patch with an exact test (the minimum of sigma over the patch rectangle against ln(255 rho));
// the warp visits only entries that can composite somewhere in the patch (a finer per-8x4-band
// test removed 20% of the evaluations but cost more instructions than it saved).  Forward and
// backward evaluate sigma / alpha through the SAME inline function, so skip / clamp / stop
// decisions replay identically; sigma, alpha and the colour accumulation follow the pinned fp32
// order of DESIGN.md §4.3 (only exp differs from the oracle: ex2.approx here, expf there).  The
// backward accumulates per (warp, Gaussian) the colour terms, sum(g) and the moments sum(g dx),
// sum(g dy), sum(g dx^2), sum(g dx dy), sum(g dy^2) (g = G dalpha).  An entry no lane composited
// is skipped; an entry composited by at most 4 lanes (VKS_RASTER_SPARSE) is finished by those
// lanes' own atomics (the outputs are linear in the sums); any other reduces its 9 sums across the
// warp with a transposed butterfly (14 shuffles instead of 45), turns the moments into the mean /
// conic gradients with the Gaussian's conic, and issues one atomic per term from 9 lanes.
#include <stdlib.h>

#include <type_traits>

#include "vks_common.cuh"

namespace vks {
namespace {


int env_choice(const char* var, int dflt, int lo, int hi) {
    const char* e = getenv(var);
    const int v = e ? atoi(e) : dflt;
    return (v >= lo && v <= hi) ? v : dflt;
}

// One warp's staged batch of 32 list entries (each warp walks the tile list on its own: no block
// barriers, so a warp never waits for a slower one and stops as soon as its own pixels are done).
struct WarpStage {  // all three arrays at a 16-byte stride: one address for the three loads
    float4 a[32];    // u, v, 0.5*a, b
    float4 b[32];    // 0.5*c, rho, c0, c1
    float4 c[32];    // c2, id (bits), position in the batch (bits), -
};

// Records path (the projection's packed raster records, include/vks.h): each warp stages two
// batches of 32 records with cp.async (three 16-byte copies per entry straight into shared
// memory, slot = lane, the next batch in flight while the current one is visited); the live
// entries are then visited in place (set bits of the warp's live mask).
#ifndef VKS_RASTER_NBUF
#define VKS_RASTER_NBUF 2  // stage buffers per warp: NBUF - 1 batches in flight
#endif
constexpr int kNB = VKS_RASTER_NBUF;
struct RecStage {
    float4 a[kNB][32];  // u, v, 0.5*a, b
    float4 b[kNB][32];  // 0.5*c, rho, c0, c1
    float4 c[kNB][32];  // c2, id (bits), -, -
};
__device__ __forceinline__ int nb_next(int b) { return b + 1 == kNB ? 0 : b + 1; }
__device__ __forceinline__ int nb_ahead(int b) { return b == 0 ? kNB - 1 : b - 1; }  // (b + kNB - 1) % kNB

template <bool REC>
using StageT = typename std::conditional<REC, RecStage, WarpStage>::type;

// one lane's record -> slot `lane` of buffer `buf` (three cp.async 16-byte copies).  CA: through L1
// (.ca), so the four warps of a tile, which stage the same entries, share L1 hits; otherwise L2
// only (.cg)
template <bool CA = true>
__device__ __forceinline__ void stage_record(RecStage& s, int buf, int lane, const float4* __restrict__ rec,
                                             uint32_t id) {
    const float4* g = rec + 3 * (size_t)id;
    if constexpr (CA) {
        cp_async16_ca(&s.a[buf][lane], g);
        cp_async16_ca(&s.b[buf][lane], g + 1);
        cp_async16_ca(&s.c[buf][lane], g + 2);
    } else {
        cp_async16(&s.a[buf][lane], g);
        cp_async16(&s.b[buf][lane], g + 1);
        cp_async16(&s.c[buf][lane], g + 2);
    }
}

struct Entry {  // one lane's gathered entry, in registers until it is stored to the stage
    float4 a, b;
    float c2;
    uint32_t id;
    int2 r;     // projection radii (kCullBox only)
};

// Patch culling modes (VKS_RASTER_CULL): a warp skips an entry when no pixel centre of its patch
// can reach alpha >= 1/255.
//   kCullNone    evaluate every entry (3SIGMA footprint, or VKS_RASTER_CULL=0)
//   kCullBox     the projection's support box (radii) widened by 1 + r/64 px
//   kCullEllipse exact: the minimum of sigma over the patch rectangle against ln(255 rho)
enum { kCullNone = 0, kCullBox = 1, kCullEllipse = 2 };

template <int CULL>
__device__ __forceinline__ Entry gather_entry(uint32_t g, uint32_t n, const float2* __restrict__ means2d,
                                              const float* __restrict__ conics, const float* __restrict__ colors,
                                              const float* __restrict__ opac, const int2* __restrict__ radii) {
    Entry e;
    VKS_DCHECK(g < n);
    (void)n;
    const float2 uv = __ldg(means2d + g);
    const float ca = __ldg(conics + 3 * (size_t)g), cb = __ldg(conics + 3 * (size_t)g + 1),
                cc = __ldg(conics + 3 * (size_t)g + 2);
    const float r0 = __ldg(colors + 3 * (size_t)g), r1 = __ldg(colors + 3 * (size_t)g + 1);
    e.c2 = __ldg(colors + 3 * (size_t)g + 2);
    const float rho = __ldg(opac + g);
    e.id = g;
    e.a = make_float4(uv.x, uv.y, 0.5f * ca, cb);
    e.b = make_float4(0.5f * cc, rho, r0, r1);
    if (CULL == kCullBox) e.r = __ldg(radii + g);
    return e;
}

// the live entries of a batch are stored compacted (slot = rank among the live lanes), with
// their position in the batch, so the visit loop is a plain counter over the slots
__device__ __forceinline__ void store_entry(WarpStage& s, int slot, int lane, const Entry& e) {
    s.a[slot] = e.a;
    s.b[slot] = e.b;
    s.c[slot] = make_float4(e.c2, __uint_as_float(e.id), __int_as_float(lane), 0.0f);
}

// sigma at one candidate point of the patch minus the bound on its fp32 evaluation error
// (the kernel's pinned evaluation and this one each err by < 1e-6 (ha dx^2 + hc dy^2), since
// |b dx dy| <= ha dx^2 + hc dy^2 for a positive-definite conic)
__device__ __forceinline__ float sigma_lower(float ha, float b, float hc, float dx, float dy) {
    const float q = ha * dx * dx + hc * dy * dy;
    return fmaf(b * dx, dy, q) - 2e-5f * q;
}

// true if no pixel centre of the warp patch [wx0, wx1] x [wy0, wy1] can composite entry (A, B).
// kCullEllipse: sigma(dx, dy) = ha dx^2 + b dx dy + hc dy^2 (dx = u - x) is convex with its
// minimum 0 at the centre; over the rectangle its minimum lies on an edge facing the centre,
// where it is a 1-D quadratic minimised at the clamped stationary point.  A pixel composites only if
// rho G >= 1/255, i.e. sigma <= ln(255 rho) (+ ex2 / log approximation slack < 1e-5), so the
// test culls only when the lower bound exceeds ln(255 rho) + 1e-3.
template <int CULL>
__device__ __forceinline__ bool culled(const Entry& e, float wx0, float wx1, float wy0, float wy1) {
    if (CULL == kCullBox) {
        // radii = ceil(sqrt(2 k' Sigma'_xx)) + 1 with k' > ln(255 rho): every pixel centre whose
        // alpha can reach 1/255 lies inside u +- rx; widen by 1 + rx/64 px more for fp32 slack.
        const float mx = (float)e.r.x * (1.0f + 1.0f / 64.0f) + 1.0f;
        const float my = (float)e.r.y * (1.0f + 1.0f / 64.0f) + 1.0f;
        return e.a.x + mx < wx0 || e.a.x - mx > wx1 || e.a.y + my < wy0 || e.a.y - my > wy1;
    } else if (CULL == kCullEllipse) {
        // only the edges facing the mean can hold the minimum (KKT: at a minimiser on an edge the
        // gradient points inwards, and convexity then puts the mean on the edge's outer side)
        const float dxl = e.a.x - wx1, dxh = e.a.x - wx0, dyl = e.a.y - wy1, dyh = e.a.y - wy0;
        const bool fx = dxl > 0.0f || dxh < 0.0f, fy = dyl > 0.0f || dyh < 0.0f;
        if (!fx && !fy) return false;  // the mean is inside the patch
        const float ha = e.a.z, b = e.a.w, hc = e.b.x;
        const float dxe = dxl > 0.0f ? dxl : dxh, dye = dyl > 0.0f ? dyl : dyh;
        const float mx = sigma_lower(ha, b, hc, dxe, fminf(fmaxf(__fdividef(-b, 2.0f * hc) * dxe, dyl), dyh));
        const float my = sigma_lower(ha, b, hc, fminf(fmaxf(__fdividef(-b, 2.0f * ha) * dye, dxl), dxh), dye);
        const float m = fminf(fx ? mx : INFINITY, fy ? my : INFINITY);
        return m > __logf(255.0f * e.b.y) + 1e-3f;
    }
    return false;
}

__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float exp2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// sigma = 1/2 a dx^2 + b dx dy + 1/2 c dy^2 in the pinned order; returns false when skipped
// (sigma < 0 or alpha < 1/255).  G = exp(-sigma) = 2^(-sigma log2 e) via ex2.approx.ftz.
__device__ __forceinline__ bool eval_alpha(const float4 A, const float4 B, float px, float py, float& dx,
                                           float& dy, float& G, float& rG, float& alpha) {
    dx = A.x - px;
    dy = A.y - py;
    const float sigma = fmaf(A.z * dx, dx, fmaf(B.x * dy, dy, (A.w * dx) * dy));
    G = exp2_ftz(sigma * -1.44269504088896341f);  // evaluated unconditionally: no branch
    rG = B.y * G;
    alpha = fminf(0.99f, rG);
    return !(sigma < 0.0f) && !(alpha < 1.0f / 255.0f);
}

// The same evaluation for a lane's two pixels (PPT = 2: rows y and y + 4, the same x) with the
// sm_100 paired fp32 instructions (FFMA2 / FMUL2 / FADD2: two IEEE results per issued instruction,
// each bit-identical to the scalar operation): dx, A.z dx and A.w dx are shared by the two
// pixels, everything else runs on (pixel 0, pixel 1) pairs; npy = -(py0, py1) (A.y - py ==
// A.y + (-py) exactly).  The raster kernels are issue-bound, so the pairs cut their issued
// instructions; the decisions equal eval_alpha's bit for bit (the 1- and 4-pixel layouts and the
// statistics kernel use the scalar form).
__device__ __forceinline__ void eval_alpha2(const float4 A, const float4 B, float px, float2 npy, float& dx,
                                            float2& dy, float2& G, float2& rG, float2& alpha, bool& ok0, bool& ok1) {
    dx = A.x - px;
    dy = __fadd2_rn(make_float2(A.y, A.y), npy);
    const float azdx = A.z * dx, awdx = A.w * dx;
    const float2 inner = __ffma2_rn(__fmul2_rn(make_float2(B.x, B.x), dy), dy, __fmul2_rn(make_float2(awdx, awdx), dy));
    const float2 sigma = __ffma2_rn(make_float2(azdx, azdx), make_float2(dx, dx), inner);
    const float2 e = __fmul2_rn(sigma, make_float2(-1.44269504088896341f, -1.44269504088896341f));
    G = make_float2(exp2_ftz(e.x), exp2_ftz(e.y));
    rG = __fmul2_rn(make_float2(B.y, B.y), G);
    alpha = make_float2(fminf(0.99f, rG.x), fminf(0.99f, rG.y));
    ok0 = !(sigma.x < 0.0f) && !(alpha.x < 1.0f / 255.0f);
    ok1 = !(sigma.y < 0.0f) && !(alpha.y < 1.0f / 255.0f);
}

// Warp patch: 8 pixels wide x 4*PPT tall; lane (lx, ly) = (lane & 7, lane >> 3) owns the PPT
// pixels (lx, ly + 4k), k < PPT.  A 16x16 tile has 8/PPT warps.
template <int PPT>
struct PixelMap {
    int x, y0;                 // first pixel of the lane
    float wx0, wx1, wy0, wy1;  // warp patch (pixel centres)
};

template <int PPT>
__device__ __forceinline__ PixelMap<PPT> pixel_map(int tile, int TX) {
    constexpr int kH = 4 * PPT;            // patch height
    constexpr int kRows = kTile / kH;      // patches per tile column
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int bx = (tile % TX) * kTile + (warp / kRows) * 8;
    const int by = (tile / TX) * kTile + (warp % kRows) * kH;
    PixelMap<PPT> m;
    m.x = bx + (lane & 7);
    m.y0 = by + (lane >> 3);
    m.wx0 = (float)bx + 0.5f;
    m.wx1 = (float)bx + 7.5f;
    m.wy0 = (float)by + 0.5f;
    m.wy1 = (float)(by + kH - 1) + 0.5f;
    return m;
}

// STATS: diagnostic variant (vks_raster_fwd_stats) that writes no image and instead accumulates
// stats[0] = list entries visited before each pixel's stop (the algorithm's evaluations),
// stats[1] = composited pairs, stats[2] = pairs actually evaluated here (after patch culling),
// stats[3] = sum of n_contrib (entries the backward replays), stats[4] = (warp, entry) pairs a
// warp processed after patch culling, stats[5] = those with at least one composited pixel.
// minimum resident blocks per SM of the records kernels at 2 pixels per thread (scaled with the
// block size for the other layouts; a register budget; the gather kernels hold more registers and
// stay unconstrained): the forward at 12 (<= 42 registers; measured
// 0.216 vs 0.224 ms on bicycle), the backward at 7 (63 registers: 0.443 vs 0.461 ms unconstrained at
// 77 registers / 6 blocks on bicycle, 1.346 vs 1.416 on stress, step 773 vs 761 views/s; 8 blocks at
// 59 registers 0.477, 10 slower still)
#ifndef VKS_RASTER_REC_CA
#define VKS_RASTER_REC_CA true
#endif
#ifndef VKS_RASTER_FWD_MINB
#define VKS_RASTER_FWD_MINB 12
#endif
#ifndef VKS_RASTER_BWD_MINB
#define VKS_RASTER_BWD_MINB 7
#endif

template <int PPT, int CULL, bool STATS = false, bool REC = false>
__global__ void __launch_bounds__(32 * 8 / PPT, REC ? (VKS_RASTER_FWD_MINB * PPT + 1) / 2 : 1) raster_fwd_kernel(vks_config cfg, vks_camera cam,
                                                                 const float2* __restrict__ means2d,
                                                                 const float* __restrict__ conics,
                                                                 const float* __restrict__ colors,
                                                                 const float* __restrict__ opac,
                                                                 const int2* __restrict__ radii,
                                                                 const float4* __restrict__ rec,
                                                                 const uint32_t* __restrict__ vals,
                                                                 const uint32_t* __restrict__ tile_offsets,
                                                                 const uint32_t* __restrict__ tile_order,
                                                                 float* __restrict__ image, float* __restrict__ T_final,
                                                                 int* __restrict__ n_contrib,
                                                                 uint32_t n, unsigned long long* __restrict__ stats = nullptr) {
    pdl_wait();
    __shared__ StageT<REC> stage[8 / PPT];
    unsigned long long n_eval = 0, n_comp = 0, n_went = 0, n_wcomp = 0;
    const int TX = tiles_x(cam);
    const int tile = tile_order ? (int)__ldg(tile_order + blockIdx.x) : (int)blockIdx.x;
    const int lane = threadIdx.x & 31;
    StageT<REC>& s = stage[threadIdx.x >> 5];
    const PixelMap<PPT> pm = pixel_map<PPT>(tile, TX);
    const float px = (float)pm.x + 0.5f;
    // a pixel is done once T < 1e-4 (T only changes when it composites, so the test is exact);
    // pixels outside the image start done (T = 0) and are never written
    float py[PPT], T[PPT], C0[PPT], C1[PPT], C2[PPT];
    int last[PPT];
#pragma unroll
    for (int k = 0; k < PPT; k++) {
        py[k] = (float)(pm.y0 + 4 * k) + 0.5f;
        T[k] = (pm.x < cam.width && pm.y0 + 4 * k < cam.height) ? 1.0f : 0.0f;
        C0[k] = C1[k] = C2[k] = 0.0f;
        last[k] = 0;
    }
    // PPT == 2, compositing (not the statistics): T and C held as (pixel 0, pixel 1) pairs
    float2 T2 = make_float2(T[0], T[PPT - 1]), C02 = make_float2(0.0f, 0.0f), C12 = C02, C22 = C02;
    const float2 npy = make_float2(-py[0], -py[PPT - 1]);
    const uint32_t start = tile_offsets[tile], end = tile_offsets[tile + 1];
    VKS_DCHECK(start <= end);
    // software pipeline: ids two batches ahead, the next batch's entries one batch ahead (gathered
    // into registers, or, REC, copied by cp.async into the other stage buffer)
    uint32_t id_next = (start + lane < end) ? __ldg(vals + start + lane) : 0u;
    Entry e_next;
    constexpr int kAhead = REC ? kNB - 1 : 1;  // batches in flight
    if constexpr (REC) {
#pragma unroll
        for (int q = 0; q < kNB - 1; q++) {  // batches 0 .. kNB - 2
            const uint32_t pq = start + 32 * q + lane;
            if (q > 0) id_next = pq < end ? __ldg(vals + pq) : 0u;
            VKS_DCHECK(pq >= end || id_next < n);
            if (pq < end) stage_record<VKS_RASTER_REC_CA>(s, q, lane, rec, id_next);
            cp_async_commit();
        }
    } else {
        if (start + lane < end) e_next = gather_entry<CULL>(id_next, n, means2d, conics, colors, opac, radii);
    }
    id_next = (start + 32 * kAhead + lane < end) ? __ldg(vals + start + 32 * kAhead + lane) : 0u;
    int buf = 0;
    for (uint32_t b = start; b < end; b += 32, buf = nb_next(buf)) {
        bool all_done = true;
        if constexpr (PPT == 2 && !STATS) {
            all_done = T2.x < 1e-4f && T2.y < 1e-4f;
        } else {
#pragma unroll
            for (int k = 0; k < PPT; k++) all_done = all_done && T[k] < 1e-4f;
        }
        if (__all_sync(VKS_FULL_MASK, all_done)) break;
        __syncwarp();  // every lane is done with the buffer the next stores / copies overwrite
        // each lane tests its own entry against the warp patch; the warp then visits, in list
        // order, only the entries that can composite somewhere in the patch
        unsigned live;
        if constexpr (REC) {
            VKS_DCHECK(b + 32 * kAhead + lane >= end || id_next < n);
            if (b + 32 * kAhead + lane < end) stage_record<VKS_RASTER_REC_CA>(s, nb_ahead(buf), lane, rec, id_next);
            cp_async_commit();
            if (b + 32 * (kAhead + 1) + lane < end) id_next = __ldg(vals + b + 32 * (kAhead + 1) + lane);
            cp_async_wait_group<kNB - 1>();  // this lane's copies of batch b have landed
            __syncwarp();              // ... and every other lane's
            bool lv = false;
            if (b + lane < end) {
                Entry e;
                e.a = s.a[buf][lane];
                e.b = s.b[buf][lane];
                lv = !culled<CULL>(e, pm.wx0, pm.wx1, pm.wy0, pm.wy1);
            }
            live = __ballot_sync(VKS_FULL_MASK, lv);
        } else {
            const bool lv = b + lane < end && !culled<CULL>(e_next, pm.wx0, pm.wx1, pm.wy0, pm.wy1);
            live = __ballot_sync(VKS_FULL_MASK, lv);
            if (lv) store_entry(s, __popc(live & lanemask_lt()), lane, e_next);
            __syncwarp();
            if (b + 32 + lane < end) e_next = gather_entry<CULL>(id_next, n, means2d, conics, colors, opac, radii);
            if (b + 64 + lane < end) id_next = __ldg(vals + b + 64 + lane);
        }
        const int nlive = __popc(live);
        const int base = (int)(b - start) + 1;
        for (int q = 0; q < nlive; q++) {  // in list order
            float4 A, B;
            float c2;
            int pos1;
            if constexpr (REC) {  // the live slots in place: lowest set bit first
                const int j = __ffs(live) - 1;
                live &= live - 1;
                A = s.a[buf][j];
                B = s.b[buf][j];
                c2 = s.c[buf][j].x;
                pos1 = base + j;
            } else {
                A = s.a[q];
                B = s.b[q];
                const float4 Cq = s.c[q];
                c2 = Cq.x;
                pos1 = base + __float_as_int(Cq.z);
            }
            if constexpr (STATS) {
                bool any = false;
#pragma unroll
                for (int k = 0; k < PPT; k++) {
                    if (T[k] < 1e-4f) continue;
                    float dx, dy, G, rG, alpha;
                    n_eval++;
                    if (!eval_alpha(A, B, px, py[k], dx, dy, G, rG, alpha)) continue;
                    n_comp++;
                    any = true;
                    T[k] = T[k] * (1.0f - alpha);
                    last[k] = pos1;
                }
                const bool wany = __any_sync(VKS_FULL_MASK, any);
                if (lane == 0) { n_went++; n_wcomp += wany; }
            } else if constexpr (PPT == 2) {
                // the same compositing on (pixel 0, pixel 1) pairs (eval_alpha2)
                float dx;
                float2 dy, G, rG, alpha;
                bool e0, e1;
                eval_alpha2(A, B, px, npy, dx, dy, G, rG, alpha, e0, e1);
                const bool ok0 = e0 && !(T2.x < 1e-4f), ok1 = e1 && !(T2.y < 1e-4f);
                const float2 a = make_float2(ok0 ? alpha.x : 0.0f, ok1 ? alpha.y : 0.0f);
                const float2 aT = __fmul2_rn(a, T2);
                C02 = __ffma2_rn(make_float2(B.z, B.z), aT, C02);
                C12 = __ffma2_rn(make_float2(B.w, B.w), aT, C12);
                C22 = __ffma2_rn(make_float2(c2, c2), aT, C22);
                T2 = __fmul2_rn(T2, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-a.x, -a.y)));
                last[0] = ok0 ? pos1 : last[0];
                last[1] = ok1 ? pos1 : last[1];
            } else {
                // branch-free: a skipped entry composites alpha = 0, which leaves C and T
                // bit-identical (C + c * 0 = C, T * (1 - 0) = T)
#pragma unroll
                for (int k = 0; k < PPT; k++) {
                    float dx, dy, G, rG, alpha;
                    const bool ok = eval_alpha(A, B, px, py[k], dx, dy, G, rG, alpha) && !(T[k] < 1e-4f);
                    const float a = ok ? alpha : 0.0f;
                    const float aT = a * T[k];
                    C0[k] = fmaf(B.z, aT, C0[k]);
                    C1[k] = fmaf(B.w, aT, C1[k]);
                    C2[k] = fmaf(c2, aT, C2[k]);
                    T[k] = T[k] * (1.0f - a);
                    last[k] = ok ? pos1 : last[k];
                }
            }
        }
    }
    if constexpr (REC) cp_async_wait_all();  // no copy outlives the warp
    if constexpr (STATS) {
        unsigned long long visited = 0, replay = 0;
#pragma unroll
        for (int k = 0; k < PPT; k++) {
            const int y = pm.y0 + 4 * k;
            if (!(pm.x < cam.width && y < cam.height)) continue;
            visited += T[k] < 1e-4f ? (unsigned long long)last[k] : (unsigned long long)(end - start);
            replay += (unsigned long long)last[k];
        }
        atomicAdd(stats + 0, visited);
        atomicAdd(stats + 1, n_comp);
        atomicAdd(stats + 2, n_eval);
        atomicAdd(stats + 3, replay);
        if (lane == 0) {
            atomicAdd(stats + 4, n_went);
            atomicAdd(stats + 5, n_wcomp);
        }
    } else {
        if constexpr (PPT == 2) {
            T[0] = T2.x; T[1] = T2.y;
            C0[0] = C02.x; C0[1] = C02.y;
            C1[0] = C12.x; C1[1] = C12.y;
            C2[0] = C22.x; C2[1] = C22.y;
        }
#pragma unroll
        for (int k = 0; k < PPT; k++) {
            const int y = pm.y0 + 4 * k;
            if (!(pm.x < cam.width && y < cam.height)) continue;
            const size_t pix = (size_t)y * cam.width + pm.x;
            image[3 * pix + 0] = __fadd_rn(C0[k], __fmul_rn(T[k], cfg.bg[0]));
            image[3 * pix + 1] = __fadd_rn(C1[k], __fmul_rn(T[k], cfg.bg[1]));
            image[3 * pix + 2] = __fadd_rn(C2[k], __fmul_rn(T[k], cfg.bg[2]));
            T_final[pix] = T[k];
            n_contrib[pix] = last[k];
        }
    }
}

// Transposed butterfly: on return lane L holds the warp sum of v[(L >> 2) & 7] (returned), and
// e holds the warp sum of the 9th term in every lane.
__device__ __forceinline__ float warp_reduce_8plus1(const float v[8], float& e, unsigned lane) {
    float a[4], b2[2];
    bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const float send = hi ? v[i] : v[i + 4];
        const float keep = hi ? v[i + 4] : v[i];
        a[i] = keep + __shfl_xor_sync(VKS_FULL_MASK, send, 16);
    }
    hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const float send = hi ? a[i] : a[i + 2];
        const float keep = hi ? a[i + 2] : a[i];
        b2[i] = keep + __shfl_xor_sync(VKS_FULL_MASK, send, 8);
    }
    hi = lane & 4;
    float c;
    {
        const float send = hi ? b2[0] : b2[1];
        const float keep = hi ? b2[1] : b2[0];
        c = keep + __shfl_xor_sync(VKS_FULL_MASK, send, 4);
    }
    c += __shfl_xor_sync(VKS_FULL_MASK, c, 2);
    c += __shfl_xor_sync(VKS_FULL_MASK, c, 1);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) e += __shfl_xor_sync(VKS_FULL_MASK, e, o);
    return c;
}

template <int PPT, int CULL, int SPARSE, bool REC = false>
__global__ void __launch_bounds__(32 * 8 / PPT, REC ? (VKS_RASTER_BWD_MINB * PPT + 1) / 2 : 1) raster_bwd_kernel(vks_config cfg, vks_camera cam,
                                                                 const float2* __restrict__ means2d,
                                                                 const float* __restrict__ conics,
                                                                 const float* __restrict__ colors,
                                                                 const float* __restrict__ opac,
                                                                 const int2* __restrict__ radii,
                                                                 const float4* __restrict__ rec,
                                                                 const uint32_t* __restrict__ vals,
                                                                 const uint32_t* __restrict__ tile_offsets,
                                                                 const uint32_t* __restrict__ tile_order,
                                                                 const float* __restrict__ T_final,
                                                                 const int* __restrict__ n_contrib,
                                                                 const float* __restrict__ dL_dimage,
                                                                 float* __restrict__ dmeans2d, float* __restrict__ dconics,
                                                                 float* __restrict__ dcolors, float* __restrict__ dopac,
                                                                 int sparse_lanes, uint32_t n) {
    pdl_wait();
    __shared__ StageT<REC> stage[8 / PPT];
    const int TX = tiles_x(cam);
    const int tile = tile_order ? (int)__ldg(tile_order + blockIdx.x) : (int)blockIdx.x;
    const unsigned lane = threadIdx.x & 31;
    StageT<REC>& s = stage[threadIdx.x >> 5];
    const PixelMap<PPT> pm = pixel_map<PPT>(tile, TX);
    const float px = (float)pm.x + 0.5f;
    const uint32_t start = tile_offsets[tile];
    VKS_DCHECK(start <= tile_offsets[tile + 1]);
    // per pixel: P = <S, w> where S is the colour composited behind the current entry (bg first):
    // dalpha only needs <c - S, w>, and <S, w> updates as P <- alpha <c, w> + (1 - alpha) P
    float py[PPT], T[PPT], w0[PPT], w1[PPT], w2[PPT], P[PPT];
    int last[PPT];
    int lmax = 0;
#pragma unroll
    for (int k = 0; k < PPT; k++) {
        const int y = pm.y0 + 4 * k;
        py[k] = (float)y + 0.5f;
        T[k] = 1.0f; w0[k] = w1[k] = w2[k] = 0.0f;
        last[k] = 0;
        if (pm.x < cam.width && y < cam.height) {
            const size_t pix = (size_t)y * cam.width + pm.x;
            T[k] = T_final[pix];
            last[k] = n_contrib[pix];
            w0[k] = dL_dimage[3 * pix];
            w1[k] = dL_dimage[3 * pix + 1];
            w2[k] = dL_dimage[3 * pix + 2];
        }
        P[k] = cfg.bg[0] * w0[k] + cfg.bg[1] * w1[k] + cfg.bg[2] * w2[k];
        lmax = max(lmax, last[k]);
    }
    const int wmax = __reduce_max_sync(VKS_FULL_MASK, lmax);  // positions >= wmax: nobody composited
    // PPT == 2: the per-pixel state as (pixel 0, pixel 1) pairs for the paired fp32 instructions
    float2 T2 = make_float2(T[0], T[PPT - 1]), P2 = make_float2(P[0], P[PPT - 1]);
    const float2 W0 = make_float2(w0[0], w0[PPT - 1]), W1 = make_float2(w1[0], w1[PPT - 1]),
                 W2 = make_float2(w2[0], w2[PPT - 1]);
    const float2 npy = make_float2(-py[0], -py[PPT - 1]);
    // per-lane destination of gradient term k after the 32-lane butterfly: lane 4k (k < 8)
    // owns term k, lane 1 the opacity term; dst(g) = base + g * stride
    const int myterm = (lane & 3) == 0 ? (int)(lane >> 2) : (lane == 1 ? 8 : -1);
    float* tbase = nullptr;
    unsigned tstride = 0;  // bytes: dst(g) = base + g * stride is one 64-bit IMAD.WIDE.U32
    // term selectors for the epilogue: term 0 -> a, term 1 -> c, both -> b (other moment),
    // conic terms 2/3/4 -> 1/2, 1, 1/2, colour terms -> 1
    const float kA = myterm == 0 ? 1.0f : 0.0f, kC = myterm == 1 ? 1.0f : 0.0f;
    const float kB = myterm == 0 || myterm == 1 ? 1.0f : 0.0f;
    const float kH = myterm == 3 ? 1.0f : (myterm == 2 || myterm == 4 ? 0.5f : 0.0f);
    const float kOne = myterm >= 5 && myterm < 8 ? 1.0f : 0.0f;
    if (myterm >= 0 && myterm < 2) { tbase = dmeans2d + myterm; tstride = 2 * sizeof(float); }
    else if (myterm >= 2 && myterm < 5) { tbase = dconics + (myterm - 2); tstride = 3 * sizeof(float); }
    else if (myterm >= 5 && myterm < 8) { tbase = dcolors + (myterm - 5); tstride = 3 * sizeof(float); }
    else if (myterm == 8) { tbase = dopac; tstride = sizeof(float); }
    // batches of 32 positions, back to front: [bs, bs+32) with bs = wmax-32, wmax-64, ...
    int bs = wmax - 32;
    int p0 = bs + (int)lane;
    uint32_t id_next = (p0 >= 0 && p0 < wmax) ? __ldg(vals + start + p0) : 0u;
    Entry e_next;
    constexpr int kAhead = REC ? kNB - 1 : 1;  // batches in flight
    if constexpr (REC) {
#pragma unroll
        for (int q = 0; q < kNB - 1; q++) {  // batches bs, bs - 32, ... (kNB - 1 of them)
            const int pq = p0 - 32 * q;
            if (q > 0) id_next = pq >= 0 ? __ldg(vals + start + pq) : 0u;
            VKS_DCHECK(!(pq >= 0 && pq < wmax) || id_next < n);
            if (pq >= 0 && pq < wmax) stage_record<VKS_RASTER_REC_CA>(s, q, (int)lane, rec, id_next);
            cp_async_commit();
        }
    } else {
        if (p0 >= 0 && p0 < wmax) e_next = gather_entry<CULL>(id_next, n, means2d, conics, colors, opac, radii);
    }
    p0 -= 32 * kAhead;
    id_next = (p0 >= 0) ? __ldg(vals + start + p0) : 0u;
    int buf = 0;
    for (; bs > -32; bs -= 32, buf = nb_next(buf)) {
        __syncwarp();
        unsigned live;
        if constexpr (REC) {
            const int p = bs - 32 * kAhead + (int)lane;  // this lane's position kAhead batches on
            VKS_DCHECK(p < 0 || id_next < n);
            if (p >= 0) stage_record<VKS_RASTER_REC_CA>(s, nb_ahead(buf), (int)lane, rec, id_next);
            cp_async_commit();
            if (p - 32 >= 0) id_next = __ldg(vals + start + p - 32);
            cp_async_wait_group<kNB - 1>();
            __syncwarp();
            const int pc = bs + (int)lane;
            bool lv = false;
            if (pc >= 0 && pc < wmax) {
                Entry e;
                e.a = s.a[buf][lane];
                e.b = s.b[buf][lane];
                lv = !culled<CULL>(e, pm.wx0, pm.wx1, pm.wy0, pm.wy1);
            }
            live = __ballot_sync(VKS_FULL_MASK, lv);
        } else {
            {
                const int p = bs + (int)lane;
                const bool ok = p >= 0 && p < wmax;
                const bool lv = ok && !culled<CULL>(e_next, pm.wx0, pm.wx1, pm.wy0, pm.wy1);
                live = __ballot_sync(VKS_FULL_MASK, lv);
                if (lv) store_entry(s, __popc(live & lanemask_lt()), lane, e_next);
            }
            __syncwarp();
            {
                const int p = bs - 32 + (int)lane;
                if (p >= 0) e_next = gather_entry<CULL>(id_next, n, means2d, conics, colors, opac, radii);
                if (p - 32 >= 0) id_next = __ldg(vals + start + p - 32);
            }
        }
        for (int q = __popc(live) - 1; q >= 0; q--) {  // back to front over the live entries
            float4 A, B, Cc;
            if constexpr (REC) {  // the live slots in place: highest set bit first
                const int j = 31 - __clz(live);
                live &= ~(1u << j);
                A = s.a[buf][j];
                B = s.b[buf][j];
                Cc = s.c[buf][j];
                Cc.z = __int_as_float(j);
            } else {
                A = s.a[q];
                B = s.b[q];
                Cc = s.c[q];
            }
            const int pos = bs + __float_as_int(Cc.z);
            const float c0 = B.z, c1 = B.w, c2 = Cc.x;
            // v[0..4]: moments sum(g dx), sum(g dy), sum(g dx^2), sum(g dx dy), sum(g dy^2) with
            // g = G dalpha (dL/dsigma = -rho g); v[5..7]: colour; e = sum(g) (dL/drho)
            float v[8], e = 0.0f;
            bool contrib = false;
            if constexpr (PPT == 2) {
                // the two pixels on paired fp32 instructions (eval_alpha2: the forward's decisions)
                float dx;
                float2 dy, G, rG, alpha;
                bool e0, e1;
                eval_alpha2(A, B, px, npy, dx, dy, G, rG, alpha, e0, e1);
                const bool ok0 = e0 && pos < last[0], ok1 = e1 && pos < last[1];
                contrib = ok0 || ok1;
                if (SPARSE && !__any_sync(VKS_FULL_MASK, contrib)) continue;
                // branch-free: an entry the pixel did not composite replays with alpha = 0, which
                // leaves T, P and every accumulator bit-identical (T * 1, 0 * x + P, + 0)
                const float2 a = make_float2(ok0 ? alpha.x : 0.0f, ok1 ? alpha.y : 0.0f);
                const float2 om = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-a.x, -a.y));
                T2 = __fmul2_rn(T2, make_float2(rcp_ftz(om.x), rcp_ftz(om.y)));  // om in [0.01, 1]
                const float2 aT = __fmul2_rn(a, T2);
                const float2 cw = __ffma2_rn(make_float2(c2, c2), W2,
                                             __ffma2_rn(make_float2(c1, c1), W1, __fmul2_rn(make_float2(c0, c0), W0)));
                const float2 d = __fadd2_rn(cw, make_float2(-P2.x, -P2.y));
                const float2 dalpha = __fmul2_rn(T2, d);
                P2 = SPARSE ? __ffma2_rn(a, d, P2) : __ffma2_rn(a, cw, __fmul2_rn(om, P2));
                // no gradient where the pixel skipped the entry or alpha was clamped
                const float2 gg = __fmul2_rn(G, dalpha);
                const float2 g = make_float2((!ok0 || rG.x > 0.99f) ? 0.0f : gg.x, (!ok1 || rG.y > 0.99f) ? 0.0f : gg.y);
                const float2 gx = __fmul2_rn(g, make_float2(dx, dx)), gy = __fmul2_rn(g, dy);
                const float2 gxx = __fmul2_rn(gx, make_float2(dx, dx)), gxy = __fmul2_rn(gx, dy), gyy = __fmul2_rn(gy, dy);
                const float2 t5 = __fmul2_rn(aT, W0), t6 = __fmul2_rn(aT, W1), t7 = __fmul2_rn(aT, W2);
                v[0] = gx.x + gx.y; v[1] = gy.x + gy.y; v[2] = gxx.x + gxx.y; v[3] = gxy.x + gxy.y;
                v[4] = gyy.x + gyy.y; v[5] = t5.x + t5.y; v[6] = t6.x + t6.y; v[7] = t7.x + t7.y;
                e = g.x + g.y;
            } else {
                // evaluate first: an entry no pixel of the warp composited leaves every T, P and
                // accumulator unchanged, so the warp skips it
                float dx[PPT], dy[PPT], G[PPT], rG[PPT], alpha[PPT];
                bool okk[PPT];
#pragma unroll
                for (int k = 0; k < PPT; k++) {
                    okk[k] = eval_alpha(A, B, px, py[k], dx[k], dy[k], G[k], rG[k], alpha[k]) && pos < last[k];
                    contrib = contrib || okk[k];
                }
                // SPARSE: an entry no pixel of the warp composited leaves every T, P and accumulator
                // unchanged, so the warp skips it
                if (SPARSE && !__any_sync(VKS_FULL_MASK, contrib)) continue;
#pragma unroll
                for (int k = 0; k < PPT; k++) {
                    // branch-free: an entry the pixel did not composite replays with alpha = 0, which
                    // leaves T, P and every accumulator bit-identical (T * 1, 0 * x + P, + 0)
                    const bool ok = okk[k];
                    const float a = ok ? alpha[k] : 0.0f;
                    const float om = 1.0f - a;
                    T[k] = T[k] * rcp_ftz(om);  // om in [0.01, 1]
                    const float aT = a * T[k];
                    const float cw = c0 * w0[k] + c1 * w1[k] + c2 * w2[k];
                    const float d = cw - P[k];
                    const float dalpha = T[k] * d;
                    P[k] = SPARSE ? fmaf(a, d, P[k]) : a * cw + om * P[k];
                    // no gradient where the pixel skipped the entry or alpha was clamped
                    const float g = (!ok || rG[k] > 0.99f) ? 0.0f : G[k] * dalpha;
                    const float gx = g * dx[k], gy = g * dy[k];
                    const float t[8] = {gx, gy, gx * dx[k], gx * dy[k], gy * dy[k], aT * w0[k], aT * w1[k], aT * w2[k]};
#pragma unroll
                    for (int q = 0; q < 8; q++) v[q] = k == 0 ? t[q] : v[q] + t[q];
                    e = k == 0 ? g : e + g;
                }
            }
            // SPARSE: an entry composited by at most `sparse_lanes` lanes is reduced by those lanes'
            // own atomics (the outputs are linear in the sums) instead of the 32-lane butterfly
            const unsigned cl = __ballot_sync(VKS_FULL_MASK, contrib);
            if (SPARSE && __popc(cl) <= sparse_lanes) {
                if (contrib) {
                    const uint32_t id = __float_as_uint(Cc.y);
                    const float nrho = -B.y;
                    atomicAdd(dmeans2d + 2 * (size_t)id, nrho * fmaf(2.0f * A.z, v[0], A.w * v[1]));
                    atomicAdd(dmeans2d + 2 * (size_t)id + 1, nrho * fmaf(2.0f * B.x, v[1], A.w * v[0]));
                    atomicAdd(dconics + 3 * (size_t)id, nrho * 0.5f * v[2]);
                    atomicAdd(dconics + 3 * (size_t)id + 1, nrho * v[3]);
                    atomicAdd(dconics + 3 * (size_t)id + 2, nrho * 0.5f * v[4]);
                    atomicAdd(dcolors + 3 * (size_t)id, v[5]);
                    atomicAdd(dcolors + 3 * (size_t)id + 1, v[6]);
                    atomicAdd(dcolors + 3 * (size_t)id + 2, v[7]);
                    atomicAdd(dopac + id, e);
                }
            } else if (cl) {
                const float r = warp_reduce_8plus1(v, e, lane);
                const float other = __shfl_xor_sync(VKS_FULL_MASK, r, 4);  // lanes 0 <-> 4: the two first moments
                // dmean = -rho (a m_x + b m_y, b m_x + c m_y), dconic = -rho (m_xx / 2, m_xy, m_yy / 2),
                // colour = r, opacity = e; branch-free with the lane's constant term selectors
                const float nrho = -B.y;
                const float cr = fmaf(nrho, fmaf(kA, 2.0f * A.z, fmaf(kC, 2.0f * B.x, kH)), kOne);
                const float out = myterm == 8 ? e : fmaf(cr, r, (nrho * kB * A.w) * other);
                if (myterm >= 0)
                    atomicAdd(reinterpret_cast<float*>(reinterpret_cast<char*>(tbase) +
                                                       (unsigned long long)__float_as_uint(Cc.y) * tstride), out);
            }
        }
    }
    if constexpr (REC) cp_async_wait_all();  // no copy outlives the warp
}

template <int PPT, int CULL, bool REC = false>
int launch_fwd(const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
               const float* colors, const float* opacities, const int32_t* radii, const float* records,
               const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order, float* image,
               float* T_final, int32_t* n_contrib, uint32_t n, cudaStream_t st) {
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    launch_k(raster_fwd_kernel<PPT, CULL, false, REC>, n_tiles, 32 * 8 / PPT, 0, st,
        cfg, cam, reinterpret_cast<const float2*>(means2d), conics, colors, opacities,
        reinterpret_cast<const int2*>(radii), reinterpret_cast<const float4*>(records), vals, tile_offsets, tile_order,
        image, T_final, n_contrib, n, nullptr);
    return LaunchCheck::check();
}

template <int PPT, int CULL, int SPARSE, bool REC = false>
int launch_bwd(const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
               const float* colors, const float* opacities, const int32_t* radii, const float* records,
               const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order, const float* T_final,
               const int32_t* n_contrib, const float* dL_dimage, float* dmeans2d, float* dconics, float* dcolors,
               float* dopacities, int sparse_lanes, uint32_t n, cudaStream_t st) {
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    launch_k(raster_bwd_kernel<PPT, CULL, SPARSE, REC>, n_tiles, 32 * 8 / PPT, 0, st,
        cfg, cam, reinterpret_cast<const float2*>(means2d), conics, colors, opacities,
        reinterpret_cast<const int2*>(radii), reinterpret_cast<const float4*>(records), vals, tile_offsets, tile_order,
        T_final, n_contrib, dL_dimage, dmeans2d, dconics, dcolors, dopacities, sparse_lanes, n);
    return LaunchCheck::check();
}

// patch culling: ellipse by default (valid for both footprints); the box test needs the support
// footprint's radii, so it falls back to no culling under 3SIGMA
int cull_choice(const vks_config& cfg) {
    const int mode = env_choice("VKS_RASTER_CULL", kCullEllipse, kCullNone, kCullEllipse);  // read per call (tests switch it)
    if (mode == kCullBox && cfg.footprint != VKS_FOOTPRINT_SUPPORT) return kCullNone;
    return mode;
}

// pixels per thread: 2 (8x8 warp patches) by default, 1 (8x4) or 4 (8x16) on request
int ppt_choice(const char* var) {
    const int v = env_choice(var, 2, 1, 4);
    return v == 3 ? 2 : v;
}

// the records path (cp.async staging of the packed records) serves every layout with the exact
// ellipse test or no culling; the diagnostic box-culling mode gathers from the separate arrays
// (it needs the radii)
bool use_records(const float* records, int ppt, int cull) {
    (void)ppt;
    return records != nullptr && cull != kCullBox;
}

template <int PPT>
int dispatch_fwd(int cull, const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
                 const float* colors, const float* opacities, const int32_t* radii, const uint32_t* vals,
                 const uint32_t* tile_offsets, const uint32_t* tile_order, float* image, float* T_final,
                 int32_t* n_contrib, uint32_t n, cudaStream_t st) {
#define VKS_FWD_ARGS cfg, cam, means2d, conics, colors, opacities, radii, nullptr, vals, tile_offsets, tile_order, \
                     image, T_final, n_contrib, n, st
    switch (cull) {
        case kCullNone: return launch_fwd<PPT, kCullNone>(VKS_FWD_ARGS);
        case kCullBox: return launch_fwd<PPT, kCullBox>(VKS_FWD_ARGS);
        default: return launch_fwd<PPT, kCullEllipse>(VKS_FWD_ARGS);
    }
#undef VKS_FWD_ARGS
}

template <int PPT>
int dispatch_bwd(int cull, const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
                 const float* colors, const float* opacities, const int32_t* radii, const float* records,
                 const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order, const float* T_final,
                 const int32_t* n_contrib, const float* dL_dimage, float* dmeans2d, float* dconics, float* dcolors,
                 float* dopacities, uint32_t n, cudaStream_t st) {
    // SPARSE (default): skip entries no pixel of the warp composited, and reduce entries composited
    // by <= VKS_RASTER_SPARSE lanes (default 4) with per-lane atomics; VKS_RASTER_BWD_SPARSE=0: the
    // 32-lane butterfly for every entry (round-1 kernel, kept for A/B measurements)
    const int sparse = env_choice("VKS_RASTER_BWD_SPARSE", 1, 0, 1);
    const int lanes = env_choice("VKS_RASTER_SPARSE", 4, 0, 32);
#define VKS_BWD_ARGS cfg, cam, means2d, conics, colors, opacities, radii, records, vals, tile_offsets, tile_order, \
                     T_final, n_contrib, dL_dimage, dmeans2d, dconics, dcolors, dopacities, lanes, n, st
    if (use_records(records, PPT, cull)) {
        if (sparse)
            return cull == kCullNone ? launch_bwd<PPT, kCullNone, 1, true>(VKS_BWD_ARGS)
                                     : launch_bwd<PPT, kCullEllipse, 1, true>(VKS_BWD_ARGS);
        return cull == kCullNone ? launch_bwd<PPT, kCullNone, 0, true>(VKS_BWD_ARGS)
                                 : launch_bwd<PPT, kCullEllipse, 0, true>(VKS_BWD_ARGS);
    }
#define VKS_BWD_CULL(SP)                                                                 \
    switch (cull) {                                                                      \
        case kCullNone: return launch_bwd<PPT, kCullNone, SP>(VKS_BWD_ARGS);             \
        case kCullBox: return launch_bwd<PPT, kCullBox, SP>(VKS_BWD_ARGS);               \
        default: return launch_bwd<PPT, kCullEllipse, SP>(VKS_BWD_ARGS);                 \
    }
    if (sparse) VKS_BWD_CULL(1)
    VKS_BWD_CULL(0)
#undef VKS_BWD_CULL
#undef VKS_BWD_ARGS
}

}  // namespace

int launch_raster_fwd_stats(const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
                            const float* colors, const float* opacities, const int32_t* radii, const float* records,
                            const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                            unsigned long long* stats, int64_t n, cudaStream_t st) {
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    const auto m2 = reinterpret_cast<const float2*>(means2d);
    const auto r2 = reinterpret_cast<const int2*>(radii);
    const auto rc = reinterpret_cast<const float4*>(records);
    const int cull = cull_choice(cfg);
    if (!use_records(records, 2, cull) && n > 0 && !conics) return VKS_ERR_INVALID_ARG;
#define VKS_STATS_ARGS cfg, cam, m2, conics, colors, opacities, r2, rc, vals, tile_offsets, tile_order, nullptr, nullptr, \
                       nullptr, (uint32_t)n, stats
    if (use_records(records, 2, cull)) {
        if (cull == kCullNone) raster_fwd_kernel<2, kCullNone, true, true><<<n_tiles, 128, 0, st>>>(VKS_STATS_ARGS);
        else raster_fwd_kernel<2, kCullEllipse, true, true><<<n_tiles, 128, 0, st>>>(VKS_STATS_ARGS);
        return LaunchCheck::check();
    }
    switch (cull) {
        case kCullNone: raster_fwd_kernel<2, kCullNone, true><<<n_tiles, 128, 0, st>>>(VKS_STATS_ARGS); break;
        case kCullBox: raster_fwd_kernel<2, kCullBox, true><<<n_tiles, 128, 0, st>>>(VKS_STATS_ARGS); break;
        default: raster_fwd_kernel<2, kCullEllipse, true><<<n_tiles, 128, 0, st>>>(VKS_STATS_ARGS);
    }
#undef VKS_STATS_ARGS
    return LaunchCheck::check();
}

int launch_raster_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const float* records, const uint32_t* vals, const uint32_t* tile_offsets,
                      const uint32_t* tile_order, float* image, float* T_final, int32_t* n_contrib, cudaStream_t st) {
    const int ppt = ppt_choice("VKS_RASTER_FWD_PPT");
    const int cull = cull_choice(cfg);
    if (!use_records(records, ppt, cull) && n > 0 && !conics) return VKS_ERR_INVALID_ARG;  // a gather mode needs them
    if (use_records(records, ppt, cull)) {
#define VKS_FWD_REC(P) return cull == kCullNone                                                                  \
        ? launch_fwd<P, kCullNone, true>(cfg, cam, means2d, conics, colors, opacities, radii, records, vals,           \
                                         tile_offsets, tile_order, image, T_final, n_contrib, (uint32_t)n, st)       \
        : launch_fwd<P, kCullEllipse, true>(cfg, cam, means2d, conics, colors, opacities, radii, records, vals,        \
                                            tile_offsets, tile_order, image, T_final, n_contrib, (uint32_t)n, st)
        if (ppt == 4) VKS_FWD_REC(4);
        if (ppt == 1) VKS_FWD_REC(1);
        VKS_FWD_REC(2);
#undef VKS_FWD_REC
    }
    if (ppt == 4) return dispatch_fwd<4>(cull, cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, tile_order, image, T_final, n_contrib, (uint32_t)n, st);
    if (ppt == 1) return dispatch_fwd<1>(cull, cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, tile_order, image, T_final, n_contrib, (uint32_t)n, st);
    return dispatch_fwd<2>(cull, cfg, cam, means2d, conics, colors, opacities, radii, vals, tile_offsets, tile_order, image, T_final, n_contrib, (uint32_t)n, st);
}

int launch_raster_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const float* records, const uint32_t* vals, const uint32_t* tile_offsets,
                      const uint32_t* tile_order, const float* T_final, const int32_t* n_contrib,
                      const float* dL_dimage, float* dmeans2d, float* dconics, float* dcolors, float* dopacities,
                      cudaStream_t st) {
    const int ppt = ppt_choice("VKS_RASTER_BWD_PPT");
    const int cull = cull_choice(cfg);
    if (!use_records(records, ppt, cull) && n > 0 && !conics) return VKS_ERR_INVALID_ARG;  // a gather mode needs them
#define VKS_RB_ARGS cull, cfg, cam, means2d, conics, colors, opacities, radii, records, vals, tile_offsets, tile_order, \
                    T_final, n_contrib, dL_dimage, dmeans2d, dconics, dcolors, dopacities, (uint32_t)n, st
    if (ppt == 4) return dispatch_bwd<4>(VKS_RB_ARGS);
    if (ppt == 1) return dispatch_bwd<1>(VKS_RB_ARGS);
    return dispatch_bwd<2>(VKS_RB_ARGS);
#undef VKS_RB_ARGS
}

}  // namespace vks
