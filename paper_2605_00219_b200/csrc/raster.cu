// raster.cu — "Rasterization Forward" and "Rasterization Backward";
// DESIGN.md §4.3-4.4 and §6.
//
// One 256-thread block per 16x16 tile; each warp owns an 8x4 pixel patch and walks the tile's
// sorted list on its own in batches of 32 staged into its shared-memory slice as packed float4
// records (software-pipelined: ids two batches ahead, records one batch ahead), so there are no
// block barriers and a warp stops as soon as its own 32 pixels are saturated.  Before evaluating a Gaussian a warp
// tests its 8x4 patch against the Gaussian's support box (support footprint only; the box is the
// projection's radii plus a safety margin, so no pixel whose alpha could reach 1/255 is skipped)
// and skips it warp-uniformly, which removes most of the evaluations that would be rejected by
// the 1/255 test anyway.  Forward and backward evaluate sigma / alpha through the SAME inline
// function, so skip / clamp / stop decisions replay identically; sigma, alpha and the colour
// accumulation follow the pinned fp32 order of DESIGN.md §4.3 (only exp differs from the oracle:
// ex2.approx here, expf there).  The backward reduces each Gaussian's 9 gradient terms across the
// warp with a transposed butterfly (14 shuffles instead of 45) and issues 2 atomic instructions per
// (warp, Gaussian) that any lane touched.
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;

// One warp's staged batch of 32 list entries (each warp walks the tile list on its own: no block
// barriers, so a warp never waits for a slower one and stops as soon as its own pixels are done).
struct WarpStage {
    float4 a[32];    // u, v, 0.5*a, b
    float4 b[32];    // 0.5*c, rho, c0, c1
    float4 box[32];  // support box of pixel centres: xmin, xmax, ymin, ymax
    float c2[32];
    uint32_t id[32];
};

struct Entry {  // one lane's gathered entry, in registers until it is stored to the stage
    float4 a, b, box;
    float c2;
    uint32_t id;
};

__device__ __forceinline__ Entry gather_entry(uint32_t g, bool cull, const float2* __restrict__ means2d,
                                              const float* __restrict__ conics, const float* __restrict__ colors,
                                              const float* __restrict__ opac, const int2* __restrict__ radii) {
    Entry e;
    const float2 uv = __ldg(means2d + g);
    const float ca = __ldg(conics + 3 * (size_t)g), cb = __ldg(conics + 3 * (size_t)g + 1),
                cc = __ldg(conics + 3 * (size_t)g + 2);
    const float r0 = __ldg(colors + 3 * (size_t)g), r1 = __ldg(colors + 3 * (size_t)g + 1);
    e.c2 = __ldg(colors + 3 * (size_t)g + 2);
    const float rho = __ldg(opac + g);
    e.id = g;
    e.a = make_float4(uv.x, uv.y, 0.5f * ca, cb);
    e.b = make_float4(0.5f * cc, rho, r0, r1);
    if (cull) {
        // radii = ceil(sqrt(2 k' Sigma'_xx)) + 1 with k' > ln(255 rho): every pixel centre whose
        // alpha can reach 1/255 lies inside u +- rx; widen by 1 + rx/64 px more for fp32 slack.
        const int2 r = __ldg(radii + g);
        const float mx = (float)r.x * (1.0f + 1.0f / 64.0f) + 1.0f;
        const float my = (float)r.y * (1.0f + 1.0f / 64.0f) + 1.0f;
        e.box = make_float4(uv.x - mx, uv.x + mx, uv.y - my, uv.y + my);
    } else {
        e.box = make_float4(-INFINITY, INFINITY, -INFINITY, INFINITY);
    }
    return e;
}

__device__ __forceinline__ void store_entry(WarpStage& s, int lane, const Entry& e) {
    s.a[lane] = e.a;
    s.b[lane] = e.b;
    s.box[lane] = e.box;
    s.c2[lane] = e.c2;
    s.id[lane] = e.id;
}

// warp patch [x0+0.5, x0+7.5] x [y0+0.5, y0+3.5] misses the support box
__device__ __forceinline__ bool culled(const float4 bx, float wx0, float wx1, float wy0, float wy1) {
    return bx.y < wx0 || bx.x > wx1 || bx.w < wy0 || bx.z > wy1;
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
    if (sigma < 0.0f) return false;
    G = exp2_ftz(sigma * -1.44269504088896341f);
    rG = B.y * G;
    alpha = fminf(0.99f, rG);
    return !(alpha < 1.0f / 255.0f);
}

struct PixelMap {
    int x, y;                  // pixel
    float wx0, wx1, wy0, wy1;  // warp patch (pixel centres)
};

__device__ __forceinline__ PixelMap pixel_map(int tile, int TX) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = (tile % TX) * kTile + (warp & 1) * 8;
    const int by = (tile / TX) * kTile + (warp >> 1) * 4;
    PixelMap m;
    m.x = bx + (lane & 7);
    m.y = by + (lane >> 3);
    m.wx0 = (float)bx + 0.5f;
    m.wx1 = (float)bx + 7.5f;
    m.wy0 = (float)by + 0.5f;
    m.wy1 = (float)by + 3.5f;
    return m;
}

__global__ void __launch_bounds__(kThreads) raster_fwd_kernel(vks_config cfg, vks_camera cam,
                                                              const float2* __restrict__ means2d,
                                                              const float* __restrict__ conics,
                                                              const float* __restrict__ colors,
                                                              const float* __restrict__ opac,
                                                              const int2* __restrict__ radii,
                                                              const uint32_t* __restrict__ vals,
                                                              const uint32_t* __restrict__ tile_offsets,
                                                              float* __restrict__ image, float* __restrict__ T_final,
                                                              int* __restrict__ n_contrib) {
    __shared__ WarpStage stage[kWarpsPerBlock];
    const int TX = tiles_x(cam);
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31;
    WarpStage& s = stage[threadIdx.x >> 5];
    const PixelMap pm = pixel_map(tile, TX);
    const bool inside = pm.x < cam.width && pm.y < cam.height;
    const bool cull = cfg.footprint == VKS_FOOTPRINT_SUPPORT;
    const float px = (float)pm.x + 0.5f, py = (float)pm.y + 0.5f;
    const uint32_t start = tile_offsets[tile], end = tile_offsets[tile + 1];
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int last = 0;
    bool done = !inside;
    // software pipeline: ids two batches ahead, gathered entries one batch ahead
    uint32_t id_next = (start + lane < end) ? __ldg(vals + start + lane) : 0u;
    Entry e_next;
    if (start + lane < end) e_next = gather_entry(id_next, cull, means2d, conics, colors, opac, radii);
    id_next = (start + 32 + lane < end) ? __ldg(vals + start + 32 + lane) : 0u;
    for (uint32_t b = start; b < end; b += 32) {
        if (__all_sync(VKS_FULL_MASK, done)) break;
        __syncwarp();
        // each lane tests its own entry against the warp patch; the warp then visits only the
        // entries whose support box meets the patch, in list order
        unsigned live = __ballot_sync(VKS_FULL_MASK, b + lane < end &&
                                                         !culled(e_next.box, pm.wx0, pm.wx1, pm.wy0, pm.wy1));
        if (b + lane < end) store_entry(s, lane, e_next);
        __syncwarp();
        if (b + 32 + lane < end) e_next = gather_entry(id_next, cull, means2d, conics, colors, opac, radii);
        if (b + 64 + lane < end) id_next = __ldg(vals + b + 64 + lane);
        while (live) {
            const int j = __ffs(live) - 1;
            live &= live - 1;
            if (done) continue;
            const float4 A = s.a[j], B = s.b[j];
            float dx, dy, G, rG, alpha;
            if (!eval_alpha(A, B, px, py, dx, dy, G, rG, alpha)) continue;
            const float aT = alpha * T;
            C0 = fmaf(B.z, aT, C0);
            C1 = fmaf(B.w, aT, C1);
            C2 = fmaf(s.c2[j], aT, C2);
            T = T * (1.0f - alpha);
            last = (int)(b - start) + j + 1;
            if (T < 1e-4f) done = true;
        }
    }
    if (!inside) return;
    const size_t pix = (size_t)pm.y * cam.width + pm.x;
    image[3 * pix + 0] = __fadd_rn(C0, __fmul_rn(T, cfg.bg[0]));
    image[3 * pix + 1] = __fadd_rn(C1, __fmul_rn(T, cfg.bg[1]));
    image[3 * pix + 2] = __fadd_rn(C2, __fmul_rn(T, cfg.bg[2]));
    T_final[pix] = T;
    n_contrib[pix] = last;
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

__global__ void __launch_bounds__(kThreads) raster_bwd_kernel(vks_config cfg, vks_camera cam,
                                                              const float2* __restrict__ means2d,
                                                              const float* __restrict__ conics,
                                                              const float* __restrict__ colors,
                                                              const float* __restrict__ opac,
                                                              const int2* __restrict__ radii,
                                                              const uint32_t* __restrict__ vals,
                                                              const uint32_t* __restrict__ tile_offsets,
                                                              const float* __restrict__ T_final,
                                                              const int* __restrict__ n_contrib,
                                                              const float* __restrict__ dL_dimage,
                                                              float* __restrict__ dmeans2d, float* __restrict__ dconics,
                                                              float* __restrict__ dcolors, float* __restrict__ dopac) {
    __shared__ WarpStage stage[kWarpsPerBlock];
    const int TX = tiles_x(cam);
    const int tile = blockIdx.x;
    const unsigned lane = threadIdx.x & 31;
    WarpStage& s = stage[threadIdx.x >> 5];
    const PixelMap pm = pixel_map(tile, TX);
    const bool inside = pm.x < cam.width && pm.y < cam.height;
    const bool cull = cfg.footprint == VKS_FOOTPRINT_SUPPORT;
    const float px = (float)pm.x + 0.5f, py = (float)pm.y + 0.5f;
    const uint32_t start = tile_offsets[tile];
    float T = 1.0f, w0 = 0.0f, w1 = 0.0f, w2 = 0.0f;
    int last = 0;
    if (inside) {
        const size_t pix = (size_t)pm.y * cam.width + pm.x;
        T = T_final[pix];
        last = n_contrib[pix];
        w0 = dL_dimage[3 * pix];
        w1 = dL_dimage[3 * pix + 1];
        w2 = dL_dimage[3 * pix + 2];
    }
    float S0 = cfg.bg[0], S1 = cfg.bg[1], S2 = cfg.bg[2];
    const int wmax = __reduce_max_sync(VKS_FULL_MASK, last);  // positions >= wmax: nobody composited
    // lane 4k (k < 8) owns gradient term k after the butterfly, lane 1 the opacity term
    const int myterm = (lane & 3) == 0 ? (int)(lane >> 2) : (lane == 1 ? 8 : -1);
    // batches of 32 positions, back to front: [bs, bs+32) with bs = wmax-32, wmax-64, ...
    int bs = wmax - 32;
    int p0 = bs + (int)lane;
    uint32_t id_next = (p0 >= 0 && p0 < wmax) ? __ldg(vals + start + p0) : 0u;
    Entry e_next;
    if (p0 >= 0 && p0 < wmax) e_next = gather_entry(id_next, cull, means2d, conics, colors, opac, radii);
    p0 -= 32;
    id_next = (p0 >= 0) ? __ldg(vals + start + p0) : 0u;
    for (; bs > -32; bs -= 32) {
        __syncwarp();
        unsigned live;
        {
            const int p = bs + (int)lane;
            const bool ok = p >= 0 && p < wmax;
            live = __ballot_sync(VKS_FULL_MASK, ok && !culled(e_next.box, pm.wx0, pm.wx1, pm.wy0, pm.wy1));
            if (ok) store_entry(s, lane, e_next);
        }
        __syncwarp();
        {
            const int p = bs - 32 + (int)lane;
            if (p >= 0) e_next = gather_entry(id_next, cull, means2d, conics, colors, opac, radii);
            if (p - 32 >= 0) id_next = __ldg(vals + start + p - 32);
        }
        while (live) {  // back to front over the entries whose support box meets the patch
            const int j = 31 - __clz(live);
            live &= ~(1u << j);
            const int pos = bs + j;
            float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            float e = 0.0f;
            bool contrib = false;
            if (pos < last) {
                const float4 A = s.a[j], B = s.b[j];
                float dx, dy, G, rG, alpha;
                if (eval_alpha(A, B, px, py, dx, dy, G, rG, alpha)) {
                    contrib = true;
                    T = __fdividef(T, 1.0f - alpha);
                    const float aT = alpha * T;
                    const float c0 = B.z, c1 = B.w, c2 = s.c2[j];
                    v[5] = aT * w0;
                    v[6] = aT * w1;
                    v[7] = aT * w2;
                    const float dalpha = T * ((c0 - S0) * w0 + (c1 - S1) * w1 + (c2 - S2) * w2);
                    S0 = alpha * c0 + (1.0f - alpha) * S0;
                    S1 = alpha * c1 + (1.0f - alpha) * S1;
                    S2 = alpha * c2 + (1.0f - alpha) * S2;
                    if (!(rG > 0.99f)) {
                        const float dsig = -rG * dalpha;
                        const float a = 2.0f * A.z, bb = A.w, c = 2.0f * B.x;
                        v[0] = (a * dx + bb * dy) * dsig;
                        v[1] = (bb * dx + c * dy) * dsig;
                        v[2] = 0.5f * dx * dx * dsig;
                        v[3] = dx * dy * dsig;
                        v[4] = 0.5f * dy * dy * dsig;
                        e = G * dalpha;
                    }
                }
            }
            if (__any_sync(VKS_FULL_MASK, contrib)) {
                const float r = warp_reduce_8plus1(v, e, lane);
                if (myterm >= 0) {
                    const uint32_t g = s.id[j];
                    float* dst;
                    float val = r;
                    if (myterm < 2) dst = dmeans2d + 2 * (size_t)g + myterm;
                    else if (myterm < 5) dst = dconics + 3 * (size_t)g + (myterm - 2);
                    else if (myterm < 8) dst = dcolors + 3 * (size_t)g + (myterm - 5);
                    else { dst = dopac + g; val = e; }
                    atomicAdd(dst, val);
                }
            }
        }
    }
}

}  // namespace

int launch_raster_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const uint32_t* vals, const uint32_t* tile_offsets, float* image, float* T_final,
                      int32_t* n_contrib, cudaStream_t st) {
    (void)n;
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    raster_fwd_kernel<<<n_tiles, kThreads, 0, st>>>(cfg, cam, reinterpret_cast<const float2*>(means2d), conics,
                                                    colors, opacities, reinterpret_cast<const int2*>(radii), vals,
                                                    tile_offsets, image, T_final, n_contrib);
    return LaunchCheck::check();
}

int launch_raster_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const uint32_t* vals, const uint32_t* tile_offsets, const float* T_final,
                      const int32_t* n_contrib, const float* dL_dimage, float* dmeans2d, float* dconics,
                      float* dcolors, float* dopacities, cudaStream_t st) {
    (void)n;
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    raster_bwd_kernel<<<n_tiles, kThreads, 0, st>>>(cfg, cam, reinterpret_cast<const float2*>(means2d), conics,
                                                    colors, opacities, reinterpret_cast<const int2*>(radii), vals,
                                                    tile_offsets, T_final, n_contrib, dL_dimage, dmeans2d, dconics,
                                                    dcolors, dopacities);
    return LaunchCheck::check();
}

}  // namespace vks
