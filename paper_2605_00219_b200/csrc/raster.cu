// raster.cu — "Rasterization Forward" and "Rasterization Backward";
// DESIGN.md §4.4-4.5 and §6.
//
// One 256-thread block per 16x16 tile, one thread per pixel.  The tile's sorted Gaussian list is
// walked in batches of 256 staged into shared memory (one coalesced gather per batch; the batch is
// reused by all 256 pixels).  The forward stops a block as soon as every pixel has T < 1e-4
// (__syncthreads_count).  Forward and backward evaluate sigma / alpha through the SAME inline
// function, so skip / clamp / stop decisions replay identically; sigma, alpha and the colour
// accumulation follow the pinned fp32 order of DESIGN.md §4.4 (only exp differs from the oracle:
// ex2.approx here, expf there).  The backward reduces each Gaussian's 9 gradient terms across the
// warp with a transposed butterfly (14 shuffles instead of 45) and issues 2 atomic instructions
// per (warp, Gaussian) that any lane touched.
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kThreads = 256;

struct Stage {
    float2 uv[kThreads];
    float ha[kThreads], b[kThreads], hc[kThreads], rho[kThreads];
    float col[3][kThreads];
    uint32_t id[kThreads];
};

__device__ __forceinline__ void stage_batch(Stage& s, int j, uint32_t g, const float2* __restrict__ means2d,
                                            const float* __restrict__ conics, const float* __restrict__ colors,
                                            const float* __restrict__ opac) {
    s.id[j] = g;
    s.uv[j] = __ldg(means2d + g);
    s.ha[j] = 0.5f * __ldg(conics + 3 * (size_t)g);
    s.b[j] = __ldg(conics + 3 * (size_t)g + 1);
    s.hc[j] = 0.5f * __ldg(conics + 3 * (size_t)g + 2);
    s.rho[j] = __ldg(opac + g);
    s.col[0][j] = __ldg(colors + 3 * (size_t)g);
    s.col[1][j] = __ldg(colors + 3 * (size_t)g + 1);
    s.col[2][j] = __ldg(colors + 3 * (size_t)g + 2);
}

// sigma = 1/2 a dx^2 + b dx dy + 1/2 c dy^2 in the pinned order; returns false when skipped
// (sigma < 0 or alpha < 1/255).  G = exp(-sigma) via ex2.approx.
__device__ __forceinline__ bool eval_alpha(const Stage& s, int j, float px, float py, float& dx, float& dy,
                                           float& G, float& rG, float& alpha) {
    dx = s.uv[j].x - px;
    dy = s.uv[j].y - py;
    const float sigma = fmaf(s.ha[j] * dx, dx, fmaf(s.hc[j] * dy, dy, (s.b[j] * dx) * dy));
    if (sigma < 0.0f) return false;
    G = __expf(-sigma);
    rG = s.rho[j] * G;
    alpha = fminf(0.99f, rG);
    return !(alpha < 1.0f / 255.0f);
}

__global__ void __launch_bounds__(kThreads) raster_fwd_kernel(vks_config cfg, vks_camera cam,
                                                              const float2* __restrict__ means2d,
                                                              const float* __restrict__ conics,
                                                              const float* __restrict__ colors,
                                                              const float* __restrict__ opac,
                                                              const uint32_t* __restrict__ vals,
                                                              const uint32_t* __restrict__ tile_offsets,
                                                              float* __restrict__ image, float* __restrict__ T_final,
                                                              int* __restrict__ n_contrib) {
    __shared__ Stage s;
    const int TX = tiles_x(cam);
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    const int x = (tile % TX) * kTile + (tid & 15);
    const int y = (tile / TX) * kTile + (tid >> 4);
    const bool inside = x < cam.width && y < cam.height;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    const uint32_t start = tile_offsets[tile], end = tile_offsets[tile + 1];
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int last = 0;
    bool done = !inside;
    for (uint32_t b = start; b < end; b += kThreads) {
        if (__syncthreads_count(done) == kThreads) break;
        if (b + tid < end) stage_batch(s, tid, __ldg(vals + b + tid), means2d, conics, colors, opac);
        __syncthreads();
        const int nb = (int)min((uint32_t)kThreads, end - b);
        if (!done) {
            for (int j = 0; j < nb; j++) {
                float dx, dy, G, rG, alpha;
                if (!eval_alpha(s, j, px, py, dx, dy, G, rG, alpha)) continue;
                const float aT = alpha * T;
                C0 = fmaf(s.col[0][j], aT, C0);
                C1 = fmaf(s.col[1][j], aT, C1);
                C2 = fmaf(s.col[2][j], aT, C2);
                T = T * (1.0f - alpha);
                last = (int)(b - start) + j + 1;
                if (T < 1e-4f) { done = true; break; }
            }
        }
    }
    if (!inside) return;
    const size_t pix = (size_t)y * cam.width + x;
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
                                                              const uint32_t* __restrict__ vals,
                                                              const uint32_t* __restrict__ tile_offsets,
                                                              const float* __restrict__ T_final,
                                                              const int* __restrict__ n_contrib,
                                                              const float* __restrict__ dL_dimage,
                                                              float* __restrict__ dmeans2d, float* __restrict__ dconics,
                                                              float* __restrict__ dcolors, float* __restrict__ dopac) {
    __shared__ Stage s;
    __shared__ int s_max;
    const int TX = tiles_x(cam);
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    const unsigned lane = tid & 31;
    const int x = (tile % TX) * kTile + (tid & 15);
    const int y = (tile / TX) * kTile + (tid >> 4);
    const bool inside = x < cam.width && y < cam.height;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    const uint32_t start = tile_offsets[tile];
    float T = 1.0f, w0 = 0.0f, w1 = 0.0f, w2 = 0.0f;
    int last = 0;
    if (inside) {
        const size_t pix = (size_t)y * cam.width + x;
        T = T_final[pix];
        last = n_contrib[pix];
        w0 = dL_dimage[3 * pix];
        w1 = dL_dimage[3 * pix + 1];
        w2 = dL_dimage[3 * pix + 2];
    }
    float S0 = cfg.bg[0], S1 = cfg.bg[1], S2 = cfg.bg[2];
    if (tid == 0) s_max = 0;
    __syncthreads();
    const int wmax = __reduce_max_sync(VKS_FULL_MASK, last);
    if (lane == 0) atomicMax(&s_max, wmax);
    __syncthreads();
    const int bmax = s_max;
    // the slot index of the 9th term: lane 4k (k < 8) owns term k, lane 1 owns the opacity term
    const int myterm = (lane & 3) == 0 ? (int)(lane >> 2) : (lane == 1 ? 8 : -1);
    for (int bend = bmax; bend > 0; bend -= kThreads) {
        const int bstart = max(0, bend - kThreads);
        __syncthreads();
        if (bstart + tid < bend) stage_batch(s, tid, __ldg(vals + start + bstart + tid), means2d, conics, colors, opac);
        __syncthreads();
        for (int j = bend - 1 - bstart; j >= 0; j--) {
            const int pos = bstart + j;
            float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            float e = 0.0f;
            bool contrib = false;
            if (pos < last) {
                float dx, dy, G, rG, alpha;
                if (eval_alpha(s, j, px, py, dx, dy, G, rG, alpha)) {
                    contrib = true;
                    T = T / (1.0f - alpha);
                    const float aT = alpha * T;
                    const float c0 = s.col[0][j], c1 = s.col[1][j], c2 = s.col[2][j];
                    v[5] = aT * w0;
                    v[6] = aT * w1;
                    v[7] = aT * w2;
                    const float dalpha = T * ((c0 - S0) * w0 + (c1 - S1) * w1 + (c2 - S2) * w2);
                    S0 = alpha * c0 + (1.0f - alpha) * S0;
                    S1 = alpha * c1 + (1.0f - alpha) * S1;
                    S2 = alpha * c2 + (1.0f - alpha) * S2;
                    if (!(rG > 0.99f)) {
                        const float dsig = -rG * dalpha;
                        const float a = 2.0f * s.ha[j], bb = s.b[j], c = 2.0f * s.hc[j];
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
                      const float* conics, const float* colors, const float* opacities,
                      const uint32_t* vals, const uint32_t* tile_offsets, float* image,
                      float* T_final, int32_t* n_contrib, cudaStream_t st) {
    (void)n;
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    raster_fwd_kernel<<<n_tiles, kThreads, 0, st>>>(cfg, cam, reinterpret_cast<const float2*>(means2d), conics,
                                                    colors, opacities, vals, tile_offsets, image, T_final,
                                                    n_contrib);
    return LaunchCheck::check();
}

int launch_raster_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities,
                      const uint32_t* vals, const uint32_t* tile_offsets, const float* T_final,
                      const int32_t* n_contrib, const float* dL_dimage, float* dmeans2d,
                      float* dconics, float* dcolors, float* dopacities, cudaStream_t st) {
    (void)n;
    const int n_tiles = tiles_x(cam) * tiles_y(cam);
    raster_bwd_kernel<<<n_tiles, kThreads, 0, st>>>(cfg, cam, reinterpret_cast<const float2*>(means2d), conics,
                                                    colors, opacities, vals, tile_offsets, T_final, n_contrib,
                                                    dL_dimage, dmeans2d, dconics, dcolors, dopacities);
    return LaunchCheck::check();
}

}  // namespace vks
