// validate.cu — VKS_FLAG_VALIDATE debug checks at the boundary (SURVEY §8(b) "Errors"):
//   * non-finite inputs (SPEC S:119 NonFiniteParameter) and zero quaternions (S:52 ZeroQuaternion)
//     -> VKS_ERR_NONFINITE, checked before the entry point computes anything;
//   * tile lists that are not a valid sorted binning (S:155 UnsortedInput): tile_offsets not a CSR
//     of [0, M), ids out of range, an entry whose Gaussian's tile rect misses its tile, or two
//     entries of a tile out of (depth bits, id) order -> VKS_ERR_UNSORTED.
// A module-scope device status word collects the failures; validate_end reads it back with one
// stream synchronisation (validate mode is a debugging aid, not meant for concurrent streams).
// Compiled with -fmad=false: the tile rect below is recomputed exactly as projection step 11.
#include <algorithm>

#include "vks_common.cuh"

namespace vks {
namespace {

__device__ unsigned int g_validate_word;

constexpr unsigned kBitNonFinite = 1u, kBitUnsorted = 2u;
constexpr int kThreads = 256;

__device__ __forceinline__ void flag_if(bool bad, unsigned bit) {
    if (__any_sync(VKS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(&g_validate_word, bit);
}

__global__ void finite_kernel(const float* __restrict__ p, int64_t count) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(p[i]);
    flag_if(bad, kBitNonFinite);
}

// quaternions: finite and of norm > 1e-12 (the projection culls the others, DESIGN.md §4.1 step 2)
__global__ void quat_kernel(const float4* __restrict__ q, int64_t n) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = q[i];
        const float nn = sqrtf(((v.x * v.x + v.y * v.y) + v.z * v.z) + v.w * v.w);
        bad |= !(nn > 1e-12f) || !isfinite(nn);
    }
    flag_if(bad, kBitNonFinite);
}

// CSR check: tile_offsets[0] == 0, non-decreasing, tile_offsets[n_tiles] == M (M < 0: not known)
// and every id of vals[0, tile_offsets[n_tiles]) < n
__global__ void csr_kernel(const uint32_t* __restrict__ tile_offsets, int n_tiles, int64_t M,
                           const uint32_t* __restrict__ vals, int64_t n) {
    bool bad = false;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = tid; t < n_tiles; t += stride) bad |= tile_offsets[t + 1] < tile_offsets[t];
    if (tid == 0) bad |= tile_offsets[0] != 0u || (M >= 0 && (int64_t)tile_offsets[n_tiles] != M);
    const int64_t end = M >= 0 ? std::min<int64_t>(tile_offsets[n_tiles], M) : (int64_t)tile_offsets[n_tiles];
    for (int64_t k = tid; k < end; k += stride) bad |= (int64_t)vals[k] >= n;
    flag_if(bad, kBitUnsorted);
}

// one block per tile: every entry's Gaussian covers the tile (rect of projection step 11) and the
// entries are strictly ascending in (f32 depth bits, id) — the stable order of the (tile | depth)
// keys with ties by id
__global__ void bins_kernel(int TX, int TY, const float2* __restrict__ means2d, const int2* __restrict__ radii,
                            const uint32_t* __restrict__ depth_bits, const uint32_t* __restrict__ vals,
                            const uint32_t* __restrict__ tile_offsets, int64_t n, int64_t M) {
    const int t = blockIdx.x, tx = t % TX, ty = t / TX;
    // bounded by M even when the CSR itself is corrupt (csr_kernel flags that)
    const uint32_t e = (uint32_t)std::min<int64_t>(tile_offsets[t + 1], M);
    const uint32_t b = std::min(tile_offsets[t], e);
    bool bad = false;
    for (uint32_t k = b + threadIdx.x; k < e; k += blockDim.x) {
        const uint32_t g = vals[k];
        if ((int64_t)g >= n) { bad = true; continue; }
        const float2 m = means2d[g];
        const int2 r = radii[g];
        const float rx = (float)r.x, ry = (float)r.y;
        const int x0 = (int)fminf(fmaxf(floorf((m.x - rx) * 0.0625f), 0.0f), (float)TX);
        const int x1 = (int)fminf(fmaxf(ceilf((m.x + rx) * 0.0625f), 0.0f), (float)TX);
        const int y0 = (int)fminf(fmaxf(floorf((m.y - ry) * 0.0625f), 0.0f), (float)TY);
        const int y1 = (int)fminf(fmaxf(ceilf((m.y + ry) * 0.0625f), 0.0f), (float)TY);
        bad |= !(r.x > 0 || r.y > 0) || tx < x0 || tx >= x1 || ty < y0 || ty >= y1;
        if (k > b) {
            const uint32_t p = vals[k - 1];
            if ((int64_t)p < n) {
                const uint32_t dp = depth_bits[p], dg = depth_bits[g];
                bad |= !(dp < dg || (dp == dg && p < g));
            }
        }
    }
    flag_if(bad, kBitUnsorted);
}

unsigned grid_for(int64_t count) {
    const int64_t want = (count + kThreads - 1) / kThreads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, 148 * 16));
}

}  // namespace

int validate_begin(cudaStream_t s) {
    void* p = nullptr;
    if (cudaError_t e = cudaGetSymbolAddress(&p, g_validate_word)) return cuda_fail(e, "validate symbol");
    if (cudaError_t e = cudaMemsetAsync(p, 0, sizeof(unsigned), s)) return cuda_fail(e, "validate reset");
    return VKS_OK;
}

int validate_finite(const float* p, int64_t count, cudaStream_t s) {
    if (count <= 0 || !p) return VKS_OK;
    finite_kernel<<<grid_for(count), kThreads, 0, s>>>(p, count);
    return check_launch("validate finite");
}

int validate_quats(const float* q, int64_t n, cudaStream_t s) {
    if (n <= 0 || !q) return VKS_OK;
    quat_kernel<<<grid_for(n), kThreads, 0, s>>>(reinterpret_cast<const float4*>(q), n);
    return check_launch("validate quats");
}

int validate_csr(const uint32_t* tile_offsets, int n_tiles, int64_t M, const uint32_t* vals, int64_t n,
                 cudaStream_t s) {
    csr_kernel<<<grid_for(std::max<int64_t>(n_tiles, 1) * 8), kThreads, 0, s>>>(tile_offsets, n_tiles, M, vals, n);
    return check_launch("validate csr");
}

int validate_bins(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii, const float* depths,
                  const uint32_t* vals, const uint32_t* tile_offsets, int64_t M, cudaStream_t s) {
    const int TX = tiles_x(cam), TY = tiles_y(cam);
    int st = validate_csr(tile_offsets, TX * TY, M, vals, n, s);
    if (st) return st;
    bins_kernel<<<TX * TY, kThreads, 0, s>>>(TX, TY, reinterpret_cast<const float2*>(means2d),
                                             reinterpret_cast<const int2*>(radii),
                                             reinterpret_cast<const uint32_t*>(depths), vals, tile_offsets, n, M);
    return check_launch("validate bins");
}

// one synchronisation: VKS_ERR_NONFINITE takes precedence over VKS_ERR_UNSORTED
int validate_end(cudaStream_t s) {
    unsigned word = 0;
    if (cudaError_t e = cudaMemcpyFromSymbolAsync(&word, g_validate_word, sizeof(word), 0, cudaMemcpyDeviceToHost, s))
        return cuda_fail(e, "validate read");
    if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_fail(e, "validate sync");
    if (word & kBitNonFinite) return VKS_ERR_NONFINITE;
    if (word & kBitUnsorted) return VKS_ERR_UNSORTED;
    return VKS_OK;
}

}  // namespace vks
