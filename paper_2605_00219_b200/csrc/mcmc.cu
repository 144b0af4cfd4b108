// mcmc.cu — SURVEY §8(f) row f3: MCMC densification at a fixed budget (PAPER
// P:36-53 "MCMC 1M densification"); include/vks.h vks_mcmc_relocate / vks_mcmc_noise; the
// readings R1-R5 are DESIGN.md §4.7.
//
// Relocation: weights_kernel (X64 opacity, dead flag, integer weight floor(rho 2^24), per-block
// sums) -> block_scan_kernel (one block: exclusive scan of the block sums, total weight, dead
// count) -> prefix_kernel (inclusive prefix W of the weights) -> sample_kernel (each dead
// Gaussian draws t = mulhi64(h, total) and binary-searches the first W_j > t; k_j += 1) ->
// copy_kernel (the dead rows take their target's parameters and the split opacity; their Adam
// moments are zeroed) -> split_kernel (the targets' own opacity).  All integer decisions are
// exact, so targets equal the oracle's.  Noise: one thread per Gaussian (fp64 Box-Muller).
#include "vks_common.cuh"

namespace vks {
namespace {

typedef unsigned long long u64;
constexpr int kMThreads = 256;
constexpr int kMItems = 4;
constexpr int kMTile = kMThreads * kMItems;

__host__ __device__ __forceinline__ u64 rng_h(u64 seed, uint32_t stream, u64 i) {
    u64 z = seed + 0x9E3779B97F4A7C15ull * ((((u64)stream) << 40) ^ i);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double rng_uniform(u64 seed, uint32_t stream, u64 i) {
    return ((double)(rng_h(seed, stream, i) >> 40) + 0.5) / 16777216.0;
}

__device__ __forceinline__ double rng_normal(u64 seed, uint32_t stream, u64 k) {
    const double u1 = rng_uniform(seed, stream, 2 * k), u2 = rng_uniform(seed, stream, 2 * k + 1);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__device__ __forceinline__ float x64_sigmoid(float o) { return (float)(1.0 / (1.0 + exp(-(double)o))); }

__device__ __forceinline__ u64 weight_of(float logit, float dead_opacity, bool& dead) {
    const float rho = x64_sigmoid(logit);
    dead = rho < dead_opacity;
    return dead ? 0ull : (u64)floor((double)rho * 16777216.0);
}

__global__ void __launch_bounds__(kMThreads) weights_kernel(int64_t n, const float* __restrict__ logits, float dead_opacity,
                                                           u64* __restrict__ bsum, u64* __restrict__ bdead) {
    __shared__ u64 s_w[kMThreads / 32], s_d[kMThreads / 32];
    const int tid = threadIdx.x;
    u64 w = 0, d = 0;
#pragma unroll
    for (int q = 0; q < kMItems; q++) {
        const int64_t i = (int64_t)blockIdx.x * kMTile + q * kMThreads + tid;
        if (i < n) {
            bool dead;
            w += weight_of(__ldg(logits + i), dead_opacity, dead);
            d += dead;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        w += __shfl_xor_sync(VKS_FULL_MASK, w, o);
        d += __shfl_xor_sync(VKS_FULL_MASK, d, o);
    }
    if ((tid & 31) == 0) { s_w[tid >> 5] = w; s_d[tid >> 5] = d; }
    __syncthreads();
    if (tid == 0) {
        u64 a = 0, b = 0;
        for (int q = 0; q < kMThreads / 32; q++) { a += s_w[q]; b += s_d[q]; }
        bsum[blockIdx.x] = a;
        bdead[blockIdx.x] = b;
    }
}

// one block: exclusive scan of the block sums in place; tot[0] = total weight, tot[1] = dead count
__global__ void __launch_bounds__(1024) block_scan_kernel(u64* __restrict__ bsum, const u64* __restrict__ bdead, int nb,
                                                         u64* __restrict__ tot, int64_t* __restrict__ n_dead) {
    __shared__ u64 s_w[32];
    __shared__ u64 s_carry, s_dead;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { s_carry = 0; s_dead = 0; }
    __syncthreads();
    u64 dead = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + tid;
        const u64 c = i < nb ? bsum[i] : 0ull;
        dead += i < nb ? bdead[i] : 0ull;
        u64 incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u64 t = __shfl_up_sync(VKS_FULL_MASK, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        u64 wpre = 0, btot = 0;
        for (int w = 0; w < 32; w++) {
            if (w < warp) wpre += s_w[w];
            btot += s_w[w];
        }
        const u64 carry = s_carry;
        if (i < nb) bsum[i] = carry + wpre + incl - c;
        __syncthreads();
        if (tid == 0) s_carry = carry + btot;
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) dead += __shfl_xor_sync(VKS_FULL_MASK, dead, o);
    if (lane == 0) atomicAdd(&s_dead, dead);
    __syncthreads();
    if (tid == 0) {
        tot[0] = s_carry;
        tot[1] = s_dead;
        if (n_dead) *n_dead = (int64_t)s_dead;
    }
}

// inclusive prefix of the weights: block-strided items (item q of thread t = element q*256 + t)
__global__ void __launch_bounds__(kMThreads) prefix_kernel(int64_t n, const float* __restrict__ logits, float dead_opacity,
                                                          const u64* __restrict__ bpre, u64* __restrict__ W) {
    __shared__ u64 s_w[kMItems][kMThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u64 incl[kMItems];
#pragma unroll
    for (int q = 0; q < kMItems; q++) {
        const int64_t i = (int64_t)blockIdx.x * kMTile + q * kMThreads + tid;
        bool dead;
        u64 x = i < n ? weight_of(__ldg(logits + i), dead_opacity, dead) : 0ull;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u64 t = __shfl_up_sync(VKS_FULL_MASK, x, d);
            if (lane >= d) x += t;
        }
        incl[q] = x;
        if (lane == 31) s_w[q][warp] = x;
    }
    __syncthreads();
    u64 run = bpre[blockIdx.x];
#pragma unroll
    for (int q = 0; q < kMItems; q++) {
        u64 pre = run;
        for (int w = 0; w < kMThreads / 32; w++) {
            if (w < warp) pre += s_w[q][w];
            run += s_w[q][w];
        }
        const int64_t i = (int64_t)blockIdx.x * kMTile + q * kMThreads + tid;
        if (i < n) W[i] = pre + incl[q];
    }
}

__global__ void __launch_bounds__(kMThreads) sample_kernel(int64_t n, const float* __restrict__ logits, float dead_opacity,
                                                          u64 seed, const u64* __restrict__ W, const u64* __restrict__ tot,
                                                          int64_t* __restrict__ target, unsigned* __restrict__ kcount) {
    const int64_t i = (int64_t)blockIdx.x * kMThreads + threadIdx.x;
    if (i >= n) return;
    bool dead;
    weight_of(__ldg(logits + i), dead_opacity, dead);
    const u64 total = tot[0];
    if (!dead || total == 0) { target[i] = -1; return; }
    const u64 t = __umul64hi(rng_h(seed, 1, (u64)i), total);
    int64_t lo = 0, hi = n - 1;  // first j with W[j] > t
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (__ldg(W + mid) > t) hi = mid; else lo = mid + 1;
    }
    VKS_DCHECK(lo >= 0 && lo < n);
    target[i] = lo;
    atomicAdd(kcount + lo, 1u);
}

__device__ __forceinline__ float split_logit(float logit_j, unsigned k) {
    const double rho = (double)x64_sigmoid(logit_j);
    const double rp = 1.0 - pow(1.0 - rho, 1.0 / (double)(k + 1));
    return (float)log(rp / (1.0 - rp));
}

struct RelocRows {
    float *means, *ls, *quats, *logits, *sh;
    float* m[5];
    float* v[5];
    int S;  // 3 * sh_coeffs
};

__global__ void __launch_bounds__(kMThreads) copy_kernel(int64_t n, const RelocRows r, const int64_t* __restrict__ target,
                                                        const unsigned* __restrict__ kcount) {
    const int64_t i = (int64_t)blockIdx.x * kMThreads + threadIdx.x;
    if (i >= n) return;
    const int64_t j = target[i];
    if (j < 0) return;
    for (int c = 0; c < 3; c++) {
        r.means[3 * i + c] = r.means[3 * j + c];
        r.ls[3 * i + c] = r.ls[3 * j + c];
    }
    for (int c = 0; c < 4; c++) r.quats[4 * i + c] = r.quats[4 * j + c];
    for (int c = 0; c < r.S; c++) r.sh[(int64_t)r.S * i + c] = r.sh[(int64_t)r.S * j + c];
    r.logits[i] = split_logit(r.logits[j], kcount[j]);  // j's logit is rewritten only by split_kernel
    const int wid[5] = {3, 3, 4, 1, r.S};
    for (int g = 0; g < 5; g++) {
        if (!r.m[g]) continue;
        for (int c = 0; c < wid[g]; c++) {
            r.m[g][(int64_t)wid[g] * i + c] = 0.0f;
            r.v[g][(int64_t)wid[g] * i + c] = 0.0f;
        }
    }
}

__global__ void __launch_bounds__(kMThreads) split_kernel(int64_t n, float* __restrict__ logits,
                                                         const unsigned* __restrict__ kcount) {
    const int64_t j = (int64_t)blockIdx.x * kMThreads + threadIdx.x;
    if (j >= n) return;
    const unsigned k = kcount[j];
    if (k) logits[j] = split_logit(logits[j], k);
}

__global__ void __launch_bounds__(kMThreads) noise_kernel(int64_t n, float lr_pos, float noise_scale, u64 seed, uint32_t step,
                                                         float* __restrict__ means, const float* __restrict__ ls,
                                                         const float4* __restrict__ quats, const float* __restrict__ logits) {
    const int64_t i = (int64_t)blockIdx.x * kMThreads + threadIdx.x;
    if (i >= n) return;
    const double rho = (double)x64_sigmoid(__ldg(logits + i));
    const double gate = 1.0 / (1.0 + exp(-100.0 * (0.005 - rho)));
    const double kk = (double)lr_pos * (double)noise_scale * gate;
    if (kk == 0.0) return;
    const float4 q = __ldg(quats + i);
    const double a = q.x, b = q.y, c = q.z, d = q.w;
    const double qn = sqrt(a * a + b * b + c * c + d * d);
    const double w = a / qn, x = b / qn, y = c / qn, z = d / qn;
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    double e[3];
    for (int k = 0; k < 3; k++) e[k] = exp((double)__ldg(ls + 3 * i + k)) * rng_normal(seed, 2 + 2 * step, 3 * (u64)i + k);
    for (int r = 0; r < 3; r++)
        means[3 * i + r] = (float)((double)means[3 * i + r] + kk * (R[3 * r] * e[0] + R[3 * r + 1] * e[1] + R[3 * r + 2] * e[2]));
}

struct McmcWs {
    u64 *W, *bsum, *bdead, *tot;
    int64_t* target;
    unsigned* kcount;
    size_t bytes;
};

McmcWs carve_mcmc(void* base, int64_t n) {
    McmcWs w{};
    const size_t nn = (size_t)(n > 0 ? n : 1), nb = (nn + kMTile - 1) / kMTile;
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    w.W = reinterpret_cast<u64*>(take(8 * nn));
    w.bsum = reinterpret_cast<u64*>(take(8 * nb));
    w.bdead = reinterpret_cast<u64*>(take(8 * nb));
    w.tot = reinterpret_cast<u64*>(take(16));
    w.target = reinterpret_cast<int64_t*>(take(8 * nn));
    w.kcount = reinterpret_cast<unsigned*>(take(4 * nn));
    w.bytes = off;
    return w;
}

}  // namespace

size_t mcmc_workspace_bytes(int64_t n) { return carve_mcmc(nullptr, n).bytes + 256; }

int launch_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, unsigned long long seed, float* means,
                         float* log_scales, float* quats, float* opacity_logits, float* sh, float* const* m,
                         float* const* v, int64_t* targets, int64_t* n_dead, void* workspace, cudaStream_t s) {
    if (n == 0) {
        if (n_dead && cudaMemsetAsync(n_dead, 0, sizeof(int64_t), s) != cudaSuccess) return VKS_ERR_CUDA;
        return VKS_OK;
    }
    McmcWs w = carve_mcmc(workspace, n);
    if (cudaMemsetAsync(w.kcount, 0, 4 * (size_t)n, s) != cudaSuccess) return VKS_ERR_CUDA;
    const unsigned nb = (unsigned)((n + kMTile - 1) / kMTile), nt = (unsigned)((n + kMThreads - 1) / kMThreads);
    weights_kernel<<<nb, kMThreads, 0, s>>>(n, opacity_logits, dead_opacity, w.bsum, w.bdead);
    block_scan_kernel<<<1, 1024, 0, s>>>(w.bsum, w.bdead, (int)nb, w.tot, n_dead);
    prefix_kernel<<<nb, kMThreads, 0, s>>>(n, opacity_logits, dead_opacity, w.bsum, w.W);
    int64_t* tg = targets ? targets : w.target;
    sample_kernel<<<nt, kMThreads, 0, s>>>(n, opacity_logits, dead_opacity, seed, w.W, w.tot, tg, w.kcount);
    RelocRows r{means, log_scales, quats, opacity_logits, sh, {}, {}, 3 * sh_coeffs};
    for (int g = 0; g < 5; g++) {
        r.m[g] = m ? m[g] : nullptr;
        r.v[g] = v ? v[g] : nullptr;
    }
    copy_kernel<<<nt, kMThreads, 0, s>>>(n, r, tg, w.kcount);
    split_kernel<<<nt, kMThreads, 0, s>>>(n, opacity_logits, w.kcount);
    return LaunchCheck::check();
}

int launch_mcmc_noise(int64_t n, float lr_pos, float noise_scale, unsigned long long seed, uint32_t step, float* means,
                      const float* log_scales, const float* quats, const float* opacity_logits, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    noise_kernel<<<(unsigned)((n + kMThreads - 1) / kMThreads), kMThreads, 0, s>>>(
        n, lr_pos, noise_scale, seed, step, means, log_scales, reinterpret_cast<const float4*>(quats), opacity_logits);
    return LaunchCheck::check();
}

}  // namespace vks
