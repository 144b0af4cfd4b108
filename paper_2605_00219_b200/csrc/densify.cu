// densify.cu — SURVEY §8(f) row f4: default densification;
// include/vks.h vks_densify_stats / vks_densify; readings R6-R9 of DESIGN.md §4.7.
//
// vks_densify_stats: one thread per Gaussian, after a view's raster backward.  vks_densify:
// kind_kernel (prune / keep / clone / split per Gaussian -> its row count 0, 1, 2, 2; per-block
// sums) -> block_count_kernel (one block: exclusive scan of the block sums, n') -> the host reads
// n' (the call's one synchronisation; VKS_ERR_CAPACITY when it exceeds the output capacity) ->
// emit_kernel (each Gaussian's output offset = block prefix + in-block prefix; writes its rows:
// copies, split children with log-scales - ln 1.6 and positions sampled from the parent, fresh
// moments for new rows).  Rows come out in input order, as the oracle's.
#include "vks_common.cuh"

namespace vks {
namespace {

typedef unsigned long long u64;
constexpr int kDThreads = 256;
constexpr int kDItems = 4;
constexpr int kDTile = kDThreads * kDItems;

__device__ __forceinline__ u64 rng_h3(u64 seed, uint32_t stream, u64 i) {
    u64 z = seed + 0x9E3779B97F4A7C15ull * ((((u64)stream) << 40) ^ i);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double normal3(u64 seed, uint32_t stream, u64 k) {
    const double u1 = ((double)(rng_h3(seed, stream, 2 * k) >> 40) + 0.5) / 16777216.0;
    const double u2 = ((double)(rng_h3(seed, stream, 2 * k + 1) >> 40) + 0.5) / 16777216.0;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

struct DensIn {
    const float *means, *ls, *quats, *logits, *sh;
    const float* m[5];
    const float* v[5];
    const float *accum, *denom;
    float gthr, sthr, pop;
    int S;  // 3 * sh_coeffs
    u64 seed;
};

struct DensOut {
    float *means, *ls, *quats, *logits, *sh;
    float* m[5];
    float* v[5];
};

// 0 prune, 1 keep, 2 clone, 3 split
__device__ __forceinline__ int kind_of(const DensIn& a, int64_t i) {
    const float rho = (float)(1.0 / (1.0 + exp(-(double)__ldg(a.logits + i))));
    if (rho < a.pop) return 0;
    const float dn = __ldg(a.denom + i);
    const float g = dn > 0.0f ? __ldg(a.accum + i) / dn : 0.0f;
    if (!(g > a.gthr)) return 1;
    float smax = (float)exp((double)__ldg(a.ls + 3 * i));
    for (int c = 1; c < 3; c++) smax = fmaxf(smax, (float)exp((double)__ldg(a.ls + 3 * i + c)));
    return smax < a.sthr ? 2 : 3;
}

__device__ __forceinline__ unsigned rows_of(int k) { return k == 0 ? 0u : (k == 1 ? 1u : 2u); }

__global__ void __launch_bounds__(kDThreads) stats_kernel(int64_t n, const float2* __restrict__ g2,
                                                         const int2* __restrict__ radii, float* __restrict__ accum,
                                                         float* __restrict__ denom) {
    const int64_t i = (int64_t)blockIdx.x * kDThreads + threadIdx.x;
    if (i >= n) return;
    const int2 r = __ldg(radii + i);
    if (r.x <= 0 && r.y <= 0) return;
    const float2 g = __ldg(g2 + i);
    accum[i] = (float)((double)accum[i] + sqrt((double)g.x * g.x + (double)g.y * g.y));
    denom[i] = denom[i] + 1.0f;
}

__global__ void __launch_bounds__(kDThreads) kind_kernel(int64_t n, const DensIn a, unsigned* __restrict__ bsum) {
    __shared__ unsigned s_w[kDThreads / 32];
    const int tid = threadIdx.x;
    unsigned c = 0;
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        const int64_t i = (int64_t)blockIdx.x * kDTile + q * kDThreads + tid;
        if (i < n) c += rows_of(kind_of(a, i));
    }
    c = __reduce_add_sync(VKS_FULL_MASK, c);
    if ((tid & 31) == 0) s_w[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        unsigned t = 0;
        for (int q = 0; q < kDThreads / 32; q++) t += s_w[q];
        bsum[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) block_count_kernel(unsigned* __restrict__ bsum, int nb, u64* __restrict__ total) {
    __shared__ u64 s_w[32];
    __shared__ u64 s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + tid;
        const u64 c = i < nb ? bsum[i] : 0u;
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
        if (i < nb) bsum[i] = (unsigned)(carry + wpre + incl - c);
        __syncthreads();
        if (tid == 0) s_carry = carry + btot;
        __syncthreads();
    }
    if (tid == 0) *total = s_carry;
}

__global__ void __launch_bounds__(kDThreads) emit_kernel(int64_t n, int64_t n_out, const DensIn a, const DensOut o,
                                                        const unsigned* __restrict__ bpre) {
    __shared__ unsigned s_w[kDItems][kDThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int kind[kDItems];
    unsigned incl[kDItems];
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        const int64_t i = (int64_t)blockIdx.x * kDTile + q * kDThreads + tid;
        kind[q] = i < n ? kind_of(a, i) : 0;
        unsigned x = rows_of(kind[q]);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned t = __shfl_up_sync(VKS_FULL_MASK, x, d);
            if (lane >= d) x += t;
        }
        incl[q] = x;
        if (lane == 31) s_w[q][warp] = x;
    }
    __syncthreads();
    u64 run = bpre[blockIdx.x];
    const int wid[5] = {3, 3, 4, 1, a.S};
#pragma unroll
    for (int q = 0; q < kDItems; q++) {
        u64 pre = run;
        for (int w = 0; w < kDThreads / 32; w++) {
            if (w < warp) pre += s_w[q][w];
            run += s_w[q][w];
        }
        const int64_t i = (int64_t)blockIdx.x * kDTile + q * kDThreads + tid;
        const int k = kind[q];
        const unsigned rows = rows_of(k);
        const int64_t o0 = (int64_t)(pre + incl[q] - rows);  // exclusive offset
        if (i >= n || rows == 0) continue;
        double R[9] = {0};
        if (k == 3) {
            const double qa = a.quats[4 * i], qb = a.quats[4 * i + 1], qc = a.quats[4 * i + 2], qd = a.quats[4 * i + 3];
            const double qn = sqrt(qa * qa + qb * qb + qc * qc + qd * qd);
            const double w = qa / qn, x = qb / qn, y = qc / qn, z = qd / qn;
            const double RR[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                                  2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                  2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
            for (int t = 0; t < 9; t++) R[t] = RR[t];
        }
        for (unsigned r = 0; r < rows; r++) {
            const int64_t oo = o0 + r;
            VKS_DCHECK(oo >= 0 && oo < n_out);
            for (int c = 0; c < 4; c++) o.quats[4 * oo + c] = a.quats[4 * i + c];
            o.logits[oo] = a.logits[i];
            for (int c = 0; c < a.S; c++) o.sh[(int64_t)a.S * oo + c] = a.sh[(int64_t)a.S * i + c];
            if (k == 3) {
                double e[3];
                for (int c = 0; c < 3; c++)
                    e[c] = exp((double)a.ls[3 * i + c]) * normal3(a.seed, 3, 6 * (u64)i + 3 * r + c);
                for (int c = 0; c < 3; c++) {
                    o.means[3 * oo + c] = (float)((double)a.means[3 * i + c] + R[3 * c] * e[0] + R[3 * c + 1] * e[1] +
                                                  R[3 * c + 2] * e[2]);
                    o.ls[3 * oo + c] = (float)((double)a.ls[3 * i + c] - log(1.6));
                }
            } else {
                for (int c = 0; c < 3; c++) {
                    o.means[3 * oo + c] = a.means[3 * i + c];
                    o.ls[3 * oo + c] = a.ls[3 * i + c];
                }
            }
            const bool fresh = (k == 2 && r == 1) || k == 3;
            for (int g = 0; g < 5; g++) {
                if (!o.m[g]) continue;
                for (int c = 0; c < wid[g]; c++) {
                    o.m[g][(int64_t)wid[g] * oo + c] = (fresh || !a.m[g]) ? 0.0f : a.m[g][(int64_t)wid[g] * i + c];
                    o.v[g][(int64_t)wid[g] * oo + c] = (fresh || !a.v[g]) ? 0.0f : a.v[g][(int64_t)wid[g] * i + c];
                }
            }
        }
    }
    (void)n_out;
}

struct DensWs {
    unsigned* bsum;
    u64* total;
    size_t bytes;
};

DensWs carve_dens(void* base, int64_t n) {
    DensWs w{};
    const size_t nb = ((size_t)(n > 0 ? n : 1) + kDTile - 1) / kDTile;
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += (bytes + 255) & ~(size_t)255; return p; };
    w.bsum = reinterpret_cast<unsigned*>(take(4 * nb));
    w.total = reinterpret_cast<u64*>(take(8));
    w.bytes = off;
    return w;
}

}  // namespace

size_t densify_workspace_bytes(int64_t n) { return carve_dens(nullptr, n).bytes + 256; }

int launch_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom,
                         cudaStream_t s) {
    if (n == 0) return VKS_OK;
    stats_kernel<<<(unsigned)((n + kDThreads - 1) / kDThreads), kDThreads, 0, s>>>(
        n, reinterpret_cast<const float2*>(dmeans2d), reinterpret_cast<const int2*>(radii), accum, denom);
    return LaunchCheck::check();
}

int launch_densify(int64_t n, int32_t sh_coeffs, const float* const* params, const float* const* m,
                   const float* const* v, const float* accum, const float* denom, float grad_threshold,
                   float size_threshold, float prune_opacity, unsigned long long seed, int64_t capacity,
                   float* const* out_params, float* const* out_m, float* const* out_v, int64_t* n_out, void* workspace,
                   cudaStream_t s) {
    DensIn a{};
    a.means = params[0]; a.ls = params[1]; a.quats = params[2]; a.logits = params[3]; a.sh = params[4];
    for (int g = 0; g < 5; g++) {
        a.m[g] = m ? m[g] : nullptr;
        a.v[g] = v ? v[g] : nullptr;
    }
    a.accum = accum; a.denom = denom;
    a.gthr = grad_threshold; a.sthr = size_threshold; a.pop = prune_opacity;
    a.S = 3 * sh_coeffs;
    a.seed = seed;
    *n_out = 0;
    if (n == 0) return VKS_OK;
    DensWs w = carve_dens(workspace, n);
    const unsigned nb = (unsigned)((n + kDTile - 1) / kDTile);
    kind_kernel<<<nb, kDThreads, 0, s>>>(n, a, w.bsum);
    block_count_kernel<<<1, 1024, 0, s>>>(w.bsum, (int)nb, w.total);
    u64 total = 0;
    if (cudaError_t e = cudaMemcpyAsync(&total, w.total, sizeof(u64), cudaMemcpyDeviceToHost, s)) return cuda_fail(e, "read n'");
    if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_fail(e, "densify sync");
    *n_out = (int64_t)total;
    if ((int64_t)total > capacity) return VKS_ERR_CAPACITY;
    DensOut o{};
    o.means = out_params[0]; o.ls = out_params[1]; o.quats = out_params[2]; o.logits = out_params[3]; o.sh = out_params[4];
    for (int g = 0; g < 5; g++) {
        o.m[g] = out_m ? out_m[g] : nullptr;
        o.v[g] = out_v ? out_v[g] : nullptr;
    }
    emit_kernel<<<nb, kDThreads, 0, s>>>(n, (int64_t)total, a, o, w.bsum);
    return LaunchCheck::check();
}

}  // namespace vks
