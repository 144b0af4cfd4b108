// adam.cu — SURVEY §8(f) row f1: the optimizer step after the path ("adam_step",
// PAPER P:76 row "Proj Bwd + Optimizer"); include/vks.h vks_adam_step.
//
// One launch over the five parameter groups.  HBM-bound (28 B per element: p, g, m, v read;
// p, m, v written): each thread owns one 16-byte chunk (4 consecutive elements) of a group and
// moves it with 128-bit loads and stores; the quaternion group's chunks are its rows, so the
// re-normalisation after the step needs no exchange.  Blocks are assigned to groups by
// contiguous block ranges.
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kAdamThreads = 256;
constexpr int kGroups = 5;

struct AdamParams {
    float* p[kGroups];
    const float* g[kGroups];
    float* m[kGroups];
    float* v[kGroups];
    int64_t count[kGroups];       // elements per group
    int64_t block0[kGroups + 1];  // first block of each group
    float lr[6];
    float b1, b2, eps, rbc1, rbc2;  // rbc = 1 / (1 - beta^t)
    int sh_coeffs;
};

__device__ __forceinline__ void adam_elem(float& p, float g, float& m, float& v, float lr, const AdamParams& a) {
    m = a.b1 * m + (1.0f - a.b1) * g;
    v = a.b2 * v + (1.0f - a.b2) * (g * g);
    const float mhat = m * a.rbc1, vhat = v * a.rbc2;
    p = p - (lr * mhat) / (sqrtf(vhat) + a.eps);
}

__device__ __forceinline__ float4 ld_stream(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st_stream(float* p, float4 x) { __stcs(reinterpret_cast<float4*>(p), x); }

__global__ void __launch_bounds__(kAdamThreads) adam_kernel(const AdamParams a) {
    const int64_t b = blockIdx.x;
    int grp = 0;
#pragma unroll
    for (int q = 1; q < kGroups; q++) grp += b >= a.block0[q];
    const int64_t chunk = (b - a.block0[grp]) * kAdamThreads + threadIdx.x;
    const int64_t e0 = chunk * 4, cnt = a.count[grp];
    if (e0 >= cnt) return;
    float* __restrict__ P = a.p[grp];
    const float* __restrict__ G = a.g[grp];
    float* __restrict__ M = a.m[grp];
    float* __restrict__ V = a.v[grp];
    float lr[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        lr[j] = a.lr[grp];
        if (grp == 4) lr[j] = ((e0 + j) / 3) % a.sh_coeffs == 0 ? a.lr[4] : a.lr[5];
    }
    if (e0 + 4 <= cnt) {  // whole chunk: 128-bit streaming accesses (every pointer 16-byte aligned)
        float4 p4 = ld_stream(P + e0);
        const float4 g4 = ld_stream(G + e0);
        float4 m4 = ld_stream(M + e0);
        float4 v4 = ld_stream(V + e0);
        adam_elem(p4.x, g4.x, m4.x, v4.x, lr[0], a);
        adam_elem(p4.y, g4.y, m4.y, v4.y, lr[1], a);
        adam_elem(p4.z, g4.z, m4.z, v4.z, lr[2], a);
        adam_elem(p4.w, g4.w, m4.w, v4.w, lr[3], a);
        if (grp == 2) {  // a quaternion row: re-normalise after the step
            const float nn = sqrtf(((p4.x * p4.x + p4.y * p4.y) + p4.z * p4.z) + p4.w * p4.w);
            if (nn > 0.0f) {
                p4.x = p4.x / nn;
                p4.y = p4.y / nn;
                p4.z = p4.z / nn;
                p4.w = p4.w / nn;
            }
        }
        st_stream(P + e0, p4);
        st_stream(M + e0, m4);
        st_stream(V + e0, v4);
    } else {  // the group's ragged tail (never a quaternion row)
        for (int j = 0; j < 4 && e0 + j < cnt; j++) {
            float p = P[e0 + j], m = M[e0 + j], v = V[e0 + j];
            adam_elem(p, __ldg(G + e0 + j), m, v, lr[j], a);
            P[e0 + j] = p;
            M[e0 + j] = m;
            V[e0 + j] = v;
        }
    }
}

}  // namespace

int launch_adam_step(const vks_adam_config& acfg, int64_t n, int32_t sh_coeffs, float* const* params,
                     const float* const* grads, float* const* m, float* const* v, cudaStream_t s) {
    AdamParams a{};
    const int64_t per_row[kGroups] = {3, 3, 4, 1, 3 * (int64_t)sh_coeffs};
    int64_t blocks = 0;
    for (int q = 0; q < kGroups; q++) {
        a.p[q] = params[q];
        a.g[q] = grads[q];
        a.m[q] = m[q];
        a.v[q] = v[q];
        a.count[q] = n * per_row[q];
        a.block0[q] = blocks;
        blocks += (a.count[q] / 4 + 1 + kAdamThreads - 1) / kAdamThreads;  // chunks incl. a ragged tail
    }
    a.block0[kGroups] = blocks;
    for (int j = 0; j < 6; j++) a.lr[j] = acfg.lr[j];
    a.b1 = acfg.beta1;
    a.b2 = acfg.beta2;
    a.eps = acfg.eps;
    a.rbc1 = (float)(1.0 / (1.0 - pow((double)acfg.beta1, (double)acfg.step)));
    a.rbc2 = (float)(1.0 / (1.0 - pow((double)acfg.beta2, (double)acfg.step)));
    a.sh_coeffs = sh_coeffs;
    if (n == 0) return VKS_OK;
    adam_kernel<<<(unsigned)blocks, kAdamThreads, 0, s>>>(a);
    return LaunchCheck::check();
}

}  // namespace vks
