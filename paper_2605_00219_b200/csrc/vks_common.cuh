// vks_common.cuh — shared device helpers of the CUDA path (never shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <utility>
#include <stdint.h>
#include <stdio.h>

#include "../../include/vks.h"

#define VKS_FULL_MASK 0xffffffffu

// Debug build (libvks_debug.so, -DVKS_DEBUG_CHECKS; the stand-in for compute-sanitizer, which this
// pool does not run): device-side bounds / invariant checks at the indexed memory accesses of the
// kernels; a failed check prints its location and traps (the launch's stream reports an error).
#ifdef VKS_DEBUG_CHECKS
#define VKS_DCHECK(cond)                                                                          \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("VKS_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,        \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                  \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define VKS_DCHECK(cond) ((void)0)
#endif

namespace vks {

constexpr int kTile = 16;

// Thread-local text of the last CUDA error seen by the library (read by vks_last_cuda_error).
inline char* last_error_buf() {
    static thread_local char buf[256] = "";
    return buf;
}
inline int cuda_fail(cudaError_t e, const char* where) {
    snprintf(last_error_buf(), 256, "%s: %s", where, cudaGetErrorString(e));
    return VKS_ERR_CUDA;
}
// check a kernel launch (clears the non-sticky launch error, keeps its text)
inline int check_launch(const char* where) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VKS_OK : cuda_fail(e, where);
}
struct LaunchCheck {
    static int check() { return check_launch("kernel launch"); }
};

__host__ __device__ inline int tiles_x(const vks_camera& c) { return (c.width + kTile - 1) / kTile; }
__host__ __device__ inline int tiles_y(const vks_camera& c) { return (c.height + kTile - 1) / kTile; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// relaxed (volatile) 32/64-bit global accesses for decoupled look-back
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Ampere-style async copies global -> shared (LDGSTS): no registers held while in flight
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
// same, with the destination already a 32-bit shared-window address
__device__ __forceinline__ void cp_async16_s(uint32_t saddr, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
}
// 16 bytes through L1 (.ca): the warps of one block that copy the same global data hit in L1
__device__ __forceinline__ void cp_async16_ca(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Per-view constants of steps 6 and 12 (FOV limits, camera centre), computed once by the launcher
// with the same IEEE fp32 operations in the same order (host code is compiled without FMA
// contraction), instead of once per Gaussian.
struct CamConst {
    float lxp, lxn, lyp, lyn;  // step 6
    float cp[3];               // step 12: campos = -R^T t
};

inline CamConst cam_const(const vks_camera& cam) {
    CamConst k;
    const float fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
    const float W = (float)cam.width, H = (float)cam.height;
    volatile float t;  // keeps every intermediate an IEEE-rounded float
    t = 0.5f * W; t = t / fx; t = 0.3f * t; const float mx = t;
    t = 0.5f * H; t = t / fy; t = 0.3f * t; const float my = t;
    t = W - cx; t = t / fx; t = t + mx; k.lxp = t;
    t = cx / fx; t = t + mx; k.lxn = t;
    t = H - cy; t = t / fy; t = t + my; k.lyp = t;
    t = cy / fy; t = t + my; k.lyn = t;
    for (int c = 0; c < 3; c++) {
        float a = cam.R[0 * 3 + c] * cam.t[0];
        t = cam.R[1 * 3 + c] * cam.t[1]; a = a + t;
        t = cam.R[2 * 3 + c] * cam.t[2]; a = a + t;
        k.cp[c] = -a;
    }
    return k;
}

}  // namespace vks

// internal launchers (implemented in the .cu files, called by api.cu)
namespace vks {
int launch_project_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, float* means2d, float* conics, float* depths, int32_t* radii,
                       int32_t* tiles_touched, float* colors, float* opacities, float* records, cudaStream_t s);
int launch_project_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, const float* colors, const int32_t* radii, const float* dmeans2d,
                       const float* dconics, const float* dcolors, const float* dopacities,
                       float* dmeans, float* dlog_scales, float* dquats, float* dopacity_logits,
                       float* dsh, cudaStream_t s);
int launch_project_fwd_batch(const vks_config& cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                             const float* means, const float* log_scales, const float* quats,
                             const float* opacity_logits, const float* sh, float* const* means2d,
                             float* const* conics, float* const* depths, int32_t* const* radii,
                             int32_t* const* tiles_touched, float* const* colors, float* opacities,
                             float* const* g2d_zero, float* const* records, cudaStream_t s);
int launch_project_bwd_batch(const vks_config& cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                             const float* means, const float* log_scales, const float* quats,
                             const float* opacity_logits, const float* sh, const float* const* colors,
                             const int32_t* const* radii, const float* const* dmeans2d, const float* const* dconics,
                             const float* const* dcolors, const float* const* dopacities, float* dmeans,
                             float* dlog_scales, float* dquats, float* dopacity_logits, float* dsh, cudaStream_t s);
int launch_adam_step(const vks_adam_config& acfg, int64_t n, int32_t sh_coeffs, float* const* params,
                     const float* const* grads, float* const* m, float* const* v, cudaStream_t s);
size_t densify_workspace_bytes(int64_t n);
int launch_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom,
                         cudaStream_t s);
int launch_densify(int64_t n, int32_t sh_coeffs, const float* const* params, const float* const* m,
                   const float* const* v, const float* accum, const float* denom, float grad_threshold,
                   float size_threshold, float prune_opacity, unsigned long long seed, int64_t capacity,
                   float* const* out_params, float* const* out_m, float* const* out_v, int64_t* n_out, void* workspace,
                   cudaStream_t s);
size_t mcmc_workspace_bytes(int64_t n);
int launch_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, unsigned long long seed, float* means,
                         float* log_scales, float* quats, float* opacity_logits, float* sh, float* const* m,
                         float* const* v, int64_t* targets, int64_t* n_dead, void* workspace, cudaStream_t s);
int launch_mcmc_noise(int64_t n, float lr_pos, float noise_scale, unsigned long long seed, uint32_t step, float* means,
                      const float* log_scales, const float* quats, const float* opacity_logits, cudaStream_t s);
size_t loss_workspace_bytes(int W, int H);
int launch_loss_grad(int W, int H, float lambda, const float* render, const float* target, float* dL, float* loss,
                     void* workspace, cudaStream_t s);
size_t bin_sort_workspace_bytes(int64_t n, int64_t capacity, int32_t n_tiles);
int run_bin_sort(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii,
                 const float* depths, const int32_t* tiles_touched, uint32_t* offsets,
                 int64_t capacity, uint64_t* keys, uint32_t* vals, uint64_t* keys_unsorted,
                 uint32_t* vals_unsorted, uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects,
                 void* workspace, size_t workspace_bytes, cudaStream_t s);
int run_bin_sort_async(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const int32_t* tiles_touched, uint32_t* offsets, int64_t capacity,
                       uint32_t* vals, uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects,
                       int32_t* status, void* workspace, size_t workspace_bytes, cudaStream_t s);
int launch_raster_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const float* records, const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                      float* image, float* T_final, int32_t* n_contrib, cudaStream_t s);
int launch_raster_fwd_stats(const vks_config& cfg, const vks_camera& cam, const float* means2d, const float* conics,
                            const float* colors, const float* opacities, const int32_t* radii, const float* records,
                            const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                            unsigned long long* stats, int64_t n, cudaStream_t s);
// VKS_FLAG_VALIDATE checks (validate.cu): begin resets the status word, the checks enqueue,
// end synchronises once and returns VKS_OK / VKS_ERR_NONFINITE / VKS_ERR_UNSORTED
int validate_begin(cudaStream_t s);
int validate_finite(const float* p, int64_t count, cudaStream_t s);
int validate_quats(const float* q, int64_t n, cudaStream_t s);
int validate_csr(const uint32_t* tile_offsets, int n_tiles, int64_t M, const uint32_t* vals, int64_t n,
                 cudaStream_t s);
int validate_bins(const vks_camera& cam, int64_t n, const float* means2d, const int32_t* radii, const float* depths,
                  const uint32_t* vals, const uint32_t* tile_offsets, int64_t M, cudaStream_t s);
int validate_end(cudaStream_t s);
int launch_raster_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means2d,
                      const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                      const float* records, const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                      const float* T_final, const int32_t* n_contrib, const float* dL_dimage, float* dmeans2d,
                      float* dconics, float* dcolors, float* dopacities, cudaStream_t s);
#ifndef VKS_PDL
#define VKS_PDL 1
#endif
// Programmatic dependent launch: the kernels of the path are launched with programmatic stream
// serialization and waits for its predecessor grid (griddepcontrol.wait; a no-op after a
// plain launch) before its first global-memory access, so its launch and block scheduling
// overlap the predecessor's tail instead of following it.
__device__ __forceinline__ void pdl_wait() {
#if VKS_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
#if VKS_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // errors: the callers' check_launch
#else
    kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
#endif
}

}  // namespace vks
