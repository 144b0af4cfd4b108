// api.cu — the C ABI declared in include/vks.h: argument validation, then one internal launcher
// per entry point.  No allocation, no global state besides a thread-local error string.
#include <stdio.h>
#include <string.h>

#include "vks_common.cuh"

namespace {

int cuda_status(int st) { return st; }

bool camera_ok(const vks_camera* c) {
    if (!c) return false;
    if (c->width <= 0 || c->height <= 0 || c->width > 65536 || c->height > 65536) return false;
    if (!(c->fx > 0.0f) || !(c->fy > 0.0f)) return false;
    return true;
}

int config_ok(const vks_config* c) {
    if (!c) return VKS_ERR_INVALID_ARG;
    if (c->sh_degree < 0 || c->sh_degree > 3) return VKS_ERR_UNSUPPORTED;
    if (c->sh_coeffs < (c->sh_degree + 1) * (c->sh_degree + 1) || c->sh_coeffs > 64) return VKS_ERR_INVALID_ARG;
    if (c->footprint != VKS_FOOTPRINT_SUPPORT && c->footprint != VKS_FOOTPRINT_3SIGMA) return VKS_ERR_UNSUPPORTED;
    if (c->flags & ~(VKS_FLAG_GRAD_OVERWRITE | VKS_FLAG_VALIDATE)) return VKS_ERR_UNSUPPORTED;
    return VKS_OK;
}

bool device_present() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
        cudaGetLastError();
        snprintf(vks::last_error_buf(), 256, "no CUDA device (libvks has no CPU fallback)");
        return false;
    }
    return true;
}

bool validating(const vks_config* c) { return (c->flags & VKS_FLAG_VALIDATE) != 0; }

// VKS_FLAG_VALIDATE: the Gaussian parameters are finite and the quaternions non-zero
int check_params(int64_t n, int32_t sh_coeffs, const float* means, const float* log_scales, const float* quats,
                 const float* opacity_logits, const float* sh, cudaStream_t s) {
    int st = vks::validate_begin(s);
    if (!st) st = vks::validate_finite(means, 3 * n, s);
    if (!st) st = vks::validate_finite(log_scales, 3 * n, s);
    if (!st) st = vks::validate_quats(quats, n, s);
    if (!st) st = vks::validate_finite(opacity_logits, n, s);
    if (!st) st = vks::validate_finite(sh, 3 * (int64_t)sh_coeffs * n, s);
    return st ? st : vks::validate_end(s);
}

// the 2D gradients a projection backward consumes are finite
int check_grads2d(int64_t n, const float* dmeans2d, const float* dconics, const float* dcolors,
                  const float* dopacities, cudaStream_t s) {
    int st = vks::validate_begin(s);
    if (!st) st = vks::validate_finite(dmeans2d, 2 * n, s);
    if (!st) st = vks::validate_finite(dconics, 3 * n, s);
    if (!st) st = vks::validate_finite(dcolors, 3 * n, s);
    if (!st) st = vks::validate_finite(dopacities, n, s);
    return st ? st : vks::validate_end(s);
}

}  // namespace

extern "C" {

const char* vks_status_string(int status) {
    switch (status) {
        case VKS_OK: return "ok";
        case VKS_ERR_INVALID_ARG: return "invalid argument";
        case VKS_ERR_CAPACITY: return "intersection capacity exceeded (regrow keys/vals to num_isects)";
        case VKS_ERR_WORKSPACE: return "workspace too small";
        case VKS_ERR_CUDA: return "CUDA error";
        case VKS_ERR_UNSUPPORTED: return "unsupported configuration";
        case VKS_ERR_NONFINITE: return "non-finite input (VKS_FLAG_VALIDATE)";
        case VKS_ERR_UNSORTED: return "tile lists are not a sorted binning (VKS_FLAG_VALIDATE / vks_bin_sort_check)";
        default: return "unknown status";
    }
}

int vks_version(void) { return VKS_VERSION; }

const char* vks_last_cuda_error(void) { return vks::last_error_buf(); }

int vks_project_fwd(const vks_config* cfg, const vks_camera* cam, int64_t n, const float* means,
                    const float* log_scales, const float* quats, const float* opacity_logits,
                    const float* sh, float* means2d, float* conics, float* depths, int32_t* radii,
                    int32_t* tiles_touched, float* colors, float* opacities, float* records,
                    vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (!camera_ok(cam) || n < 0) return VKS_ERR_INVALID_ARG;
    // conics may be NULL when the records (which carry them) are written
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits || !sh || !means2d || (!conics && !records) ||
                  !depths || !radii || !tiles_touched || !colors || !opacities))
        return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(quats) & 15) || (reinterpret_cast<uintptr_t>(means2d) & 7) ||
        (reinterpret_cast<uintptr_t>(radii) & 7) || (reinterpret_cast<uintptr_t>(records) & 15))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg) && (st = check_params(n, cfg->sh_coeffs, means, log_scales, quats, opacity_logits, sh,
                                              (cudaStream_t)stream)))
        return st;
    return cuda_status(vks::launch_project_fwd(*cfg, *cam, n, means, log_scales, quats, opacity_logits, sh,
                                               means2d, conics, depths, radii, tiles_touched, colors,
                                               opacities, records, (cudaStream_t)stream));
}

size_t vks_bin_sort_workspace_bytes(int64_t n, int64_t capacity, int32_t n_tiles) {
    if (n < 0 || capacity < 0 || n_tiles <= 0) return 0;
    return vks::bin_sort_workspace_bytes(n, capacity, n_tiles);
}

int vks_bin_sort(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                 const float* depths, const int32_t* tiles_touched, uint32_t* offsets, int64_t capacity,
                 uint64_t* keys, uint32_t* vals, uint64_t* keys_unsorted, uint32_t* vals_unsorted,
                 uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects, void* workspace,
                 size_t workspace_bytes, vks_stream_t stream) {
    if (!camera_ok(cam) || n < 0 || capacity < 0 || !num_isects || !tile_offsets) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || !radii || !depths || !tiles_touched || !offsets)) return VKS_ERR_INVALID_ARG;
    if (capacity > 0 && !vals) return VKS_ERR_INVALID_ARG;  // keys is optional
    if (!workspace) return VKS_ERR_WORKSPACE;
    if ((reinterpret_cast<uintptr_t>(means2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7))
        return VKS_ERR_INVALID_ARG;
    if (n >= (1ll << 32)) return VKS_ERR_UNSUPPORTED;  // Gaussian ids are u32
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::run_bin_sort(*cam, n, means2d, radii, depths, tiles_touched, offsets, capacity, keys,
                                         vals, keys_unsorted, vals_unsorted, tile_offsets, tile_order, num_isects,
                                         workspace,
                                         workspace_bytes, (cudaStream_t)stream));
}

int vks_bin_sort_async(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const int32_t* tiles_touched, uint32_t* offsets, int64_t capacity,
                       uint32_t* vals, uint32_t* tile_offsets, uint32_t* tile_order, int64_t* num_isects,
                       int32_t* status, void* workspace, size_t workspace_bytes, vks_stream_t stream) {
    if (!camera_ok(cam) || n < 0 || capacity < 0 || !num_isects || !status || !tile_offsets) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || !radii || !depths || !tiles_touched || !offsets)) return VKS_ERR_INVALID_ARG;
    if (capacity > 0 && !vals) return VKS_ERR_INVALID_ARG;
    if (!workspace) return VKS_ERR_WORKSPACE;
    if ((reinterpret_cast<uintptr_t>(means2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7) ||
        (reinterpret_cast<uintptr_t>(num_isects) & 7) || (reinterpret_cast<uintptr_t>(status) & 3))
        return VKS_ERR_INVALID_ARG;
    if (n >= (1ll << 32)) return VKS_ERR_UNSUPPORTED;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::run_bin_sort_async(*cam, n, means2d, radii, depths, tiles_touched, offsets, capacity, vals,
                                               tile_offsets, tile_order, num_isects, status, workspace,
                                               workspace_bytes, (cudaStream_t)stream));
}

int vks_bin_sort_check(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const uint32_t* vals, const uint32_t* tile_offsets, int64_t num_isects,
                       vks_stream_t stream) {
    if (!camera_ok(cam) || n < 0 || num_isects < 0 || !tile_offsets) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || !radii || !depths)) return VKS_ERR_INVALID_ARG;
    if (num_isects > 0 && !vals) return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(means2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    int st = vks::validate_begin((cudaStream_t)stream);
    if (!st) st = vks::validate_bins(*cam, n, means2d, radii, depths, vals, tile_offsets, num_isects, (cudaStream_t)stream);
    return st ? st : vks::validate_end((cudaStream_t)stream);
}

int vks_raster_fwd(const vks_config* cfg, const vks_camera* cam, int64_t n, const float* means2d,
                   const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                   const float* records, const uint32_t* vals, const uint32_t* tile_offsets,
                   const uint32_t* tile_order, float* image, float* T_final, int32_t* n_contrib,
                   vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (!camera_ok(cam) || n < 0) return VKS_ERR_INVALID_ARG;
    if (!tile_offsets || !image || !T_final || !n_contrib) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || (!conics && !records) || !colors || !opacities || !radii)) return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(means2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7) ||
        (reinterpret_cast<uintptr_t>(records) & 15))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg)) {  // the tile lists index [0, n) through a CSR (S:155 UnsortedInput)
        st = vks::validate_begin((cudaStream_t)stream);
        if (!st) st = vks::validate_csr(tile_offsets, vks::tiles_x(*cam) * vks::tiles_y(*cam), -1, vals, n,
                                        (cudaStream_t)stream);
        if (!st) st = vks::validate_end((cudaStream_t)stream);
        if (st) return st;
    }
    return cuda_status(vks::launch_raster_fwd(*cfg, *cam, n, means2d, conics, colors, opacities, radii, records, vals,
                                              tile_offsets, tile_order, image, T_final, n_contrib,
                                              (cudaStream_t)stream));
}

int vks_raster_fwd_stats(const vks_config* cfg, const vks_camera* cam, int64_t n, const float* means2d,
                         const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                         const float* records, const uint32_t* vals, const uint32_t* tile_offsets,
                         const uint32_t* tile_order, uint64_t* stats, vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (!camera_ok(cam) || n < 0 || !tile_offsets || !stats) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || (!conics && !records) || !colors || !opacities || !radii)) return VKS_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(records) & 15) return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    return vks::launch_raster_fwd_stats(*cfg, *cam, means2d, conics, colors, opacities, radii, records, vals, tile_offsets,
                                        tile_order, reinterpret_cast<unsigned long long*>(stats), n,
                                        (cudaStream_t)stream);
}

int vks_raster_bwd(const vks_config* cfg, const vks_camera* cam, int64_t n, const float* means2d,
                   const float* conics, const float* colors, const float* opacities, const int32_t* radii,
                   const float* records, const uint32_t* vals, const uint32_t* tile_offsets,
                   const uint32_t* tile_order, const float* T_final, const int32_t* n_contrib,
                   const float* dL_dimage, float* dmeans2d, float* dconics, float* dcolors,
                   float* dopacities, vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (!camera_ok(cam) || n < 0) return VKS_ERR_INVALID_ARG;
    if (!tile_offsets || !T_final || !n_contrib || !dL_dimage) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means2d || (!conics && !records) || !colors || !opacities || !radii || !dmeans2d || !dconics ||
                  !dcolors || !dopacities))
        return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(means2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7) ||
        (reinterpret_cast<uintptr_t>(records) & 15))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg)) {  // finite upstream gradient, tile lists a CSR over [0, n)
        st = vks::validate_begin((cudaStream_t)stream);
        if (!st) st = vks::validate_finite(dL_dimage, 3 * (int64_t)cam->width * cam->height, (cudaStream_t)stream);
        if (!st) st = vks::validate_csr(tile_offsets, vks::tiles_x(*cam) * vks::tiles_y(*cam), -1, vals, n,
                                        (cudaStream_t)stream);
        if (!st) st = vks::validate_end((cudaStream_t)stream);
        if (st) return st;
    }
    return cuda_status(vks::launch_raster_bwd(*cfg, *cam, n, means2d, conics, colors, opacities, radii, records, vals,
                                              tile_offsets, tile_order, T_final, n_contrib, dL_dimage, dmeans2d,
                                              dconics,
                                              dcolors, dopacities, (cudaStream_t)stream));
}

int vks_project_bwd(const vks_config* cfg, const vks_camera* cam, int64_t n, const float* means,
                    const float* log_scales, const float* quats, const float* opacity_logits,
                    const float* sh, const float* colors, const int32_t* radii, const float* dmeans2d, const float* dconics,
                    const float* dcolors, const float* dopacities, float* dmeans, float* dlog_scales,
                    float* dquats, float* dopacity_logits, float* dsh, vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (!camera_ok(cam) || n < 0) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits || !sh || !colors || !radii || !dmeans2d ||
                  !dconics || !dcolors || !dopacities || !dmeans || !dlog_scales || !dquats ||
                  !dopacity_logits || !dsh))
        return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(quats) & 15) || (reinterpret_cast<uintptr_t>(dquats) & 15) ||
        (reinterpret_cast<uintptr_t>(dmeans2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg) &&
        ((st = check_params(n, cfg->sh_coeffs, means, log_scales, quats, opacity_logits, sh, (cudaStream_t)stream)) ||
         (st = check_grads2d(n, dmeans2d, dconics, dcolors, dopacities, (cudaStream_t)stream))))
        return st;
    return cuda_status(vks::launch_project_bwd(*cfg, *cam, n, means, log_scales, quats, opacity_logits, sh, colors, radii,
                                               dmeans2d, dconics, dcolors, dopacities, dmeans, dlog_scales,
                                               dquats, dopacity_logits, dsh, (cudaStream_t)stream));
}

int vks_project_fwd_batch(const vks_config* cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                          const float* means, const float* log_scales, const float* quats,
                          const float* opacity_logits, const float* sh, float* const* means2d,
                          float* const* conics, float* const* depths, int32_t* const* radii,
                          int32_t* const* tiles_touched, float* const* colors, float* opacities,
                          float* const* g2d_zero, float* const* records, vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (n_views < 1 || n_views > 16 || !cams || n < 0) return VKS_ERR_INVALID_ARG;
    if (records)
        for (int v = 0; v < n_views; v++)
            if (n > 0 && (!records[v] || (reinterpret_cast<uintptr_t>(records[v]) & 15))) return VKS_ERR_INVALID_ARG;
    if (!means2d || !conics || !depths || !radii || !tiles_touched || !colors) return VKS_ERR_INVALID_ARG;
    if (g2d_zero)
        for (int v = 0; v < n_views; v++)
            if (n > 0 && (!g2d_zero[v] || (reinterpret_cast<uintptr_t>(g2d_zero[v]) & 7))) return VKS_ERR_INVALID_ARG;
    for (int v = 0; v < n_views; v++) {
        if (!camera_ok(cams + v) || cams[v].width != cams[0].width || cams[v].height != cams[0].height)
            return VKS_ERR_INVALID_ARG;
        if (n > 0 && (!means2d[v] || (!conics[v] && !records) || !depths[v] || !radii[v] || !tiles_touched[v] ||
                      !colors[v]))
            return VKS_ERR_INVALID_ARG;
        if ((reinterpret_cast<uintptr_t>(means2d[v]) & 7) || (reinterpret_cast<uintptr_t>(radii[v]) & 7))
            return VKS_ERR_INVALID_ARG;
    }
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits || !sh || !opacities)) return VKS_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(quats) & 15) return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg) && (st = check_params(n, cfg->sh_coeffs, means, log_scales, quats, opacity_logits, sh,
                                              (cudaStream_t)stream)))
        return st;
    return cuda_status(vks::launch_project_fwd_batch(*cfg, n_views, cams, n, means, log_scales, quats, opacity_logits,
                                                     sh, means2d, conics, depths, radii, tiles_touched, colors,
                                                     opacities, g2d_zero, records, (cudaStream_t)stream));
}

int vks_project_bwd_batch(const vks_config* cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                          const float* means, const float* log_scales, const float* quats,
                          const float* opacity_logits, const float* sh, const float* const* colors,
                          const int32_t* const* radii, const float* const* dmeans2d, const float* const* dconics,
                          const float* const* dcolors, const float* const* dopacities, float* dmeans,
                          float* dlog_scales, float* dquats, float* dopacity_logits, float* dsh,
                          vks_stream_t stream) {
    int st = config_ok(cfg);
    if (st) return st;
    if (n_views < 1 || n_views > 16 || !cams || n < 0) return VKS_ERR_INVALID_ARG;
    if (!colors || !radii || !dmeans2d || !dconics || !dcolors || !dopacities) return VKS_ERR_INVALID_ARG;
    for (int v = 0; v < n_views; v++) {
        if (!camera_ok(cams + v)) return VKS_ERR_INVALID_ARG;
        if (n > 0 && (!colors[v] || !radii[v] || !dmeans2d[v] || !dconics[v] || !dcolors[v] || !dopacities[v]))
            return VKS_ERR_INVALID_ARG;
        if ((reinterpret_cast<uintptr_t>(dmeans2d[v]) & 7) || (reinterpret_cast<uintptr_t>(radii[v]) & 7))
            return VKS_ERR_INVALID_ARG;
    }
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits || !sh || !dmeans || !dlog_scales || !dquats ||
                  !dopacity_logits || !dsh))
        return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(quats) & 15) || (reinterpret_cast<uintptr_t>(dquats) & 15))
        return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    if (validating(cfg)) {
        if ((st = check_params(n, cfg->sh_coeffs, means, log_scales, quats, opacity_logits, sh, (cudaStream_t)stream)))
            return st;
        for (int v = 0; v < n_views; v++)
            if ((st = check_grads2d(n, dmeans2d[v], dconics[v], dcolors[v], dopacities[v], (cudaStream_t)stream)))
                return st;
    }
    return cuda_status(vks::launch_project_bwd_batch(*cfg, n_views, cams, n, means, log_scales, quats, opacity_logits,
                                                     sh, colors, radii, dmeans2d, dconics, dcolors, dopacities,
                                                     dmeans, dlog_scales, dquats, dopacity_logits, dsh,
                                                     (cudaStream_t)stream));
}

int vks_adam_step(const vks_adam_config* acfg, int64_t n, int32_t sh_coeffs, float* const* params,
                  const float* const* grads, float* const* m, float* const* v, vks_stream_t stream) {
    if (!acfg || n < 0 || sh_coeffs < 1 || sh_coeffs > 64 || !params || !grads || !m || !v) return VKS_ERR_INVALID_ARG;
    if (acfg->step < 1 || !(acfg->beta1 >= 0.0f && acfg->beta1 < 1.0f) || !(acfg->beta2 >= 0.0f && acfg->beta2 < 1.0f) ||
        !(acfg->eps >= 0.0f))
        return VKS_ERR_INVALID_ARG;
    for (int q = 0; q < 5; q++) {
        const void* ptrs[4] = {params[q], grads[q], m[q], v[q]};
        for (const void* p : ptrs)
            if (n > 0 && (!p || (reinterpret_cast<uintptr_t>(p) & 15))) return VKS_ERR_INVALID_ARG;
    }
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_adam_step(*acfg, n, sh_coeffs, params, grads, m, v, (cudaStream_t)stream));
}

size_t vks_loss_workspace_bytes(int32_t width, int32_t height) {
    if (width < 1 || height < 1 || width > 65536 || height > 65536) return 0;
    return vks::loss_workspace_bytes(width, height);
}

int vks_loss_grad(int32_t width, int32_t height, float lambda, const float* render, const float* target,
                  float* dL_dimage, float* loss, void* workspace, size_t workspace_bytes, vks_stream_t stream) {
    if (width < 1 || height < 1 || width > 65536 || height > 65536) return VKS_ERR_INVALID_ARG;
    if (!(lambda >= 0.0f && lambda <= 1.0f)) return VKS_ERR_INVALID_ARG;
    if (lambda != 0.0f && (width < 11 || height < 11)) return VKS_ERR_INVALID_ARG;
    if (!render || !target || !dL_dimage || !workspace) return VKS_ERR_INVALID_ARG;
    if (workspace_bytes < vks::loss_workspace_bytes(width, height) || (reinterpret_cast<uintptr_t>(workspace) & 255))
        return VKS_ERR_WORKSPACE;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_loss_grad(width, height, lambda, render, target, dL_dimage, loss, workspace,
                                             (cudaStream_t)stream));
}

size_t vks_mcmc_workspace_bytes(int64_t n) {
    if (n < 0) return 0;
    return vks::mcmc_workspace_bytes(n);
}

int vks_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, uint64_t seed, float* means,
                      float* log_scales, float* quats, float* opacity_logits, float* sh, float* const* m,
                      float* const* v, int64_t* targets, int64_t* n_dead, void* workspace, size_t workspace_bytes,
                      vks_stream_t stream) {
    if (n < 0 || n >= ((int64_t)1 << 40) || sh_coeffs < 1 || sh_coeffs > 64) return VKS_ERR_INVALID_ARG;
    if (!(dead_opacity >= 0.0f && dead_opacity < 1.0f)) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits || !sh || !workspace)) return VKS_ERR_INVALID_ARG;
    if ((m == nullptr) != (v == nullptr)) return VKS_ERR_INVALID_ARG;
    if (m)
        for (int g = 0; g < 5; g++)
            if (n > 0 && (!m[g] || !v[g])) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (workspace_bytes < vks::mcmc_workspace_bytes(n) || (reinterpret_cast<uintptr_t>(workspace) & 255)))
        return VKS_ERR_WORKSPACE;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_mcmc_relocate(n, sh_coeffs, dead_opacity, seed, means, log_scales, quats,
                                                 opacity_logits, sh, m, v, targets, n_dead, workspace,
                                                 (cudaStream_t)stream));
}

int vks_mcmc_noise(int64_t n, float lr_pos, float noise_scale, uint64_t seed, uint32_t step, float* means,
                   const float* log_scales, const float* quats, const float* opacity_logits, vks_stream_t stream) {
    if (n < 0) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!means || !log_scales || !quats || !opacity_logits)) return VKS_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(quats) & 15) return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_mcmc_noise(n, lr_pos, noise_scale, seed, step, means, log_scales, quats,
                                              opacity_logits, (cudaStream_t)stream));
}

int vks_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom,
                      vks_stream_t stream) {
    if (n < 0) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (!dmeans2d || !radii || !accum || !denom)) return VKS_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(dmeans2d) & 7) || (reinterpret_cast<uintptr_t>(radii) & 7)) return VKS_ERR_INVALID_ARG;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_densify_stats(n, dmeans2d, radii, accum, denom, (cudaStream_t)stream));
}

size_t vks_densify_workspace_bytes(int64_t n) {
    if (n < 0) return 0;
    return vks::densify_workspace_bytes(n);
}

int vks_densify(int64_t n, int32_t sh_coeffs, const float* const* params, const float* const* m, const float* const* v,
                const float* accum, const float* denom, float grad_threshold, float size_threshold, float prune_opacity,
                uint64_t seed, int64_t capacity, float* const* out_params, float* const* out_m, float* const* out_v,
                int64_t* n_out, void* workspace, size_t workspace_bytes, vks_stream_t stream) {
    if (n < 0 || n >= ((int64_t)1 << 31) || sh_coeffs < 1 || sh_coeffs > 64 || capacity < 0 || !n_out)
        return VKS_ERR_INVALID_ARG;
    if (!params || !out_params) return VKS_ERR_INVALID_ARG;
    if ((m == nullptr) != (v == nullptr) || (out_m == nullptr) != (out_v == nullptr)) return VKS_ERR_INVALID_ARG;
    for (int g = 0; g < 5; g++) {
        if (n > 0 && (!params[g] || !out_params[g])) return VKS_ERR_INVALID_ARG;
        if (n > 0 && m && (!m[g] || !v[g])) return VKS_ERR_INVALID_ARG;
        if (n > 0 && out_m && (!out_m[g] || !out_v[g])) return VKS_ERR_INVALID_ARG;
    }
    if (n > 0 && (!accum || !denom || !workspace)) return VKS_ERR_INVALID_ARG;
    if (n > 0 && (workspace_bytes < vks::densify_workspace_bytes(n) || (reinterpret_cast<uintptr_t>(workspace) & 255)))
        return VKS_ERR_WORKSPACE;
    if (!device_present()) return VKS_ERR_CUDA;
    return cuda_status(vks::launch_densify(n, sh_coeffs, params, m, v, accum, denom, grad_threshold, size_threshold,
                                           prune_opacity, seed, capacity, out_params, out_m, out_v, n_out, workspace,
                                           (cudaStream_t)stream));
}

}  // extern "C"
