/*
 * vks.h — C ABI of the B200-native VkSplat hot path (libvks.so, sm_100a).
 *
 * The five entry points are the per-iteration stages the paper times
 * (§2 "Timing breakdown"; one call per table row or group):
 *
 *   vks_project_fwd  <- "Projection Forward"
 *   vks_bin_sort     <- "Index Offset", "Generate Keys", "Sorting", "Tile Ranges"
 *                       (grouped as "tiling/sorting")
 *   vks_raster_fwd   <- "Rasterization Forward"
 *   vks_raster_bwd   <- "Rasterization Backward"
 *   vks_project_bwd  <- "Proj Bwd + Optimizer", projection part
 *
 * The paper prints no formulas (PAPER.md is the supplementary timing/metric
 * tables only).  The operations follow the SPEC written from the paper
 * and the readings listed in
 * DESIGN.md §4 (e.g. support footprint, FOV clamp, SH degree 3).
 *
 * Conventions (all calls):
 *  - Every array argument is a DEVICE pointer (caller-owned; e.g. a torch
 *    tensor's data_ptr) unless marked HOST.  All arrays are dense, row-major,
 *    fp32 / int32 / uint32 / uint64 as typed, 16-byte aligned base pointers.
 *  - `stream` is a cudaStream_t (CUstream); every call only enqueues work on
 *    it and returns, except vks_bin_sort which synchronises `stream` once to
 *    read the intersection count.
 *  - The library never allocates or frees device memory and keeps no pointer
 *    between calls.  It is re-entrant; calls on different streams may overlap.
 *  - Gradient outputs ACCUMULATE (+=): the caller zeroes them (2D grads once
 *    per view, parameter grads once per batch of views).
 *  - Errors: synchronous argument checks return VKS_ERR_INVALID_ARG /
 *    VKS_ERR_UNSUPPORTED without launching anything; a failed launch returns
 *    VKS_ERR_CUDA; asynchronous device faults surface at the next sync
 *    (CUDA convention).  There is no CPU fallback: without a CUDA device
 *    every compute call returns VKS_ERR_CUDA.
 *
 * Coordinates: OpenCV camera axes (x right, y down, z forward); pixel (x,y)
 * has centre (x+0.5, y+0.5); tiles are 16x16, row-major ids
 * t = ty*TX + tx with TX = ceil(W/16), TY = ceil(H/16).
 */
#ifndef VKS_H
#define VKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VKS_VERSION 1
#define VKS_TILE 16

typedef struct CUstream_st* vks_stream_t; /* == cudaStream_t */

/* Pinhole camera, world->camera p_cam = R p_world + t. */
typedef struct {
    float R[9];      /* row-major rotation */
    float t[3];
    float fx, fy, cx, cy;
    int32_t width, height; /* 1 .. 65536 */
} vks_camera;

enum { VKS_FOOTPRINT_SUPPORT = 0, VKS_FOOTPRINT_3SIGMA = 1 };

typedef struct {
    int32_t sh_degree;  /* active SH degree D in 0..3 (north_star: degree 3) */
    int32_t sh_coeffs;  /* coefficients stored per Gaussian, >= (D+1)^2; sh row = 3*sh_coeffs floats */
    float near_plane;   /* cull if !(t.z > near) (0.01) */
    float bg[3];        /* background colour (default 0) */
    int32_t fov_clamp;  /* 1 = clamp tx/tz, ty/tz to 1.3x the image half-FOV inside J (gsplat/3DGS) */
    int32_t footprint;  /* VKS_FOOTPRINT_SUPPORT (default): exact alpha>=1/255 support bbox;
                           VKS_FOOTPRINT_3SIGMA: ceil(3 sqrt(lambda_max)) square */
    uint32_t flags;     /* VKS_FLAG_* bits, 0 = defaults */
} vks_config;

/* vks_project_bwd WRITES its parameter gradients instead of accumulating them, and writes zeros
 * to the rows of Gaussians with radii == 0 (first view of a batch: no memset of the buffer). */
#define VKS_FLAG_GRAD_OVERWRITE 1u
/* Debug mode (SURVEY §8(b) "Errors"): before computing, the entry point checks its inputs on the
 * device and synchronises `stream` once to read the result —
 *   vks_project_fwd(_batch), vks_project_bwd(_batch): every parameter finite and every quaternion
 *     of norm > 1e-12, else VKS_ERR_NONFINITE (S:119 NonFiniteParameter, S:52 ZeroQuaternion);
 *     the backward also checks its 2D gradients;
 *   vks_raster_fwd / vks_raster_bwd: tile_offsets a CSR (starts at 0, non-decreasing) whose entries
 *     index [0, n), else VKS_ERR_UNSORTED (S:155 UnsortedInput); the backward also checks that
 *     dL_dimage is finite (VKS_ERR_NONFINITE).
 * Nothing is written when a check fails.  Without the flag, non-finite Gaussians are culled by the
 * projection and nothing is checked.  Uses a module-scope device status word:
 * not for concurrent streams. */
#define VKS_FLAG_VALIDATE 2u

enum {
    VKS_OK = 0,
    VKS_ERR_INVALID_ARG = 1,
    VKS_ERR_CAPACITY = 2,   /* vks_bin_sort: M > capacity; *num_isects holds M (regrow and re-call) */
    VKS_ERR_WORKSPACE = 3,  /* workspace too small */
    VKS_ERR_CUDA = 4,       /* launch / runtime failure (incl. no CUDA device) */
    VKS_ERR_UNSUPPORTED = 5, /* configuration outside the library's limits (e.g. M >= 2^30 keys) */
    VKS_ERR_NONFINITE = 6,   /* VKS_FLAG_VALIDATE: a non-finite input (S:119 NonFiniteParameter) */
    VKS_ERR_UNSORTED = 7     /* VKS_FLAG_VALIDATE / vks_bin_sort_check: not a sorted binning */
};

const char* vks_status_string(int status);
int vks_version(void);
/* last CUDA error string seen by this thread (for VKS_ERR_CUDA) */
const char* vks_last_cuda_error(void);

/*
 * vks_project_fwd — "Projection Forward".
 * Per Gaussian i: t = R mu + t; cull !(t.z > near); q-hat = q/|q| (w,x,y,z);
 * Sigma' = J (R Rq S)(R Rq S)^T J^T + 0.3 I; conic = Sigma'^-1 as (a,b,c);
 * mean2d = (fx tx/tz + cx, fy ty/tz + cy); depth = tz; opacity = sigmoid(o);
 * colour = max(0, sum_l Y_l(d) f_l + 0.5) (3DGS real SH); footprint radii and
 * tiles_touched = #16x16 tiles of the footprint rect clipped to the image.
 *   n                Gaussians (>= 0)
 *   means [n,3], log_scales [n,3], quats [n,4] (w,x,y,z, need not be unit),
 *   opacity_logits [n], sh [n, sh_coeffs, 3]
 *   -> means2d [n,2], conics [n,3], depths [n], radii [n,2] int32,
 *      tiles_touched [n] int32, colors [n,3], opacities [n]
 * Rows with tiles_touched == 0 (culled / off-image) have radii = (0,0); their
 * other outputs are unspecified (currently written as zeros: whole-row stores keep
 * every DRAM sector fully written, which avoids read-modify-write fills).  fp32,
 * operation order pinned (bit-exact with the oracle's O1).
 *   records [n,12] fp32 (nullable, 16-byte aligned): the packed raster record of every row with
 *      tiles_touched > 0 — the values the rasterizer stages per list entry, copied from the
 *      outputs above: (u, v, a/2, b), (c/2, opacity, c0, c1), (c2, bits of the row index i, 0, 0),
 *      one 48-byte row per Gaussian.  Passed to
 *      vks_raster_fwd / vks_raster_bwd, the rasterizer copies each tile's batches of entries into
 *      shared memory with cp.async (three 16-byte copies per entry) instead of gathering eight
 *      scalars from the separate arrays; results are identical.  Rows with tiles_touched == 0 are
 *      written as zeros (each warp stores its 32 rows as three coalesced 512-byte runs).  With
 *      records given, conics may be NULL (not written; the records carry a/2, b, c/2).
 */
int vks_project_fwd(const vks_config* cfg, const vks_camera* cam, int64_t n,
                    const float* means, const float* log_scales, const float* quats,
                    const float* opacity_logits, const float* sh,
                    float* means2d, float* conics, float* depths, int32_t* radii,
                    int32_t* tiles_touched, float* colors, float* opacities, float* records,
                    vks_stream_t stream);

/*
 * vks_bin_sort_workspace_bytes — device workspace needed by vks_bin_sort for
 * n Gaussians, a key capacity `capacity` and n_tiles tiles (~60 B per Gaussian + 16 B
 * per key slot).  Returns 0 for n < 0 or n_tiles < 1.
 */
size_t vks_bin_sort_workspace_bytes(int64_t n, int64_t capacity, int32_t n_tiles);

/*
 * vks_bin_sort — "Index Offset" + "Generate Keys" + "Sorting" + "Tile Ranges"
 * (S:124-159).
 *   offsets [n] u32      <- exclusive prefix sum of tiles_touched
 *   *num_isects (HOST)   <- M = sum tiles_touched
 *   for each i with tiles_touched > 0 and each tile (ty outer, tx inner) of its
 *   rect: slot offsets[i]+k gets key = (tile << 32) | f32bits(depth_i), val = i
 *   keys/vals [capacity] <- the M pairs stable-sorted ascending by key (u64); keys is
 *                           nullable (the rasterizer needs only vals and tile_offsets)
 *   tile_offsets [n_tiles+1] u32 <- CSR: #entries with tile id < t
 *   tile_order [n_tiles] u32 (nullable) <- the tile ids ordered by decreasing list length
 *                           (approximately: log-spaced length classes) — a scheduling hint for
 *                           the rasterizer (heaviest tiles first); results never depend on it
 *   keys_unsorted / vals_unsorted (nullable, debug; [capacity] like keys/vals): the pre-sort pairs.
 * Tile grids of >= 2^20 tiles return VKS_ERR_INVALID_ARG.
 * If M > capacity returns VKS_ERR_CAPACITY after writing offsets and *num_isects, touching no
 * other output; the call is idempotent, so the caller regrows and calls again.  M >= 2^30 is a
 * hard limit of the sort (30-bit look-back counts): VKS_ERR_UNSUPPORTED, *num_isects = M, no
 * capacity helps.  Synchronises `stream` once (to read M).
 * workspace: device memory of >= vks_bin_sort_workspace_bytes(n, capacity, n_tiles), 256-byte
 * aligned (else VKS_ERR_WORKSPACE).
 */
int vks_bin_sort(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                 const float* depths, const int32_t* tiles_touched, uint32_t* offsets,
                 int64_t capacity, uint64_t* keys, uint32_t* vals, uint64_t* keys_unsorted,
                 uint32_t* vals_unsorted, uint32_t* tile_offsets, uint32_t* tile_order,
                 int64_t* num_isects,
                 void* workspace, size_t workspace_bytes, vks_stream_t stream);

/*
 * vks_bin_sort_async — vks_bin_sort without the host synchronisation (stream-ordered and
 * CUDA-graph capturable): the same tile lists (ids in (depth bits, id) order per tile) and CSR
 * tile_offsets, bit-identical, but M is written to the DEVICE word *num_isects (int64, 8-byte
 * aligned) together with a DEVICE status word *status (int32): VKS_OK; VKS_ERR_CAPACITY if
 * M > capacity, or VKS_ERR_UNSUPPORTED if M >= 2^30 — then every tile list is left empty
 * (tile_offsets all zero, so a rasterizer launched behind it reads nothing) and the caller regrows
 * and re-runs.  Every kernel is launched for the host-side bounds (n Gaussians, `capacity` keys)
 * and reads the actual counts on the device; the launch sequence depends only on (n, capacity,
 * camera size).  No u64 keys and no debug outputs.  capacity >= 2^30: VKS_ERR_UNSUPPORTED.
 * Other arguments, the workspace and its size as for vks_bin_sort.
 */
int vks_bin_sort_async(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const int32_t* tiles_touched, uint32_t* offsets,
                       int64_t capacity, uint32_t* vals, uint32_t* tile_offsets, uint32_t* tile_order,
                       int64_t* num_isects, int32_t* status, void* workspace, size_t workspace_bytes,
                       vks_stream_t stream);

/*
 * vks_bin_sort_check — debug verification of a binning ("Tile Ranges" errors, S:155 UnsortedInput):
 * checks that tile_offsets [n_tiles+1] is a CSR of [0, num_isects) (starts at 0, non-decreasing,
 * ends at num_isects), that every id vals[k] < n, that the tile rect of Gaussian vals[k] (projection
 * step 11 from means2d / radii) contains the tile k belongs to, and that the entries of every tile
 * are strictly ascending in (f32 bits of depths[id], id) — i.e. the sort of the (tile | depth) keys
 * with ties by id.  Returns VKS_OK or VKS_ERR_UNSORTED; synchronises `stream` once; writes nothing.
 * Inputs as produced by vks_project_fwd / vks_bin_sort (device pointers).
 */
int vks_bin_sort_check(const vks_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                       const float* depths, const uint32_t* vals, const uint32_t* tile_offsets,
                       int64_t num_isects, vks_stream_t stream);

/*
 * vks_raster_fwd — "Rasterization Forward".
 * Per pixel, front to back over its tile's sorted list:
 *   sigma = 1/2 a dx^2 + b dx dy + 1/2 c dy^2 (dx = u - (x+.5));  skip sigma < 0;
 *   alpha = min(0.99, rho e^-sigma); skip alpha < 1/255;  C += c alpha T;
 *   T *= 1 - alpha;  stop once T < 1e-4.   out = C + T bg.
 *   -> image [H,W,3], T_final [H,W], n_contrib [H,W] int32 (1-based position,
 *      within the tile's list, of the last composited entry; 0 = none).
 * means2d/conics/colors/opacities/radii as produced by vks_project_fwd, vals/tile_offsets (and
 * the optional tile_order: the order in which tiles are scheduled; nullptr = tile id order) as
 * produced by vks_bin_sort.  Before evaluating an entry, each warp tests whether any pixel centre
 * of its 8x8 patch can reach alpha >= 1/255 (exact minimum of sigma over the patch against
 * ln(255 rho), with an fp32 error margin) and skips the entry warp-uniformly if none can; radii
 * (the support box) are read only by the diagnostic box-culling mode (VKS_RASTER_CULL=1).
 * records (nullable, 16-byte aligned): vks_project_fwd's packed raster records of the same view;
 * when given, each warp's batches of 32 entries are copied into shared memory with cp.async
 * (double-buffered, the next batch in flight while one is composited) instead of gathered from
 * means2d / conics / colors / opacities; identical results.  With records, conics may be NULL
 * (VKS_ERR_INVALID_ARG if the diagnostic box-culling mode VKS_RASTER_CULL=1, which gathers from
 * the separate arrays, is selected then).
 */
int vks_raster_fwd(const vks_config* cfg, const vks_camera* cam, int64_t n,
                   const float* means2d, const float* conics, const float* colors,
                   const float* opacities, const int32_t* radii, const float* records,
                   const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                   float* image, float* T_final, int32_t* n_contrib,
                   vks_stream_t stream);

/*
 * vks_raster_fwd_stats — diagnostic twin of vks_raster_fwd for the roofline model:
 * runs the same compositing without writing the image and ACCUMULATES into the device counters
 *   stats[0] += list entries visited before each pixel's stop (the algorithm's evaluations)
 *   stats[1] += composited (pixel, Gaussian) pairs
 *   stats[2] += pairs actually evaluated by the kernel (after its patch culling)
 *   stats[3] += sum of n_contrib (entries the backward replays)
 *   stats[4] += (warp, entry) pairs processed after patch culling
 *   stats[5] += of those, pairs with at least one composited pixel
 * stats must hold 6 uint64 counters.  records (nullable) as for vks_raster_fwd (same counts).
 */
int vks_raster_fwd_stats(const vks_config* cfg, const vks_camera* cam, int64_t n,
                         const float* means2d, const float* conics, const float* colors,
                         const float* opacities, const int32_t* radii, const float* records,
                         const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                         uint64_t* stats, vks_stream_t stream);

/*
 * vks_raster_bwd — "Rasterization Backward".
 * Replays each pixel back to front from n_contrib, recovering T by division,
 * and ACCUMULATES exact gradients of the forward w.r.t. mean2d, conic (a,b,c
 * as independent scalars), colour and opacity (0 where alpha was clamped).
 *   dL_dimage [H,W,3] -> dmeans2d [n,2], dconics [n,3], dcolors [n,3], dopacities [n] (+=)
 * tile_order and records as for vks_raster_fwd (nullable).
 */
int vks_raster_bwd(const vks_config* cfg, const vks_camera* cam, int64_t n,
                   const float* means2d, const float* conics, const float* colors,
                   const float* opacities, const int32_t* radii, const float* records,
                   const uint32_t* vals, const uint32_t* tile_offsets, const uint32_t* tile_order,
                   const float* T_final, const int32_t* n_contrib, const float* dL_dimage,
                   float* dmeans2d, float* dconics, float* dcolors, float* dopacities,
                   vks_stream_t stream);

/*
 * vks_project_bwd — projection part of "Proj Bwd + Optimizer".
 * Chain rule from the 2D gradients to the parameters for every Gaussian with
 * radii != 0 (others untouched): conic inversion, Sigma' = J W Sigma W^T J^T
 * (+0.3 passes the gradient), exact FOV-clamp derivative, quaternion
 * normalisation, exp / sigmoid activations, SH colour (clamped channels give 0).
 * colors / radii are vks_project_fwd's outputs for the same view: colour == 0 marks a clamped
 * channel, radii != 0 a rasterised Gaussian.
 *   -> dmeans [n,3], dlog_scales [n,3], dquats [n,4], dopacity_logits [n],
 *      dsh [n, sh_coeffs, 3]   (+=; with VKS_FLAG_GRAD_OVERWRITE: =, and zero rows for radii == 0)
 */
int vks_project_bwd(const vks_config* cfg, const vks_camera* cam, int64_t n,
                    const float* means, const float* log_scales, const float* quats,
                    const float* opacity_logits, const float* sh, const float* colors,
                    const int32_t* radii,
                    const float* dmeans2d, const float* dconics, const float* dcolors,
                    const float* dopacities, float* dmeans, float* dlog_scales, float* dquats,
                    float* dopacity_logits, float* dsh, vks_stream_t stream);

/*
 * vks_project_fwd_batch — "Projection Forward" of a batch of views in one pass over the
 * parameters: the camera-independent part of DESIGN.md §4.1 (unit quaternion, rotation, X64
 * scales and opacity, the footprint's X64 log) once per Gaussian, the SH row read once, then
 * every view's steps exactly as vks_project_fwd — each view's outputs are bit-identical to a
 * vks_project_fwd call for that view (except the opacities, below).
 *   n_views in [1, 16] (VKS_ERR_INVALID_ARG otherwise); cams: HOST array of n_views cameras, all
 *   with the same width and height
 *   means2d, conics, depths, radii, tiles_touched, colors: HOST arrays of n_views DEVICE
 *     pointers, each laid out as the matching vks_project_fwd output
 *   opacities [n]: one array for the batch (the opacity is view-independent); rows the
 *     footprint test culls are unspecified
 *   g2d_zero (nullable): HOST array of n_views DEVICE pointers, each a view's [9n] fp32 block of
 *     2D-gradient accumulators (dmeans2d [n,2] | dconics [n,3] | dcolors [n,3] | dopacities [n],
 *     8-byte aligned) that vks_raster_bwd will add into: zeroed here, in the same pass, instead
 *     of by a separate memset
 *   records (nullable): HOST array of n_views DEVICE pointers, each a view's [n,12] packed raster
 *     records as for vks_project_fwd (16-byte aligned); with records, conics[v] may be NULL
 */
int vks_project_fwd_batch(const vks_config* cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                          const float* means, const float* log_scales, const float* quats,
                          const float* opacity_logits, const float* sh, float* const* means2d,
                          float* const* conics, float* const* depths, int32_t* const* radii,
                          int32_t* const* tiles_touched, float* const* colors, float* opacities,
                          float* const* g2d_zero, float* const* records, vks_stream_t stream);

/*
 * vks_project_bwd_batch — the projection backward of a batch of views in one pass: the sum over
 * the views of vks_project_bwd (P:76 projection part; a training step's views share one set of
 * parameter gradients).  Each view's chain is exactly vks_project_bwd's;
 * every parameter row and SH row is read once and every gradient row written once, instead of
 * one read-modify-write of the whole gradient buffer per view.
 *   n_views in [1, 16] (VKS_ERR_INVALID_ARG otherwise)
 *   cams: HOST array of n_views cameras
 *   colors, radii, dmeans2d, dconics, dcolors, dopacities: HOST arrays of n_views DEVICE
 *     pointers — each view's vks_project_fwd colours / radii and vks_raster_bwd 2D gradients,
 *     laid out as for vks_project_bwd
 *   -> dmeans, dlog_scales, dquats, dopacity_logits, dsh as vks_project_bwd, holding the sum
 *      over the views (+=; with VKS_FLAG_GRAD_OVERWRITE: =, and zero rows for Gaussians no view
 *      rasterises)
 */
int vks_project_bwd_batch(const vks_config* cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                          const float* means, const float* log_scales, const float* quats,
                          const float* opacity_logits, const float* sh,
                          const float* const* colors, const int32_t* const* radii,
                          const float* const* dmeans2d, const float* const* dconics,
                          const float* const* dcolors, const float* const* dopacities,
                          float* dmeans, float* dlog_scales, float* dquats, float* dopacity_logits,
                          float* dsh, vks_stream_t stream);

/* ---- the optimizer step after the path ---------------------------------
 *
 * vks_adam_step — Adam with bias correction per parameter group ("adam_step":
 * "standard Adam with bias correction per parameter group"; PAPER P:76 row "Proj Bwd +
 * Optimizer"), quaternions re-normalised after the step.  For step t = acfg->step >= 1,
 * element-wise in fp32:
 *     m <- b1 m + (1 - b1) g;   v <- b2 v + (1 - b2) g^2
 *     p <- p - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 * Groups (index into params / grads / m / v): 0 means [n,3], 1 log_scales [n,3], 2 quats [n,4]
 * (then q <- q / |q| per row), 3 opacity_logits [n], 4 sh [n, sh_coeffs, 3]; lr[0..3] per
 * group, lr[4] for SH coefficient 0 and lr[5] for the others.
 *   params, m, v: HOST arrays of 5 DEVICE fp32 pointers, updated in place (zero moments for a
 *     new Gaussian); grads: HOST array of 5 DEVICE pointers (e.g. the slices of the allreduced
 *     gradient buffer).  Every device pointer 16-byte aligned.
 * Errors (before any launch): VKS_ERR_INVALID_ARG for a null or unaligned pointer, n < 0,
 * step < 1, sh_coeffs outside [1, 64], a beta outside [0, 1) or eps < 0.  Asynchronous on
 * `stream`.  HBM-bound: 28 B per element (p, g, m, v in; p, m, v out).
 */
typedef struct {
    float lr[6];
    float beta1, beta2, eps;
    int32_t step;
} vks_adam_config;

int vks_adam_step(const vks_adam_config* acfg, int64_t n, int32_t sh_coeffs, float* const* params,
                  const float* const* grads, float* const* m, float* const* v, vks_stream_t stream);

/* ---- the loss gradient before the path --------------------------------
 *
 * vks_loss_grad — "Loss Gradient" (SSIM S:482):
 *   loss = (1 - lambda) mean_{pixels, channels} |render - target| + lambda (1 - SSIM)
 *   SSIM = mean over the 3 channels and the VALID window centres (no padding) of
 *          S = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx2 + sy2 + C2)),
 *   window statistics over the normalised 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
 *   C2 = 0.03^2;  dL_dimage = the exact gradient of `loss` with respect to render (L1
 *   subgradient sign(0) = 0) — the dL/dimage input of vks_raster_bwd.
 *   render, target: device [height, width, 3] fp32 (HWC, as vks_raster_fwd's image)
 *   dL_dimage: device [height, width, 3] fp32, written; loss: device fp32 [1], written (nullable)
 *   workspace: device, 256-byte aligned, >= vks_loss_workspace_bytes(width, height) bytes
 *     (one fp64 42x42 partial slot per 32x32 tile of window centres and channel: ~41 B per pixel)
 * Errors (before any launch): VKS_ERR_INVALID_ARG for a null pointer, a size outside [1, 65536],
 * lambda outside [0, 1], or lambda > 0 with width or height < 11; VKS_ERR_WORKSPACE.
 * Asynchronous on `stream`; deterministic.
 */
size_t vks_loss_workspace_bytes(int32_t width, int32_t height);
int vks_loss_grad(int32_t width, int32_t height, float lambda, const float* render, const float* target,
                  float* dL_dimage, float* loss, void* workspace, size_t workspace_bytes, vks_stream_t stream);

/* ---- MCMC densification at a fixed budget ------------------------------
 *
 * Counter-based generator (DESIGN.md §4.7 R1): h(seed, stream, i) = splitmix64(seed +
 * 0x9E3779B97F4A7C15 * ((stream << 40) ^ i)); uniform ((h >> 40) + 0.5) / 2^24; normal = Box-Muller
 * of the uniforms of counters 2k, 2k+1.
 *
 * vks_mcmc_relocate — relocation of "dead" Gaussians (SPEC S:273 densify_mcmc):
 * rho_i = sigmoid(opacity_logit_i) (evaluated in fp64, rounded to fp32); dead_i = rho_i <
 * dead_opacity; integer weights w_j = dead_j ? 0 : floor(rho_j 2^24); each dead i draws
 * t = mulhi64(h(seed, 1, i), sum w) and takes the first j with inclusive prefix W_j > t
 * (probability w_j / sum w), copies j's means, log_scales, quats and sh, and j with its k_j copies
 * all get rho' = 1 - (1 - rho_j)^(1/(k_j+1)) (appearance-conserving: (1 - rho')^(k_j+1) = 1 - rho_j),
 * logit' = log(rho'/(1 - rho')).  The copies' Adam moments are zeroed.  Count unchanged (the
 * budget).  Targets are exact integer decisions: identical to the CPU oracle's.
 *   parameters: device fp32 rows as vks_project_fwd's inputs, updated in place
 *   m, v: HOST arrays of 5 DEVICE pointers (the vks_adam_step groups) or both NULL
 *   targets: device int64 [n] (nullable) <- j for dead i, -1 otherwise
 *   n_dead: device int64 [1] (nullable) <- number of dead Gaussians
 *   workspace: device, 256-byte aligned, >= vks_mcmc_workspace_bytes(n) (~28 B per Gaussian)
 * Errors: VKS_ERR_INVALID_ARG (null pointer, n < 0, sh_coeffs outside [1, 64], dead_opacity
 * outside [0, 1), exactly one of m / v NULL); VKS_ERR_WORKSPACE.  Asynchronous on `stream`.
 *
 * vks_mcmc_noise — positional noise after an optimizer step (R5): means_i += lr_pos *
 * noise_scale * gate(rho_i) * Rq_i diag(exp(log_scales_i)) eps_i, gate(rho) = sigmoid(100 (0.005 -
 * rho)), eps_i = the normals of counters 3i .. 3i+2 of stream 2 + 2 step (fp64 arithmetic).
 * quats 16-byte aligned.  Asynchronous on `stream`.
 */
size_t vks_mcmc_workspace_bytes(int64_t n);
int vks_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, uint64_t seed, float* means,
                      float* log_scales, float* quats, float* opacity_logits, float* sh, float* const* m,
                      float* const* v, int64_t* targets, int64_t* n_dead, void* workspace, size_t workspace_bytes,
                      vks_stream_t stream);
int vks_mcmc_noise(int64_t n, float lr_pos, float noise_scale, uint64_t seed, uint32_t step, float* means,
                   const float* log_scales, const float* quats, const float* opacity_logits, vks_stream_t stream);

/* ---- default densification --------------------------------------------
 *
 * vks_densify_stats — screen-gradient statistics ("mean accumulated screen-gradient
 * norm"; DESIGN.md §4.7 R6), after a view's vks_raster_bwd: for every Gaussian the view rasterised
 * (radii != 0): accum += |dmeans2d| (Euclidean, pixels), denom += 1.
 *   dmeans2d [n,2] fp32, radii [n,2] i32 (8-byte aligned), accum / denom [n] fp32 (in place).
 *
 * vks_densify — one densification event (R7-R9).  Per Gaussian (rho = sigmoid(logit)
 * in fp64, rounded to fp32): rho < prune_opacity -> removed; else with g = accum / denom (0 when
 * denom = 0) and smax = the largest exp(log_scale): g > grad_threshold and smax < size_threshold
 * -> cloned (the row, then an identical copy); g > grad_threshold and smax >= size_threshold ->
 * split (two children: log_scales - ln 1.6, means + Rq diag(s) eps with eps the normals of
 * counters 6i + 3c .. 6i + 3c + 2 of stream 3 of the vks_mcmc generator, everything else copied);
 * otherwise kept.  Rows are written in input order (a copy or second child right after its
 * source); new rows get zero Adam moments, kept rows keep theirs.
 *   params: HOST array of 5 DEVICE pointers (means, log_scales, quats, opacity_logits, sh as
 *     vks_project_fwd's inputs); m, v: HOST arrays of 5 DEVICE pointers (vks_adam_step groups) or
 *     both NULL; out_params / out_m / out_v likewise, each with room for `capacity` rows
 *     (outputs never alias inputs)
 *   *n_out (HOST) <- n', the new count.  If n' > capacity: VKS_ERR_CAPACITY, nothing else
 *     written (grow the outputs, e.g. x1.5 as S:312, and call again).  Synchronises `stream`
 *     once (to read n').
 *   workspace: device, 256-byte aligned, >= vks_densify_workspace_bytes(n).
 * Opacity reset (every 3000 iterations) is a clamp of the logits the caller applies.
 */
int vks_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom,
                      vks_stream_t stream);
size_t vks_densify_workspace_bytes(int64_t n);
int vks_densify(int64_t n, int32_t sh_coeffs, const float* const* params, const float* const* m, const float* const* v,
                const float* accum, const float* denom, float grad_threshold, float size_threshold, float prune_opacity,
                uint64_t seed, int64_t capacity, float* const* out_params, float* const* out_m, float* const* out_v,
                int64_t* n_out, void* workspace, size_t workspace_bytes, vks_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VKS_H */
