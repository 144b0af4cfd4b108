/*
 * vko.h — CPU ORACLE for the VkSplat hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load, call or execute anything under oracle/.  The product
 * path (paper_2605_00219_b200/) never links or imports it, and the two share no
 * code, headers, constants or helpers.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, SURVEY §8c = /root/repo/SURVEY.md):
 *   - projection forward  ("Projection Forward")
 *   - index offsets       ("Index Offset";       S:124-132; §8c.3)
 *   - key generation      ("Generate Keys";      S:133-141; §8c.3)
 *   - stable sort         ("Sorting";            S:142-150; §8c.3)
 *   - tile ranges         ("Tile Ranges";        S:151-159; §8c.3)
 *   - compositing fwd     ("Rasterization Forward"; §8c.1, §8c.4)
 *     UNTILED: every pixel walks all candidates in global (depth, id) order.
 *   - compositing bwd     ("Rasterization Backward"; §8c.5)
 *   - projection bwd      ("Proj Bwd + Optimizer", projection part; §8c.6)
 *
 * Precision: O1 = fp32 forward with the operation order pinned in DESIGN.md §4
 * (the kernel's precision, because fp32 values decide integers: footprints,
 * tile rects, keys, skip/stop decisions).  O2 = the same formulas in fp64, and
 * every backward accumulates in fp64.  O3 = brute force (no bounding box).
 *
 * Parity pins: see tests/test_oracle_*.py.  "VkSplat's actual kernel
 * behaviour" is parity unpinned: the paper publishes timings only.
 */
#ifndef VKO_H
#define VKO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    float R[9];      /* world->camera rotation, row-major; OpenCV axes (x right, y down, z fwd) */
    float t[3];      /* p_cam = R p_world + t */
    float fx, fy, cx, cy;
    int32_t width, height;
} vko_camera;

typedef struct {
    int32_t sh_degree;   /* 0..3, active degree; K = (D+1)^2 coefficients used */
    int32_t sh_coeffs;   /* stored coefficients per Gaussian (row stride / 3), >= K */
    float near_plane;    /* 0.01 */
    float bg[3];         /* background colour (north_star: empty scene gives bg) */
    int32_t fov_clamp;   /* 1: gsplat/3DGS 1.3x tan-FOV clamp inside J */
    int32_t footprint;   /* 0 = exact alpha-support bbox (default), 1 = 3-sigma square */
} vko_config;

enum { VKO_FOOTPRINT_SUPPORT = 0, VKO_FOOTPRINT_3SIGMA = 1 };

/* per-Gaussian flag bits written by the projection */
enum {
    VKO_F_PROJECTABLE = 1 << 0, /* passed near / quaternion / det / finiteness / (support: rho) culls */
    VKO_F_VISIBLE = 1 << 1,     /* tiles_touched > 0 */
    VKO_F_CLAMP_R = 1 << 2,     /* colour channel clamped at 0 (raw <= 0) */
    VKO_F_CLAMP_G = 1 << 3,
    VKO_F_CLAMP_B = 1 << 4,
    VKO_F_FOVX_HI = 1 << 5,     /* tx/tz > lim_x+ : clamped at the upper x limit */
    VKO_F_FOVX_LO = 1 << 6,
    VKO_F_FOVY_HI = 1 << 7,
    VKO_F_FOVY_LO = 1 << 8
};

/* O1 projection (fp32, pinned order).  Outputs of non-visible rows: radii=0,
 * tiles=0, other fields are still written (garbage allowed, compared only on
 * visible rows).  cov2d [n,3] = (A,B,C) incl. +0.3 (nullable). */
void vko_project_fwd_f32(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const float* means, const float* log_scales, const float* quats,
                         const float* opacity_logits, const float* sh,
                         float* means2d, float* conics, float* depths, int32_t* radii,
                         int32_t* tiles_touched, float* colors, float* opacities,
                         float* cov2d, int32_t* flags, int nthreads);

/* O2 projection (fp64) of the same formulas; same layout, double outputs. */
void vko_project_fwd_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const double* means, const double* log_scales, const double* quats,
                         const double* opacity_logits, const double* sh,
                         double* means2d, double* conics, double* depths, int32_t* radii,
                         int32_t* tiles_touched, double* colors, double* opacities,
                         double* cov2d, int32_t* flags);

/* Binning (integer, exact). */
int64_t vko_scan_offsets(int64_t n, const int32_t* tiles_touched, uint32_t* offsets);
void vko_gen_keys(const vko_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                  const float* depths, const int32_t* tiles_touched, const uint32_t* offsets,
                  uint64_t* keys, uint32_t* vals);
void vko_sort_pairs(int64_t m, uint64_t* keys, uint32_t* vals);
void vko_tile_ranges(int64_t m, const uint64_t* keys, int32_t n_tiles, uint32_t* tile_offsets);

/* Forward + (optional) backward compositing, untiled.
 * Runs its own O1 projection from the parameters.
 *   dL_dimage [H,W,3] nullable -> no backward.
 *   row_mask [H] nullable -> all rows; else only rows with row_mask[y]!=0 are rendered
 *   brute != 0 -> O3: every candidate is tested at every pixel (no bbox).
 * Outputs: image [H,W,3], T_final [H,W], last_id [H,W] (-1 = none),
 *          fragile [H,W] (1 = a decision lies within the fast-exp window, §8c.9),
 *          stats [8]: 0 footprint violations, 1 evaluations, 2 composited,
 *                     3 fragile pixels, 4 candidates, 5 rows rendered
 * Backward outputs (fp64, overwritten): dmeans2d [n,2], dconics [n,3],
 *   dcolors [n,3], dopacities [n]; mass [n,9] nullable = sum |terms|.        */
int vko_render_f32(const vko_config* cfg, const vko_camera* cam, int64_t n,
                   const float* means, const float* log_scales, const float* quats,
                   const float* opacity_logits, const float* sh,
                   const float* dL_dimage, const uint8_t* row_mask, int brute,
                   float* image, float* T_final, int32_t* last_id, uint8_t* fragile,
                   int64_t* stats, double* dmeans2d, double* dconics, double* dcolors,
                   double* dopacities, double* mass, int nthreads);

/* fp64 forward render for finite differences (O2): image [H,W,3] double,
 * decision hash per pixel [H,W] (uint64; folds skip/clamp/stop decisions) and
 * projection flags [n].  If dL_dimage != NULL also returns the fp64 backward
 * (exact gradient of this fp64 forward) in the d* outputs. */
int vko_render_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                   const double* means, const double* log_scales, const double* quats,
                   const double* opacity_logits, const double* sh,
                   const double* dL_dimage, double* image, uint64_t* decision_hash,
                   int32_t* proj_flags, double* dmeans2d, double* dconics, double* dcolors,
                   double* dopacities);

/* Projection backward (O2, fp64).  Discrete decisions (cull,
 * FOV clamp, colour clamp) come from the O1 fp32 projection of the same
 * parameters.  Gradients are OVERWRITTEN (not accumulated). */
void vko_project_bwd(const vko_config* cfg, const vko_camera* cam, int64_t n,
                     const float* means, const float* log_scales, const float* quats,
                     const float* opacity_logits, const float* sh,
                     const double* dmeans2d, const double* dconics, const double* dcolors,
                     const double* dopacities,
                     double* dmeans, double* dlog_scales, double* dquats,
                     double* dopacity_logits, double* dsh, int nthreads);

/* Mass of the projection backward (non-negative inputs = masses of the 2D gradients; outputs =
 * sum of |terms| of each parameter gradient along the SURVEY §8c.6 chain, stage by stage).  Used
 * to classify condition-limited elements (DESIGN.md §7 P5); pinned by tests/test_oracle_mass.py. */
void vko_project_bwd_mass(const vko_config* cfg, const vko_camera* cam, int64_t n,
                          const float* means, const float* log_scales, const float* quats,
                          const float* opacity_logits, const float* sh,
                          const double* m_dmeans2d, const double* m_dconics, const double* m_dcolors,
                          const double* m_dopacities, double* m_dmeans, double* m_dlog_scales,
                          double* m_dquats, double* m_dopacity_logits, double* m_dsh, int nthreads);

/* fp64-parameter variant (for FD on double parameters); decisions from the
 * fp64 projection. */
void vko_project_bwd_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const double* means, const double* log_scales, const double* quats,
                         const double* opacity_logits, const double* sh,
                         const double* dmeans2d, const double* dconics, const double* dcolors,
                         const double* dopacities,
                         double* dmeans, double* dlog_scales, double* dquats,
                         double* dopacity_logits, double* dsh);

/* ---- the optimizer step after the path ------------------------------ */

/* Adam with bias correction on one parameter group of n fp32 elements (SPEC S:252-259
 * "adam_step": "standard Adam with bias correction per parameter group"; PAPER P:76 row "Proj
 * Bwd + Optimizer").  For step t >= 1, element-wise, in fp64 with one rounding to fp32 at the end:
 *     m <- b1 m + (1 - b1) g
 *     v <- b2 v + (1 - b2) g^2
 *     p <- p - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
 * Parity pins (tests/test_oracle_pins.py): SPEC S:259 worked example, zero-gradient identity
 * (S:258), the closed form of a constant gradient, S:260 (x^2 decreases). */
void vko_adam_group(int64_t n, float* p, float* m, float* v, const float* g, double lr, double b1,
                    double b2, double eps, int32_t t);

/* Quaternion re-normalisation after the step ("rotations re-normalized after the step"):
 * each row of 4 divided by its fp64 norm (rows of norm 0 left unchanged). */
void vko_quat_renorm(int64_t n, float* q);

/* ---- the loss gradient before the path ------------------------------ */

/* "Loss Gradient" (SSIM definition):
 *   loss = (1 - lambda) mean_{pixels, channels} |r - t| + lambda (1 - SSIM(r, t))
 *   SSIM = mean over channels and VALID window centres (no padding) of
 *          S = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)(sx2 + sy2 + C2)),
 *   window statistics with the normalised 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
 *   C2 = 0.03^2; sx2 = E[x^2] - mx^2, sxy = E[xy] - mx my.
 *   dL_dr = the exact gradient (L1 subgradient sign(0) = 0), written as fp64.
 * Images HWC fp32 [H, W, 3]; SSIM needs H, W >= 11 unless lambda = 0.  fp64 throughout; the
 * window sums are direct (121 terms), the gradient scatters each centre's partials
 * (dS/dmx, dS/dE[x^2], dS/dE[xy]) back over its window.  Returns the loss. */
double vko_loss_grad(int32_t W, int32_t H, double lambda, const float* render, const float* target,
                     double* dL_dr, double* ssim_out);

/* ---- MCMC densification (fixed budget) ------------------------------- */

/* Counter-based generator shared (as a definition, not as code) with the CUDA path (DESIGN.md
 * §4.7 reading R1): h(seed, stream, i) = splitmix64(seed + 0x9E3779B97F4A7C15 * ((stream << 40) ^ i)),
 * uniform u = ((h >> 40) + 0.5) / 2^24, normal = Box-Muller of the uniforms of counters 2i, 2i+1. */
uint64_t vko_rng(uint64_t seed, uint32_t stream, uint64_t i);

/* Relocation (SPEC S:273 densify_mcmc; "MCMC 1M densification"; readings R3-R4 of
 * DESIGN.md §4.7): rho_i = X64 sigmoid(logit_i); dead_i = rho_i < dead_opacity; weights
 * w_j = dead_j ? 0 : floor(rho_j 2^24); every dead i draws t = mulhi64(h(seed, 1, i), sum w) and
 * takes the first j with inclusive prefix W_j > t (probability w_j / sum w); it copies j's means,
 * log_scales, quats and sh, and j and its k_j copies all get rho' = 1 - (1 - rho_j)^(1/(k_j+1))
 * (appearance-conserving: (1 - rho')^(k_j+1) = 1 - rho_j), logit' = log(rho'/(1 - rho')) (X64);
 * the copies' Adam moments (m, v: flat [n * (11 + 3K)] group-major like the parameters, nullable)
 * are zeroed.  targets[i] = j for dead i, -1 otherwise.  Returns the number of dead. */
int64_t vko_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, uint64_t seed, float* means,
                          float* log_scales, float* quats, float* opacity_logits, float* sh, float* m, float* v,
                          int64_t* targets);

/* Positional noise after an optimizer step (reading R5): means_i += lr_pos * noise_scale *
 * gate(rho_i) * Rq_i diag(exp(log_scales_i)) eps_i, gate(rho) = 1 / (1 + exp(-100 (0.005 - rho))),
 * eps_i = the normals of counters 3i, 3i+1, 3i+2 of stream 2 + 2 step (fp64). */
void vko_mcmc_noise(int64_t n, float lr_pos, float noise_scale, uint64_t seed, uint32_t step, float* means,
                    const float* log_scales, const float* quats, const float* opacity_logits);

/* ---- default densification ---------------------------------------------- */

/* Screen-gradient statistics ("mean accumulated screen-gradient norm"; reading R6):
 * for every Gaussian the view rasterised (radii > 0): accum += |dL/dmean2d| (Euclidean, pixels),
 * denom += 1. */
void vko_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom);

/* One densification event (readings R7-R9 of DESIGN.md §4.7).  Per Gaussian i
 * (rho = X64 sigmoid): prune if rho < prune_opacity; else with g = accum / denom (0 if denom = 0)
 * and smax = max exp(log_scales): g > grad_threshold and smax < size_threshold -> clone (the row,
 * then an identical copy), g > grad_threshold and smax >= size_threshold -> split (two children:
 * log_scales - ln 1.6, means + Rq diag(s) eps with eps the normals of counters 6i + 3c .. of stream
 * 3 (child c = 0, 1), other parameters copied), else keep.  Rows are emitted in i order (a clone's
 * copy and a split's second child right after); new rows (copies, children) get zero moments, kept
 * rows keep theirs.  m, v: flat group-major [n (11 + 3K)] (nullable; outputs likewise with n').
 * Returns n'; writes the outputs only if n' <= cap. */
int64_t vko_densify(int64_t n, int32_t sh_coeffs, const float* means, const float* log_scales, const float* quats,
                    const float* opacity_logits, const float* sh, const float* m, const float* v,
                    const float* accum, const float* denom, float grad_threshold, float size_threshold,
                    float prune_opacity, uint64_t seed, int64_t cap, float* o_means, float* o_log_scales,
                    float* o_quats, float* o_opacity_logits, float* o_sh, float* o_m, float* o_v);

#ifdef __cplusplus
}
#endif
#endif
