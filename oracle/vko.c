/*
 * vko.c — CPU ORACLE drivers.  TEST INFRASTRUCTURE ONLY (see vko.h): only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  It shares no code with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (no fast-math, no FTZ) -shared.
 */
#define _GNU_SOURCE
#include "vko.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* O1: fp32 instantiation                                              */
#define REAL float
#define PIN float
#define SFX _f32
#define L(x) x##f
#define SQRT sqrtf
#define CEIL ceilf
#define FLOOR floorf
#define FMIN fminf
#define FMAX fmaxf
#define FMA fmaf
#define EXPR expf
#define VKO_IS_F32 1
#include "vko_generic.inc"
#undef REAL
#undef PIN
#undef SFX
#undef L
#undef SQRT
#undef CEIL
#undef FLOOR
#undef FMIN
#undef FMAX
#undef FMA
#undef EXPR
#undef VKO_IS_F32

/* ------------------------------------------------------------------ */
/* O2: fp64 instantiation                                              */
#define REAL double
#define PIN double
#define SFX _f64
#define L(x) x
#define SQRT sqrt
#define CEIL ceil
#define FLOOR floor
#define FMIN fmin
#define FMAX fmax
#define FMA fma
#define EXPR exp
#define VKO_IS_F32 0
#include "vko_generic.inc"
#undef REAL
#undef PIN
#undef SFX
#undef L
#undef SQRT
#undef CEIL
#undef FLOOR
#undef FMIN
#undef FMAX
#undef FMA
#undef EXPR
#undef VKO_IS_F32

/* ------------------------------------------------------------------ */
/* plain pthread parallel-for over [0, n) with dynamic chunks           */
typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end, int tid);
typedef struct {
    range_fn fn;
    void* ctx;
    int64_t n, chunk;
    int64_t next;
    pthread_mutex_t mu;
    int tid;
} pfor_t;

static int resolve_threads(int nthreads) {
    if (nthreads > 0) return nthreads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

typedef struct { pfor_t* p; int tid; } pfor_arg;

static void* pfor_worker(void* argp) {
    pfor_arg* a = (pfor_arg*)argp;
    pfor_t* p = a->p;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t b = p->next;
        p->next += p->chunk;
        pthread_mutex_unlock(&p->mu);
        if (b >= p->n) break;
        int64_t e = b + p->chunk < p->n ? b + p->chunk : p->n;
        p->fn(p->ctx, b, e, a->tid);
    }
    return NULL;
}

static void parallel_for(int64_t n, int64_t chunk, int nthreads, range_fn fn, void* ctx) {
    if (n <= 0) return;
    nthreads = resolve_threads(nthreads);
    if (chunk < 1) chunk = 1;
    pfor_t p = {fn, ctx, n, chunk, 0, PTHREAD_MUTEX_INITIALIZER, 0};
    if (nthreads == 1 || n <= chunk) {
        fn(ctx, 0, n, 0);
        return;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    pfor_arg* args = (pfor_arg*)malloc(sizeof(pfor_arg) * nthreads);
    for (int i = 0; i < nthreads; i++) {
        args[i].p = &p;
        args[i].tid = i;
        pthread_create(&th[i], NULL, pfor_worker, &args[i]);
    }
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(th);
    free(args);
}

/* ------------------------------------------------------------------ */
/* projection drivers                                                  */
typedef struct {
    const vko_config* cfg;
    const vko_camera* cam;
    const float *means, *ls, *q, *o, *sh;
    proj_t_f32* P;
} projctx_f32;

static void proj_range_f32(void* vp, int64_t b, int64_t e, int tid) {
    (void)tid;
    projctx_f32* c = (projctx_f32*)vp;
    const int64_t S = c->cfg->sh_coeffs * 3;
    for (int64_t i = b; i < e; i++)
        project_one_f32(c->cfg, c->cam, c->means + 3 * i, c->ls + 3 * i, c->q + 4 * i, c->o[i],
                        c->sh + S * i, &c->P[i]);
}

static proj_t_f32* project_all_f32(const vko_config* cfg, const vko_camera* cam, int64_t n,
                                   const float* means, const float* ls, const float* q,
                                   const float* o, const float* sh, int nthreads) {
    proj_t_f32* P = (proj_t_f32*)malloc(sizeof(proj_t_f32) * (n > 0 ? n : 1));
    projctx_f32 c = {cfg, cam, means, ls, q, o, sh, P};
    parallel_for(n, 4096, nthreads, proj_range_f32, &c);
    return P;
}

static proj_t_f64* project_all_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                                   const double* means, const double* ls, const double* q,
                                   const double* o, const double* sh) {
    proj_t_f64* P = (proj_t_f64*)malloc(sizeof(proj_t_f64) * (n > 0 ? n : 1));
    const int64_t S = cfg->sh_coeffs * 3;
    for (int64_t i = 0; i < n; i++)
        project_one_f64(cfg, cam, means + 3 * i, ls + 3 * i, q + 4 * i, o[i], sh + S * i, &P[i]);
    return P;
}

#define WRITE_PROJ(P, i)                                                        \
    do {                                                                        \
        means2d[2 * (i)] = P.u; means2d[2 * (i) + 1] = P.v;                      \
        conics[3 * (i)] = P.a; conics[3 * (i) + 1] = P.b; conics[3 * (i) + 2] = P.c; \
        depths[i] = P.depth;                                                    \
        int vis_ = (P.flags & VKO_F_VISIBLE) != 0;                              \
        radii[2 * (i)] = vis_ ? P.rx : 0; radii[2 * (i) + 1] = vis_ ? P.ry : 0; \
        tiles_touched[i] = vis_ ? P.tiles : 0;                                  \
        colors[3 * (i)] = P.color[0]; colors[3 * (i) + 1] = P.color[1];          \
        colors[3 * (i) + 2] = P.color[2];                                       \
        opacities[i] = P.rho;                                                   \
        if (cov2d) { cov2d[3 * (i)] = P.A; cov2d[3 * (i) + 1] = P.B; cov2d[3 * (i) + 2] = P.C; } \
        if (flags) flags[i] = P.flags;                                          \
    } while (0)

void vko_project_fwd_f32(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const float* means, const float* log_scales, const float* quats,
                         const float* opacity_logits, const float* sh, float* means2d,
                         float* conics, float* depths, int32_t* radii, int32_t* tiles_touched,
                         float* colors, float* opacities, float* cov2d, int32_t* flags,
                         int nthreads) {
    proj_t_f32* P = project_all_f32(cfg, cam, n, means, log_scales, quats, opacity_logits, sh, nthreads);
    for (int64_t i = 0; i < n; i++) WRITE_PROJ(P[i], i);
    free(P);
}

void vko_project_fwd_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const double* means, const double* log_scales, const double* quats,
                         const double* opacity_logits, const double* sh, double* means2d,
                         double* conics, double* depths, int32_t* radii, int32_t* tiles_touched,
                         double* colors, double* opacities, double* cov2d, int32_t* flags) {
    proj_t_f64* P = project_all_f64(cfg, cam, n, means, log_scales, quats, opacity_logits, sh);
    for (int64_t i = 0; i < n; i++) WRITE_PROJ(P[i], i);
    free(P);
}

/* ------------------------------------------------------------------ */
/* binning                                    */

/* exclusive prefix sum, sequential loop */
int64_t vko_scan_offsets(int64_t n, const int32_t* tiles_touched, uint32_t* offsets) {
    int64_t acc = 0;
    for (int64_t i = 0; i < n; i++) {
        offsets[i] = (uint32_t)acc;
        acc += tiles_touched[i];
    }
    return acc;
}

/* key = (tile << 32) | f32bits(depth), val = i, slots offsets[i]+k, rows
 * outer, columns inner. The rect is recomputed from mean2d and radii
 * exactly as in projection step 11. */
void vko_gen_keys(const vko_camera* cam, int64_t n, const float* means2d, const int32_t* radii,
                  const float* depths, const int32_t* tiles_touched, const uint32_t* offsets,
                  uint64_t* keys, uint32_t* vals) {
    const int TX = (cam->width + 15) / 16, TY = (cam->height + 15) / 16;
    for (int64_t i = 0; i < n; i++) {
        if (tiles_touched[i] <= 0) continue;
        float u = means2d[2 * i], v = means2d[2 * i + 1];
        float rx = (float)radii[2 * i], ry = (float)radii[2 * i + 1];
        int x0 = (int)fminf(fmaxf(floorf((u - rx) * 0.0625f), 0.0f), (float)TX);
        int x1 = (int)fminf(fmaxf(ceilf((u + rx) * 0.0625f), 0.0f), (float)TX);
        int y0 = (int)fminf(fmaxf(floorf((v - ry) * 0.0625f), 0.0f), (float)TY);
        int y1 = (int)fminf(fmaxf(ceilf((v + ry) * 0.0625f), 0.0f), (float)TY);
        uint32_t dbits;
        memcpy(&dbits, &depths[i], 4);
        int64_t slot = offsets[i];
        for (int ty = y0; ty < y1; ty++)
            for (int tx = x0; tx < x1; tx++) {
                uint64_t tile = (uint64_t)(ty * TX + tx);
                keys[slot] = (tile << 32) | (uint64_t)dbits;
                vals[slot] = (uint32_t)i;
                slot++;
            }
    }
}

typedef struct { uint64_t key; uint32_t val; uint32_t pos; } kv_t;

static int kv_cmp(const void* pa, const void* pb) {
    const kv_t* a = (const kv_t*)pa;
    const kv_t* b = (const kv_t*)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->pos < b->pos ? -1 : (a->pos > b->pos ? 1 : 0); /* stability */
}

/* stable ascending sort by u64 key: library comparison sort on (key, slot) */
void vko_sort_pairs(int64_t m, uint64_t* keys, uint32_t* vals) {
    if (m <= 0) return;
    kv_t* t = (kv_t*)malloc(sizeof(kv_t) * m);
    for (int64_t i = 0; i < m; i++) { t[i].key = keys[i]; t[i].val = vals[i]; t[i].pos = (uint32_t)i; }
    qsort(t, (size_t)m, sizeof(kv_t), kv_cmp);
    for (int64_t i = 0; i < m; i++) { keys[i] = t[i].key; vals[i] = t[i].val; }
    free(t);
}

/* CSR tile ranges: tile_offsets[t] = #{entries with tile < t} */
void vko_tile_ranges(int64_t m, const uint64_t* keys, int32_t n_tiles, uint32_t* tile_offsets) {
    int64_t j = 0;
    for (int32_t t = 0; t <= n_tiles; t++) {
        while (j < m && (int64_t)(keys[j] >> 32) < t) j++;
        tile_offsets[t] = (uint32_t)j;
    }
}

/* ------------------------------------------------------------------ */
/* untiled render driver, generic over precision          */

typedef struct { float depth; int32_t id; } dk_t;
typedef struct { double depth; int32_t id; } dk64_t;

static int dk_cmp(const void* pa, const void* pb) {
    const dk_t* a = (const dk_t*)pa;
    const dk_t* b = (const dk_t*)pb;
    if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}
static int dk64_cmp(const void* pa, const void* pb) {
    const dk64_t* a = (const dk64_t*)pa;
    const dk64_t* b = (const dk64_t*)pb;
    if (a->depth != b->depth) return a->depth < b->depth ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

/* The oracle's OWN conservative pixel box for a candidate: the ellipse
 * sigma <= k'' of its fp32 conic, k'' = ln(255 rho)*1.01 + 0.01, plus 2 px.
 * It only accelerates candidate gathering; correctness of the bound is
 * checked against the brute-force O3 in tests. */
typedef struct { int32_t x0, x1, y0, y1; } pbox_t; /* inclusive pixel bounds, x0 > x1 = empty */

static pbox_t oracle_box(double u, double v, double a, double b, double c, double rho, int W, int H, int brute) {
    pbox_t r = {0, W - 1, 0, H - 1};
    if (brute) return r;
    if (!(rho >= 1.0 / 255.0)) { r.x0 = 1; r.x1 = 0; return r; }
    double k = log(255.0 * rho) * 1.01 + 0.01;
    double det = a * c - b * b;
    if (!(det > 0) || !(a > 0) || !(c > 0)) return r; /* degenerate: whole image */
    double hx = sqrt(2.0 * k * c / det) + 2.0, hy = sqrt(2.0 * k * a / det) + 2.0;
    double fx0 = floor(u - hx), fx1 = ceil(u + hx), fy0 = floor(v - hy), fy1 = ceil(v + hy);
    if (fx1 < 0 || fy1 < 0 || fx0 > W - 1 || fy0 > H - 1) { r.x0 = 1; r.x1 = 0; return r; }
    r.x0 = fx0 < 0 ? 0 : (int32_t)fx0;
    r.x1 = fx1 > W - 1 ? W - 1 : (int32_t)fx1;
    r.y0 = fy0 < 0 ? 0 : (int32_t)fy0;
    r.y1 = fy1 > H - 1 ? H - 1 : (int32_t)fy1;
    return r;
}

#define BAND 16

#define DEFINE_RENDER(SFXN, REALT, PROJT, ENTRYT, COMPOSITE, BACKWARD, ISF32)                  \
    typedef struct {                                                                          \
        const vko_config* cfg;                                                                \
        const vko_camera* cam;                                                                \
        const PROJT* P;                                                                       \
        int64_t ncand;                                                                        \
        const int32_t* cand; /* global ids in (depth,id) order */                             \
        const pbox_t* box;   /* per candidate */                                              \
        const REALT* dL;     /* [H,W,3] or NULL */                                            \
        const uint8_t* row_mask;                                                              \
        int brute;                                                                            \
        REALT* image; float* T_final_f; double* T_final_d; int32_t* last_id; uint8_t* fragile; \
        uint64_t* dhash;                                                                      \
        int32_t** band_cand; int64_t* band_n; double** band_g; double** band_m;               \
        int want_mass;                                                                        \
        int64_t* st_viol; int64_t* st_eval; int64_t* st_comp; int64_t* st_frag; int64_t* st_rows; \
        pthread_mutex_t* mu;                                                                  \
    } rctx##SFXN;                                                                             \
                                                                                              \
    static void band_range##SFXN(void* vp, int64_t bb, int64_t be, int tid) {                 \
        (void)tid;                                                                            \
        rctx##SFXN* c = (rctx##SFXN*)vp;                                                      \
        const int W = c->cam->width, H = c->cam->height;                                     \
        for (int64_t band = bb; band < be; band++) {                                          \
            int ys = (int)band * BAND, ye = ys + BAND < H ? ys + BAND : H;                     \
            int any = 0;                                                                      \
            for (int y = ys; y < ye; y++) any |= !c->row_mask || c->row_mask[y];              \
            c->band_n[band] = 0;                                                              \
            c->band_cand[band] = NULL; c->band_g[band] = NULL; c->band_m[band] = NULL;        \
            if (!any) continue;                                                               \
            /* candidates of this band, in global (depth,id) order */                         \
            int64_t nb = 0;                                                                   \
            for (int64_t i = 0; i < c->ncand; i++)                                            \
                if (c->box[i].x0 <= c->box[i].x1 && c->box[i].y0 < ye && c->box[i].y1 >= ys) nb++; \
            int32_t* bc = (int32_t*)malloc(sizeof(int32_t) * (nb > 0 ? nb : 1));              \
            int32_t* bci = (int32_t*)malloc(sizeof(int32_t) * (nb > 0 ? nb : 1));             \
            nb = 0;                                                                           \
            for (int64_t i = 0; i < c->ncand; i++)                                            \
                if (c->box[i].x0 <= c->box[i].x1 && c->box[i].y0 < ye && c->box[i].y1 >= ys) { \
                    bc[nb] = c->cand[i]; bci[nb] = (int32_t)i; nb++;                          \
                }                                                                             \
            double* bg_ = NULL; double* bm_ = NULL;                                           \
            if (c->dL) {                                                                      \
                bg_ = (double*)calloc((size_t)(nb > 0 ? nb : 1) * 9, sizeof(double));         \
                if (c->want_mass) bm_ = (double*)calloc((size_t)(nb > 0 ? nb : 1) * 9, sizeof(double)); \
            }                                                                                 \
            int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (W + 1));                       \
            int64_t cap = 0; int32_t* lists = NULL;                                           \
            ENTRYT* ent = NULL; int64_t entcap = 0;                                           \
            int64_t viol = 0, ev = 0, comp = 0, frag = 0, rows = 0;                           \
            for (int y = ys; y < ye; y++) {                                                   \
                if (c->row_mask && !c->row_mask[y]) continue;                                 \
                rows++;                                                                       \
                const int ty = y / 16;                                                        \
                memset(cnt, 0, sizeof(int64_t) * (W + 1));                                    \
                for (int64_t j = 0; j < nb; j++) {                                            \
                    const pbox_t* bx = &c->box[bci[j]];                                       \
                    if (bx->y0 > y || bx->y1 < y) continue;                                   \
                    const PROJT* g = &c->P[bc[j]];                                            \
                    for (int x = bx->x0; x <= bx->x1; x++) {                                  \
                        if (c->cfg->footprint == VKO_FOOTPRINT_3SIGMA) {                      \
                            int tx = x / 16;                                                  \
                            if (!(g->flags & VKO_F_VISIBLE) || tx < g->x0 || tx >= g->x1 ||   \
                                ty < g->y0 || ty >= g->y1) continue;                          \
                        }                                                                     \
                        cnt[x + 1]++;                                                         \
                    }                                                                         \
                }                                                                             \
                for (int x = 0; x < W; x++) cnt[x + 1] += cnt[x];                             \
                if (cnt[W] > cap) { cap = cnt[W]; lists = (int32_t*)realloc(lists, sizeof(int32_t) * cap); } \
                int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * W);                        \
                for (int x = 0; x < W; x++) fill[x] = cnt[x];                                 \
                for (int64_t j = 0; j < nb; j++) {                                            \
                    const pbox_t* bx = &c->box[bci[j]];                                       \
                    if (bx->y0 > y || bx->y1 < y) continue;                                   \
                    const PROJT* g = &c->P[bc[j]];                                            \
                    for (int x = bx->x0; x <= bx->x1; x++) {                                  \
                        if (c->cfg->footprint == VKO_FOOTPRINT_3SIGMA) {                      \
                            int tx = x / 16;                                                  \
                            if (!(g->flags & VKO_F_VISIBLE) || tx < g->x0 || tx >= g->x1 ||   \
                                ty < g->y0 || ty >= g->y1) continue;                          \
                        }                                                                     \
                        lists[fill[x]++] = (int32_t)j;                                        \
                    }                                                                         \
                }                                                                             \
                free(fill);                                                                   \
                for (int x = 0; x < W; x++) {                                                 \
                    int64_t len = cnt[x + 1] - cnt[x];                                        \
                    if (len > entcap) { entcap = len; ent = (ENTRYT*)realloc(ent, sizeof(ENTRYT) * entcap); } \
                    REALT out[3]; REALT Tf; int64_t last; int fr = 0; uint64_t hh = 0;         \
                    const REALT px = (REALT)x + (REALT)0.5, py = (REALT)y + (REALT)0.5;       \
                    int nent = COMPOSITE(c->P, bc, lists + cnt[x], len, px, py, out, &Tf, &last, ent, \
                                         ISF32 ? &fr : NULL, &hh, &ev);                       \
                    comp += nent;                                                             \
                    const int64_t pix = (int64_t)y * W + x;                                   \
                    for (int ch = 0; ch < 3; ch++)                                            \
                        c->image[3 * pix + ch] = out[ch] + Tf * (REALT)c->cfg->bg[ch];        \
                    if (c->T_final_f) c->T_final_f[pix] = (float)Tf;                          \
                    if (c->T_final_d) c->T_final_d[pix] = (double)Tf;                         \
                    if (c->last_id) c->last_id[pix] = last >= 0 ? bc[lists[cnt[x] + last]] : -1; \
                    if (c->fragile) c->fragile[pix] = (uint8_t)fr;                            \
                    if (c->dhash) c->dhash[pix] = hh;                                         \
                    frag += fr;                                                               \
                    /* footprint violation: composited outside the tile rect */               \
                    const int tx = x / 16;                                                    \
                    for (int e = 0; e < nent; e++) {                                          \
                        const PROJT* g = &c->P[bc[ent[e].idx]];                               \
                        if (!(g->flags & VKO_F_VISIBLE) || tx < g->x0 || tx >= g->x1 || ty < g->y0 || \
                            ty >= g->y1) viol++;                                              \
                    }                                                                         \
                    if (c->dL) {                                                              \
                        double wv[3] = {(double)c->dL[3 * pix], (double)c->dL[3 * pix + 1],   \
                                        (double)c->dL[3 * pix + 2]};                          \
                        double bgd[3] = {(double)c->cfg->bg[0], (double)c->cfg->bg[1], (double)c->cfg->bg[2]}; \
                        BACKWARD(c->P, bc, ent, nent, px, py, wv, bgd, bg_, bm_);             \
                    }                                                                         \
                }                                                                             \
            }                                                                                 \
            free(cnt); free(lists); free(ent); free(bci);                                     \
            c->band_cand[band] = bc; c->band_n[band] = nb; c->band_g[band] = bg_; c->band_m[band] = bm_; \
            pthread_mutex_lock(c->mu);                                                        \
            *c->st_viol += viol; *c->st_eval += ev; *c->st_comp += comp; *c->st_frag += frag; \
            *c->st_rows += rows;                                                              \
            pthread_mutex_unlock(c->mu);                                                      \
        }                                                                                     \
    }

DEFINE_RENDER(_f32, float, proj_t_f32, entry_t_f32, composite_f32, backward_pixel_f32, 1)
DEFINE_RENDER(_f64, double, proj_t_f64, entry_t_f64, composite_f64, backward_pixel_f64, 0)

/* common tail: reduce per-band gradient partials in band order (deterministic) */
static void reduce_bands(int64_t nbands, int32_t** band_cand, int64_t* band_n, double** band_g,
                         double** band_m, int64_t n, double* dmeans2d, double* dconics,
                         double* dcolors, double* dopacities, double* mass) {
    if (dmeans2d) memset(dmeans2d, 0, sizeof(double) * 2 * n);
    if (dconics) memset(dconics, 0, sizeof(double) * 3 * n);
    if (dcolors) memset(dcolors, 0, sizeof(double) * 3 * n);
    if (dopacities) memset(dopacities, 0, sizeof(double) * n);
    if (mass) memset(mass, 0, sizeof(double) * 9 * n);
    for (int64_t b = 0; b < nbands; b++) {
        if (band_g[b]) {
            for (int64_t j = 0; j < band_n[b]; j++) {
                const int64_t g = band_cand[b][j];
                const double* v = band_g[b] + 9 * j;
                if (dmeans2d) { dmeans2d[2 * g] += v[0]; dmeans2d[2 * g + 1] += v[1]; }
                if (dconics) { dconics[3 * g] += v[2]; dconics[3 * g + 1] += v[3]; dconics[3 * g + 2] += v[4]; }
                if (dcolors) { dcolors[3 * g] += v[5]; dcolors[3 * g + 1] += v[6]; dcolors[3 * g + 2] += v[7]; }
                if (dopacities) dopacities[g] += v[8];
                if (mass && band_m[b])
                    for (int k = 0; k < 9; k++) mass[9 * g + k] += band_m[b][9 * j + k];
            }
        }
        free(band_cand[b]); free(band_g[b]); free(band_m[b]);
    }
}

int vko_render_f32(const vko_config* cfg, const vko_camera* cam, int64_t n, const float* means,
                   const float* log_scales, const float* quats, const float* opacity_logits,
                   const float* sh, const float* dL_dimage, const uint8_t* row_mask, int brute,
                   float* image, float* T_final, int32_t* last_id, uint8_t* fragile,
                   int64_t* stats, double* dmeans2d, double* dconics, double* dcolors,
                   double* dopacities, double* mass, int nthreads) {
    const int W = cam->width, H = cam->height;
    proj_t_f32* P = project_all_f32(cfg, cam, n, means, log_scales, quats, opacity_logits, sh, nthreads);
    /* candidates: every projectable Gaussian, in ascending (f32 depth, id) */
    int64_t nc = 0;
    for (int64_t i = 0; i < n; i++) nc += (P[i].flags & VKO_F_PROJECTABLE) != 0;
    dk_t* dk = (dk_t*)malloc(sizeof(dk_t) * (nc > 0 ? nc : 1));
    nc = 0;
    for (int64_t i = 0; i < n; i++)
        if (P[i].flags & VKO_F_PROJECTABLE) { dk[nc].depth = P[i].depth; dk[nc].id = (int32_t)i; nc++; }
    qsort(dk, (size_t)nc, sizeof(dk_t), dk_cmp);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (nc > 0 ? nc : 1));
    pbox_t* box = (pbox_t*)malloc(sizeof(pbox_t) * (nc > 0 ? nc : 1));
    for (int64_t i = 0; i < nc; i++) {
        const proj_t_f32* g = &P[dk[i].id];
        cand[i] = dk[i].id;
        box[i] = oracle_box(g->u, g->v, g->a, g->b, g->c, g->rho, W, H, brute);
    }
    free(dk);
    const int64_t nbands = (H + BAND - 1) / BAND;
    int32_t** band_cand = (int32_t**)calloc(nbands > 0 ? nbands : 1, sizeof(int32_t*));
    int64_t* band_n = (int64_t*)calloc(nbands > 0 ? nbands : 1, sizeof(int64_t));
    double** band_g = (double**)calloc(nbands > 0 ? nbands : 1, sizeof(double*));
    double** band_m = (double**)calloc(nbands > 0 ? nbands : 1, sizeof(double*));
    int64_t viol = 0, ev = 0, comp = 0, frag = 0, rows = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    /* unrendered rows keep background / T=1 / -1 */
    for (int64_t p = 0; p < (int64_t)W * H; p++) {
        for (int ch = 0; ch < 3; ch++) image[3 * p + ch] = cfg->bg[ch];
        if (T_final) T_final[p] = 1.0f;
        if (last_id) last_id[p] = -1;
        if (fragile) fragile[p] = 0;
    }
    rctx_f32 c = {cfg, cam, P, nc, cand, box, dL_dimage, row_mask, brute, image, T_final, NULL,
                  last_id, fragile, NULL, band_cand, band_n, band_g, band_m, mass != NULL,
                  &viol, &ev, &comp, &frag, &rows, &mu};
    parallel_for(nbands, 1, nthreads, band_range_f32, &c);
    reduce_bands(nbands, band_cand, band_n, band_g, band_m, n, dL_dimage ? dmeans2d : NULL,
                 dL_dimage ? dconics : NULL, dL_dimage ? dcolors : NULL,
                 dL_dimage ? dopacities : NULL, dL_dimage ? mass : NULL);
    if (stats) {
        stats[0] = viol; stats[1] = ev; stats[2] = comp; stats[3] = frag; stats[4] = nc; stats[5] = rows;
        stats[6] = 0; stats[7] = 0;
    }
    free(band_cand); free(band_n); free(band_g); free(band_m);
    free(cand); free(box); free(P);
    return 0;
}

int vko_render_f64(const vko_config* cfg, const vko_camera* cam, int64_t n, const double* means,
                   const double* log_scales, const double* quats, const double* opacity_logits,
                   const double* sh, const double* dL_dimage, double* image,
                   uint64_t* decision_hash, int32_t* proj_flags, double* dmeans2d,
                   double* dconics, double* dcolors, double* dopacities) {
    const int W = cam->width, H = cam->height;
    proj_t_f64* P = project_all_f64(cfg, cam, n, means, log_scales, quats, opacity_logits, sh);
    int64_t nc = 0;
    for (int64_t i = 0; i < n; i++) {
        if (proj_flags) proj_flags[i] = P[i].flags;
        nc += (P[i].flags & VKO_F_PROJECTABLE) != 0;
    }
    dk64_t* dk = (dk64_t*)malloc(sizeof(dk64_t) * (nc > 0 ? nc : 1));
    nc = 0;
    for (int64_t i = 0; i < n; i++)
        if (P[i].flags & VKO_F_PROJECTABLE) { dk[nc].depth = P[i].depth; dk[nc].id = (int32_t)i; nc++; }
    qsort(dk, (size_t)nc, sizeof(dk64_t), dk64_cmp);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (nc > 0 ? nc : 1));
    pbox_t* box = (pbox_t*)malloc(sizeof(pbox_t) * (nc > 0 ? nc : 1));
    for (int64_t i = 0; i < nc; i++) {
        cand[i] = dk[i].id;
        box[i] = oracle_box(0, 0, 0, 0, 0, 1, W, H, 1); /* fp64 FD path: brute force */
    }
    free(dk);
    const int64_t nbands = (H + BAND - 1) / BAND;
    int32_t** band_cand = (int32_t**)calloc(nbands > 0 ? nbands : 1, sizeof(int32_t*));
    int64_t* band_n = (int64_t*)calloc(nbands > 0 ? nbands : 1, sizeof(int64_t));
    double** band_g = (double**)calloc(nbands > 0 ? nbands : 1, sizeof(double*));
    double** band_m = (double**)calloc(nbands > 0 ? nbands : 1, sizeof(double*));
    int64_t viol = 0, ev = 0, comp = 0, frag = 0, rows = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    rctx_f64 c = {cfg, cam, P, nc, cand, box, dL_dimage, NULL, 1, image, NULL, NULL, NULL, NULL,
                  decision_hash, band_cand, band_n, band_g, band_m, 0,
                  &viol, &ev, &comp, &frag, &rows, &mu};
    parallel_for(nbands, 1, 1, band_range_f64, &c);
    reduce_bands(nbands, band_cand, band_n, band_g, band_m, n, dL_dimage ? dmeans2d : NULL,
                 dL_dimage ? dconics : NULL, dL_dimage ? dcolors : NULL,
                 dL_dimage ? dopacities : NULL, NULL);
    free(band_cand); free(band_n); free(band_g); free(band_m);
    free(cand); free(box); free(P);
    return 0;
}

/* ------------------------------------------------------------------ */
/* projection backward, fp64                             */

static const double C0d = 0.28209479177387814, C1d = 0.4886025119029199;
static const double C2d[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
static const double C3d[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

/* gradient of each basis function w.r.t. the (unit) direction (x,y,z) */
static void sh_basis_grad(double x, double y, double z, int K, double Y[16], double dY[16][3]) {
    memset(dY, 0, sizeof(double) * 48);
    Y[0] = C0d;
    if (K > 1) {
        Y[1] = -C1d * y; dY[1][1] = -C1d;
        Y[2] = C1d * z;  dY[2][2] = C1d;
        Y[3] = -C1d * x; dY[3][0] = -C1d;
    }
    if (K > 4) {
        double xx = x * x, yy = y * y, zz = z * z;
        Y[4] = C2d[0] * x * y; dY[4][0] = C2d[0] * y; dY[4][1] = C2d[0] * x;
        Y[5] = C2d[1] * y * z; dY[5][1] = C2d[1] * z; dY[5][2] = C2d[1] * y;
        Y[6] = C2d[2] * (2 * zz - xx - yy);
        dY[6][0] = -2 * C2d[2] * x; dY[6][1] = -2 * C2d[2] * y; dY[6][2] = 4 * C2d[2] * z;
        Y[7] = C2d[3] * x * z; dY[7][0] = C2d[3] * z; dY[7][2] = C2d[3] * x;
        Y[8] = C2d[4] * (xx - yy); dY[8][0] = 2 * C2d[4] * x; dY[8][1] = -2 * C2d[4] * y;
    }
    if (K > 9) {
        double xx = x * x, yy = y * y, zz = z * z;
        Y[9] = C3d[0] * y * (3 * xx - yy);
        dY[9][0] = 6 * C3d[0] * x * y; dY[9][1] = C3d[0] * (3 * xx - 3 * yy);
        Y[10] = C3d[1] * x * y * z;
        dY[10][0] = C3d[1] * y * z; dY[10][1] = C3d[1] * x * z; dY[10][2] = C3d[1] * x * y;
        Y[11] = C3d[2] * y * (4 * zz - xx - yy);
        dY[11][0] = -2 * C3d[2] * x * y; dY[11][1] = C3d[2] * (4 * zz - xx - 3 * yy);
        dY[11][2] = 8 * C3d[2] * y * z;
        Y[12] = C3d[3] * z * (2 * zz - 3 * xx - 3 * yy);
        dY[12][0] = -6 * C3d[3] * x * z; dY[12][1] = -6 * C3d[3] * y * z;
        dY[12][2] = C3d[3] * (6 * zz - 3 * xx - 3 * yy);
        Y[13] = C3d[4] * x * (4 * zz - xx - yy);
        dY[13][0] = C3d[4] * (4 * zz - 3 * xx - yy); dY[13][1] = -2 * C3d[4] * x * y;
        dY[13][2] = 8 * C3d[4] * x * z;
        Y[14] = C3d[5] * z * (xx - yy);
        dY[14][0] = 2 * C3d[5] * x * z; dY[14][1] = -2 * C3d[5] * y * z; dY[14][2] = C3d[5] * (xx - yy);
        Y[15] = C3d[6] * x * (xx - 3 * yy);
        dY[15][0] = C3d[6] * (3 * xx - 3 * yy); dY[15][1] = -6 * C3d[6] * x * y;
    }
}

/* one Gaussian; decisions (cull, FOV clamp, colour clamp) from `flags` */
static void proj_bwd_one(const vko_config* cfg, const vko_camera* cam, int32_t flags,
                         const double mu[3], const double ls[3], const double q[4], double o,
                         const double* sh, const double dm2[2], const double dcon[3],
                         const double dcol[3], double drho, double dmu[3], double dls[3],
                         double dq[4], double* dlogit, double* dsh) {
    double R[9], ct[3];
    for (int i = 0; i < 9; i++) R[i] = cam->R[i];
    for (int i = 0; i < 3; i++) ct[i] = cam->t[i];
    const double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    const double W = cam->width, H = cam->height;
    const int K = (cfg->sh_degree + 1) * (cfg->sh_degree + 1);
    double t[3];
    for (int j = 0; j < 3; j++) t[j] = R[3 * j] * mu[0] + R[3 * j + 1] * mu[1] + R[3 * j + 2] * mu[2] + ct[j];
    const double tx = t[0], ty = t[1], tz = t[2];
    double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    double Rq[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                    2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                    2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double M[9], Mc[9];
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) M[3 * j + k] = Rq[3 * j + k] * s[k];
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++)
            Mc[3 * j + k] = R[3 * j] * M[k] + R[3 * j + 1] * M[3 + k] + R[3 * j + 2] * M[6 + k];
    /* FOV clamp, branch from the fp32 decision */
    double Lx = 0, Ly = 0;
    int clx = 0, cly = 0;
    if (cfg->fov_clamp) {
        double lxp = (W - cx) / fx + 0.3 * (0.5 * W / fx), lxn = cx / fx + 0.3 * (0.5 * W / fx);
        double lyp = (H - cy) / fy + 0.3 * (0.5 * H / fy), lyn = cy / fy + 0.3 * (0.5 * H / fy);
        if (flags & VKO_F_FOVX_HI) { clx = 1; Lx = lxp; }
        else if (flags & VKO_F_FOVX_LO) { clx = 1; Lx = -lxn; }
        if (flags & VKO_F_FOVY_HI) { cly = 1; Ly = lyp; }
        else if (flags & VKO_F_FOVY_LO) { cly = 1; Ly = -lyn; }
    }
    const double txc = clx ? tz * Lx : tx, tyc = cly ? tz * Ly : ty;
    const double J00 = fx / tz, J02 = -fx * txc / (tz * tz), J11 = fy / tz, J12 = -fy * tyc / (tz * tz);
    double K0[3], K1[3];
    for (int k = 0; k < 3; k++) {
        K0[k] = J00 * Mc[k] + J02 * Mc[6 + k];
        K1[k] = J11 * Mc[3 + k] + J12 * Mc[6 + k];
    }
    const double A = K0[0] * K0[0] + K0[1] * K0[1] + K0[2] * K0[2] + 0.3;
    const double B = K0[0] * K1[0] + K0[1] * K1[1] + K0[2] * K1[2];
    const double C = K1[0] * K1[0] + K1[1] * K1[1] + K1[2] * K1[2] + 0.3;
    const double det = A * C - B * B, det2 = det * det;
    /* opacity: d logit = d rho * rho (1 - rho) */
    const double rho = 1.0 / (1.0 + exp(-o));
    *dlogit = drho * rho * (1 - rho);
    /* colour: masked by the forward clamp; dsh = Y dcolour; direction term */
    double cp[3];
    for (int k = 0; k < 3; k++) cp[k] = -(R[k] * ct[0] + R[3 + k] * ct[1] + R[6 + k] * ct[2]);
    double d[3] = {mu[0] - cp[0], mu[1] - cp[1], mu[2] - cp[2]};
    double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dh[3] = {d[0] / dl, d[1] / dl, d[2] / dl};
    double Y[16], dY[16][3];
    sh_basis_grad(dh[0], dh[1], dh[2], K, Y, dY);
    double dce[3];
    for (int ch = 0; ch < 3; ch++) dce[ch] = (flags & (VKO_F_CLAMP_R << ch)) ? 0.0 : dcol[ch];
    double ddh[3] = {0, 0, 0};
    for (int l = 0; l < K; l++)
        for (int ch = 0; ch < 3; ch++) {
            dsh[3 * l + ch] = Y[l] * dce[ch];
            for (int k = 0; k < 3; k++) ddh[k] += dce[ch] * sh[3 * l + ch] * dY[l][k];
        }
    double proj = dh[0] * ddh[0] + dh[1] * ddh[1] + dh[2] * ddh[2];
    for (int k = 0; k < 3; k++) dmu[k] = (ddh[k] - dh[k] * proj) / dl;
    /* conic (a,b,c) = (C,-B,A)/det  ->  (A,B,C) */
    const double da = dcon[0], db = dcon[1], dc = dcon[2];
    const double dA = da * (-C * C / det2) + db * (B * C / det2) + dc * (1 / det - A * C / det2);
    const double dB = da * (2 * B * C / det2) + db * (-1 / det - 2 * B * B / det2) + dc * (2 * A * B / det2);
    const double dC = da * (1 / det - A * C / det2) + db * (A * B / det2) + dc * (-A * A / det2);
    /* Sigma' = K K^T + 0.3 I :  dK = 2 G2 K */
    double dK0[3], dK1[3];
    for (int k = 0; k < 3; k++) {
        dK0[k] = 2 * dA * K0[k] + dB * K1[k];
        dK1[k] = dB * K0[k] + 2 * dC * K1[k];
    }
    /* K = J Mc */
    double dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0;
    for (int k = 0; k < 3; k++) {
        dJ00 += dK0[k] * Mc[k];
        dJ02 += dK0[k] * Mc[6 + k];
        dJ11 += dK1[k] * Mc[3 + k];
        dJ12 += dK1[k] * Mc[6 + k];
    }
    double dMc[9];
    for (int k = 0; k < 3; k++) {
        dMc[k] = J00 * dK0[k];
        dMc[3 + k] = J11 * dK1[k];
        dMc[6 + k] = J02 * dK0[k] + J12 * dK1[k];
    }
    /* Mc = R M */
    double dM[9];
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++)
            dM[3 * j + k] = R[j] * dMc[k] + R[3 + j] * dMc[3 + k] + R[6 + j] * dMc[6 + k];
    /* M = Rq diag(s) */
    double D[9];
    for (int k = 0; k < 3; k++) {
        double ds = 0;
        for (int j = 0; j < 3; j++) {
            ds += dM[3 * j + k] * Rq[3 * j + k];
            D[3 * j + k] = dM[3 * j + k] * s[k];
        }
        dls[k] = ds * s[k];
    }
    double dqh[4];
    dqh[0] = 2 * (-z * D[1] + y * D[2] + z * D[3] - x * D[5] - y * D[6] + x * D[7]);
    dqh[1] = 2 * (y * D[1] + z * D[2] + y * D[3] - 2 * x * D[4] - w * D[5] + z * D[6] + w * D[7] - 2 * x * D[8]);
    dqh[2] = 2 * (-2 * y * D[0] + x * D[1] + w * D[2] + x * D[3] + z * D[5] - w * D[6] + z * D[7] - 2 * y * D[8]);
    dqh[3] = 2 * (-2 * z * D[0] - w * D[1] + x * D[2] + w * D[3] - 2 * z * D[4] + y * D[5] + x * D[6] + y * D[7]);
    const double qd = w * dqh[0] + x * dqh[1] + y * dqh[2] + z * dqh[3];
    const double qh[4] = {w, x, y, z};
    for (int k = 0; k < 4; k++) dq[k] = (dqh[k] - qh[k] * qd) / qn;
    /* t: from mean2d and from J */
    double dt[3] = {0, 0, 0};
    const double tz2 = tz * tz, tz3 = tz2 * tz;
    dt[0] += fx / tz * dm2[0];
    dt[1] += fy / tz * dm2[1];
    dt[2] += -fx * tx / tz2 * dm2[0] - fy * ty / tz2 * dm2[1];
    dt[2] += -fx / tz2 * dJ00 - fy / tz2 * dJ11;
    if (!clx) { dt[0] += -fx / tz2 * dJ02; dt[2] += 2 * fx * tx / tz3 * dJ02; }
    else { dt[2] += fx * Lx / tz2 * dJ02; }
    if (!cly) { dt[1] += -fy / tz2 * dJ12; dt[2] += 2 * fy * ty / tz3 * dJ12; }
    else { dt[2] += fy * Ly / tz2 * dJ12; }
    /* t = R mu + t_cam */
    for (int k = 0; k < 3; k++) dmu[k] += R[k] * dt[0] + R[3 + k] * dt[1] + R[6 + k] * dt[2];
}

/* "Mass" of the projection backward (sum |terms| per gradient entry): the
 * chain of SURVEY §8c.6 (proj_bwd_one above), stage by stage, with every local coefficient replaced
 * by its absolute value, i.e. |J_stage|^T applied to non-negative input masses; the two
 * normalisations are written as two terms each (dq = (dq^ - q^<q^,dq^>)/|q|, the same for the SH
 * direction), so they contribute (|I| + |q^||q^|^T)/|q|.  Inputs: masses of the 2D gradients.
 * Outputs bound |gradient| (triangle inequality) and scale the rounding error of any fp32
 * evaluation of the chain.  Pinned in tests/test_oracle_mass.py against an independent rebuild of
 * the chain from autograd stage Jacobians (equal to 1e-9) and the bound property. */
static void proj_bwd_mass_one(const vko_config* cfg, const vko_camera* cam, int32_t flags,
                              const double mu[3], const double ls[3], const double q[4], double o,
                              const double* sh, const double mdm2[2], const double mdcon[3],
                              const double mdcol[3], double mdrho, double mmu[3], double mls[3],
                              double mq[4], double* mlogit, double* msh) {
    double R[9], ct[3];
    for (int i = 0; i < 9; i++) R[i] = cam->R[i];
    for (int i = 0; i < 3; i++) ct[i] = cam->t[i];
    const double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
    const double W = cam->width, H = cam->height;
    const int K = (cfg->sh_degree + 1) * (cfg->sh_degree + 1);
    double t[3];
    for (int j = 0; j < 3; j++) t[j] = R[3 * j] * mu[0] + R[3 * j + 1] * mu[1] + R[3 * j + 2] * mu[2] + ct[j];
    const double tx = t[0], ty = t[1], tz = t[2];
    double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    double Rq[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                    2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                    2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double M[9], Mc[9];
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) M[3 * j + k] = Rq[3 * j + k] * s[k];
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++)
            Mc[3 * j + k] = R[3 * j] * M[k] + R[3 * j + 1] * M[3 + k] + R[3 * j + 2] * M[6 + k];
    double Lx = 0, Ly = 0;
    int clx = 0, cly = 0;
    if (cfg->fov_clamp) {
        double lxp = (W - cx) / fx + 0.3 * (0.5 * W / fx), lxn = cx / fx + 0.3 * (0.5 * W / fx);
        double lyp = (H - cy) / fy + 0.3 * (0.5 * H / fy), lyn = cy / fy + 0.3 * (0.5 * H / fy);
        if (flags & VKO_F_FOVX_HI) { clx = 1; Lx = lxp; }
        else if (flags & VKO_F_FOVX_LO) { clx = 1; Lx = -lxn; }
        if (flags & VKO_F_FOVY_HI) { cly = 1; Ly = lyp; }
        else if (flags & VKO_F_FOVY_LO) { cly = 1; Ly = -lyn; }
    }
    const double txc = clx ? tz * Lx : tx, tyc = cly ? tz * Ly : ty;
    const double J00 = fx / tz, J02 = -fx * txc / (tz * tz), J11 = fy / tz, J12 = -fy * tyc / (tz * tz);
    double K0[3], K1[3];
    for (int k = 0; k < 3; k++) {
        K0[k] = J00 * Mc[k] + J02 * Mc[6 + k];
        K1[k] = J11 * Mc[3 + k] + J12 * Mc[6 + k];
    }
    const double A = K0[0] * K0[0] + K0[1] * K0[1] + K0[2] * K0[2] + 0.3;
    const double B = K0[0] * K1[0] + K0[1] * K1[1] + K0[2] * K1[2];
    const double C = K1[0] * K1[0] + K1[1] * K1[1] + K1[2] * K1[2] + 0.3;
    const double det = A * C - B * B, det2 = det * det;
    const double rho = 1.0 / (1.0 + exp(-o));
    *mlogit = mdrho * rho * (1 - rho);
    double cp[3];
    for (int k = 0; k < 3; k++) cp[k] = -(R[k] * ct[0] + R[3 + k] * ct[1] + R[6 + k] * ct[2]);
    double d[3] = {mu[0] - cp[0], mu[1] - cp[1], mu[2] - cp[2]};
    double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double dh[3] = {d[0] / dl, d[1] / dl, d[2] / dl};
    double Y[16], dY[16][3];
    sh_basis_grad(dh[0], dh[1], dh[2], K, Y, dY);
    double mce[3];
    for (int ch = 0; ch < 3; ch++) mce[ch] = (flags & (VKO_F_CLAMP_R << ch)) ? 0.0 : mdcol[ch];
    double mdh[3] = {0, 0, 0};
    for (int l = 0; l < K; l++) {
        double mg = 0;
        for (int ch = 0; ch < 3; ch++) {
            msh[3 * l + ch] = fabs(Y[l]) * mce[ch];
            mg += mce[ch] * fabs(sh[3 * l + ch]);
        }
        for (int k = 0; k < 3; k++) mdh[k] += mg * fabs(dY[l][k]);
    }
    const double mpr = fabs(dh[0]) * mdh[0] + fabs(dh[1]) * mdh[1] + fabs(dh[2]) * mdh[2];
    for (int k = 0; k < 3; k++) mmu[k] = (mdh[k] + fabs(dh[k]) * mpr) / dl;
    const double ma = mdcon[0], mb = mdcon[1], mc = mdcon[2];
    const double mA = (C * C * ma + fabs(B * C) * mb + B * B * mc) / det2;
    const double mB = (2 * fabs(B * C) * ma + (A * C + B * B) * mb + 2 * fabs(A * B) * mc) / det2;
    const double mC = (B * B * ma + fabs(A * B) * mb + A * A * mc) / det2;
    double mK0[3], mK1[3];
    for (int k = 0; k < 3; k++) {
        mK0[k] = 2 * mA * fabs(K0[k]) + mB * fabs(K1[k]);
        mK1[k] = mB * fabs(K0[k]) + 2 * mC * fabs(K1[k]);
    }
    double mJ00 = 0, mJ02 = 0, mJ11 = 0, mJ12 = 0, mMc[9];
    for (int k = 0; k < 3; k++) {
        mJ00 += mK0[k] * fabs(Mc[k]);
        mJ02 += mK0[k] * fabs(Mc[6 + k]);
        mJ11 += mK1[k] * fabs(Mc[3 + k]);
        mJ12 += mK1[k] * fabs(Mc[6 + k]);
        mMc[k] = fabs(J00) * mK0[k];
        mMc[3 + k] = fabs(J11) * mK1[k];
        mMc[6 + k] = fabs(J02) * mK0[k] + fabs(J12) * mK1[k];
    }
    double mD[9];
    for (int k = 0; k < 3; k++) {
        double ms = 0;
        for (int j = 0; j < 3; j++) {
            const double mM = fabs(R[j]) * mMc[k] + fabs(R[3 + j]) * mMc[3 + k] + fabs(R[6 + j]) * mMc[6 + k];
            ms += mM * fabs(Rq[3 * j + k]);
            mD[3 * j + k] = mM * s[k];
        }
        mls[k] = ms * s[k];
    }
    const double aw = fabs(w), ax = fabs(x), ay = fabs(y), az = fabs(z);
    double mqh[4];
    mqh[0] = 2 * (az * mD[1] + ay * mD[2] + az * mD[3] + ax * mD[5] + ay * mD[6] + ax * mD[7]);
    mqh[1] = 2 * (ay * mD[1] + az * mD[2] + ay * mD[3] + 2 * ax * mD[4] + aw * mD[5] + az * mD[6] + aw * mD[7] + 2 * ax * mD[8]);
    mqh[2] = 2 * (2 * ay * mD[0] + ax * mD[1] + aw * mD[2] + ax * mD[3] + az * mD[5] + aw * mD[6] + az * mD[7] + 2 * ay * mD[8]);
    mqh[3] = 2 * (2 * az * mD[0] + aw * mD[1] + ax * mD[2] + aw * mD[3] + 2 * az * mD[4] + ay * mD[5] + ax * mD[6] + ay * mD[7]);
    const double mqd = aw * mqh[0] + ax * mqh[1] + ay * mqh[2] + az * mqh[3];
    const double aq[4] = {aw, ax, ay, az};
    for (int k = 0; k < 4; k++) mq[k] = (mqh[k] + aq[k] * mqd) / qn;
    const double tz2 = tz * tz, tz3 = tz2 * tz;
    double mt[3];
    mt[0] = fx / tz * mdm2[0];
    mt[1] = fy / tz * mdm2[1];
    mt[2] = fabs(fx * tx) / tz2 * mdm2[0] + fabs(fy * ty) / tz2 * mdm2[1] + fx / tz2 * mJ00 + fy / tz2 * mJ11;
    if (!clx) { mt[0] += fx / tz2 * mJ02; mt[2] += 2 * fabs(fx * tx) / tz3 * mJ02; }
    else { mt[2] += fabs(fx * Lx) / tz2 * mJ02; }
    if (!cly) { mt[1] += fy / tz2 * mJ12; mt[2] += 2 * fabs(fy * ty) / tz3 * mJ12; }
    else { mt[2] += fabs(fy * Ly) / tz2 * mJ12; }
    for (int k = 0; k < 3; k++) mmu[k] += fabs(R[k]) * mt[0] + fabs(R[3 + k]) * mt[1] + fabs(R[6 + k]) * mt[2];
}

typedef struct {
    const vko_config* cfg;
    const vko_camera* cam;
    const float *means, *ls, *q, *o, *sh;
    const double *dm2, *dcon, *dcol, *dop;
    double *dmeans, *dls, *dq, *dol, *dsh;
} pmctx;

static void pmass_range(void* vp, int64_t b, int64_t e, int tid) {
    (void)tid;
    pmctx* c = (pmctx*)vp;
    const int64_t S = c->cfg->sh_coeffs * 3;
    double* shd = (double*)malloc(sizeof(double) * S);
    for (int64_t i = b; i < e; i++) {
        memset(c->dmeans + 3 * i, 0, 3 * sizeof(double));
        memset(c->dls + 3 * i, 0, 3 * sizeof(double));
        memset(c->dq + 4 * i, 0, 4 * sizeof(double));
        c->dol[i] = 0;
        memset(c->dsh + S * i, 0, S * sizeof(double));
        proj_t_f32 P;
        project_one_f32(c->cfg, c->cam, c->means + 3 * i, c->ls + 3 * i, c->q + 4 * i, c->o[i],
                        c->sh + S * i, &P);
        if (!(P.flags & VKO_F_VISIBLE)) continue;
        double mu[3], ls[3], q[4];
        for (int k = 0; k < 3; k++) { mu[k] = c->means[3 * i + k]; ls[k] = c->ls[3 * i + k]; }
        for (int k = 0; k < 4; k++) q[k] = c->q[4 * i + k];
        for (int k = 0; k < S; k++) shd[k] = c->sh[S * i + k];
        proj_bwd_mass_one(c->cfg, c->cam, P.flags, mu, ls, q, c->o[i], shd, c->dm2 + 2 * i,
                          c->dcon + 3 * i, c->dcol + 3 * i, c->dop[i], c->dmeans + 3 * i,
                          c->dls + 3 * i, c->dq + 4 * i, &c->dol[i], c->dsh + S * i);
    }
    free(shd);
}

void vko_project_bwd_mass(const vko_config* cfg, const vko_camera* cam, int64_t n, const float* means,
                          const float* log_scales, const float* quats, const float* opacity_logits,
                          const float* sh, const double* m_dmeans2d, const double* m_dconics,
                          const double* m_dcolors, const double* m_dopacities, double* m_dmeans,
                          double* m_dlog_scales, double* m_dquats, double* m_dopacity_logits,
                          double* m_dsh, int nthreads) {
    pmctx c = {cfg, cam, means, log_scales, quats, opacity_logits, sh, m_dmeans2d, m_dconics,
               m_dcolors, m_dopacities, m_dmeans, m_dlog_scales, m_dquats, m_dopacity_logits, m_dsh};
    parallel_for(n, 4096, nthreads, pmass_range, &c);
}

typedef struct {
    const vko_config* cfg;
    const vko_camera* cam;
    const float *means, *ls, *q, *o, *sh;
    const double *dm2, *dcon, *dcol, *dop;
    double *dmeans, *dls, *dq, *dol, *dsh;
} pbctx;

static void pbwd_range(void* vp, int64_t b, int64_t e, int tid) {
    (void)tid;
    pbctx* c = (pbctx*)vp;
    const int64_t S = c->cfg->sh_coeffs * 3;
    double* shd = (double*)malloc(sizeof(double) * S);
    for (int64_t i = b; i < e; i++) {
        memset(c->dmeans + 3 * i, 0, 3 * sizeof(double));
        memset(c->dls + 3 * i, 0, 3 * sizeof(double));
        memset(c->dq + 4 * i, 0, 4 * sizeof(double));
        c->dol[i] = 0;
        memset(c->dsh + S * i, 0, S * sizeof(double));
        proj_t_f32 P;
        project_one_f32(c->cfg, c->cam, c->means + 3 * i, c->ls + 3 * i, c->q + 4 * i, c->o[i],
                        c->sh + S * i, &P);
        if (!(P.flags & VKO_F_VISIBLE)) continue; /* never rasterised: no gradient */
        double mu[3], ls[3], q[4];
        for (int k = 0; k < 3; k++) { mu[k] = c->means[3 * i + k]; ls[k] = c->ls[3 * i + k]; }
        for (int k = 0; k < 4; k++) q[k] = c->q[4 * i + k];
        for (int k = 0; k < S; k++) shd[k] = c->sh[S * i + k];
        proj_bwd_one(c->cfg, c->cam, P.flags, mu, ls, q, c->o[i], shd, c->dm2 + 2 * i,
                     c->dcon + 3 * i, c->dcol + 3 * i, c->dop[i], c->dmeans + 3 * i,
                     c->dls + 3 * i, c->dq + 4 * i, &c->dol[i], c->dsh + S * i);
    }
    free(shd);
}

void vko_project_bwd(const vko_config* cfg, const vko_camera* cam, int64_t n, const float* means,
                     const float* log_scales, const float* quats, const float* opacity_logits,
                     const float* sh, const double* dmeans2d, const double* dconics,
                     const double* dcolors, const double* dopacities, double* dmeans,
                     double* dlog_scales, double* dquats, double* dopacity_logits, double* dsh,
                     int nthreads) {
    pbctx c = {cfg, cam, means, log_scales, quats, opacity_logits, sh, dmeans2d, dconics, dcolors,
               dopacities, dmeans, dlog_scales, dquats, dopacity_logits, dsh};
    parallel_for(n, 4096, nthreads, pbwd_range, &c);
}

void vko_project_bwd_f64(const vko_config* cfg, const vko_camera* cam, int64_t n,
                         const double* means, const double* log_scales, const double* quats,
                         const double* opacity_logits, const double* sh, const double* dmeans2d,
                         const double* dconics, const double* dcolors, const double* dopacities,
                         double* dmeans, double* dlog_scales, double* dquats,
                         double* dopacity_logits, double* dsh) {
    const int64_t S = cfg->sh_coeffs * 3;
    for (int64_t i = 0; i < n; i++) {
        memset(dmeans + 3 * i, 0, 3 * sizeof(double));
        memset(dlog_scales + 3 * i, 0, 3 * sizeof(double));
        memset(dquats + 4 * i, 0, 4 * sizeof(double));
        dopacity_logits[i] = 0;
        memset(dsh + S * i, 0, S * sizeof(double));
        proj_t_f64 P;
        project_one_f64(cfg, cam, means + 3 * i, log_scales + 3 * i, quats + 4 * i,
                        opacity_logits[i], sh + S * i, &P);
        if (!(P.flags & VKO_F_PROJECTABLE)) continue;
        proj_bwd_one(cfg, cam, P.flags, means + 3 * i, log_scales + 3 * i, quats + 4 * i,
                     opacity_logits[i], sh + S * i, dmeans2d + 2 * i, dconics + 3 * i,
                     dcolors + 3 * i, dopacities[i], dmeans + 3 * i, dlog_scales + 3 * i,
                     dquats + 4 * i, &dopacity_logits[i], dsh + S * i);
    }
}

/* ---- optimizer: Adam with bias correction, S:252-259 -------------------- */
void vko_adam_group(int64_t n, float* p, float* m, float* v, const float* g, double lr, double b1,
                    double b2, double eps, int32_t t) {
    const double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < n; i++) {
        const double gi = (double)g[i];
        const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
        const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
        const double mhat = mi / bc1, vhat = vi / bc2;
        p[i] = (float)((double)p[i] - lr * mhat / (sqrt(vhat) + eps));
        m[i] = (float)mi;
        v[i] = (float)vi;
    }
}

void vko_quat_renorm(int64_t n, float* q) {
    for (int64_t i = 0; i < n; i++) {
        const double a = q[4 * i], b = q[4 * i + 1], c = q[4 * i + 2], d = q[4 * i + 3];
        const double nn = sqrt(a * a + b * b + c * c + d * d);
        if (!(nn > 0.0)) continue;
        q[4 * i] = (float)(a / nn);
        q[4 * i + 1] = (float)(b / nn);
        q[4 * i + 2] = (float)(c / nn);
        q[4 * i + 3] = (float)(d / nn);
    }
}

/* ---- loss gradient: L1 + lambda D-SSIM, S:178-186, S:482 ------------------ */
static void ssim_window(double w[11][11]) {
    double g[11], sum = 0.0;
    for (int i = 0; i < 11; i++) {
        const double d = (double)(i - 5);
        g[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += g[i];
    }
    for (int i = 0; i < 11; i++)
        for (int j = 0; j < 11; j++) w[i][j] = (g[i] / sum) * (g[j] / sum);
}

double vko_loss_grad(int32_t W, int32_t H, double lambda, const float* render, const float* target,
                     double* dL_dr, double* ssim_out) {
    const int64_t np = (int64_t)W * H;
    double l1 = 0.0;
    for (int64_t i = 0; i < 3 * np; i++) {
        const double d = (double)render[i] - (double)target[i];
        l1 += fabs(d);
        dL_dr[i] = (1.0 - lambda) * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / (double)(3 * np);
    }
    l1 /= (double)(3 * np);
    double ssim = 1.0;
    if (lambda != 0.0) {
        const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
        double w[11][11];
        ssim_window(w);
        const int Wv = W - 10, Hv = H - 10;
        const double nv = 3.0 * (double)Wv * (double)Hv;
        double acc = 0.0;
        for (int c = 0; c < 3; c++)
            for (int py = 0; py < Hv; py++)
                for (int px = 0; px < Wv; px++) {
                    double mx = 0, my = 0, exx = 0, eyy = 0, exy = 0;
                    for (int i = 0; i < 11; i++)
                        for (int j = 0; j < 11; j++) {
                            const int64_t q = ((int64_t)(py + i) * W + (px + j)) * 3 + c;
                            const double x = render[q], y = target[q], ww = w[i][j];
                            mx += ww * x; my += ww * y;
                            exx += ww * x * x; eyy += ww * y * y; exy += ww * x * y;
                        }
                    const double sx2 = exx - mx * mx, sy2 = eyy - my * my, sxy = exy - mx * my;
                    const double l1n = 2 * mx * my + C1, l2n = mx * mx + my * my + C1;
                    const double c1n = 2 * sxy + C2, c2n = sx2 + sy2 + C2;
                    const double S = (l1n * c1n) / (l2n * c2n);
                    acc += S;
                    /* partials with respect to mx, E[x^2], E[xy] (the other window sums held) */
                    const double dB = -S / c2n;                 /* dS/dE[x^2] = dS/dsx2 */
                    const double dC = 2.0 * l1n / (l2n * c2n);  /* dS/dE[xy]  = dS/dsxy */
                    const double dA = 2.0 * my * c1n / (l2n * c2n) - 2.0 * mx * S / l2n
                                    - 2.0 * mx * dB - my * dC;  /* total dS/dmx */
                    const double k = -lambda / nv;
                    for (int i = 0; i < 11; i++)
                        for (int j = 0; j < 11; j++) {
                            const int64_t q = ((int64_t)(py + i) * W + (px + j)) * 3 + c;
                            const double x = render[q], y = target[q];
                            dL_dr[q] += k * w[i][j] * (dA + 2.0 * dB * x + dC * y);
                        }
                }
        ssim = acc / nv;
    }
    if (ssim_out) *ssim_out = ssim;
    return (1.0 - lambda) * l1 + lambda * (1.0 - ssim);
}

/* ---- MCMC densification: S:273, readings R1-R5 of DESIGN.md §4.7 ----------- */
uint64_t vko_rng(uint64_t seed, uint32_t stream, uint64_t i) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((((uint64_t)stream) << 40) ^ i);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double rng_uniform(uint64_t seed, uint32_t stream, uint64_t i) {
    return ((double)(vko_rng(seed, stream, i) >> 40) + 0.5) / 16777216.0;
}

static double rng_normal(uint64_t seed, uint32_t stream, uint64_t k) {
    const double u1 = rng_uniform(seed, stream, 2 * k), u2 = rng_uniform(seed, stream, 2 * k + 1);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

static float x64_sigmoid(float o) { return (float)(1.0 / (1.0 + exp(-(double)o))); }

int64_t vko_mcmc_relocate(int64_t n, int32_t sh_coeffs, float dead_opacity, uint64_t seed, float* means,
                          float* log_scales, float* quats, float* opacity_logits, float* sh, float* m, float* v,
                          int64_t* targets) {
    float* rho = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    uint64_t* W = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    int64_t* k = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    uint64_t total = 0;
    int64_t dead = 0;
    for (int64_t i = 0; i < n; i++) {
        rho[i] = x64_sigmoid(opacity_logits[i]);
        const int is_dead = rho[i] < dead_opacity;
        dead += is_dead;
        total += is_dead ? 0 : (uint64_t)floor((double)rho[i] * 16777216.0);
        W[i] = total;
    }
    for (int64_t i = 0; i < n; i++) {
        targets[i] = -1;
        if (!(rho[i] < dead_opacity) || total == 0) continue;
        const uint64_t t = (uint64_t)(((unsigned __int128)vko_rng(seed, 1, (uint64_t)i) * total) >> 64);
        int64_t lo = 0, hi = n - 1;  /* first j with W[j] > t */
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (W[mid] > t) hi = mid; else lo = mid + 1;
        }
        targets[i] = lo;
        k[lo]++;
    }
    const int64_t S = 3 * (int64_t)sh_coeffs, F = 11 + S;
    for (int64_t i = 0; i < n; i++) {  /* copies first (they read the targets' original rows) */
        const int64_t j = targets[i];
        if (j < 0) continue;
        memcpy(means + 3 * i, means + 3 * j, 3 * sizeof(float));
        memcpy(log_scales + 3 * i, log_scales + 3 * j, 3 * sizeof(float));
        memcpy(quats + 4 * i, quats + 4 * j, 4 * sizeof(float));
        memcpy(sh + S * i, sh + S * j, (size_t)S * sizeof(float));
        const double rp = 1.0 - pow(1.0 - (double)rho[j], 1.0 / (double)(k[j] + 1));
        opacity_logits[i] = (float)log(rp / (1.0 - rp));
        if (m && v) {
            const int64_t off[5] = {0, 3 * n, 6 * n, 10 * n, 11 * n}, w[5] = {3, 3, 4, 1, S};
            for (int g = 0; g < 5; g++)
                for (int64_t c = 0; c < w[g]; c++) {
                    m[off[g] + w[g] * i + c] = 0.0f;
                    v[off[g] + w[g] * i + c] = 0.0f;
                }
        }
        (void)F;
    }
    for (int64_t j = 0; j < n; j++) {
        if (k[j] == 0) continue;
        const double rp = 1.0 - pow(1.0 - (double)rho[j], 1.0 / (double)(k[j] + 1));
        opacity_logits[j] = (float)log(rp / (1.0 - rp));
    }
    free(rho); free(W); free(k);
    return dead;
}

void vko_mcmc_noise(int64_t n, float lr_pos, float noise_scale, uint64_t seed, uint32_t step, float* means,
                    const float* log_scales, const float* quats, const float* opacity_logits) {
    for (int64_t i = 0; i < n; i++) {
        const double rho = x64_sigmoid(opacity_logits[i]);
        const double gate = 1.0 / (1.0 + exp(-100.0 * (0.005 - rho)));
        const double a = quats[4 * i], b = quats[4 * i + 1], c = quats[4 * i + 2], d = quats[4 * i + 3];
        const double qn = sqrt(a * a + b * b + c * c + d * d);
        const double w = a / qn, x = b / qn, y = c / qn, z = d / qn;
        const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                             2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                             2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        double e[3];
        for (int q = 0; q < 3; q++) e[q] = exp((double)log_scales[3 * i + q]) * rng_normal(seed, 2 + 2 * step, 3 * (uint64_t)i + q);
        const double kk = (double)lr_pos * (double)noise_scale * gate;
        for (int r = 0; r < 3; r++)
            means[3 * i + r] = (float)((double)means[3 * i + r] + kk * (R[3 * r] * e[0] + R[3 * r + 1] * e[1] + R[3 * r + 2] * e[2]));
    }
}

/* ---- default densification: S:261-269, readings R6-R9 ----------------------- */
void vko_densify_stats(int64_t n, const float* dmeans2d, const int32_t* radii, float* accum, float* denom) {
    for (int64_t i = 0; i < n; i++) {
        if (radii[2 * i] <= 0 && radii[2 * i + 1] <= 0) continue;
        const double gx = dmeans2d[2 * i], gy = dmeans2d[2 * i + 1];
        accum[i] = (float)((double)accum[i] + sqrt(gx * gx + gy * gy));
        denom[i] = denom[i] + 1.0f;
    }
}

static int densify_kind(int64_t i, const float* log_scales, const float* opacity_logits, const float* accum,
                        const float* denom, float gthr, float sthr, float pop) {
    const float rho = x64_sigmoid(opacity_logits[i]);
    if (rho < pop) return 0;                                     /* prune */
    const float g = denom[i] > 0.0f ? accum[i] / denom[i] : 0.0f;
    if (!(g > gthr)) return 1;                                   /* keep */
    float smax = (float)exp((double)log_scales[3 * i]);
    for (int c = 1; c < 3; c++) smax = fmaxf(smax, (float)exp((double)log_scales[3 * i + c]));
    return smax < sthr ? 2 : 3;                                  /* clone : split */
}

int64_t vko_densify(int64_t n, int32_t sh_coeffs, const float* means, const float* log_scales, const float* quats,
                    const float* opacity_logits, const float* sh, const float* m, const float* v,
                    const float* accum, const float* denom, float grad_threshold, float size_threshold,
                    float prune_opacity, uint64_t seed, int64_t cap, float* o_means, float* o_log_scales,
                    float* o_quats, float* o_opacity_logits, float* o_sh, float* o_m, float* o_v) {
    const int64_t S = 3 * (int64_t)sh_coeffs;
    int64_t np = 0;
    for (int64_t i = 0; i < n; i++) {
        const int k = densify_kind(i, log_scales, opacity_logits, accum, denom, grad_threshold, size_threshold,
                                   prune_opacity);
        np += k == 0 ? 0 : (k == 1 ? 1 : 2);
    }
    if (np > cap) return np;
    const int64_t wid[5] = {3, 3, 4, 1, S};
    int64_t o = 0;
    for (int64_t i = 0; i < n; i++) {
        const int k = densify_kind(i, log_scales, opacity_logits, accum, denom, grad_threshold, size_threshold,
                                   prune_opacity);
        const int rows = k == 0 ? 0 : (k == 1 ? 1 : 2);
        for (int r = 0; r < rows; r++, o++) {
            memcpy(o_means + 3 * o, means + 3 * i, 3 * sizeof(float));
            memcpy(o_log_scales + 3 * o, log_scales + 3 * i, 3 * sizeof(float));
            memcpy(o_quats + 4 * o, quats + 4 * i, 4 * sizeof(float));
            o_opacity_logits[o] = opacity_logits[i];
            memcpy(o_sh + S * o, sh + S * i, (size_t)S * sizeof(float));
            if (k == 3) {  /* split child r */
                const double a = quats[4 * i], b = quats[4 * i + 1], c = quats[4 * i + 2], d = quats[4 * i + 3];
                const double qn = sqrt(a * a + b * b + c * c + d * d);
                const double w = a / qn, x = b / qn, y = c / qn, z = d / qn;
                const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
                double e[3];
                for (int q = 0; q < 3; q++)
                    e[q] = exp((double)log_scales[3 * i + q]) * rng_normal(seed, 3, 6 * (uint64_t)i + 3 * r + q);
                for (int q = 0; q < 3; q++) {
                    o_means[3 * o + q] = (float)((double)means[3 * i + q] + R[3 * q] * e[0] + R[3 * q + 1] * e[1] +
                                                 R[3 * q + 2] * e[2]);
                    o_log_scales[3 * o + q] = (float)((double)log_scales[3 * i + q] - log(1.6));
                }
            }
            if (o_m && o_v) {
                const int fresh = (k == 2 && r == 1) || k == 3;
                int64_t off = 0, offo = 0;
                for (int g = 0; g < 5; g++) {
                    for (int64_t c = 0; c < wid[g]; c++) {
                        o_m[offo + wid[g] * o + c] = (fresh || !m) ? 0.0f : m[off + wid[g] * i + c];
                        o_v[offo + wid[g] * o + c] = (fresh || !v) ? 0.0f : v[off + wid[g] * i + c];
                    }
                    off += wid[g] * n;
                    offo += wid[g] * np;
                }
            }
        }
    }
    return np;
}
