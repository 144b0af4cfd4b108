// project.cu — "Projection Forward"; the backward lives in project_bwd.cu.  Compiled with -fmad=false: every fp32 + - * / below is one IEEE-rounded operation in
// the order written, which is the order pinned in DESIGN.md §4.1 (the oracle's O1 follows the
// same written specification independently), so projection outputs are bit-exact with O1.
// Transcendentals on the key path are evaluated as (float)f((double)x).
//
// Layout: SoA parameter rows (means [N,3], log_scales [N,3], quats [N,4], opacity_logits [N],
// sh [N,KS,3]); one thread per Gaussian; SH rows of a warp's 32 Gaussians are staged through
// shared memory with coalesced 16-byte loads, and only for lanes that survived culling (the SH
// bytes of culled Gaussians are never read).
#include "vks_common.cuh"
#include "vks_sh.cuh"

namespace vks {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// 3DGS real spherical-harmonics constants (closed forms in DESIGN.md §4.1 step 12)
using namespace sh;  // the SH basis constants (vks_sh.cuh)

struct Params {
    vks_camera cam;
    vks_config cfg;
    CamConst cc;
    int64_t n;
    const float* __restrict__ means;
    const float* __restrict__ ls;
    const float4* __restrict__ quats;
    const float* __restrict__ ologit;
    const float* __restrict__ sh;
    // forward outputs
    float2* __restrict__ means2d;
    float* __restrict__ conics;
    float* __restrict__ depths;
    int2* __restrict__ radii;
    int* __restrict__ tiles;
    float* __restrict__ colors;
    float* __restrict__ opac;
    float4* __restrict__ rec;  // nullable: packed raster records [n][3] (store_records_warp)
};

// The packed raster records (include/vks.h, vks_project_fwd `records`): per visible Gaussian the
// values the rasterizer stages per list entry, in its order — (u, v, a/2, b), (c/2, rho, c0, c1),
// (c2, id bits, 0, 0).  A warp writes its 32 rows (1.5 KB) through a shared-memory buffer as three
// fully coalesced 512-byte stores (48-byte rows stored lane by lane leave every 32-byte sector
// half-written per instruction); culled rows get zeros, rows >= n nothing.  Every lane of the warp
// calls it.
constexpr int kRecWarpF4 = 96;  // float4 per warp buffer
__device__ __forceinline__ void store_records_warp(float4* __restrict__ rec, int64_t g0, int64_t n, float4* sb, bool vis,
                                                   float u, float v, float a, float b, float c, float rho,
                                                   const float col[3]) {
    const int lane = (int)lane_id();
    const float4 z = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    sb[3 * lane + 0] = vis ? make_float4(u, v, 0.5f * a, b) : z;
    sb[3 * lane + 1] = vis ? make_float4(0.5f * c, rho, col[0], col[1]) : z;
    sb[3 * lane + 2] = vis ? make_float4(col[2], __uint_as_float((uint32_t)(g0 + lane)), 0.0f, 0.0f) : z;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const int j = lane + 32 * k;
        if (g0 + j / 3 < n) rec[3 * g0 + j] = sb[j];
    }
    __syncwarp();
}

__device__ __forceinline__ float dot3(const float* a, const float* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// Steps 1-9 and 12a of DESIGN.md §4.1 (everything but the footprint and the colour).
struct Core {
    float t[3];
    float w, x, y, z, qn;
    float Rq[9], s[3], Mc[9];
    int fovx, fovy;  // +1 clamped at the upper limit, -1 at the lower, 0 free
    float Lx, Ly;    // the limit value when clamped (signed)
    float J00, J02, J11, J12;
    float K0[3], K1[3];
    float A, B, C, det, a, b, c;
    float u, v, rho;
};

__device__ __forceinline__ bool project_core(const vks_camera& cam, const vks_config& cfg, const CamConst& cc,
                                             const float mu[3], const float ls[3], float4 q,
                                             float o, Core& k) {
    const float* R = cam.R;
    const float fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
    // 1. camera-space mean; cull !(t.z > near)
    k.t[0] = dot3(R + 0, mu) + cam.t[0];
    k.t[1] = dot3(R + 3, mu) + cam.t[1];
    k.t[2] = dot3(R + 6, mu) + cam.t[2];
    const float tx = k.t[0], ty = k.t[1], tz = k.t[2];
    if (!(tz > cfg.near_plane) || !isfinite(tz)) return false;
    // 2. unit quaternion (w,x,y,z)
    k.qn = sqrtf(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
    if (!(k.qn > 1e-12f)) return false;
    const float w = q.x / k.qn, x = q.y / k.qn, y = q.z / k.qn, z = q.w / k.qn;
    k.w = w; k.x = x; k.y = y; k.z = z;
    // 3. rotation of the unit quaternion
    k.Rq[0] = 1.0f - 2.0f * (y * y + z * z);
    k.Rq[1] = 2.0f * (x * y - w * z);
    k.Rq[2] = 2.0f * (x * z + w * y);
    k.Rq[3] = 2.0f * (x * y + w * z);
    k.Rq[4] = 1.0f - 2.0f * (x * x + z * z);
    k.Rq[5] = 2.0f * (y * z - w * x);
    k.Rq[6] = 2.0f * (x * z - w * y);
    k.Rq[7] = 2.0f * (y * z + w * x);
    k.Rq[8] = 1.0f - 2.0f * (x * x + y * y);
    // 4. scales (X64) and M = Rq diag(s); 5. Mc = R M
    float M[9];
#pragma unroll
    for (int j = 0; j < 3; j++) k.s[j] = (float)exp((double)ls[j]);
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int c = 0; c < 3; c++) M[j * 3 + c] = k.Rq[j * 3 + c] * k.s[c];
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int c = 0; c < 3; c++)
            k.Mc[j * 3 + c] = (R[j * 3 + 0] * M[0 * 3 + c] + R[j * 3 + 1] * M[1 * 3 + c]) + R[j * 3 + 2] * M[2 * 3 + c];
    // 6. FOV clamp
    float txc = tx, tyc = ty;
    k.fovx = k.fovy = 0;
    k.Lx = k.Ly = 0.0f;
    if (cfg.fov_clamp) {
        const float lxp = cc.lxp, lxn = cc.lxn, lyp = cc.lyp, lyn = cc.lyn;
        const float rxz = tx / tz, ryz = ty / tz;
        txc = tz * fminf(lxp, fmaxf(-lxn, rxz));
        tyc = tz * fminf(lyp, fmaxf(-lyn, ryz));
        if (rxz > lxp) { k.fovx = 1; k.Lx = lxp; }
        else if (rxz < -lxn) { k.fovx = -1; k.Lx = -lxn; }
        if (ryz > lyp) { k.fovy = 1; k.Ly = lyp; }
        else if (ryz < -lyn) { k.fovy = -1; k.Ly = -lyn; }
    }
    // 7. J and K = J Mc
    k.J00 = fx / tz;
    k.J02 = -(fx * txc) / (tz * tz);
    k.J11 = fy / tz;
    k.J12 = -(fy * tyc) / (tz * tz);
#pragma unroll
    for (int c = 0; c < 3; c++) {
        k.K0[c] = k.J00 * k.Mc[0 * 3 + c] + k.J02 * k.Mc[2 * 3 + c];
        k.K1[c] = k.J11 * k.Mc[1 * 3 + c] + k.J12 * k.Mc[2 * 3 + c];
    }
    // 8. 2D covariance + low-pass, conic
    k.A = dot3(k.K0, k.K0) + 0.3f;
    k.B = dot3(k.K0, k.K1);
    k.C = dot3(k.K1, k.K1) + 0.3f;
    k.det = k.A * k.C - k.B * k.B;
    if (!(k.det > 0.0f)) return false;
    k.a = k.C / k.det;
    k.b = -k.B / k.det;
    k.c = k.A / k.det;
    // 9. mean2d (unclamped t)
    k.u = (fx * tx) / tz + cx;
    k.v = (fy * ty) / tz + cy;
    // 12a. opacity (X64 sigmoid)
    k.rho = (float)(1.0 / (1.0 + exp(-(double)o)));
    if (!isfinite(k.u) || !isfinite(k.v) || !isfinite(k.a) || !isfinite(k.b) || !isfinite(k.c) ||
        !isfinite(k.rho))
        return false;
    return true;
}

// 10-11. footprint half-extents and the clipped tile rect
__device__ __forceinline__ bool footprint_rect(const Core& k, const vks_config& cfg, int TX, int TY,
                                               float& rxf, float& ryf, int& x0, int& x1, int& y0,
                                               int& y1) {
    if (cfg.footprint == VKS_FOOTPRINT_SUPPORT) {
        if (!(k.rho >= 1.0f / 255.0f)) return false;
        const float kk = (float)log(255.0 * (double)k.rho);
        const float kp = kk * 1.001f + 1e-3f;
        rxf = ceilf(sqrtf((2.0f * kp) * k.A)) + 1.0f;
        ryf = ceilf(sqrtf((2.0f * kp) * k.C)) + 1.0f;
    } else {
        const float h = 0.5f * (k.A - k.C);
        const float l1 = 0.5f * (k.A + k.C) + sqrtf(h * h + k.B * k.B);
        rxf = ceilf(3.0f * sqrtf(l1));
        ryf = rxf;
    }
    rxf = fminf(rxf, 16777216.0f);
    ryf = fminf(ryf, 16777216.0f);
    x0 = (int)fminf(fmaxf(floorf((k.u - rxf) * 0.0625f), 0.0f), (float)TX);
    x1 = (int)fminf(fmaxf(ceilf((k.u + rxf) * 0.0625f), 0.0f), (float)TX);
    y0 = (int)fminf(fmaxf(floorf((k.v - ryf) * 0.0625f), 0.0f), (float)TY);
    y1 = (int)fminf(fmaxf(ceilf((k.v + ryf) * 0.0625f), 0.0f), (float)TY);
    return (x1 - x0) * (y1 - y0) > 0;
}

// 12b. view direction and SH basis (3DGS order, pinned evaluation order)
__device__ __forceinline__ void view_dir(const CamConst& cc, const float mu[3], float dh[3], float& dl) {
    float d[3];
#pragma unroll
    for (int c = 0; c < 3; c++) d[c] = mu[c] - cc.cp[c];
    dl = sqrtf(dot3(d, d));
#pragma unroll
    for (int c = 0; c < 3; c++) dh[c] = d[c] / dl;
}

__device__ __forceinline__ void sh_basis(float x, float y, float z, int K, float Y[16]) {
    Y[0] = C0;
    if (K <= 1) return;
    Y[1] = -C1 * y;
    Y[2] = C1 * z;
    Y[3] = -C1 * x;
    if (K <= 4) return;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    Y[4] = C20 * xy;
    Y[5] = C21 * yz;
    Y[6] = C22 * ((2.0f * zz - xx) - yy);
    Y[7] = C23 * xz;
    Y[8] = C24 * (xx - yy);
    if (K <= 9) return;
    Y[9] = (C30 * y) * (3.0f * xx - yy);
    Y[10] = (C31 * xy) * z;
    Y[11] = (C32 * y) * ((4.0f * zz - xx) - yy);
    Y[12] = (C33 * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
    Y[13] = (C34 * x) * ((4.0f * zz - xx) - yy);
    Y[14] = (C35 * z) * (xx - yy);
    Y[15] = (C36 * x) * (xx - 3.0f * yy);
}

// ---- warp-cooperative staging of SH rows ------------------------------------------------
// KS = stored coefficients per Gaussian (compile time); S = 3*KS floats per row; the smem row
// stride SP is chosen so per-lane row reads are bank-conflict free.
template <int KS>
struct ShLayout {
    static constexpr int S = 3 * KS;
    static constexpr bool kVec = (S % 4) == 0;
    static constexpr int SP = (S == 48) ? 52 : S;  // 52 = 13 float4: conflict-free 128-bit LDS
    static constexpr int kWarpFloats = 32 * SP;
};

// the single-view kernel reuses the warp's SH staging buffer for its 96-float4 record buffer
template <int KS>
constexpr bool rec_in_sh() {
    if constexpr (KS > 0) return ShLayout<KS>::kWarpFloats * sizeof(float) >= 96 * sizeof(float4) &&
                                 (ShLayout<KS>::kWarpFloats % 4) == 0;
    return false;
}

// staged rows readable as float4 (16-byte aligned, whole float4 per row)
template <int KS>
constexpr bool vec_rows() {
    if constexpr (KS > 0) return ShLayout<KS>::kVec && ShLayout<KS>::SP % 4 == 0;
    return false;
}

// issue async copies of the SH rows of lanes in `mask` (row base `g0` = first Gaussian of the
// warp) into the warp's smem slice; the caller commits / waits
template <int KS>
__device__ __forceinline__ void sh_stage_async(const float* __restrict__ src, int64_t g0, unsigned mask, float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec && (Lay::S / 4) % 4 == 0) {
        // 4 lanes per row, V/4 float4 each: lane l takes row l/4 + 8 it and columns l%4 + 4 m;
        // every instruction moves 8 rows x 64 contiguous bytes, addresses advance by constants
        constexpr int V = Lay::S / 4;
        constexpr int M = V / 4;
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V + (lane >> 2) * V + (lane & 3);
        uint32_t d = smem_addr(buf) + 4u * ((lane >> 2) * Lay::SP + 4 * (lane & 3));
#pragma unroll
        for (int it = 0; it < 4; it++) {
            if ((mask >> ((lane >> 2) + 8 * it)) & 1u) {
#pragma unroll
                for (int m = 0; m < M; m++) cp_async16_s(d + 64u * m, s4 + 4 * m);
            }
            s4 += 8 * V;
            d += 4u * 8 * Lay::SP;
        }
    } else if constexpr (Lay::kVec) {
        constexpr int V = Lay::S / 4;  // float4 per row
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V;
        // chunk j = lane + 32 it of the warp's 32 x V float4: row r = j / V, column c = j % V,
        // advanced incrementally (32 = (32 / V) V + 32 % V)
        int r = (int)lane / V, c = (int)lane - r * V;
#pragma unroll
        for (int it = 0; it < V; it++) {
            if ((mask >> r) & 1u) cp_async16(buf + r * Lay::SP + 4 * c, s4 + (lane + 32 * it));
            c += 32 % V;
            r += 32 / V;
            if (c >= V) { c -= V; r += 1; }
        }
    } else {
        const float* s1 = src + g0 * Lay::S;
        for (int j = lane; j < 32 * Lay::S; j += 32) {
            const int r = j / Lay::S, c = j - r * Lay::S;
            if ((mask >> r) & 1u) cp_async4(buf + r * Lay::SP + c, s1 + j);
        }
    }
}

// ------------------------------------------------------------------------------------------
// forward: KS = compile-time stored SH coefficients (1,4,9,16) or 0 = generic (runtime stride)
template <int KS>
__global__ void __launch_bounds__(kThreads) project_fwd_kernel(const Params p) {
    pdl_wait();
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;  // first Gaussian of this warp
    const bool valid = i < p.n;
    const int TX = tiles_x(p.cam), TY = tiles_y(p.cam);

    Core k;
    float mu[3] = {0, 0, 0}, ls[3] = {0, 0, 0}, o = 0.0f;
    float4 q = make_float4(0, 0, 0, 0);
    float rxf = 0, ryf = 0;
    int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    bool near_ok = false;
    if (valid) {  // every parameter load issued at once (one DRAM round trip)
#pragma unroll
        for (int c = 0; c < 3; c++) {
            mu[c] = __ldg(p.means + 3 * i + c);
            ls[c] = __ldg(p.ls + 3 * i + c);
        }
        q = __ldg(p.quats + i);
        o = __ldg(p.ologit + i);
        const float tz = dot3(p.cam.R + 6, mu) + p.cam.t[2];
        near_ok = tz > p.cfg.near_plane;
    }
    bool vis = near_ok && project_core(p.cam, p.cfg, p.cc, mu, ls, q, o, k) &&
               footprint_rect(k, p.cfg, TX, TY, rxf, ryf, x0, x1, y0, y1);
    // SH rows only of the Gaussians that touch a tile (in front of the camera but outside the
    // view is ~1/3 of the near-plane survivors on the ring views: their rows are never read)
    const int K = (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);
    float col[3] = {0, 0, 0};
    const unsigned vmask = __ballot_sync(VKS_FULL_MASK, vis);
    float* buf = nullptr;
    if constexpr (KS > 0) {
        buf = smem + warp * ShLayout<KS>::kWarpFloats;
        if (vmask) {
            sh_stage_async<KS>(p.sh, g0, vmask, buf);
            cp_async_commit();
        }
    }
    float Y[16];
    if (vis) {  // the SH basis of the view direction while the rows are in flight
        float dh[3], dl;
        view_dir(p.cc, mu, dh, dl);
        sh_basis(dh[0], dh[1], dh[2], K, Y);
    }
    if constexpr (KS > 0) {
        if (vmask) cp_async_wait_all();
        __syncwarp();
    }
    if (vmask && vis) {
        const float* f;
        if constexpr (KS > 0) f = buf + lane * ShLayout<KS>::SP;
        else f = p.sh + 3 * (int64_t)p.cfg.sh_coeffs * i;
        float acc[3];
        if constexpr (vec_rows<KS>()) {
            // 128-bit shared-memory reads of the staged row; element e = 3 l + ch, each channel
            // still accumulated in ascending l (the pinned order)
            const float4* f4 = reinterpret_cast<const float4*>(f);
#pragma unroll
            for (int m = 0; m < ShLayout<KS>::S / 4; m++) {
                const float4 qv = f4[m];
                const float e4[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int e = 4 * m + t, l = e / 3, ch = e % 3;
                    if (l == 0) acc[ch] = Y[0] * e4[t];
                    else if (l < K) acc[ch] = acc[ch] + Y[l] * e4[t];
                }
            }
        } else {
#pragma unroll
            for (int ch = 0; ch < 3; ch++) {
                acc[ch] = Y[0] * f[ch];
#pragma unroll
                for (int l = 1; l < 16; l++)
                    if (l < K) acc[ch] = acc[ch] + Y[l] * f[3 * l + ch];
            }
        }
        bool ok = true;
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            const float raw = acc[ch] + 0.5f;
            ok = ok && isfinite(raw);
            col[ch] = raw > 0.0f ? raw : 0.0f;
        }
        vis = ok;
    }
    if (p.rec) {
        // the warp's SH staging buffer is free once the colours are formed (rows of >= 12 floats
        // hold the 96 float4); smaller layouts get a buffer of their own after the SH region
        float4* sb;
        if constexpr (rec_in_sh<KS>()) {
            __syncwarp();  // every lane has read its SH row
            sb = reinterpret_cast<float4*>(buf);
        } else {
            sb = reinterpret_cast<float4*>(smem + (KS > 0 ? kWarps * ShLayout<KS>::kWarpFloats : 0)) + warp * kRecWarpF4;
        }
        store_records_warp(p.rec, g0, p.n, sb, vis, k.u, k.v, k.a, k.b, k.c, k.rho, col);
    }
    if (!valid) return;
    if (vis) {
        p.means2d[i] = make_float2(k.u, k.v);
        if (p.conics) {
            p.conics[3 * i + 0] = k.a;
            p.conics[3 * i + 1] = k.b;
            p.conics[3 * i + 2] = k.c;
        }
        p.depths[i] = k.t[2];
        p.radii[i] = make_int2((int)rxf, (int)ryf);
        p.tiles[i] = (x1 - x0) * (y1 - y0);
        p.colors[3 * i + 0] = col[0];
        p.colors[3 * i + 1] = col[1];
        p.colors[3 * i + 2] = col[2];
        p.opac[i] = k.rho;
    } else {  // full rows: partial-sector writes would make L2 fetch the sector from DRAM first
        p.means2d[i] = make_float2(0.0f, 0.0f);
        if (p.conics) {
            p.conics[3 * i + 0] = 0.0f;
            p.conics[3 * i + 1] = 0.0f;
            p.conics[3 * i + 2] = 0.0f;
        }
        p.depths[i] = 0.0f;
        p.radii[i] = make_int2(0, 0);
        p.tiles[i] = 0;
        p.colors[3 * i + 0] = 0.0f;
        p.colors[3 * i + 1] = 0.0f;
        p.colors[3 * i + 2] = 0.0f;
        p.opac[i] = 0.0f;
    }
}

// ------------------------------------------------------------------------------------------
// Batched forward: a step's views in one pass over the parameters.  Everything of §4.1 that
// does not depend on the camera — the unit quaternion, Rq, the X64 scales, M = Rq diag(s), the
// X64 opacity and the footprint's X64 log(255 rho) — is computed once per Gaussian, the SH row
// staged once; the per-view part is the single-view kernel's, operation for operation, so every
// view's outputs are bit-identical to vks_project_fwd's.
constexpr int kMaxFwdViews = 16;

struct FwdViewOut {
    vks_camera cam;
    CamConst cc;
    float2* means2d;
    float* conics;
    float* depths;
    int2* radii;
    int* tiles;
    float* colors;
    float4* rec;  // nullable: packed raster records [n][3]
    float* g2d;  // nullable: the view's 2D-gradient accumulators [9n] (dmeans2d | dconics | dcolors | dopacities), zeroed
};

struct BatchFwdParams {
    vks_config cfg;
    int64_t n;
    int nv;
    const float* __restrict__ means;
    const float* __restrict__ ls;
    const float4* __restrict__ quats;
    const float* __restrict__ ologit;
    const float* __restrict__ sh;
    float* __restrict__ opac;  // view-independent: one array
    FwdViewOut v[kMaxFwdViews];
};

// camera-independent part (steps 2-4, 12a and the footprint's k), pinned exactly as project_core
struct GCore {
    float M[9];
    float rho, kk;
    bool ok;
};

__device__ __forceinline__ void gauss_core(const vks_config& cfg, const float ls[3], float4 q, float o, GCore& G) {
    const float qn = sqrtf(((q.x * q.x + q.y * q.y) + q.z * q.z) + q.w * q.w);
    G.ok = qn > 1e-12f;
    const float w = q.x / qn, x = q.y / qn, y = q.z / qn, z = q.w / qn;
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * (y * y + z * z);
    Rq[1] = 2.0f * (x * y - w * z);
    Rq[2] = 2.0f * (x * z + w * y);
    Rq[3] = 2.0f * (x * y + w * z);
    Rq[4] = 1.0f - 2.0f * (x * x + z * z);
    Rq[5] = 2.0f * (y * z - w * x);
    Rq[6] = 2.0f * (x * z - w * y);
    Rq[7] = 2.0f * (y * z + w * x);
    Rq[8] = 1.0f - 2.0f * (x * x + y * y);
    float sc[3];
#pragma unroll
    for (int j = 0; j < 3; j++) sc[j] = (float)exp((double)ls[j]);
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int c = 0; c < 3; c++) G.M[j * 3 + c] = Rq[j * 3 + c] * sc[c];
    G.rho = (float)(1.0 / (1.0 + exp(-(double)o)));
    G.ok = G.ok && isfinite(G.rho);
    G.kk = 0.0f;
    if (cfg.footprint == VKS_FOOTPRINT_SUPPORT) {
        G.ok = G.ok && G.rho >= 1.0f / 255.0f;
        G.kk = G.ok ? (float)log(255.0 * (double)G.rho) : 0.0f;
    }
}

// the camera-dependent part (steps 1, 5-9) given G
__device__ __forceinline__ bool view_core(const vks_camera& cam, const vks_config& cfg, const CamConst& cc,
                                          const float mu[3], const GCore& G, Core& k) {
    const float* R = cam.R;
    const float fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
    k.t[0] = dot3(R + 0, mu) + cam.t[0];
    k.t[1] = dot3(R + 3, mu) + cam.t[1];
    k.t[2] = dot3(R + 6, mu) + cam.t[2];
    const float tx = k.t[0], ty = k.t[1], tz = k.t[2];
    if (!(tz > cfg.near_plane) || !isfinite(tz)) return false;
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int c = 0; c < 3; c++)
            k.Mc[j * 3 + c] = (R[j * 3 + 0] * G.M[0 * 3 + c] + R[j * 3 + 1] * G.M[1 * 3 + c]) + R[j * 3 + 2] * G.M[2 * 3 + c];
    float txc = tx, tyc = ty;
    if (cfg.fov_clamp) {
        const float rxz = tx / tz, ryz = ty / tz;
        txc = tz * fminf(cc.lxp, fmaxf(-cc.lxn, rxz));
        tyc = tz * fminf(cc.lyp, fmaxf(-cc.lyn, ryz));
    }
    k.J00 = fx / tz;
    k.J02 = -(fx * txc) / (tz * tz);
    k.J11 = fy / tz;
    k.J12 = -(fy * tyc) / (tz * tz);
#pragma unroll
    for (int c = 0; c < 3; c++) {
        k.K0[c] = k.J00 * k.Mc[0 * 3 + c] + k.J02 * k.Mc[2 * 3 + c];
        k.K1[c] = k.J11 * k.Mc[1 * 3 + c] + k.J12 * k.Mc[2 * 3 + c];
    }
    k.A = dot3(k.K0, k.K0) + 0.3f;
    k.B = dot3(k.K0, k.K1);
    k.C = dot3(k.K1, k.K1) + 0.3f;
    k.det = k.A * k.C - k.B * k.B;
    if (!(k.det > 0.0f)) return false;
    k.a = k.C / k.det;
    k.b = -k.B / k.det;
    k.c = k.A / k.det;
    k.u = (fx * tx) / tz + cx;
    k.v = (fy * ty) / tz + cy;
    k.rho = G.rho;
    return isfinite(k.u) && isfinite(k.v) && isfinite(k.a) && isfinite(k.b) && isfinite(k.c);
}

// footprint half-extents and rect (steps 10-11) with the footprint's k from G
__device__ __forceinline__ bool footprint_rect_g(const Core& k, float kk, const vks_config& cfg, int TX, int TY,
                                                 float& rxf, float& ryf, int& x0, int& x1, int& y0, int& y1) {
    if (cfg.footprint == VKS_FOOTPRINT_SUPPORT) {
        const float kp = kk * 1.001f + 1e-3f;
        rxf = ceilf(sqrtf((2.0f * kp) * k.A)) + 1.0f;
        ryf = ceilf(sqrtf((2.0f * kp) * k.C)) + 1.0f;
    } else {
        const float h = 0.5f * (k.A - k.C);
        const float l1 = 0.5f * (k.A + k.C) + sqrtf(h * h + k.B * k.B);
        rxf = ceilf(3.0f * sqrtf(l1));
        ryf = rxf;
    }
    rxf = fminf(rxf, 16777216.0f);
    ryf = fminf(ryf, 16777216.0f);
    x0 = (int)fminf(fmaxf(floorf((k.u - rxf) * 0.0625f), 0.0f), (float)TX);
    x1 = (int)fminf(fmaxf(ceilf((k.u + rxf) * 0.0625f), 0.0f), (float)TX);
    y0 = (int)fminf(fmaxf(floorf((k.v - ryf) * 0.0625f), 0.0f), (float)TY);
    y1 = (int)fminf(fmaxf(ceilf((k.v + ryf) * 0.0625f), 0.0f), (float)TY);
    return (x1 - x0) * (y1 - y0) > 0;
}

template <int KS>
#ifdef VKS_PFWD_MINB  // measurement builds only: a residency target for the batched forward
#define VKS_PFWD_LB kThreads, VKS_PFWD_MINB
#else
#define VKS_PFWD_LB kThreads
#endif
__global__ void __launch_bounds__(VKS_PFWD_LB) project_fwd_batch_kernel(const BatchFwdParams p) {
    pdl_wait();
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;
    const bool valid = i < p.n;
    const int K = (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);
    float mu[3] = {0, 0, 0}, ls[3] = {0, 0, 0}, o = 0.0f;
    float4 q = make_float4(1, 0, 0, 0);
    if (valid) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
            mu[c] = __ldg(p.means + 3 * i + c);
            ls[c] = __ldg(p.ls + 3 * i + c);
        }
        q = __ldg(p.quats + i);
        o = __ldg(p.ologit + i);
    }
    // SH rows of the warp's Gaussians staged once for all views, issued with the parameter loads
    // (every row in range, not only those gauss_core keeps: one DRAM round trip instead of two
    // dependent ones; a dropped Gaussian's row is never read)
    const unsigned gmask = __ballot_sync(VKS_FULL_MASK, valid);
    float* buf = nullptr;
    if constexpr (KS > 0) {
        buf = smem + warp * ShLayout<KS>::kWarpFloats;
        if (gmask) sh_stage_async<KS>(p.sh, g0, gmask, buf);
        cp_async_commit();
    }
    GCore G;
    gauss_core(p.cfg, ls, q, o, G);
    G.ok = G.ok && valid;
    if (valid) p.opac[i] = G.ok ? G.rho : 0.0f;
    if constexpr (KS > 0) {
        cp_async_wait_all();
        __syncwarp();
    }
    const int TX = tiles_x(p.v[0].cam), TY = tiles_y(p.v[0].cam);
    for (int v = 0; v < p.nv; v++) {
        const FwdViewOut& V = p.v[v];
        Core k;
        float rxf = 0, ryf = 0;
        int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
        bool vis = G.ok && view_core(V.cam, p.cfg, V.cc, mu, G, k) &&
                   footprint_rect_g(k, G.kk, p.cfg, TX, TY, rxf, ryf, x0, x1, y0, y1);
        float col[3] = {0, 0, 0};
        if (vis) {
            float dh[3], dl, Y[16];
            view_dir(V.cc, mu, dh, dl);
            sh_basis(dh[0], dh[1], dh[2], K, Y);
            const float* f;
            if constexpr (KS > 0) f = buf + lane * ShLayout<KS>::SP;
            else f = p.sh + 3 * (int64_t)p.cfg.sh_coeffs * i;
            float acc[3];
            if constexpr (vec_rows<KS>()) {
                const float4* f4 = reinterpret_cast<const float4*>(f);
#pragma unroll
                for (int m = 0; m < ShLayout<KS>::S / 4; m++) {
                    const float4 qv = f4[m];
                    const float e4[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                    for (int t = 0; t < 4; t++) {
                        const int e = 4 * m + t, l = e / 3, ch = e % 3;
                        if (l == 0) acc[ch] = Y[0] * e4[t];
                        else if (l < K) acc[ch] = acc[ch] + Y[l] * e4[t];
                    }
                }
            } else {
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    acc[ch] = Y[0] * f[ch];
#pragma unroll
                    for (int l = 1; l < 16; l++)
                        if (l < K) acc[ch] = acc[ch] + Y[l] * f[3 * l + ch];
                }
            }
            bool ok = true;
#pragma unroll
            for (int ch = 0; ch < 3; ch++) {
                const float raw = acc[ch] + 0.5f;
                ok = ok && isfinite(raw);
                col[ch] = raw > 0.0f ? raw : 0.0f;
            }
            vis = ok;
        }
        if (V.rec) {
            float4* sb = reinterpret_cast<float4*>(smem + (KS > 0 ? kWarps * ShLayout<KS>::kWarpFloats : 0)) +
                         warp * kRecWarpF4;
            store_records_warp(V.rec, g0, p.n, sb, vis, k.u, k.v, k.a, k.b, k.c, G.rho, col);
        }
        if (!valid) continue;
        if (V.g2d) {  // the raster backward's accumulators, cleared here instead of by a separate pass
            reinterpret_cast<float2*>(V.g2d)[i] = make_float2(0.0f, 0.0f);
            float* dcon = V.g2d + 2 * p.n + 3 * i;
            float* dcol = V.g2d + 5 * p.n + 3 * i;
            dcon[0] = 0.0f; dcon[1] = 0.0f; dcon[2] = 0.0f;
            dcol[0] = 0.0f; dcol[1] = 0.0f; dcol[2] = 0.0f;
            V.g2d[8 * p.n + i] = 0.0f;
        }
        if (vis) {
            V.means2d[i] = make_float2(k.u, k.v);
            if (V.conics) {
                V.conics[3 * i + 0] = k.a;
                V.conics[3 * i + 1] = k.b;
                V.conics[3 * i + 2] = k.c;
            }
            V.depths[i] = k.t[2];
            V.radii[i] = make_int2((int)rxf, (int)ryf);
            V.tiles[i] = (x1 - x0) * (y1 - y0);
            V.colors[3 * i + 0] = col[0];
            V.colors[3 * i + 1] = col[1];
            V.colors[3 * i + 2] = col[2];
        } else {  // whole rows (no read-for-merge of partial DRAM sectors)
            V.means2d[i] = make_float2(0.0f, 0.0f);
            if (V.conics) {
                V.conics[3 * i + 0] = 0.0f;
                V.conics[3 * i + 1] = 0.0f;
                V.conics[3 * i + 2] = 0.0f;
            }
            V.depths[i] = 0.0f;
            V.radii[i] = make_int2(0, 0);
            V.tiles[i] = 0;
            V.colors[3 * i + 0] = 0.0f;
            V.colors[3 * i + 1] = 0.0f;
            V.colors[3 * i + 2] = 0.0f;
        }
    }
}

template <int KS>
int launch_fwd_batch_t(const BatchFwdParams& p, cudaStream_t s) {
    size_t sm = 0;
    if constexpr (KS > 0) sm = sizeof(float) * kWarps * ShLayout<KS>::kWarpFloats;
    if (p.nv > 0) {
        bool rec = false;
        for (int v = 0; v < p.nv; v++) rec = rec || p.v[v].rec != nullptr;
        if (rec) sm += sizeof(float4) * kWarps * kRecWarpF4;  // the records' staging buffers
    }
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(project_fwd_batch_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm);
        if (e != cudaSuccess) return VKS_ERR_CUDA;
    }
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    launch_k(project_fwd_batch_kernel<KS>, blocks, kThreads, sm, s, p);
    return LaunchCheck::check();
}

template <int KS>
size_t smem_bytes() {
    if constexpr (KS > 0) return sizeof(float) * kWarps * ShLayout<KS>::kWarpFloats;
    return 0;
}

template <int KS>
int launch_fwd_t(const Params& p, cudaStream_t s) {
    const size_t sm = smem_bytes<KS>() + (p.rec && !rec_in_sh<KS>() ? sizeof(float4) * kWarps * kRecWarpF4 : 0);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(project_fwd_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return VKS_ERR_CUDA;
    }
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    launch_k(project_fwd_kernel<KS>, blocks, kThreads, sm, s, p);
    return LaunchCheck::check();
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

int launch_project_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, float* means2d, float* conics, float* depths, int32_t* radii,
                       int32_t* tiles_touched, float* colors, float* opacities, float* records, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    Params p{};
    p.cam = cam; p.cfg = cfg; p.n = n;
    p.cc = cam_const(cam);
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh;
    p.means2d = reinterpret_cast<float2*>(means2d); p.conics = conics; p.depths = depths;
    p.radii = reinterpret_cast<int2*>(radii); p.tiles = tiles_touched; p.colors = colors;
    p.opac = opacities;
    p.rec = reinterpret_cast<float4*>(records);
    const bool al = aligned16(sh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_fwd_t<16>(p, s) : launch_fwd_t<0>(p, s);
        case 9: return launch_fwd_t<9>(p, s);
        case 4: return al ? launch_fwd_t<4>(p, s) : launch_fwd_t<0>(p, s);
        case 1: return launch_fwd_t<1>(p, s);
        default: return launch_fwd_t<0>(p, s);
    }
}

int launch_project_fwd_batch(const vks_config& cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                             const float* means, const float* log_scales, const float* quats,
                             const float* opacity_logits, const float* sh, float* const* means2d,
                             float* const* conics, float* const* depths, int32_t* const* radii,
                             int32_t* const* tiles_touched, float* const* colors, float* opacities,
                             float* const* g2d_zero, float* const* records, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    if (n_views < 1 || n_views > kMaxFwdViews) return VKS_ERR_INVALID_ARG;
    BatchFwdParams p{};
    p.cfg = cfg; p.n = n; p.nv = n_views;
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh; p.opac = opacities;
    for (int v = 0; v < n_views; v++) {
        FwdViewOut& V = p.v[v];
        V.cam = cams[v];
        V.cc = cam_const(cams[v]);
        V.means2d = reinterpret_cast<float2*>(means2d[v]);
        V.conics = conics[v];
        V.depths = depths[v];
        V.radii = reinterpret_cast<int2*>(radii[v]);
        V.tiles = tiles_touched[v];
        V.colors = colors[v];
        V.g2d = g2d_zero ? g2d_zero[v] : nullptr;
        V.rec = records ? reinterpret_cast<float4*>(records[v]) : nullptr;
    }
    const bool al = aligned16(sh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_fwd_batch_t<16>(p, s) : launch_fwd_batch_t<0>(p, s);
        case 9: return launch_fwd_batch_t<9>(p, s);
        case 4: return al ? launch_fwd_batch_t<4>(p, s) : launch_fwd_batch_t<0>(p, s);
        case 1: return launch_fwd_batch_t<1>(p, s);
        default: return launch_fwd_batch_t<0>(p, s);
    }
}

}  // namespace vks
