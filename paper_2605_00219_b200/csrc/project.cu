// project.cu — "Projection Forward" and the projection part of "Proj Bwd + Optimizer"
// (P:76).  Compiled with -fmad=false: every fp32 + - * / below is one IEEE-rounded operation in
// the order written, which is the order pinned in DESIGN.md §4.1 (the oracle's O1 follows the
// same written specification independently), so projection outputs are bit-exact with O1.
// Transcendentals on the key path are evaluated as (float)f((double)x).
//
// Layout: SoA parameter rows (means [N,3], log_scales [N,3], quats [N,4], opacity_logits [N],
// sh [N,KS,3]); one thread per Gaussian; SH rows of a warp's 32 Gaussians are staged through
// shared memory with coalesced 16-byte loads, and only for lanes that survived culling (the SH
// bytes of culled Gaussians are never read).
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// 3DGS real spherical-harmonics constants (closed forms in DESIGN.md §4.1 step 12)
#define C0 0.28209479177387814f
#define C1 0.4886025119029199f
#define C20 1.0925484305920792f
#define C21 -1.0925484305920792f
#define C22 0.31539156525252005f
#define C23 -1.0925484305920792f
#define C24 0.5462742152960396f
#define C30 -0.5900435899266435f
#define C31 2.890611442640554f
#define C32 -0.4570457994644658f
#define C33 0.3731763325901154f
#define C34 -0.4570457994644658f
#define C35 1.445305721320277f
#define C36 -0.5900435899266435f

struct Params {
    vks_camera cam;
    vks_config cfg;
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
    // backward
    const int2* __restrict__ radii_in;
    const float2* __restrict__ dm2;
    const float* __restrict__ dcon;
    const float* __restrict__ dcol;
    const float* __restrict__ dop;
    float* __restrict__ dmeans;
    float* __restrict__ dls;
    float4* __restrict__ dquats;
    float* __restrict__ dologit;
    float* __restrict__ dsh;
};

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

__device__ __forceinline__ bool project_core(const vks_camera& cam, const vks_config& cfg,
                                             const float mu[3], const float ls[3], float4 q,
                                             float o, Core& k) {
    const float* R = cam.R;
    const float fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
    const float W = (float)cam.width, H = (float)cam.height;
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
        const float lxp = (W - cx) / fx + 0.3f * ((0.5f * W) / fx);
        const float lxn = cx / fx + 0.3f * ((0.5f * W) / fx);
        const float lyp = (H - cy) / fy + 0.3f * ((0.5f * H) / fy);
        const float lyn = cy / fy + 0.3f * ((0.5f * H) / fy);
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
__device__ __forceinline__ void view_dir(const vks_camera& cam, const float mu[3], float dh[3], float& dl) {
    const float* R = cam.R;
    float cp[3], d[3];
#pragma unroll
    for (int c = 0; c < 3; c++) cp[c] = -((R[0 * 3 + c] * cam.t[0] + R[1 * 3 + c] * cam.t[1]) + R[2 * 3 + c] * cam.t[2]);
#pragma unroll
    for (int c = 0; c < 3; c++) d[c] = mu[c] - cp[c];
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

// d Y_l / d(x,y,z) (backward only; not on the bit-exact path)
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, int K, float dY[16][3]) {
#pragma unroll
    for (int l = 0; l < 16; l++) dY[l][0] = dY[l][1] = dY[l][2] = 0.0f;
    if (K > 1) {
        dY[1][1] = -C1;
        dY[2][2] = C1;
        dY[3][0] = -C1;
    }
    if (K > 4) {
        dY[4][0] = C20 * y; dY[4][1] = C20 * x;
        dY[5][1] = C21 * z; dY[5][2] = C21 * y;
        dY[6][0] = -2.0f * C22 * x; dY[6][1] = -2.0f * C22 * y; dY[6][2] = 4.0f * C22 * z;
        dY[7][0] = C23 * z; dY[7][2] = C23 * x;
        dY[8][0] = 2.0f * C24 * x; dY[8][1] = -2.0f * C24 * y;
    }
    if (K > 9) {
        const float xx = x * x, yy = y * y, zz = z * z;
        dY[9][0] = 6.0f * C30 * x * y; dY[9][1] = C30 * (3.0f * xx - 3.0f * yy);
        dY[10][0] = C31 * y * z; dY[10][1] = C31 * x * z; dY[10][2] = C31 * x * y;
        dY[11][0] = -2.0f * C32 * x * y; dY[11][1] = C32 * (4.0f * zz - xx - 3.0f * yy); dY[11][2] = 8.0f * C32 * y * z;
        dY[12][0] = -6.0f * C33 * x * z; dY[12][1] = -6.0f * C33 * y * z; dY[12][2] = C33 * (6.0f * zz - 3.0f * xx - 3.0f * yy);
        dY[13][0] = C34 * (4.0f * zz - 3.0f * xx - yy); dY[13][1] = -2.0f * C34 * x * y; dY[13][2] = 8.0f * C34 * x * z;
        dY[14][0] = 2.0f * C35 * x * z; dY[14][1] = -2.0f * C35 * y * z; dY[14][2] = C35 * (xx - yy);
        dY[15][0] = C36 * (3.0f * xx - 3.0f * yy); dY[15][1] = -6.0f * C36 * x * y;
    }
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

// copy rows of lanes in `mask` from global (row base `g0` = first Gaussian of the warp) to smem
template <int KS>
__device__ __forceinline__ void sh_stage_in(const float* __restrict__ src, int64_t g0, int64_t n,
                                            unsigned mask, float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec) {
        constexpr int V = Lay::S / 4;  // float4 per row
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V;
        for (int j = lane; j < 32 * V; j += 32) {
            const int r = j / V, c = j - r * V;
            if ((mask >> r) & 1u) {
                float4 v = __ldg(s4 + j);
                *reinterpret_cast<float4*>(buf + r * Lay::SP + 4 * c) = v;
            }
        }
    } else {
        const float* s1 = src + g0 * Lay::S;
        for (int j = lane; j < 32 * Lay::S; j += 32) {
            const int r = j / Lay::S, c = j - r * Lay::S;
            if ((mask >> r) & 1u) buf[r * Lay::SP + c] = __ldg(s1 + j);
        }
    }
    (void)n;
}

template <int KS>
__device__ __forceinline__ void sh_stage_out(float* __restrict__ dst, int64_t g0, unsigned mask,
                                             const float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec) {
        constexpr int V = Lay::S / 4;
        float4* d4 = reinterpret_cast<float4*>(dst) + g0 * V;
        for (int j = lane; j < 32 * V; j += 32) {
            const int r = j / V, c = j - r * V;
            if ((mask >> r) & 1u) d4[j] = *reinterpret_cast<const float4*>(buf + r * Lay::SP + 4 * c);
        }
    } else {
        float* d1 = dst + g0 * Lay::S;
        for (int j = lane; j < 32 * Lay::S; j += 32) {
            const int r = j / Lay::S, c = j - r * Lay::S;
            if ((mask >> r) & 1u) d1[j] = buf[r * Lay::SP + c];
        }
    }
}

__device__ __forceinline__ void load_params(const Params& p, int64_t i, float mu[3], float ls[3],
                                            float4& q, float& o) {
#pragma unroll
    for (int c = 0; c < 3; c++) {
        mu[c] = __ldg(p.means + 3 * i + c);
        ls[c] = __ldg(p.ls + 3 * i + c);
    }
    q = __ldg(p.quats + i);
    o = __ldg(p.ologit + i);
}

// ------------------------------------------------------------------------------------------
// forward: KS = compile-time stored SH coefficients (1,4,9,16) or 0 = generic (runtime stride)
template <int KS>
__global__ void __launch_bounds__(kThreads) project_fwd_kernel(const Params p) {
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;  // first Gaussian of this warp
    const bool valid = i < p.n;
    const int TX = tiles_x(p.cam), TY = tiles_y(p.cam);

    Core k;
    float mu[3], ls[3], o = 0.0f;
    float4 q = make_float4(0, 0, 0, 0);
    float rxf = 0, ryf = 0;
    int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    bool vis = false;
    if (valid) {
        mu[0] = __ldg(p.means + 3 * i);
        mu[1] = __ldg(p.means + 3 * i + 1);
        mu[2] = __ldg(p.means + 3 * i + 2);
        // cheap near-plane test first: skip the other parameter loads of Gaussians behind the camera
        const float tz = dot3(p.cam.R + 6, mu) + p.cam.t[2];
        if (tz > p.cfg.near_plane) {
#pragma unroll
            for (int c = 0; c < 3; c++) ls[c] = __ldg(p.ls + 3 * i + c);
            q = __ldg(p.quats + i);
            o = __ldg(p.ologit + i);
            vis = project_core(p.cam, p.cfg, mu, ls, q, o, k) &&
                  footprint_rect(k, p.cfg, TX, TY, rxf, ryf, x0, x1, y0, y1);
        }
    }
    // colour (only for survivors; SH rows staged through smem)
    const int K = (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);
    float col[3] = {0, 0, 0};
    const unsigned vmask = __ballot_sync(VKS_FULL_MASK, vis);
    if (vmask) {
        const float* f;
        if constexpr (KS > 0) {
            float* buf = smem + warp * ShLayout<KS>::kWarpFloats;
            sh_stage_in<KS>(p.sh, g0, p.n, vmask, buf);
            __syncwarp();
            f = buf + lane * ShLayout<KS>::SP;
        } else {
            f = p.sh + 3 * (int64_t)p.cfg.sh_coeffs * i;
        }
        if (vis) {
            float dh[3], dl;
            view_dir(p.cam, mu, dh, dl);
            float Y[16];
            sh_basis(dh[0], dh[1], dh[2], K, Y);
            bool ok = true;
#pragma unroll
            for (int ch = 0; ch < 3; ch++) {
                float acc = Y[0] * f[ch];
#pragma unroll
                for (int l = 1; l < 16; l++)
                    if (l < K) acc = acc + Y[l] * f[3 * l + ch];
                const float raw = acc + 0.5f;
                ok = ok && isfinite(raw);
                col[ch] = raw > 0.0f ? raw : 0.0f;
            }
            vis = ok;
        }
    }
    if (!valid) return;
    if (vis) {
        p.means2d[i] = make_float2(k.u, k.v);
        p.conics[3 * i + 0] = k.a;
        p.conics[3 * i + 1] = k.b;
        p.conics[3 * i + 2] = k.c;
        p.depths[i] = k.t[2];
        p.radii[i] = make_int2((int)rxf, (int)ryf);
        p.tiles[i] = (x1 - x0) * (y1 - y0);
        p.colors[3 * i + 0] = col[0];
        p.colors[3 * i + 1] = col[1];
        p.colors[3 * i + 2] = col[2];
        p.opac[i] = k.rho;
    } else {
        p.radii[i] = make_int2(0, 0);
        p.tiles[i] = 0;
    }
}

// ------------------------------------------------------------------------------------------
// backward: fp32 chain rule, accumulate (+=)
// OVERWRITE: write the gradients (zero rows for radii == 0) instead of accumulating (+=)
template <int KS, bool OVERWRITE>
__global__ void __launch_bounds__(kThreads) project_bwd_kernel(const Params p) {
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;
    bool act = i < p.n;
    if (act) {
        const int2 r = p.radii_in[i];
        act = (r.x != 0) || (r.y != 0);
    }
    Core k;
    float mu[3] = {0, 0, 0}, ls[3] = {0, 0, 0}, o = 0.0f;
    float4 q = make_float4(1, 0, 0, 0);
    if (act) {
        load_params(p, i, mu, ls, q, o);
        act = project_core(p.cam, p.cfg, mu, ls, q, o, k);  // always true for radii != 0
    }
    const unsigned amask = __ballot_sync(VKS_FULL_MASK, act);
    if (OVERWRITE && i < p.n && !act) {  // never rasterised: zero rows
        const int S0 = 3 * p.cfg.sh_coeffs;
#pragma unroll
        for (int c = 0; c < 3; c++) { p.dmeans[3 * i + c] = 0.0f; p.dls[3 * i + c] = 0.0f; }
        p.dquats[i] = make_float4(0, 0, 0, 0);
        p.dologit[i] = 0.0f;
        if (KS == 0)
            for (int j = 0; j < S0; j++) p.dsh[(int64_t)S0 * i + j] = 0.0f;
    }
    if (!amask) {
        if constexpr (OVERWRITE && KS > 0) {
            // whole warp inactive: zero its SH rows with coalesced stores
            const int64_t nrow = min((int64_t)32, p.n - g0);
            float4* d4 = reinterpret_cast<float4*>(p.dsh + g0 * 3 * KS);
            if constexpr ((3 * KS) % 4 == 0) {
                for (int j = lane; j < nrow * (3 * KS / 4); j += 32) d4[j] = make_float4(0, 0, 0, 0);
            } else {
                for (int j = lane; j < nrow * 3 * KS; j += 32) p.dsh[g0 * 3 * KS + j] = 0.0f;
            }
        }
        return;
    }
    const int K = (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);
    const int S = 3 * p.cfg.sh_coeffs;

    float dmu[3] = {0, 0, 0};
    float dcol[3] = {0, 0, 0};
    float dhv[3] = {0, 0, 0}, dl = 1.0f;
    float Y[16];
    if (act) {
        dcol[0] = p.dcol[3 * i]; dcol[1] = p.dcol[3 * i + 1]; dcol[2] = p.dcol[3 * i + 2];
        view_dir(p.cam, mu, dhv, dl);
        sh_basis(dhv[0], dhv[1], dhv[2], K, Y);
    }
    // SH: stage f rows in, compute clamp flags + direction gradient, stage dsh rows in, add, out
    float* buf = nullptr;
    const float* f;
    if constexpr (KS > 0) {
        buf = smem + warp * ShLayout<KS>::kWarpFloats;
        sh_stage_in<KS>(p.sh, g0, p.n, amask, buf);
        __syncwarp();
        f = buf + lane * ShLayout<KS>::SP;
    } else {
        f = p.sh + (int64_t)S * i;
    }
    float dce[3] = {0, 0, 0};
    float ddh[3] = {0, 0, 0};
    if (act) {
        float dY[16][3];
        sh_basis_grad(dhv[0], dhv[1], dhv[2], K, dY);
#pragma unroll
        for (int ch = 0; ch < 3; ch++) {
            // clamp decision with the forward's exact fp32 sequence
            float acc = Y[0] * f[ch];
#pragma unroll
            for (int l = 1; l < 16; l++)
                if (l < K) acc = acc + Y[l] * f[3 * l + ch];
            const float raw = acc + 0.5f;
            dce[ch] = raw > 0.0f ? dcol[ch] : 0.0f;
        }
#pragma unroll
        for (int l = 1; l < 16; l++) {
            if (l < K) {
                const float g = dce[0] * f[3 * l] + dce[1] * f[3 * l + 1] + dce[2] * f[3 * l + 2];
                ddh[0] += g * dY[l][0];
                ddh[1] += g * dY[l][1];
                ddh[2] += g * dY[l][2];
            }
        }
    }
    if constexpr (KS > 0) {
        __syncwarp();
        if (!OVERWRITE) sh_stage_in<KS>(p.dsh, g0, p.n, amask, buf);
        __syncwarp();
        if (act) {
            float* dfp = buf + lane * ShLayout<KS>::SP;
#pragma unroll
            for (int l = 0; l < KS; l++) {
                const float yl = l < K ? Y[l] : 0.0f;
#pragma unroll
                for (int ch = 0; ch < 3; ch++) {
                    if (OVERWRITE) dfp[3 * l + ch] = yl * dce[ch];
                    else dfp[3 * l + ch] += yl * dce[ch];
                }
            }
        }
        __syncwarp();
        // rows of inactive lanes in an active warp: OVERWRITE must still zero them
        const unsigned omask = OVERWRITE ? __ballot_sync(VKS_FULL_MASK, i < p.n) : amask;
        if (OVERWRITE && !act && i < p.n) {
            float* dfp = buf + lane * ShLayout<KS>::SP;
            for (int j = 0; j < 3 * KS; j++) dfp[j] = 0.0f;
        }
        __syncwarp();
        sh_stage_out<KS>(p.dsh, g0, omask, buf);
    } else {
        if (act) {
            float* dfp = p.dsh + (int64_t)S * i;
            for (int l = 0; l < S / 3; l++) {
                const float yl = l < K ? Y[l] : 0.0f;
                for (int ch = 0; ch < 3; ch++) {
                    if (OVERWRITE) dfp[3 * l + ch] = yl * dce[ch];
                    else dfp[3 * l + ch] += yl * dce[ch];
                }
            }
        }
    }
    if (!act) return;
    {
        const float pr = dhv[0] * ddh[0] + dhv[1] * ddh[1] + dhv[2] * ddh[2];
#pragma unroll
        for (int c = 0; c < 3; c++) dmu[c] = (ddh[c] - dhv[c] * pr) / dl;
    }
    // opacity: sigmoid chain
    const float drho = p.dop[i];
    if (OVERWRITE) p.dologit[i] = drho * k.rho * (1.0f - k.rho);
    else p.dologit[i] += drho * k.rho * (1.0f - k.rho);
    // conic (a,b,c) = (C, -B, A)/det  ->  (A, B, C)
    const float da = p.dcon[3 * i], db = p.dcon[3 * i + 1], dc = p.dcon[3 * i + 2];
    const float id = 1.0f / k.det, id2 = id * id;
    const float A = k.A, B = k.B, C = k.C;
    // d(Sigma'^-1): written without the 1/det - AC/det^2 cancellation (= -B^2/det^2)
    const float dA = (-C * C * da + B * C * db - B * B * dc) * id2;
    const float dB = (2.0f * B * C * da - (A * C + B * B) * db + 2.0f * A * B * dc) * id2;
    const float dC = (-B * B * da + A * B * db - A * A * dc) * id2;
    // Sigma' = K K^T + 0.3 I
    float dK0[3], dK1[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        dK0[c] = 2.0f * dA * k.K0[c] + dB * k.K1[c];
        dK1[c] = dB * k.K0[c] + 2.0f * dC * k.K1[c];
    }
    // K = J Mc
    float dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0, dMc[9];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        dJ00 += dK0[c] * k.Mc[c];
        dJ02 += dK0[c] * k.Mc[6 + c];
        dJ11 += dK1[c] * k.Mc[3 + c];
        dJ12 += dK1[c] * k.Mc[6 + c];
        dMc[c] = k.J00 * dK0[c];
        dMc[3 + c] = k.J11 * dK1[c];
        dMc[6 + c] = k.J02 * dK0[c] + k.J12 * dK1[c];
    }
    // Mc = R M ;  M = Rq diag(s)
    const float* R = p.cam.R;
    float D[9], dlsv[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float ds = 0.0f;
#pragma unroll
        for (int j = 0; j < 3; j++) {
            const float dM = R[j] * dMc[c] + R[3 + j] * dMc[3 + c] + R[6 + j] * dMc[6 + c];
            ds += dM * k.Rq[3 * j + c];
            D[3 * j + c] = dM * k.s[c];
        }
        dlsv[c] = ds * k.s[c];
    }
    const float w = k.w, x = k.x, y = k.y, z = k.z;
    float dq0 = 2.0f * (-z * D[1] + y * D[2] + z * D[3] - x * D[5] - y * D[6] + x * D[7]);
    float dq1 = 2.0f * (y * D[1] + z * D[2] + y * D[3] - 2.0f * x * D[4] - w * D[5] + z * D[6] + w * D[7] - 2.0f * x * D[8]);
    float dq2 = 2.0f * (-2.0f * y * D[0] + x * D[1] + w * D[2] + x * D[3] + z * D[5] - w * D[6] + z * D[7] - 2.0f * y * D[8]);
    float dq3 = 2.0f * (-2.0f * z * D[0] - w * D[1] + x * D[2] + w * D[3] - 2.0f * z * D[4] + y * D[5] + x * D[6] + y * D[7]);
    const float qd = w * dq0 + x * dq1 + y * dq2 + z * dq3;
    const float iqn = 1.0f / k.qn;
    // t: from mean2d and from J (exact FOV-clamp derivative)
    const float2 dm = p.dm2[i];
    const float fx = p.cam.fx, fy = p.cam.fy;
    const float tx = k.t[0], ty = k.t[1], tz = k.t[2];
    const float itz = 1.0f / tz, itz2 = itz * itz, itz3 = itz2 * itz;
    float dt0 = fx * itz * dm.x;
    float dt1 = fy * itz * dm.y;
    float dt2 = -fx * tx * itz2 * dm.x - fy * ty * itz2 * dm.y - fx * itz2 * dJ00 - fy * itz2 * dJ11;
    if (k.fovx == 0) { dt0 += -fx * itz2 * dJ02; dt2 += 2.0f * fx * tx * itz3 * dJ02; }
    else { dt2 += fx * k.Lx * itz2 * dJ02; }
    if (k.fovy == 0) { dt1 += -fy * itz2 * dJ12; dt2 += 2.0f * fy * ty * itz3 * dJ12; }
    else { dt2 += fy * k.Ly * itz2 * dJ12; }
#pragma unroll
    for (int c = 0; c < 3; c++) dmu[c] += R[c] * dt0 + R[3 + c] * dt1 + R[6 + c] * dt2;
#pragma unroll
    for (int c = 0; c < 3; c++) {
        if (OVERWRITE) { p.dmeans[3 * i + c] = dmu[c]; p.dls[3 * i + c] = dlsv[c]; }
        else { p.dmeans[3 * i + c] += dmu[c]; p.dls[3 * i + c] += dlsv[c]; }
    }
    float4 dqv = OVERWRITE ? make_float4(0, 0, 0, 0) : p.dquats[i];
    dqv.x += (dq0 - w * qd) * iqn;
    dqv.y += (dq1 - x * qd) * iqn;
    dqv.z += (dq2 - y * qd) * iqn;
    dqv.w += (dq3 - z * qd) * iqn;
    p.dquats[i] = dqv;
}

template <int KS>
size_t smem_bytes() {
    if constexpr (KS > 0) return sizeof(float) * kWarps * ShLayout<KS>::kWarpFloats;
    return 0;
}

template <int KS>
int launch_fwd_t(const Params& p, cudaStream_t s) {
    const size_t sm = smem_bytes<KS>();
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(project_fwd_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return VKS_ERR_CUDA;
    }
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    project_fwd_kernel<KS><<<blocks, kThreads, sm, s>>>(p);
    return LaunchCheck::check();
}

template <int KS, bool OW>
int launch_bwd_t2(const Params& p, cudaStream_t s) {
    const size_t sm = smem_bytes<KS>();
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(project_bwd_kernel<KS, OW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return VKS_ERR_CUDA;
    }
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    project_bwd_kernel<KS, OW><<<blocks, kThreads, sm, s>>>(p);
    return LaunchCheck::check();
}

template <int KS>
int launch_bwd_t(const Params& p, cudaStream_t s) {
    return (p.cfg.flags & VKS_FLAG_GRAD_OVERWRITE) ? launch_bwd_t2<KS, true>(p, s) : launch_bwd_t2<KS, false>(p, s);
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

int launch_project_fwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, float* means2d, float* conics, float* depths, int32_t* radii,
                       int32_t* tiles_touched, float* colors, float* opacities, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    Params p{};
    p.cam = cam; p.cfg = cfg; p.n = n;
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh;
    p.means2d = reinterpret_cast<float2*>(means2d); p.conics = conics; p.depths = depths;
    p.radii = reinterpret_cast<int2*>(radii); p.tiles = tiles_touched; p.colors = colors;
    p.opac = opacities;
    const bool al = aligned16(sh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_fwd_t<16>(p, s) : launch_fwd_t<0>(p, s);
        case 9: return launch_fwd_t<9>(p, s);
        case 4: return al ? launch_fwd_t<4>(p, s) : launch_fwd_t<0>(p, s);
        case 1: return launch_fwd_t<1>(p, s);
        default: return launch_fwd_t<0>(p, s);
    }
}

int launch_project_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, const int32_t* radii, const float* dmeans2d,
                       const float* dconics, const float* dcolors, const float* dopacities,
                       float* dmeans, float* dlog_scales, float* dquats, float* dopacity_logits,
                       float* dsh, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    Params p{};
    p.cam = cam; p.cfg = cfg; p.n = n;
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh;
    p.radii_in = reinterpret_cast<const int2*>(radii);
    p.dm2 = reinterpret_cast<const float2*>(dmeans2d); p.dcon = dconics; p.dcol = dcolors;
    p.dop = dopacities; p.dmeans = dmeans; p.dls = dlog_scales;
    p.dquats = reinterpret_cast<float4*>(dquats); p.dologit = dopacity_logits; p.dsh = dsh;
    const bool al = aligned16(sh) && aligned16(dsh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_bwd_t<16>(p, s) : launch_bwd_t<0>(p, s);
        case 9: return launch_bwd_t<9>(p, s);
        case 4: return al ? launch_bwd_t<4>(p, s) : launch_bwd_t<0>(p, s);
        case 1: return launch_bwd_t<1>(p, s);
        default: return launch_bwd_t<0>(p, s);
    }
}

}  // namespace vks
