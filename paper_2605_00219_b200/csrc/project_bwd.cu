// project_bwd.cu — projection part of "Proj Bwd + Optimizer".
//
// One thread per Gaussian with radii != 0 (everything else is untouched, or zeroed under
// VKS_FLAG_GRAD_OVERWRITE).  The chain rule runs in ordinary fp32 (FMA contraction allowed): only
// the two discrete decisions must replay the forward exactly, and both are taken from bit-exact
// sources — the colour clamp from the forward's own output (colour == 0 <=> raw <= 0), the FOV
// clamp by recomputing t and tx/tz with explicitly rounded intrinsics in the pinned order of
// DESIGN.md §4.1 steps 1 and 6.  All parameter / 2D-gradient loads are issued up front; SH rows of
// a warp are staged through shared memory with coalesced 16-byte loads (active lanes only).
#include "vks_common.cuh"
#include "vks_sh.cuh"

namespace vks {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

using namespace sh;  // the SH basis constants (vks_sh.cuh)

struct Params {
    vks_camera cam;
    vks_config cfg;
    int64_t n;
    const float* __restrict__ means;
    const float* __restrict__ ls;
    const float4* __restrict__ quats;
    const float* __restrict__ ologit;
    const float* __restrict__ sh;
    const float* __restrict__ colors;
    const int2* __restrict__ radii;
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

template <int KS>
struct ShLayout {
    static constexpr int S = 3 * KS;
    static constexpr bool kVec = (S % 4) == 0;
    static constexpr int SP = (S == 48) ? 52 : S;
    static constexpr int kWarpFloats = 32 * SP;
};

template <int KS>
__device__ __forceinline__ void stage_in(const float* __restrict__ src, int64_t g0, unsigned mask, float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec && (Lay::S / 4) % 4 == 0) {
        // 4 lanes per row (see stage_in_async)
        constexpr int V = Lay::S / 4, M = V / 4;
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V + (lane >> 2) * V + (lane & 3);
        float* d = buf + (lane >> 2) * Lay::SP + 4 * (lane & 3);
#pragma unroll
        for (int it = 0; it < 4; it++) {
            if ((mask >> ((lane >> 2) + 8 * it)) & 1u) {
#pragma unroll
                for (int m = 0; m < M; m++) *reinterpret_cast<float4*>(d + 16 * m) = __ldg(s4 + 4 * m);
            }
            s4 += 8 * V;
            d += 8 * Lay::SP;
        }
    } else if constexpr (Lay::kVec) {
        constexpr int V = Lay::S / 4;
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V;
        int r = (int)lane / V, c = (int)lane - r * V;  // chunk lane + 32 it: row / column, incremental
#pragma unroll 4
        for (int it = 0; it < V; it++) {
            if ((mask >> r) & 1u) *reinterpret_cast<float4*>(buf + r * Lay::SP + 4 * c) = __ldg(s4 + (lane + 32 * it));
            c += 32 % V;
            r += 32 / V;
            if (c >= V) { c -= V; r += 1; }
        }
    } else {
        const float* s1 = src + g0 * Lay::S;
        for (int j = lane; j < 32 * Lay::S; j += 32) {
            const int r = j / Lay::S, c = j - r * Lay::S;
            if ((mask >> r) & 1u) buf[r * Lay::SP + c] = __ldg(s1 + j);
        }
    }
}

template <int KS>
__device__ __forceinline__ void stage_in_async(const float* __restrict__ src, int64_t g0, unsigned mask, float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec && (Lay::S / 4) % 4 == 0) {
        // 4 lanes per row, V/4 float4 each: lane l takes row l/4 + 8 it and columns l%4 + 4 m;
        // every instruction moves 8 rows x 64 contiguous bytes, addresses advance by constants
        constexpr int V = Lay::S / 4, M = V / 4;
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
        constexpr int V = Lay::S / 4;
        const float4* s4 = reinterpret_cast<const float4*>(src) + g0 * V;
        int r = (int)lane / V, c = (int)lane - r * V;
#pragma unroll 4
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
    cp_async_commit();
}

template <int KS>
__device__ __forceinline__ void stage_out(float* __restrict__ dst, int64_t g0, unsigned mask, const float* buf) {
    using Lay = ShLayout<KS>;
    const unsigned lane = lane_id();
    if constexpr (Lay::kVec) {
        // (stores keep 512 contiguous bytes per instruction: the 4-lanes-per-row layout of the
        // loads made this HBM-bound kernel slower when used for the gradient stores)
        constexpr int V = Lay::S / 4;
        float4* d4 = reinterpret_cast<float4*>(dst) + g0 * V;
        int r = (int)lane / V, c = (int)lane - r * V;
#pragma unroll 4
        for (int it = 0; it < V; it++) {
            if ((mask >> r) & 1u) d4[lane + 32 * it] = *reinterpret_cast<const float4*>(buf + r * Lay::SP + 4 * c);
            c += 32 % V;
            r += 32 / V;
            if (c >= V) { c -= V; r += 1; }
        }
    } else {
        float* d1 = dst + g0 * Lay::S;
        for (int j = lane; j < 32 * Lay::S; j += 32) {
            const int r = j / Lay::S, c = j - r * Lay::S;
            if ((mask >> r) & 1u) d1[j] = buf[r * Lay::SP + c];
        }
    }
}

// pinned dot3 ((a0 b0 + a1 b1) + a2 b2) with explicit rounding (immune to FMA contraction)
__device__ __forceinline__ float pdot3(const float* a, const float* b) {
    return __fadd_rn(__fadd_rn(__fmul_rn(a[0], b[0]), __fmul_rn(a[1], b[1])), __fmul_rn(a[2], b[2]));
}

// FOV-clamp decision of DESIGN.md §4.1 steps 1 and 6, bit-identical to the forward
__device__ __forceinline__ void fov_decision(const vks_camera& cam, const float mu[3], float& tx, float& ty,
                                             float& tz, int& fx_, int& fy_, float& Lx, float& Ly) {
    tx = __fadd_rn(pdot3(cam.R + 0, mu), cam.t[0]);
    ty = __fadd_rn(pdot3(cam.R + 3, mu), cam.t[1]);
    tz = __fadd_rn(pdot3(cam.R + 6, mu), cam.t[2]);
    const float W = (float)cam.width, H = (float)cam.height;
    const float lxp = __fadd_rn(__fdiv_rn(__fsub_rn(W, cam.cx), cam.fx),
                                __fmul_rn(0.3f, __fdiv_rn(__fmul_rn(0.5f, W), cam.fx)));
    const float lxn = __fadd_rn(__fdiv_rn(cam.cx, cam.fx), __fmul_rn(0.3f, __fdiv_rn(__fmul_rn(0.5f, W), cam.fx)));
    const float lyp = __fadd_rn(__fdiv_rn(__fsub_rn(H, cam.cy), cam.fy),
                                __fmul_rn(0.3f, __fdiv_rn(__fmul_rn(0.5f, H), cam.fy)));
    const float lyn = __fadd_rn(__fdiv_rn(cam.cy, cam.fy), __fmul_rn(0.3f, __fdiv_rn(__fmul_rn(0.5f, H), cam.fy)));
    const float rxz = __fdiv_rn(tx, tz), ryz = __fdiv_rn(ty, tz);
    fx_ = fy_ = 0;
    Lx = Ly = 0.0f;
    if (rxz > lxp) { fx_ = 1; Lx = lxp; } else if (rxz < -lxn) { fx_ = -1; Lx = -lxn; }
    if (ryz > lyp) { fy_ = 1; Ly = lyp; } else if (ryz < -lyn) { fy_ = -1; Ly = -lyn; }
}

__device__ __forceinline__ void sh_basis_and_grad(float x, float y, float z, int K, float Y[16], float dY[16][3]) {
#pragma unroll
    for (int l = 0; l < 16; l++) { Y[l] = 0.0f; dY[l][0] = dY[l][1] = dY[l][2] = 0.0f; }
    Y[0] = C0;
    if (K > 1) {
        Y[1] = -C1 * y; dY[1][1] = -C1;
        Y[2] = C1 * z;  dY[2][2] = C1;
        Y[3] = -C1 * x; dY[3][0] = -C1;
    }
    if (K > 4) {
        const float xx = x * x, yy = y * y, zz = z * z;
        Y[4] = C20 * x * y; dY[4][0] = C20 * y; dY[4][1] = C20 * x;
        Y[5] = C21 * y * z; dY[5][1] = C21 * z; dY[5][2] = C21 * y;
        Y[6] = C22 * (2.0f * zz - xx - yy); dY[6][0] = -2.0f * C22 * x; dY[6][1] = -2.0f * C22 * y; dY[6][2] = 4.0f * C22 * z;
        Y[7] = C23 * x * z; dY[7][0] = C23 * z; dY[7][2] = C23 * x;
        Y[8] = C24 * (xx - yy); dY[8][0] = 2.0f * C24 * x; dY[8][1] = -2.0f * C24 * y;
    }
    if (K > 9) {
        const float xx = x * x, yy = y * y, zz = z * z;
        Y[9] = C30 * y * (3.0f * xx - yy);
        dY[9][0] = 6.0f * C30 * x * y; dY[9][1] = C30 * (3.0f * xx - 3.0f * yy);
        Y[10] = C31 * x * y * z;
        dY[10][0] = C31 * y * z; dY[10][1] = C31 * x * z; dY[10][2] = C31 * x * y;
        Y[11] = C32 * y * (4.0f * zz - xx - yy);
        dY[11][0] = -2.0f * C32 * x * y; dY[11][1] = C32 * (4.0f * zz - xx - 3.0f * yy); dY[11][2] = 8.0f * C32 * y * z;
        Y[12] = C33 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
        dY[12][0] = -6.0f * C33 * x * z; dY[12][1] = -6.0f * C33 * y * z; dY[12][2] = C33 * (6.0f * zz - 3.0f * xx - 3.0f * yy);
        Y[13] = C34 * x * (4.0f * zz - xx - yy);
        dY[13][0] = C34 * (4.0f * zz - 3.0f * xx - yy); dY[13][1] = -2.0f * C34 * x * y; dY[13][2] = 8.0f * C34 * x * z;
        Y[14] = C35 * z * (xx - yy);
        dY[14][0] = 2.0f * C35 * x * z; dY[14][1] = -2.0f * C35 * y * z; dY[14][2] = C35 * (xx - yy);
        Y[15] = C36 * x * (xx - 3.0f * yy);
        dY[15][0] = C36 * (3.0f * xx - 3.0f * yy); dY[15][1] = -6.0f * C36 * x * y;
    }
}

template <int KS, bool OVERWRITE>
__global__ void __launch_bounds__(kThreads) project_bwd_kernel(const Params p) {
    pdl_wait();
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;
    const bool valid = i < p.n;
    bool act = false;
    if (valid) {
        const int2 r = p.radii[i];
        act = (r.x != 0) || (r.y != 0);
    }
    // ---- all loads up front
    float mu[3] = {0, 0, 0}, ls[3] = {0, 0, 0}, o = 0.0f, dcl[3] = {0, 0, 0}, col[3] = {0, 0, 0};
    float da = 0, db = 0, dc = 0, drho = 0;
    float2 dm = make_float2(0, 0);
    float4 q = make_float4(1, 0, 0, 0);
    if (act) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
            mu[c] = __ldg(p.means + 3 * i + c);
            ls[c] = __ldg(p.ls + 3 * i + c);
            dcl[c] = __ldg(p.dcol + 3 * i + c);
            col[c] = __ldg(p.colors + 3 * i + c);
        }
        q = __ldg(p.quats + i);
        o = __ldg(p.ologit + i);
        dm = __ldg(p.dm2 + i);
        da = __ldg(p.dcon + 3 * i);
        db = __ldg(p.dcon + 3 * i + 1);
        dc = __ldg(p.dcon + 3 * i + 2);
        drho = __ldg(p.dop + i);
    }
    const unsigned amask = __ballot_sync(VKS_FULL_MASK, act);
    if (!amask) {
        if (OVERWRITE && valid) {
#pragma unroll
            for (int c = 0; c < 3; c++) { p.dmeans[3 * i + c] = 0.0f; p.dls[3 * i + c] = 0.0f; }
            p.dquats[i] = make_float4(0, 0, 0, 0);
            p.dologit[i] = 0.0f;
            const int64_t nrow = min((int64_t)32, p.n - g0);
            if constexpr (KS > 0 && (3 * KS) % 4 == 0) {
                float4* d4 = reinterpret_cast<float4*>(p.dsh + g0 * 3 * KS);
                for (int j = lane; j < nrow * (3 * KS / 4); j += 32) d4[j] = make_float4(0, 0, 0, 0);
            } else {
                const int S = 3 * p.cfg.sh_coeffs;
                for (int j = lane; j < nrow * S; j += 32) p.dsh[g0 * S + j] = 0.0f;
            }
        }
        return;
    }
    const int K = (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);
    const int S = 3 * p.cfg.sh_coeffs;
    float* buf = nullptr;
    const float* f;
    if constexpr (KS > 0) {
        buf = smem + warp * ShLayout<KS>::kWarpFloats;
        stage_in_async<KS>(p.sh, g0, amask, buf);  // lands while the geometry chain runs
    }
    // ---- geometry (independent of SH; overlaps the staged loads)
    const float* R = p.cam.R;
    const float fx = p.cam.fx, fy = p.cam.fy;
    float tx, ty, tz, Lx, Ly;
    int fovx, fovy;
    fov_decision(p.cam, mu, tx, ty, tz, fovx, fovy, Lx, Ly);
    const float qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    const float iqn = 1.0f / qn;
    const float w = q.x * iqn, x = q.y * iqn, y = q.z * iqn, z = q.w * iqn;
    const float Rq[9] = {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y - w * z), 2.0f * (x * z + w * y),
                         2.0f * (x * y + w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z - w * x),
                         2.0f * (x * z - w * y), 2.0f * (y * z + w * x), 1.0f - 2.0f * (x * x + y * y)};
    const float s[3] = {__expf(ls[0]), __expf(ls[1]), __expf(ls[2])};
    float Mc[9];
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
        for (int c = 0; c < 3; c++)
            Mc[3 * j + c] = (R[3 * j] * Rq[c] + R[3 * j + 1] * Rq[3 + c] + R[3 * j + 2] * Rq[6 + c]) * s[c];
    const float itz = 1.0f / tz, itz2 = itz * itz, itz3 = itz2 * itz;
    const float txc = fovx ? tz * Lx : tx, tyc = fovy ? tz * Ly : ty;
    const float J00 = fx * itz, J02 = -fx * txc * itz2, J11 = fy * itz, J12 = -fy * tyc * itz2;
    float K0[3], K1[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        K0[c] = J00 * Mc[c] + J02 * Mc[6 + c];
        K1[c] = J11 * Mc[3 + c] + J12 * Mc[6 + c];
    }
    const float A = K0[0] * K0[0] + K0[1] * K0[1] + K0[2] * K0[2] + 0.3f;
    const float B = K0[0] * K1[0] + K0[1] * K1[1] + K0[2] * K1[2];
    const float C = K1[0] * K1[0] + K1[1] * K1[1] + K1[2] * K1[2] + 0.3f;
    const float id = 1.0f / (A * C - B * B), id2 = id * id;
    // conic -> (A,B,C), written without the 1/det - AC/det^2 cancellation
    const float dA = (-C * C * da + B * C * db - B * B * dc) * id2;
    const float dB = (2.0f * B * C * da - (A * C + B * B) * db + 2.0f * A * B * dc) * id2;
    const float dC = (-B * B * da + A * B * db - A * A * dc) * id2;
    float dK0[3], dK1[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        dK0[c] = 2.0f * dA * K0[c] + dB * K1[c];
        dK1[c] = dB * K0[c] + 2.0f * dC * K1[c];
    }
    float dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0, dMc[9];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        dJ00 += dK0[c] * Mc[c];
        dJ02 += dK0[c] * Mc[6 + c];
        dJ11 += dK1[c] * Mc[3 + c];
        dJ12 += dK1[c] * Mc[6 + c];
        dMc[c] = J00 * dK0[c];
        dMc[3 + c] = J11 * dK1[c];
        dMc[6 + c] = J02 * dK0[c] + J12 * dK1[c];
    }
    float D[9], dlsv[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float ds = 0.0f;
#pragma unroll
        for (int j = 0; j < 3; j++) {
            const float dM = R[j] * dMc[c] + R[3 + j] * dMc[3 + c] + R[6 + j] * dMc[6 + c];
            ds += dM * Rq[3 * j + c];
            D[3 * j + c] = dM * s[c];
        }
        dlsv[c] = ds * s[c];
    }
    const float dq0 = 2.0f * (-z * D[1] + y * D[2] + z * D[3] - x * D[5] - y * D[6] + x * D[7]);
    const float dq1 = 2.0f * (y * D[1] + z * D[2] + y * D[3] - 2.0f * x * D[4] - w * D[5] + z * D[6] + w * D[7] - 2.0f * x * D[8]);
    const float dq2 = 2.0f * (-2.0f * y * D[0] + x * D[1] + w * D[2] + x * D[3] + z * D[5] - w * D[6] + z * D[7] - 2.0f * y * D[8]);
    const float dq3 = 2.0f * (-2.0f * z * D[0] - w * D[1] + x * D[2] + w * D[3] - 2.0f * z * D[4] + y * D[5] + x * D[6] + y * D[7]);
    const float qd = w * dq0 + x * dq1 + y * dq2 + z * dq3;
    float dt0 = fx * itz * dm.x;
    float dt1 = fy * itz * dm.y;
    float dt2 = -fx * tx * itz2 * dm.x - fy * ty * itz2 * dm.y - fx * itz2 * dJ00 - fy * itz2 * dJ11;
    if (fovx == 0) { dt0 += -fx * itz2 * dJ02; dt2 += 2.0f * fx * tx * itz3 * dJ02; }
    else { dt2 += fx * Lx * itz2 * dJ02; }
    if (fovy == 0) { dt1 += -fy * itz2 * dJ12; dt2 += 2.0f * fy * ty * itz3 * dJ12; }
    else { dt2 += fy * Ly * itz2 * dJ12; }
    const float rho = 1.0f / (1.0f + __expf(-o));
    // ---- SH: colour clamp from the forward's colour (0 <=> raw <= 0), direction gradient, dsh
    float dce[3];
#pragma unroll
    for (int c = 0; c < 3; c++) dce[c] = col[c] > 0.0f ? dcl[c] : 0.0f;
    float cp[3], d[3];
#pragma unroll
    for (int c = 0; c < 3; c++) cp[c] = -(R[c] * p.cam.t[0] + R[3 + c] * p.cam.t[1] + R[6 + c] * p.cam.t[2]);
#pragma unroll
    for (int c = 0; c < 3; c++) d[c] = mu[c] - cp[c];
    const float idl = rsqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    const float dh[3] = {d[0] * idl, d[1] * idl, d[2] * idl};
    float Y[16], dY[16][3];
    sh_basis_and_grad(dh[0], dh[1], dh[2], K, Y, dY);
    if constexpr (KS > 0) {
        cp_async_wait_all();
        __syncwarp();
        f = buf + lane * ShLayout<KS>::SP;
    } else {
        f = p.sh + (int64_t)S * i;
    }
    float ddh0 = 0, ddh1 = 0, ddh2 = 0;
    if (act) {
#pragma unroll
        for (int l = 1; l < 16; l++) {
            if (l < K) {
                const float g = dce[0] * f[3 * l] + dce[1] * f[3 * l + 1] + dce[2] * f[3 * l + 2];
                ddh0 += g * dY[l][0];
                ddh1 += g * dY[l][1];
                ddh2 += g * dY[l][2];
            }
        }
    }
    if constexpr (KS > 0) {
        __syncwarp();
        if (!OVERWRITE) stage_in<KS>(p.dsh, g0, amask, buf);
        __syncwarp();
        float* dfp = buf + lane * ShLayout<KS>::SP;
        if (act) {
#pragma unroll
            for (int l = 0; l < KS; l++) {
                const float yl = l < K ? Y[l] : 0.0f;
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    if (OVERWRITE) dfp[3 * l + c] = yl * dce[c];
                    else dfp[3 * l + c] += yl * dce[c];
                }
            }
        } else if (OVERWRITE && valid) {
#pragma unroll
            for (int j = 0; j < 3 * KS; j++) dfp[j] = 0.0f;
        }
        __syncwarp();
        const unsigned omask = OVERWRITE ? __ballot_sync(VKS_FULL_MASK, valid) : amask;
        stage_out<KS>(p.dsh, g0, omask, buf);
    } else {
        if (act || (OVERWRITE && valid)) {
            float* dfp = p.dsh + (int64_t)S * i;
            for (int l = 0; l < S / 3; l++) {
                const float yl = (act && l < K) ? Y[l] : 0.0f;
                for (int c = 0; c < 3; c++) {
                    if (OVERWRITE) dfp[3 * l + c] = yl * dce[c];
                    else dfp[3 * l + c] += yl * dce[c];
                }
            }
        }
    }
    if (!valid) return;
    if (!act) {
        if (OVERWRITE) {
#pragma unroll
            for (int c = 0; c < 3; c++) { p.dmeans[3 * i + c] = 0.0f; p.dls[3 * i + c] = 0.0f; }
            p.dquats[i] = make_float4(0, 0, 0, 0);
            p.dologit[i] = 0.0f;
        }
        return;
    }
    const float pr = dh[0] * ddh0 + dh[1] * ddh1 + dh[2] * ddh2;
    const float dmu0 = (ddh0 - dh[0] * pr) * idl + R[0] * dt0 + R[3] * dt1 + R[6] * dt2;
    const float dmu1 = (ddh1 - dh[1] * pr) * idl + R[1] * dt0 + R[4] * dt1 + R[7] * dt2;
    const float dmu2 = (ddh2 - dh[2] * pr) * idl + R[2] * dt0 + R[5] * dt1 + R[8] * dt2;
    const float dlo = drho * rho * (1.0f - rho);
    const float4 dqv = make_float4((dq0 - w * qd) * iqn, (dq1 - x * qd) * iqn, (dq2 - y * qd) * iqn,
                                   (dq3 - z * qd) * iqn);
    if (OVERWRITE) {
        p.dmeans[3 * i] = dmu0; p.dmeans[3 * i + 1] = dmu1; p.dmeans[3 * i + 2] = dmu2;
        p.dls[3 * i] = dlsv[0]; p.dls[3 * i + 1] = dlsv[1]; p.dls[3 * i + 2] = dlsv[2];
        p.dquats[i] = dqv;
        p.dologit[i] = dlo;
    } else {
        p.dmeans[3 * i] += dmu0; p.dmeans[3 * i + 1] += dmu1; p.dmeans[3 * i + 2] += dmu2;
        p.dls[3 * i] += dlsv[0]; p.dls[3 * i + 1] += dlsv[1]; p.dls[3 * i + 2] += dlsv[2];
        float4 o4 = p.dquats[i];
        o4.x += dqv.x; o4.y += dqv.y; o4.z += dqv.z; o4.w += dqv.w;
        p.dquats[i] = o4;
        p.dologit[i] += dlo;
    }
}

// ------------------------------------------------------------------------------------------
// Batched projection backward: the parameter gradients of V views summed in one pass.  Every
// Gaussian's parameters and SH row are read once and its gradient row written once (instead of
// V read-modify-writes of the 1.37 GB gradient buffer); per view only that view's 2D gradients,
// colour and radii are read.  Each view's chain is the single-view kernel's; only the summation
// over views is regrouped: linear view-independent factors (ρ(1-ρ), s, the quaternion-norm
// projection) are applied once to the summed raw gradients.
constexpr int kMaxBatchViews = 16;

struct ViewIn {
    vks_camera cam;
    CamConst cc;  // FOV limits (pinned, host-computed exactly as the forward) and camera centre
    const float* colors;
    const int2* radii;
    const float2* dm2;
    const float* dcon;
    const float* dcol;
    const float* dop;
};

struct BatchParams {
    vks_config cfg;
    int64_t n;
    int nv;
    const float* __restrict__ means;
    const float* __restrict__ ls;
    const float4* __restrict__ quats;
    const float* __restrict__ ologit;
    const float* __restrict__ sh;
    float* __restrict__ dmeans;
    float* __restrict__ dls;
    float4* __restrict__ dquats;
    float* __restrict__ dologit;
    float* __restrict__ dsh;
    ViewIn v[kMaxBatchViews];
};

// SH rows readable / writable as float4 in shared memory
template <int KS>
constexpr bool vec4_rows() {
    if constexpr (KS > 0) return (3 * KS) % 4 == 0 && ShLayout<KS>::SP % 4 == 0;
    return false;
}

// one view's per-Gaussian inputs (prefetched one view ahead)
struct ViewLoads {
    float dcl[3], col[3], da, db, dc, dr;
    float2 dm;
};

__device__ __forceinline__ void load_view(const ViewIn& V, int64_t i, bool on, ViewLoads& L) {
    if (on) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
            L.dcl[c] = __ldg(V.dcol + 3 * i + c);
            L.col[c] = __ldg(V.colors + 3 * i + c);
        }
        L.dm = __ldg(V.dm2 + i);
        L.da = __ldg(V.dcon + 3 * i);
        L.db = __ldg(V.dcon + 3 * i + 1);
        L.dc = __ldg(V.dcon + 3 * i + 2);
        L.dr = __ldg(V.dop + i);
    } else {
#pragma unroll
        for (int c = 0; c < 3; c++) L.dcl[c] = L.col[c] = 0.0f;
        L.dm = make_float2(0.0f, 0.0f);
        L.da = L.db = L.dc = L.dr = 0.0f;
    }
}

template <int KS, bool OVERWRITE, bool KFULL>
__global__ void __launch_bounds__(kThreads) project_bwd_batch_kernel(const BatchParams p) {
    pdl_wait();
    extern __shared__ float smem[];
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int64_t g0 = i - lane;
    const bool valid = i < p.n;
    // the SH rows (staged once) and the parameters are requested with the radii, for every row in
    // range (nearly every Gaussian is seen by some view of a batch): one DRAM round trip instead
    // of radii -> visibility -> parameters
    const unsigned vmask = __ballot_sync(VKS_FULL_MASK, valid);
    float* shv = nullptr;
    if constexpr (KS > 0) {
        shv = smem + warp * 2 * ShLayout<KS>::kWarpFloats;
        if (vmask) stage_in_async<KS>(p.sh, g0, vmask, shv);
    }
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
    // visibility in each view (radii != 0)
    unsigned vis = 0;
    if (valid) {
        for (int v = 0; v < p.nv; v++) {
            const int2 r = __ldg(p.v[v].radii + i);
            if (r.x != 0 || r.y != 0) vis |= 1u << v;
        }
    }
    const bool act = vis != 0;
    const unsigned amask = __ballot_sync(VKS_FULL_MASK, act);
    const int K = KFULL ? KS : (p.cfg.sh_degree + 1) * (p.cfg.sh_degree + 1);  // KFULL: compile-time
    const int S = 3 * p.cfg.sh_coeffs;
    // shared memory per warp: the SH rows and the dSH accumulator rows
    float* acc = nullptr;
    if constexpr (KS > 0) {
        float* accw = shv + ShLayout<KS>::kWarpFloats;
        acc = accw + lane * ShLayout<KS>::SP;
#pragma unroll
        for (int j = 0; j < 3 * KS; j++) acc[j] = 0.0f;
    } else if (valid && OVERWRITE) {
        for (int j = 0; j < S; j++) p.dsh[(int64_t)S * i + j] = 0.0f;
    }
    float dmu[3] = {0, 0, 0}, dsv[3] = {0, 0, 0}, dqr[4] = {0, 0, 0, 0}, drho = 0.0f;
    if (amask) {
        // view-independent part of the chain
        const float qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
        const float iqn = 1.0f / qn;
        const float w = q.x * iqn, x = q.y * iqn, y = q.z * iqn, z = q.w * iqn;
        const float Rq[9] = {1.0f - 2.0f * (y * y + z * z), 2.0f * (x * y - w * z), 2.0f * (x * z + w * y),
                             2.0f * (x * y + w * z), 1.0f - 2.0f * (x * x + z * z), 2.0f * (y * z - w * x),
                             2.0f * (x * z - w * y), 2.0f * (y * z + w * x), 1.0f - 2.0f * (x * x + y * y)};
        const float s[3] = {__expf(ls[0]), __expf(ls[1]), __expf(ls[2])};
        float Ms[9];  // Rq diag(s): view-independent, so each view's Mc = R Ms is 27 multiply-adds
#pragma unroll
        for (int j = 0; j < 9; j++) Ms[j] = Rq[j] * s[j % 3];
        const float* f;
        if constexpr (KS > 0) {
            cp_async_wait_all();
            __syncwarp();
            f = shv + lane * ShLayout<KS>::SP;
        } else {
            f = p.sh + (int64_t)S * i;
        }
        ViewLoads cur;
        load_view(p.v[0], i, vis & 1u, cur);
        for (int v = 0; v < p.nv; v++) {
            const bool on = (vis >> v) & 1u;
            ViewLoads nxt;  // next view's inputs in flight while this view computes
            if (v + 1 < p.nv) load_view(p.v[v + 1], i, (vis >> (v + 1)) & 1u, nxt);
            if (__any_sync(VKS_FULL_MASK, on)) {
                const ViewIn& V = p.v[v];
                const float* R = V.cam.R;
                const float fx = V.cam.fx, fy = V.cam.fy;
                // FOV decision of the forward (steps 1, 6), bit-identical: pinned t, tx/tz vs limits
                const float tx = __fadd_rn(pdot3(R + 0, mu), V.cam.t[0]);
                const float ty = __fadd_rn(pdot3(R + 3, mu), V.cam.t[1]);
                const float tz = __fadd_rn(pdot3(R + 6, mu), V.cam.t[2]);
                // the comparisons need the IEEE-rounded tx/tz only near a limit: an approximate ratio
                // (relative error < 1e-6) decides every case further than 1e-5 from the limits
                const float rtz = __fdividef(1.0f, tz);
                float rxz = tx * rtz, ryz = ty * rtz;
                const bool nearx = fabsf(rxz - V.cc.lxp) <= 1e-5f * fabsf(V.cc.lxp) + 1e-30f ||
                                   fabsf(rxz + V.cc.lxn) <= 1e-5f * fabsf(V.cc.lxn) + 1e-30f;
                const bool neary = fabsf(ryz - V.cc.lyp) <= 1e-5f * fabsf(V.cc.lyp) + 1e-30f ||
                                   fabsf(ryz + V.cc.lyn) <= 1e-5f * fabsf(V.cc.lyn) + 1e-30f;
                if (nearx) rxz = __fdiv_rn(tx, tz);
                if (neary) ryz = __fdiv_rn(ty, tz);
                int fovx = 0, fovy = 0;
                float Lx = 0.0f, Ly = 0.0f;
                if (rxz > V.cc.lxp) { fovx = 1; Lx = V.cc.lxp; } else if (rxz < -V.cc.lxn) { fovx = -1; Lx = -V.cc.lxn; }
                if (ryz > V.cc.lyp) { fovy = 1; Ly = V.cc.lyp; } else if (ryz < -V.cc.lyn) { fovy = -1; Ly = -V.cc.lyn; }
                float Mc[9];
#pragma unroll
                for (int j = 0; j < 3; j++)
#pragma unroll
                    for (int c = 0; c < 3; c++)
                        Mc[3 * j + c] = R[3 * j] * Ms[c] + R[3 * j + 1] * Ms[3 + c] + R[3 * j + 2] * Ms[6 + c];
                const float itz = 1.0f / tz, itz2 = itz * itz, itz3 = itz2 * itz;
                const float txc = fovx ? tz * Lx : tx, tyc = fovy ? tz * Ly : ty;
                const float J00 = fx * itz, J02 = -fx * txc * itz2, J11 = fy * itz, J12 = -fy * tyc * itz2;
                float K0[3], K1[3];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    K0[c] = J00 * Mc[c] + J02 * Mc[6 + c];
                    K1[c] = J11 * Mc[3 + c] + J12 * Mc[6 + c];
                }
                const float A = K0[0] * K0[0] + K0[1] * K0[1] + K0[2] * K0[2] + 0.3f;
                const float B = K0[0] * K1[0] + K0[1] * K1[1] + K0[2] * K1[2];
                const float C = K1[0] * K1[0] + K1[1] * K1[1] + K1[2] * K1[2] + 0.3f;
                const float id = 1.0f / (A * C - B * B), id2 = id * id;
                const float da = cur.da, db = cur.db, dc = cur.dc;
                const float dA = (-C * C * da + B * C * db - B * B * dc) * id2;
                const float dB = (2.0f * B * C * da - (A * C + B * B) * db + 2.0f * A * B * dc) * id2;
                const float dC = (-B * B * da + A * B * db - A * A * dc) * id2;
                float dK0[3], dK1[3];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    dK0[c] = 2.0f * dA * K0[c] + dB * K1[c];
                    dK1[c] = dB * K0[c] + 2.0f * dC * K1[c];
                }
                float dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0, dMc[9];
#pragma unroll
                for (int c = 0; c < 3; c++) {
                    dJ00 += dK0[c] * Mc[c];
                    dJ02 += dK0[c] * Mc[6 + c];
                    dJ11 += dK1[c] * Mc[3 + c];
                    dJ12 += dK1[c] * Mc[6 + c];
                    dMc[c] = J00 * dK0[c];
                    dMc[3 + c] = J11 * dK1[c];
                    dMc[6 + c] = J02 * dK0[c] + J12 * dK1[c];
                }
                float D[9];
#pragma unroll
                for (int c = 0; c < 3; c++) {
#pragma unroll
                    for (int j = 0; j < 3; j++) {
                        const float dM = R[j] * dMc[c] + R[3 + j] * dMc[3 + c] + R[6 + j] * dMc[6 + c];
                        dsv[c] += dM * Rq[3 * j + c];  // x s[c] once at the end
                        D[3 * j + c] = dM * s[c];
                    }
                }
                dqr[0] += 2.0f * (-z * D[1] + y * D[2] + z * D[3] - x * D[5] - y * D[6] + x * D[7]);
                dqr[1] += 2.0f * (y * D[1] + z * D[2] + y * D[3] - 2.0f * x * D[4] - w * D[5] + z * D[6] +
                                  w * D[7] - 2.0f * x * D[8]);
                dqr[2] += 2.0f * (-2.0f * y * D[0] + x * D[1] + w * D[2] + x * D[3] + z * D[5] - w * D[6] +
                                  z * D[7] - 2.0f * y * D[8]);
                dqr[3] += 2.0f * (-2.0f * z * D[0] - w * D[1] + x * D[2] + w * D[3] - 2.0f * z * D[4] +
                                  y * D[5] + x * D[6] + y * D[7]);
                const float2 dm = cur.dm;
                float dt0 = fx * itz * dm.x;
                float dt1 = fy * itz * dm.y;
                float dt2 = -fx * tx * itz2 * dm.x - fy * ty * itz2 * dm.y - fx * itz2 * dJ00 - fy * itz2 * dJ11;
                if (fovx == 0) { dt0 += -fx * itz2 * dJ02; dt2 += 2.0f * fx * tx * itz3 * dJ02; }
                else { dt2 += fx * Lx * itz2 * dJ02; }
                if (fovy == 0) { dt1 += -fy * itz2 * dJ12; dt2 += 2.0f * fy * ty * itz3 * dJ12; }
                else { dt2 += fy * Ly * itz2 * dJ12; }
                drho += cur.dr;
                // SH: colour clamp from the forward's colour, direction gradient, dsh += Y (x) dce
                float dce[3];
#pragma unroll
                for (int c = 0; c < 3; c++) dce[c] = cur.col[c] > 0.0f ? cur.dcl[c] : 0.0f;
                float d[3];
#pragma unroll
                for (int c = 0; c < 3; c++) d[c] = mu[c] - V.cc.cp[c];
                const float idl = rsqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                const float dh[3] = {d[0] * idl, d[1] * idl, d[2] * idl};
                float Y[16], dY[16][3];
                sh_basis_and_grad(dh[0], dh[1], dh[2], K, Y, dY);
                if (on) {
                    float ddh0 = 0, ddh1 = 0, ddh2 = 0;
                    if constexpr (vec4_rows<KS>()) {
                        // 128-bit shared-memory reads of the SH row and read-modify-writes of the
                        // dSH row; element e = 3 l + ch
                        const float4* f4 = reinterpret_cast<const float4*>(f);
                        float4* a4 = reinterpret_cast<float4*>(acc);
                        float g = 0.0f;  // <dce, f_l> of the current l (elements arrive in e order)
#pragma unroll
                        for (int m = 0; m < 3 * KS / 4; m++) {
                            const float4 fv = f4[m];
                            const float fe[4] = {fv.x, fv.y, fv.z, fv.w};
                            float4 av = a4[m];
                            float ae[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                const int e = 4 * m + t, l = e / 3, c = e % 3;
                                if (l < K) {
                                    g += dce[c] * fe[t];
                                    ae[t] += Y[l] * dce[c];
                                    if (c == 2) {
                                        if (l > 0) {
                                            ddh0 += g * dY[l][0];
                                            ddh1 += g * dY[l][1];
                                            ddh2 += g * dY[l][2];
                                        }
                                        g = 0.0f;
                                    }
                                }
                            }
                            a4[m] = make_float4(ae[0], ae[1], ae[2], ae[3]);
                        }
                    } else {
#pragma unroll
                        for (int l = 1; l < 16; l++) {
                            if (l < K) {
                                const float g = dce[0] * f[3 * l] + dce[1] * f[3 * l + 1] + dce[2] * f[3 * l + 2];
                                ddh0 += g * dY[l][0];
                                ddh1 += g * dY[l][1];
                                ddh2 += g * dY[l][2];
                            }
                        }
                    }
                    if constexpr (vec4_rows<KS>()) {
                        // (accumulated above)
                    } else if constexpr (KS > 0) {
#pragma unroll
                        for (int l = 0; l < KS; l++) {
                            if (l < K) {
#pragma unroll
                                for (int c = 0; c < 3; c++) acc[3 * l + c] += Y[l] * dce[c];
                            }
                        }
                    } else {
                        for (int l = 0; l < K; l++)
                            for (int c = 0; c < 3; c++) p.dsh[(int64_t)S * i + 3 * l + c] += Y[l] * dce[c];
                    }
                    const float pr = dh[0] * ddh0 + dh[1] * ddh1 + dh[2] * ddh2;
                    dmu[0] += (ddh0 - dh[0] * pr) * idl + R[0] * dt0 + R[3] * dt1 + R[6] * dt2;
                    dmu[1] += (ddh1 - dh[1] * pr) * idl + R[1] * dt0 + R[4] * dt1 + R[7] * dt2;
                    dmu[2] += (ddh2 - dh[2] * pr) * idl + R[2] * dt0 + R[5] * dt1 + R[8] * dt2;
                }
            }
            if (v + 1 < p.nv) cur = nxt;
        }
        // view-independent factors applied once to the summed raw gradients
        const float rho = 1.0f / (1.0f + __expf(-o));
        drho *= rho * (1.0f - rho);
#pragma unroll
        for (int c = 0; c < 3; c++) dsv[c] *= s[c];
        const float qd = w * dqr[0] + x * dqr[1] + y * dqr[2] + z * dqr[3];
        dqr[0] = (dqr[0] - w * qd) * iqn;
        dqr[1] = (dqr[1] - x * qd) * iqn;
        dqr[2] = (dqr[2] - y * qd) * iqn;
        dqr[3] = (dqr[3] - z * qd) * iqn;
    }
    // ---- outputs: every row under OVERWRITE (zeros where no view sees the Gaussian), else the
    // rows some view sees
    if constexpr (KS > 0) {
        float* accw = smem + warp * 2 * ShLayout<KS>::kWarpFloats + ShLayout<KS>::kWarpFloats;
        if (!OVERWRITE && act) {  // += onto the old row
            const float* src = p.dsh + (int64_t)3 * KS * i;
#pragma unroll
            for (int j = 0; j < 3 * KS; j++) acc[j] += src[j];
        }
        __syncwarp();
        const unsigned omask = OVERWRITE ? __ballot_sync(VKS_FULL_MASK, valid) : amask;
        stage_out<KS>(p.dsh, g0, omask, accw);
    }
    if (!valid || (!OVERWRITE && !act)) return;
    if (OVERWRITE) {
        p.dmeans[3 * i] = dmu[0]; p.dmeans[3 * i + 1] = dmu[1]; p.dmeans[3 * i + 2] = dmu[2];
        p.dls[3 * i] = dsv[0]; p.dls[3 * i + 1] = dsv[1]; p.dls[3 * i + 2] = dsv[2];
        p.dquats[i] = make_float4(dqr[0], dqr[1], dqr[2], dqr[3]);
        p.dologit[i] = drho;
    } else {
        p.dmeans[3 * i] += dmu[0]; p.dmeans[3 * i + 1] += dmu[1]; p.dmeans[3 * i + 2] += dmu[2];
        p.dls[3 * i] += dsv[0]; p.dls[3 * i + 1] += dsv[1]; p.dls[3 * i + 2] += dsv[2];
        float4 o4 = p.dquats[i];
        o4.x += dqr[0]; o4.y += dqr[1]; o4.z += dqr[2]; o4.w += dqr[3];
        p.dquats[i] = o4;
        p.dologit[i] += drho;
    }
}

template <int KS, bool OW, bool KF>
int launch_batch_t(const BatchParams& p, cudaStream_t s) {
    size_t sm = 0;
    if constexpr (KS > 0) sm = sizeof(float) * kWarps * 2 * ShLayout<KS>::kWarpFloats;
    if (sm > 48 * 1024 &&
        cudaFuncSetAttribute(project_bwd_batch_kernel<KS, OW, KF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess)
        return VKS_ERR_CUDA;
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    launch_k(project_bwd_batch_kernel<KS, OW, KF>, blocks, kThreads, sm, s, p);
    return LaunchCheck::check();
}

template <int KS>
int launch_batch_k(const BatchParams& p, cudaStream_t s) {
    const bool ow = p.cfg.flags & VKS_FLAG_GRAD_OVERWRITE;
    if (KS == 16 && p.cfg.sh_degree == 3)  // every stored coefficient used: K known at compile time
        return ow ? launch_batch_t<KS, true, true>(p, s) : launch_batch_t<KS, false, true>(p, s);
    return ow ? launch_batch_t<KS, true, false>(p, s) : launch_batch_t<KS, false, false>(p, s);
}

template <int KS, bool OW>
int launch_t(const Params& p, cudaStream_t s) {
    size_t sm = 0;
    if constexpr (KS > 0) sm = sizeof(float) * kWarps * ShLayout<KS>::kWarpFloats;
    if (sm > 48 * 1024 &&
        cudaFuncSetAttribute(project_bwd_kernel<KS, OW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return VKS_ERR_CUDA;
    const unsigned blocks = (unsigned)((p.n + kThreads - 1) / kThreads);
    launch_k(project_bwd_kernel<KS, OW>, blocks, kThreads, sm, s, p);
    return LaunchCheck::check();
}

template <int KS>
int launch_bwd_k(const Params& p, cudaStream_t s) {
    return (p.cfg.flags & VKS_FLAG_GRAD_OVERWRITE) ? launch_t<KS, true>(p, s) : launch_t<KS, false>(p, s);
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

}  // namespace

int launch_project_bwd(const vks_config& cfg, const vks_camera& cam, int64_t n, const float* means,
                       const float* log_scales, const float* quats, const float* opacity_logits,
                       const float* sh, const float* colors, const int32_t* radii, const float* dmeans2d,
                       const float* dconics, const float* dcolors, const float* dopacities, float* dmeans,
                       float* dlog_scales, float* dquats, float* dopacity_logits, float* dsh, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    Params p{};
    p.cam = cam; p.cfg = cfg; p.n = n;
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh; p.colors = colors;
    p.radii = reinterpret_cast<const int2*>(radii);
    p.dm2 = reinterpret_cast<const float2*>(dmeans2d); p.dcon = dconics; p.dcol = dcolors;
    p.dop = dopacities; p.dmeans = dmeans; p.dls = dlog_scales;
    p.dquats = reinterpret_cast<float4*>(dquats); p.dologit = dopacity_logits; p.dsh = dsh;
    const bool al = aligned16(sh) && aligned16(dsh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_bwd_k<16>(p, s) : launch_bwd_k<0>(p, s);
        case 9: return launch_bwd_k<9>(p, s);
        case 4: return al ? launch_bwd_k<4>(p, s) : launch_bwd_k<0>(p, s);
        case 1: return launch_bwd_k<1>(p, s);
        default: return launch_bwd_k<0>(p, s);
    }
}

int launch_project_bwd_batch(const vks_config& cfg, int32_t n_views, const vks_camera* cams, int64_t n,
                             const float* means, const float* log_scales, const float* quats,
                             const float* opacity_logits, const float* sh, const float* const* colors,
                             const int32_t* const* radii, const float* const* dmeans2d, const float* const* dconics,
                             const float* const* dcolors, const float* const* dopacities, float* dmeans,
                             float* dlog_scales, float* dquats, float* dopacity_logits, float* dsh, cudaStream_t s) {
    if (n == 0) return VKS_OK;
    if (n_views < 1 || n_views > kMaxBatchViews) return VKS_ERR_INVALID_ARG;
    BatchParams p{};
    p.cfg = cfg; p.n = n; p.nv = n_views;
    p.means = means; p.ls = log_scales; p.quats = reinterpret_cast<const float4*>(quats);
    p.ologit = opacity_logits; p.sh = sh;
    p.dmeans = dmeans; p.dls = dlog_scales; p.dquats = reinterpret_cast<float4*>(dquats);
    p.dologit = dopacity_logits; p.dsh = dsh;
    for (int v = 0; v < n_views; v++) {
        ViewIn& V = p.v[v];
        V.cam = cams[v];
        V.cc = cam_const(cams[v]);
        V.colors = colors[v];
        V.radii = reinterpret_cast<const int2*>(radii[v]);
        V.dm2 = reinterpret_cast<const float2*>(dmeans2d[v]);
        V.dcon = dconics[v];
        V.dcol = dcolors[v];
        V.dop = dopacities[v];
    }
    const bool al = aligned16(sh) && aligned16(dsh);
    switch (cfg.sh_coeffs) {
        case 16: return al ? launch_batch_k<16>(p, s) : launch_batch_k<0>(p, s);
        case 9: return launch_batch_k<9>(p, s);
        case 4: return al ? launch_batch_k<4>(p, s) : launch_batch_k<0>(p, s);
        case 1: return launch_batch_k<1>(p, s);
        default: return launch_batch_k<0>(p, s);
    }
}

}  // namespace vks
