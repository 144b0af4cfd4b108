// loss.cu — SURVEY §8(f) row f2: the loss gradient before the path ("Loss Gradient", PAPER P:74;
// SPEC S:178-186, SSIM definition); include/vks.h vks_loss_grad.
//
//   loss = (1 - lambda) mean|r - t| + lambda (1 - SSIM),   SSIM = mean over channels and valid
//   11x11 windows (Gaussian, sigma 1.5) of S = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)
//   (sx2 + sy2 + C2)).
// Three kernels: ssim_fwd_kernel (per 32x32 tile of window centres and channel: the separable
// window sums of x, y, x^2, y^2, xy — horizontal into shared memory, then vertical — and S with
// its partials dS/dmx, dS/dE[x^2], dS/dE[xy] per centre), ssim_bwd_kernel (per 32x32 pixel tile
// and channel: the transposed separable window sums of the three partial maps, the L1
// subgradient, dL/dr), loss_finalize_kernel (one block: the block partial sums -> loss,
// deterministic).  The window sums, S, the partials and the transposed pass are fp64: the
// variances E[x^2] - mx^2 cancel down to ~C2 = 9e-4, and fp32 statistics would put up to ~1e-3
// relative error into the gradient.  Each thread produces four adjacent outputs of a pass from a
// sliding register window (14 inputs for 4 outputs of an 11-tap pass: 3.5 shared-memory loads and
// products per output instead of 11), so the kernels are bound by the fp64 FMAs, not by 64-bit
// shared-memory traffic (round 1: one output per thread, 0.17 ms for 1237x822, mio-throttled).
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kT = 32;                        // tile of centres (fwd) / pixels (bwd), square
constexpr int kR = 5, kWin = 11;                  // window radius / width
constexpr int kI = kT + 2 * kR;                   // tile + halo (42)
constexpr int kIP = kI + 3;                       // float row pitch 45: the 4 rows x 8 column groups of
                                                  // a warp's sliding-window loads hit 32 distinct banks
#ifndef VKS_LOSS_RUN
#define VKS_LOSS_RUN 4
#endif
#ifndef VKS_LOSS_THREADS
#define VKS_LOSS_THREADS 512  // 2 blocks x 16 warps per SM (70-75 KB of shared memory per block):
#endif                        // 0.153 ms vs 0.159 with 256 threads, 0.167 with 2 outputs per thread
constexpr int kRun = VKS_LOSS_RUN;                // outputs per thread and pass
constexpr int kLossThreads = VKS_LOSS_THREADS;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;
#ifndef VKS_LOSS_MAP_T
#define VKS_LOSS_MAP_T double  // storage type of the partial maps between the two kernels
#endif
typedef VKS_LOSS_MAP_T map_t;

struct Gauss {
    double g[kWin];
};

Gauss window() {
    Gauss w;
    double s = 0.0;
    for (int i = 0; i < kWin; i++) {
        const double d = (double)(i - kR);
        w.g[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        s += w.g[i];
    }
    for (int i = 0; i < kWin; i++) w.g[i] /= s;
    return w;
}

// dynamic shared memory of the two kernels.  64-bit rows are padded to an odd pitch: a warp
// stores four rows x eight runs (elements 4g + o of each row), and with pitch 33 / 43 doubles
// those 32 stores / loads spread over all 16 bank pairs (two wavefronts, the minimum for 256 B)
constexpr int kHP = kT + 1, kMP = kI + 1;
struct FwdSmem {
    float sx[kI][kIP], sy[kI][kIP];   // input tile + halo
    double hs[5][kI][kHP];            // horizontal window sums of x, y, x^2, y^2, xy
    double red[kLossThreads / 32];
};
struct BwdSmem {
    double sm[3][kI][kMP];            // partial maps of the centres that reach the tile
    double hs[3][kI][kHP];            // their horizontal transposed sums
    double red[kLossThreads / 32];
};

// block (x: centre tile, y: centre tile, z: channel).  Centre p's window covers pixels p .. p+10.
__global__ void __launch_bounds__(kLossThreads, kLossThreads >= 512 ? 2 : 3) ssim_fwd_kernel(int W, int H, const float* __restrict__ render,
                                                               const float* __restrict__ target, const Gauss w,
                                                               map_t* __restrict__ A, map_t* __restrict__ B,
                                                               map_t* __restrict__ Cm, double* __restrict__ s_part) {
    extern __shared__ __align__(16) unsigned char loss_smem[];
    FwdSmem& S = *reinterpret_cast<FwdSmem*>(loss_smem);
    const int tid = threadIdx.x, c = blockIdx.z;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const int cx0 = blockIdx.x * kT, cy0 = blockIdx.y * kT;
    {   // every load of the tile in flight before the first shared-memory store
        constexpr int kIt = (kI * kI + kLossThreads - 1) / kLossThreads;
        float vx[kIt], vy[kIt];
#pragma unroll
        for (int it = 0; it < kIt; it++) {
            const int k = tid + it * kLossThreads;
            const int r = k / kI, q = k % kI;
            const int py = cy0 + r, px = cx0 + q;
            const bool in = k < kI * kI && px < W && py < H;
            const size_t o = ((size_t)py * W + px) * 3 + c;
            vx[it] = in ? __ldg(render + o) : 0.0f;
            vy[it] = in ? __ldg(target + o) : 0.0f;
        }
#pragma unroll
        for (int it = 0; it < kIt; it++) {
            const int k = tid + it * kLossThreads;
            if (k < kI * kI) {
                S.sx[k / kI][k % kI] = vx[it];
                S.sy[k / kI][k % kI] = vy[it];
            }
        }
    }
    __syncthreads();
    // horizontal sums: item = (row, run of 4 centre columns); inputs j0 .. j0 + 13 of the row
    for (int k = tid; k < kI * (kT / kRun); k += kLossThreads) {
        const int r = k / (kT / kRun), j0 = kRun * (k % (kT / kRun));
        double acc[kRun][5];
#pragma unroll
        for (int o = 0; o < kRun; o++)
#pragma unroll
            for (int q = 0; q < 5; q++) acc[o][q] = 0.0;
#pragma unroll
        for (int i = 0; i < kWin + kRun - 1; i++) {
            const double x = S.sx[r][j0 + i], y = S.sy[r][j0 + i];
            const double xx = x * x, yy = y * y, xy = x * y;
#pragma unroll
            for (int o = 0; o < kRun; o++) {
                const int t = i - o;  // tap of output o
                if (t >= 0 && t < kWin) {
                    const double g = w.g[t];
                    acc[o][0] += g * x;
                    acc[o][1] += g * y;
                    acc[o][2] += g * xx;
                    acc[o][3] += g * yy;
                    acc[o][4] += g * xy;
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kRun; o++)
#pragma unroll
            for (int q = 0; q < 5; q++) S.hs[q][r][j0 + o] = acc[o][q];
    }
    __syncthreads();
    // vertical sums -> S and partials: item = (column, run of 4 centre rows); rows i0 .. i0 + 13
    double ssum = 0.0;
    for (int k = tid; k < kT * (kT / kRun); k += kLossThreads) {
        const int j = k % kT, i0 = kRun * (k / kT);
        double st[kRun][5];
#pragma unroll
        for (int o = 0; o < kRun; o++)
#pragma unroll
            for (int q = 0; q < 5; q++) st[o][q] = 0.0;
#pragma unroll
        for (int i = 0; i < kWin + kRun - 1; i++) {
            double hv[5];
#pragma unroll
            for (int q = 0; q < 5; q++) hv[q] = S.hs[q][i0 + i][j];
#pragma unroll
            for (int o = 0; o < kRun; o++) {
                const int t = i - o;
                if (t >= 0 && t < kWin) {
#pragma unroll
                    for (int q = 0; q < 5; q++) st[o][q] += w.g[t] * hv[q];
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kRun; o++) {
            const int px = cx0 + j, py = cy0 + i0 + o;
            if (px >= Wv || py >= Hv) continue;
            const double mx = st[o][0], my = st[o][1], exx = st[o][2], eyy = st[o][3], exy = st[o][4];
            const double sx2 = exx - mx * mx, sy2 = eyy - my * my, sxy = exy - mx * my;
            const double l1 = 2 * mx * my + kC1, l2 = mx * mx + my * my + kC1;
            const double c1 = 2 * sxy + kC2, c2 = sx2 + sy2 + kC2;
            const double inv = 1.0 / (l2 * c2);  // the one fp64 division: 1/l2 = c2 inv, 1/c2 = l2 inv
            const double Sv = l1 * c1 * inv;
            const double dB = -Sv * (l2 * inv), dC = 2.0 * l1 * inv;
            const double dA = 2.0 * my * c1 * inv - 2.0 * mx * Sv * (c2 * inv) - 2.0 * mx * dB - my * dC;
            const size_t off = ((size_t)c * Hv + py) * Wv + px;
            A[off] = (map_t)dA;
            B[off] = (map_t)dB;
            Cm[off] = (map_t)dC;
            ssum += Sv;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ssum += __shfl_xor_sync(VKS_FULL_MASK, ssum, o);
    if ((tid & 31) == 0) S.red[tid >> 5] = ssum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) t += S.red[q];
        s_part[((size_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

// block (x, y: pixel tile, z: channel).  dL_q = (1 - lambda) sign(r - t) / (3 N)
//   - lambda / (3 Nv) sum_{centres p: q in window(p)} w(q - p) (A_p + 2 B_p r_q + C_p t_q)
__global__ void __launch_bounds__(kLossThreads, kLossThreads >= 512 ? 2 : 3) ssim_bwd_kernel(int W, int H, float lambda, const float* __restrict__ render,
                                                               const float* __restrict__ target, const Gauss w,
                                                               const map_t* __restrict__ A, const map_t* __restrict__ B,
                                                               const map_t* __restrict__ Cm, float* __restrict__ dL,
                                                               double* __restrict__ l1_part) {
    extern __shared__ __align__(16) unsigned char loss_smem[];
    BwdSmem& S = *reinterpret_cast<BwdSmem*>(loss_smem);
    const int tid = threadIdx.x, c = blockIdx.z;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
    const int qx0 = blockIdx.x * kT, qy0 = blockIdx.y * kT;
    const double inv_n = 1.0 / (3.0 * (double)W * (double)H);
    const double k_ssim = ssim ? -(double)lambda / (3.0 * (double)Wv * (double)Hv) : 0.0;
    double l1 = 0.0;
    if (ssim) {
        // centres p = q - i (i in [0, 10]) for q in the tile: rows qy0-10 .. qy0+31, same columns
        // every load of the region in flight before the first shared-memory store (in halves:
        // 3 x 4 doubles in registers per thread)
        constexpr int kIt = (kI * kI + kLossThreads - 1) / kLossThreads;  // 7
        constexpr int kHalf = (kIt + 1) / 2;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            double va[kHalf], vb[kHalf], vc[kHalf];
#pragma unroll
            for (int u = 0; u < kHalf; u++) {
                const int k = tid + (h * kHalf + u) * kLossThreads;
                const int r = k / kI, sc = k % kI;
                const int py = qy0 - 2 * kR + r, px = qx0 - 2 * kR + sc;
                const bool in = k < kI * kI && px >= 0 && py >= 0 && px < Wv && py < Hv;
                const size_t o = ((size_t)c * Hv + py) * Wv + px;
                va[u] = in ? (double)__ldg(A + o) : 0.0;
                vb[u] = in ? (double)__ldg(B + o) : 0.0;
                vc[u] = in ? (double)__ldg(Cm + o) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kHalf; u++) {
                const int k = tid + (h * kHalf + u) * kLossThreads;
                if (k < kI * kI) {
                    S.sm[0][k / kI][k % kI] = va[u];
                    S.sm[1][k / kI][k % kI] = vb[u];
                    S.sm[2][k / kI][k % kI] = vc[u];
                }
            }
        }
        __syncthreads();
        // horizontal transposed sums: item = (row, run of 4 pixel columns); centre columns
        // j0 .. j0 + 13 of the row, pixel j0 + o takes centre column j0 + o + t with weight g[10 - t]
        for (int k = tid; k < kI * (kT / kRun); k += kLossThreads) {
            const int r = k / (kT / kRun), j0 = kRun * (k % (kT / kRun));
            double acc[kRun][3];
#pragma unroll
            for (int o = 0; o < kRun; o++) acc[o][0] = acc[o][1] = acc[o][2] = 0.0;
#pragma unroll
            for (int i = 0; i < kWin + kRun - 1; i++) {
                const double v0 = S.sm[0][r][j0 + i], v1 = S.sm[1][r][j0 + i], v2 = S.sm[2][r][j0 + i];
#pragma unroll
                for (int o = 0; o < kRun; o++) {
                    const int t = i - o;
                    if (t >= 0 && t < kWin) {
                        const double g = w.g[2 * kR - t];
                        acc[o][0] += g * v0;
                        acc[o][1] += g * v1;
                        acc[o][2] += g * v2;
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < kRun; o++)
#pragma unroll
                for (int q = 0; q < 3; q++) S.hs[q][r][j0 + o] = acc[o][q];
        }
        __syncthreads();
    }
    // vertical transposed sums + the pixel gradient: item = (column, run of 4 pixel rows)
    for (int k = tid; k < kT * (kT / kRun); k += kLossThreads) {
        const int j = k % kT, i0 = kRun * (k / kT);
        double acc[kRun][3];
#pragma unroll
        for (int o = 0; o < kRun; o++) acc[o][0] = acc[o][1] = acc[o][2] = 0.0;
        if (ssim) {
#pragma unroll
            for (int i = 0; i < kWin + kRun - 1; i++) {
                const double v0 = S.hs[0][i0 + i][j], v1 = S.hs[1][i0 + i][j], v2 = S.hs[2][i0 + i][j];
#pragma unroll
                for (int o = 0; o < kRun; o++) {
                    const int t = i - o;
                    if (t >= 0 && t < kWin) {
                        const double g = w.g[2 * kR - t];
                        acc[o][0] += g * v0;
                        acc[o][1] += g * v1;
                        acc[o][2] += g * v2;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kRun; o++) {
            const int qx = qx0 + j, qy = qy0 + i0 + o;
            if (qx >= W || qy >= H) continue;
            const size_t off = ((size_t)qy * W + qx) * 3 + c;
            const double x = __ldg(render + off), y = __ldg(target + off);
            const double d = x - y;
            l1 += fabs(d);
            double g = (1.0 - (double)lambda) * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;
            if (ssim) g += k_ssim * (acc[o][0] + 2.0 * acc[o][1] * x + acc[o][2] * y);
            dL[off] = (float)g;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) l1 += __shfl_xor_sync(VKS_FULL_MASK, l1, o);
    if ((tid & 31) == 0) S.red[tid >> 5] = l1;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) t += S.red[q];
        l1_part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kLossThreads) loss_finalize_kernel(int W, int H, float lambda, const double* __restrict__ s_part,
                                                                    int ns, const double* __restrict__ l1_part, int nl,
                                                                    float* __restrict__ loss) {
    __shared__ double red[2][kLossThreads / 32];
    const int tid = threadIdx.x;
    double s = 0.0, l = 0.0;
    for (int i = tid; i < ns; i += kLossThreads) s += s_part[i];
    for (int i = tid; i < nl; i += kLossThreads) l += l1_part[i];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        s += __shfl_xor_sync(VKS_FULL_MASK, s, o);
        l += __shfl_xor_sync(VKS_FULL_MASK, l, o);
    }
    if ((tid & 31) == 0) { red[0][tid >> 5] = s; red[1][tid >> 5] = l; }
    __syncthreads();
    if (tid == 0) {
        double Ssum = 0.0, L = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) { Ssum += red[0][q]; L += red[1][q]; }
        const int Wv = W - 2 * kR, Hv = H - 2 * kR;
        const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
        const double l1 = L / (3.0 * (double)W * (double)H);
        const double ss = ssim ? Ssum / (3.0 * (double)Wv * (double)Hv) : 1.0;
        *loss = (float)((1.0 - (double)lambda) * l1 + (double)lambda * (1.0 - ss));
    }
}

struct LossWs {
    map_t *A, *B, *C;
    double *s_part, *l1_part;
    size_t bytes;
};

LossWs carve_loss(void* base, int W, int H) {
    LossWs w{};
    const int Wv = W - 2 * kR > 0 ? W - 2 * kR : 0, Hv = H - 2 * kR > 0 ? H - 2 * kR : 0;
    const size_t maps = (size_t)3 * Wv * Hv;
    const size_t nfwd = (size_t)3 * ((Wv + kT - 1) / kT) * ((Hv + kT - 1) / kT);
    const size_t nbwd = (size_t)3 * ((W + kT - 1) / kT) * ((H + kT - 1) / kT);
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t n) { double* p = b ? reinterpret_cast<double*>(b + off) : nullptr; off += (8 * n + 255) & ~(size_t)255; return p; };
    w.A = reinterpret_cast<map_t*>(take(maps));  // (sized for doubles whatever map_t is)
    w.B = reinterpret_cast<map_t*>(take(maps));
    w.C = reinterpret_cast<map_t*>(take(maps));
    w.s_part = take(nfwd > 0 ? nfwd : 1);
    w.l1_part = take(nbwd);
    w.bytes = off;
    return w;
}

}  // namespace

size_t loss_workspace_bytes(int W, int H) { return carve_loss(nullptr, W, H).bytes + 256; }

int launch_loss_grad(int W, int H, float lambda, const float* render, const float* target, float* dL, float* loss,
                     void* workspace, cudaStream_t s) {
    LossWs ws = carve_loss(workspace, W, H);
    const Gauss w = window();
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
    int ns = 0;
    // shared memory beyond 48 KB: the attributes are set on every call (per-device state)
    if (cudaFuncSetAttribute(ssim_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwdSmem)) ||
        cudaFuncSetAttribute(ssim_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BwdSmem)))
        return cuda_fail(cudaGetLastError(), "loss smem attribute");
    if (ssim) {
        const dim3 g((Wv + kT - 1) / kT, (Hv + kT - 1) / kT, 3);
        ssim_fwd_kernel<<<g, kLossThreads, sizeof(FwdSmem), s>>>(W, H, render, target, w, ws.A, ws.B, ws.C, ws.s_part);
        ns = (int)(g.x * g.y * g.z);
        if (int e = LaunchCheck::check()) return e;
    }
    const dim3 gb((W + kT - 1) / kT, (H + kT - 1) / kT, 3);
    ssim_bwd_kernel<<<gb, kLossThreads, sizeof(BwdSmem), s>>>(W, H, lambda, render, target, w, ws.A, ws.B, ws.C, dL,
                                                              ws.l1_part);
    if (int e = LaunchCheck::check()) return e;
    if (loss) {
        loss_finalize_kernel<<<1, kLossThreads, 0, s>>>(W, H, lambda, ws.s_part, ns, ws.l1_part,
                                                        (int)(gb.x * gb.y * gb.z), loss);
        return LaunchCheck::check();
    }
    return VKS_OK;
}

}  // namespace vks
