// loss.cu — SURVEY §8(f) row f2: the loss gradient before the path ("Loss Gradient", PAPER P:74;
// SPEC S:178-186, SSIM definition); include/vks.h vks_loss_grad.
//
//   loss = (1 - lambda) mean|r - t| + lambda (1 - SSIM),   SSIM = mean over channels and valid
//   11x11 windows (Gaussian, sigma 1.5) of S = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)
//   (sx2 + sy2 + C2)).
// Three kernels: ssim_fwd_kernel (per 32x16 tile of window centres and channel: separable window
// sums of x, y, x^2, y^2, xy in shared memory, then S and its partials dS/dmx, dS/dE[x^2],
// dS/dE[xy] per centre), ssim_bwd_kernel (per 32x16 pixel tile and channel: the transposed
// separable window sums of the three partial maps, the L1 subgradient, dL/dr),
// loss_finalize_kernel (one block: the block partial sums -> loss, deterministic).  The window
// sums, S, the partials and the transposed pass are fp64: the variances E[x^2] - mx^2 cancel down
// to ~C2 = 9e-4, and fp32 statistics would put up to ~1e-3 relative error into the gradient (fp32
// horizontal sums measured 0.189 vs 0.204 ms for 1237x822: not worth their 1e-6 absolute error).
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kTW = 32, kTH = 16;                 // tile of centres (fwd) / pixels (bwd)
constexpr int kR = 5, kWin = 11;                  // window radius / width
constexpr int kIW = kTW + 2 * kR, kIH = kTH + 2 * kR;  // input tile with halo
constexpr int kLossThreads = 256;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

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

// block (x: centre tile, y: centre tile, z: channel).  Centre p's window covers pixels p .. p+10.
__global__ void __launch_bounds__(kLossThreads) ssim_fwd_kernel(int W, int H, const float* __restrict__ render,
                                                               const float* __restrict__ target, const Gauss w,
                                                               double* __restrict__ A, double* __restrict__ B,
                                                               double* __restrict__ Cm, double* __restrict__ s_part) {
    __shared__ float sx[kIH][kIW], sy[kIH][kIW];
    __shared__ double hs[5][kIH][kTW];
    __shared__ double red[kLossThreads / 32];
    const int tid = threadIdx.x, c = blockIdx.z;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const int cx0 = blockIdx.x * kTW, cy0 = blockIdx.y * kTH;
    for (int k = tid; k < kIH * kIW; k += kLossThreads) {
        const int r = k / kIW, q = k % kIW;
        const int py = cy0 + r, px = cx0 + q;
        const bool in = px < W && py < H;
        const size_t o = ((size_t)py * W + px) * 3 + c;
        sx[r][q] = in ? __ldg(render + o) : 0.0f;
        sy[r][q] = in ? __ldg(target + o) : 0.0f;
    }
    __syncthreads();
    for (int k = tid; k < kIH * kTW; k += kLossThreads) {  // horizontal window sums
        const int r = k / kTW, j = k % kTW;
        double a = 0, b = 0, aa = 0, bb = 0, ab = 0;
#pragma unroll
        for (int i = 0; i < kWin; i++) {
            const double x = sx[r][j + i], y = sy[r][j + i], g = w.g[i];
            a += g * x;
            b += g * y;
            aa += g * x * x;
            bb += g * y * y;
            ab += g * x * y;
        }
        hs[0][r][j] = a; hs[1][r][j] = b; hs[2][r][j] = aa; hs[3][r][j] = bb; hs[4][r][j] = ab;
    }
    __syncthreads();
    double ssum = 0.0;
    // vertical sums -> S and partials; two vertically adjacent centres per thread share 10 of the
    // 12 rows they read (halves the 64-bit shared-memory traffic)
    for (int k = tid; k < (kTH / 2) * kTW; k += kLossThreads) {
        const int i0 = 2 * (k / kTW), j = k % kTW;
        double st[2][5] = {};
#pragma unroll
        for (int t = 0; t < kWin + 1; t++) {
            double hv[5];
#pragma unroll
            for (int q = 0; q < 5; q++) hv[q] = hs[q][i0 + t][j];
            if (t < kWin) {
#pragma unroll
                for (int q = 0; q < 5; q++) st[0][q] += w.g[t] * hv[q];
            }
            if (t > 0) {
#pragma unroll
                for (int q = 0; q < 5; q++) st[1][q] += w.g[t - 1] * hv[q];
            }
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int px = cx0 + j, py = cy0 + i0 + h;
            if (px >= Wv || py >= Hv) continue;
            const double mx = st[h][0], my = st[h][1], exx = st[h][2], eyy = st[h][3], exy = st[h][4];
            const double sx2 = exx - mx * mx, sy2 = eyy - my * my, sxy = exy - mx * my;
            const double l1 = 2 * mx * my + kC1, l2 = mx * mx + my * my + kC1;
            const double c1 = 2 * sxy + kC2, c2 = sx2 + sy2 + kC2;
            const double inv = 1.0 / (l2 * c2);  // the one fp64 division: 1/l2 = c2 inv, 1/c2 = l2 inv
            const double S = l1 * c1 * inv;
            const double dB = -S * (l2 * inv), dC = 2.0 * l1 * inv;
            const double dA = 2.0 * my * c1 * inv - 2.0 * mx * S * (c2 * inv) - 2.0 * mx * dB - my * dC;
            const size_t o = ((size_t)c * Hv + py) * Wv + px;
            A[o] = dA;
            B[o] = dB;
            Cm[o] = dC;
            ssum += S;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ssum += __shfl_xor_sync(VKS_FULL_MASK, ssum, o);
    if ((tid & 31) == 0) red[tid >> 5] = ssum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) t += red[q];
        s_part[((size_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

// block (x, y: pixel tile); all three channels.  dL_q = (1 - lambda) sign(r - t) / (3 N)
//   - lambda / (3 Nv) sum_{centres p: q in window(p)} w(q - p) (A_p + 2 B_p r_q + C_p t_q)
__global__ void __launch_bounds__(kLossThreads) ssim_bwd_kernel(int W, int H, float lambda, const float* __restrict__ render,
                                                               const float* __restrict__ target, const Gauss w,
                                                               const double* __restrict__ A, const double* __restrict__ B,
                                                               const double* __restrict__ Cm, float* __restrict__ dL,
                                                               double* __restrict__ l1_part) {
    __shared__ double sm[3][kIH][kIW];  // partial maps of the centres that reach the tile
    __shared__ double hs[3][kIH][kTW];
    __shared__ double red[kLossThreads / 32];
    const int tid = threadIdx.x;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
    const int qx0 = blockIdx.x * kTW, qy0 = blockIdx.y * kTH;
    const double inv_n = 1.0 / (3.0 * (double)W * (double)H);
    const double k_ssim = ssim ? -(double)lambda / (3.0 * (double)Wv * (double)Hv) : 0.0;
    double l1 = 0.0;
    {
        const int c = blockIdx.z;
        if (ssim) {
            // centres p = q - i (i in [0, 10]) for q in the tile: rows qy0-10 .. qy0+kTH-1
            for (int k = tid; k < kIH * kIW; k += kLossThreads) {
                const int r = k / kIW, s = k % kIW;
                const int py = qy0 - 2 * kR + r, px = qx0 - 2 * kR + s;
                const bool in = px >= 0 && py >= 0 && px < Wv && py < Hv;
                const size_t o = ((size_t)c * Hv + py) * Wv + px;
                sm[0][r][s] = in ? A[o] : 0.0;
                sm[1][r][s] = in ? B[o] : 0.0;
                sm[2][r][s] = in ? Cm[o] : 0.0;
            }
            __syncthreads();
            for (int k = tid; k < kIH * (kTW / 2); k += kLossThreads) {  // horizontal transposed sums
                const int r = k / (kTW / 2), j0 = 2 * (k % (kTW / 2));   // two adjacent columns
                double o0[3] = {}, o1[3] = {};
#pragma unroll
                for (int t = 0; t < kWin + 1; t++) {  // centre columns j0 .. j0 + 11 in tile coordinates
                    const double v0 = sm[0][r][j0 + t], v1 = sm[1][r][j0 + t], v2 = sm[2][r][j0 + t];
                    if (t < kWin) {
                        const double g = w.g[2 * kR - t];
                        o0[0] += g * v0; o0[1] += g * v1; o0[2] += g * v2;
                    }
                    if (t > 0) {
                        const double g = w.g[2 * kR + 1 - t];
                        o1[0] += g * v0; o1[1] += g * v1; o1[2] += g * v2;
                    }
                }
#pragma unroll
                for (int q = 0; q < 3; q++) {
                    hs[q][r][j0] = o0[q];
                    hs[q][r][j0 + 1] = o1[q];
                }
            }
            __syncthreads();
        }
        for (int k = tid; k < (kTH / 2) * kTW; k += kLossThreads) {  // two vertically adjacent pixels
            const int i0 = 2 * (k / kTW), j = k % kTW;
            double acc[2][3] = {};
            if (ssim) {
#pragma unroll
                for (int t = 0; t < kWin + 1; t++) {  // centre rows i0 .. i0 + 11 in tile coordinates
                    const double v0 = hs[0][i0 + t][j], v1 = hs[1][i0 + t][j], v2 = hs[2][i0 + t][j];
                    if (t < kWin) {
                        const double g = w.g[2 * kR - t];
                        acc[0][0] += g * v0; acc[0][1] += g * v1; acc[0][2] += g * v2;
                    }
                    if (t > 0) {
                        const double g = w.g[2 * kR + 1 - t];
                        acc[1][0] += g * v0; acc[1][1] += g * v1; acc[1][2] += g * v2;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int qx = qx0 + j, qy = qy0 + i0 + h;
                if (qx >= W || qy >= H) continue;
                const size_t o = ((size_t)qy * W + qx) * 3 + c;
                const double x = __ldg(render + o), y = __ldg(target + o);
                const double d = x - y;
                l1 += fabs(d);
                double g = (1.0 - (double)lambda) * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;
                if (ssim) g += k_ssim * (acc[h][0] + 2.0 * acc[h][1] * x + acc[h][2] * y);
                dL[o] = (float)g;
            }
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) l1 += __shfl_xor_sync(VKS_FULL_MASK, l1, o);
    if ((tid & 31) == 0) red[tid >> 5] = l1;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) t += red[q];
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
        double S = 0.0, L = 0.0;
        for (int q = 0; q < kLossThreads / 32; q++) { S += red[0][q]; L += red[1][q]; }
        const int Wv = W - 2 * kR, Hv = H - 2 * kR;
        const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
        const double l1 = L / (3.0 * (double)W * (double)H);
        const double ss = ssim ? S / (3.0 * (double)Wv * (double)Hv) : 1.0;
        *loss = (float)((1.0 - (double)lambda) * l1 + (double)lambda * (1.0 - ss));
    }
}

struct LossWs {
    double *A, *B, *C, *s_part, *l1_part;
    size_t bytes;
};

LossWs carve_loss(void* base, int W, int H) {
    LossWs w{};
    const int Wv = W - 2 * kR > 0 ? W - 2 * kR : 0, Hv = H - 2 * kR > 0 ? H - 2 * kR : 0;
    const size_t maps = (size_t)3 * Wv * Hv;
    const size_t nfwd = (size_t)3 * ((Wv + kTW - 1) / kTW) * ((Hv + kTH - 1) / kTH);
    const size_t nbwd = (size_t)3 * ((W + kTW - 1) / kTW) * ((H + kTH - 1) / kTH);
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t n) { double* p = b ? reinterpret_cast<double*>(b + off) : nullptr; off += (8 * n + 255) & ~(size_t)255; return p; };
    w.A = take(maps);
    w.B = take(maps);
    w.C = take(maps);
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
    if (ssim) {
        const dim3 g((Wv + kTW - 1) / kTW, (Hv + kTH - 1) / kTH, 3);
        ssim_fwd_kernel<<<g, kLossThreads, 0, s>>>(W, H, render, target, w, ws.A, ws.B, ws.C, ws.s_part);
        ns = (int)(g.x * g.y * g.z);
        if (int e = LaunchCheck::check()) return e;
    }
    const dim3 gb((W + kTW - 1) / kTW, (H + kTH - 1) / kTH, 3);
    ssim_bwd_kernel<<<gb, kLossThreads, 0, s>>>(W, H, lambda, render, target, w, ws.A, ws.B, ws.C, dL, ws.l1_part);
    if (int e = LaunchCheck::check()) return e;
    if (loss) {
        loss_finalize_kernel<<<1, kLossThreads, 0, s>>>(W, H, lambda, ws.s_part, ns, ws.l1_part,
                                                        (int)(gb.x * gb.y * gb.z), loss);
        return LaunchCheck::check();
    }
    return VKS_OK;
}

}  // namespace vks
