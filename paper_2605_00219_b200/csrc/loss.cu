// loss.cu — SURVEY §8(f) row f2: the loss gradient before the path ("Loss Gradient", PAPER P:74;
// SPEC S:178-186, SSIM definition); include/vks.h vks_loss_grad.
//
//   loss = (1 - lambda) mean|r - t| + lambda (1 - SSIM),   SSIM = mean over channels and valid
//   11x11 windows (Gaussian, sigma 1.5) of S = (2 mx my + C1)(2 sxy + C2) / ((mx^2 + my^2 + C1)
//   (sx2 + sy2 + C2)).
// Three kernels: ssim_fused_kernel (per 32x32 tile of window centres and channel: the separable
// window sums of x, y, x^2, y^2, xy — horizontal into shared memory, then vertical — S with its
// partials A = dS/dmx, B = dS/dE[x^2], C = dS/dE[xy] per centre, then the transposed separable
// sums of A, B, C over the 42x42 pixel region the tile's windows reach and each pixel's partial
// A + 2 B x + C y, into a per-tile slot), loss_combine_kernel (per pixel: the L1 subgradient plus
// the <= 2x2 tile partials in a fixed order, dL/dr) and loss_finalize_kernel (one block: the block
// partial sums -> loss, deterministic).  The window sums, S, the partials and the transposed sums
// are fp64: the variances E[x^2] - mx^2 cancel down to ~C2 = 9e-4, and fp32 statistics would put
// up to ~1e-3 relative error into the gradient.  Each thread produces four adjacent outputs of a
// pass from a sliding register window (14 inputs for 4 outputs of an 11-tap pass: 3.5 shared-
// memory loads and products per output instead of 11).  Round 1/2 ran the transposed sums in a
// second kernel over 32x32 pixel tiles, reading fp64 maps of A, B, C (72 B per pixel) with a
// 10-pixel halo back from HBM: 0.154 ms for 1237x822, the second kernel at 25% of the fp64 pipe.
#include "vks_common.cuh"

namespace vks {
namespace {

constexpr int kT = 32;                             // tile of window centres, square
constexpr int kR = 5, kWin = 11;                  // window radius / width
constexpr int kI = kT + 2 * kR;                   // tile + halo (42)
constexpr int kIP = kI + 3;                       // float row pitch 45: the 4 rows x 8 column groups of
                                                  // a warp's sliding-window loads hit 32 distinct banks
#ifndef VKS_LOSS_RUN
#define VKS_LOSS_RUN 4
#endif
constexpr int kRun = VKS_LOSS_RUN;                // outputs per thread and pass
constexpr int kLossThreads = 512;             // 2 blocks x 16 warps per SM (75 KB of shared memory each)
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

// dynamic shared memory of the fused kernel: two regions reused phase by phase.  64-bit rows
// have an odd pitch, so a warp reading one element of 32 consecutive rows (stride 33 or 45
// doubles) spreads over all 16 bank pairs; 32 consecutive columns of a row are contiguous.
constexpr int kHP = kT + 1;       // 33
constexpr int kXP = kI + 1;       // 43
constexpr int kUP = kI + 3;       // 45
constexpr int kLen = 16, kVLen = 14;  // rolling-window run lengths: 2 x 16 centre rows, 3 x 14 pixel cols / rows
struct FusedSmem {
    union {                                 // region A
        double hs[5][kI][kHP];              // horizontal window sums of x, y, x^2, y^2, xy  (P1 -> P2)
        double abc[3][kT][kHP];             // the centres' partials A, B, C                 (P3 -> P4)
        double vt[3][kI][kXP];              // transposed window sums of A, B, C per pixel   (P5 -> P6)
    } a;
    union {                                 // region B
        struct {
            float sx[kI][kIP], sy[kI][kIP];  // input tile + halo                             (P0 -> P1)
        } in;
        double st[5][kT][kHP];              // window statistics per centre                  (P2 -> P3)
        double ht[3][kT][kUP];              // horizontal transposed sums of A, B, C         (P4 -> P5)
    } b;
    double red[kLossThreads / 32];
};
static_assert(kLossThreads >= kI * (kT / kRun) && kLossThreads >= kT * 5 * 2 && kLossThreads >= kT * 3 * 3 &&
              kLossThreads >= kI * 3 * 3 && 2 * kLen == kT && 3 * kVLen == kI,
              "one item per thread in every phase");

// block (x: centre tile, y: centre tile, z: channel).  Centre p's window covers pixels p .. p+10,
// so the block's 32x32 centres reach the 42x42 pixel region starting at the tile origin.  The
// block computes the window statistics, S and its partials A, B, C for its centres, then the
// transposed window sums of A, B, C over the region and, per pixel q,
//   part_b(q) = sum_{centres p of the block} w(q - p) (A_p + 2 B_p x_q + C_p y_q)
// into its own 42x42 slot of `part` (fp64).  A pixel is reached by at most 2x2 blocks;
// loss_combine_kernel adds their slots in a fixed order (deterministic).  The vertical and the
// transposed passes run one (column or row, quantity, run) per thread with the 11-tap window
// rolling in registers: 26 (24) shared-memory loads for 16 (14) outputs.
__global__ void __launch_bounds__(kLossThreads, 2) ssim_fused_kernel(int W, int H, const float* __restrict__ render,
                                                                    const float* __restrict__ target, const Gauss w,
                                                                    double* __restrict__ part,
                                                                    double* __restrict__ s_part) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char loss_smem[];
    FusedSmem& S = *reinterpret_cast<FusedSmem*>(loss_smem);
    const int tid = threadIdx.x, c = blockIdx.z;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const int cx0 = blockIdx.x * kT, cy0 = blockIdx.y * kT;
    {   // P0: every load of the tile in flight before the first shared-memory store
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
                S.b.in.sx[k / kI][k % kI] = vx[it];
                S.b.in.sy[k / kI][k % kI] = vy[it];
            }
        }
    }
    __syncthreads();
    // P1 horizontal sums: item = (row, run of 4 centre columns); inputs j0 .. j0 + 13 of the row
    if (tid < kI * (kT / kRun)) {
        const int r = tid / (kT / kRun), j0 = kRun * (tid % (kT / kRun));
        double acc[kRun][5];
#pragma unroll
        for (int o = 0; o < kRun; o++)
#pragma unroll
            for (int q = 0; q < 5; q++) acc[o][q] = 0.0;
#pragma unroll
        for (int i = 0; i < kWin + kRun - 1; i++) {
            const double x = S.b.in.sx[r][j0 + i], y = S.b.in.sy[r][j0 + i];
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
            for (int q = 0; q < 5; q++) S.a.hs[q][r][j0 + o] = acc[o][q];
    }
    __syncthreads();
    // P2 vertical sums: item = (centre column j, statistic q, half h): centre rows 16h .. 16h + 15
    // from hs rows 16h .. 16h + 25
    if (tid < kT * 5 * 2) {
        const int j = tid % kT, q = (tid / kT) % 5, i0 = kLen * (tid / (kT * 5));
        double acc[kLen];
#pragma unroll
        for (int o = 0; o < kLen; o++) acc[o] = 0.0;
#pragma unroll
        for (int i = 0; i < kLen + kWin - 1; i++) {
            const double v = S.a.hs[q][i0 + i][j];
#pragma unroll
            for (int o = 0; o < kLen; o++) {
                const int t = i - o;
                if (t >= 0 && t < kWin) acc[o] += w.g[t] * v;
            }
        }
#pragma unroll
        for (int o = 0; o < kLen; o++) S.b.st[q][i0 + o][j] = acc[o];
    }
    __syncthreads();
    // P3 S and its partials per centre (two centres per thread); centres outside the valid range
    // contribute nothing
    double ssum = 0.0;
#pragma unroll
    for (int m = 0; m < kT * kT / kLossThreads; m++) {
        const int k = tid + m * kLossThreads, i = k / kT, j = k % kT;
        double pa = 0.0, pb = 0.0, pc = 0.0;
        if (cx0 + j < Wv && cy0 + i < Hv) {
            const double mx = S.b.st[0][i][j], my = S.b.st[1][i][j];
            const double exx = S.b.st[2][i][j], eyy = S.b.st[3][i][j], exy = S.b.st[4][i][j];
            const double sx2 = exx - mx * mx, sy2 = eyy - my * my, sxy = exy - mx * my;
            const double l1 = 2 * mx * my + kC1, l2 = mx * mx + my * my + kC1;
            const double c1 = 2 * sxy + kC2, c2 = sx2 + sy2 + kC2;
            const double inv = 1.0 / (l2 * c2);  // the one fp64 division: 1/l2 = c2 inv, 1/c2 = l2 inv
            const double Sv = l1 * c1 * inv;
            const double dB = -Sv * (l2 * inv), dC = 2.0 * l1 * inv;
            pa = 2.0 * my * c1 * inv - 2.0 * mx * Sv * (c2 * inv) - 2.0 * mx * dB - my * dC;
            pb = dB;
            pc = dC;
            ssum += Sv;
        }
        S.a.abc[0][i][j] = pa;
        S.a.abc[1][i][j] = pb;
        S.a.abc[2][i][j] = pc;
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
    // P4 horizontal transposed sums: item = (centre row r, partial m, third): pixel columns
    // u0 .. u0 + 13 (u0 = 14 third) take centre columns u - 10 .. u inside the tile: centre
    // u0 - 10 + jj feeds output o with weight g[10 + o - jj]
    if (tid < kT * 3 * 3) {
        const int r = tid % kT, m = (tid / kT) % 3, u0 = kVLen * (tid / (kT * 3));
        double acc[kVLen];
#pragma unroll
        for (int o = 0; o < kVLen; o++) acc[o] = 0.0;
#pragma unroll
        for (int jj = 0; jj < kVLen + kWin - 1; jj++) {
            const int j = u0 - 2 * kR + jj;
            const double v = (j >= 0 && j < kT) ? S.a.abc[m][r][j] : 0.0;
#pragma unroll
            for (int o = 0; o < kVLen; o++) {
                const int t = 2 * kR + o - jj;
                if (t >= 0 && t < kWin) acc[o] += w.g[t] * v;
            }
        }
#pragma unroll
        for (int o = 0; o < kVLen; o++) S.b.ht[m][r][u0 + o] = acc[o];
    }
    __syncthreads();
    // P5 vertical transposed sums: item = (pixel column u, partial m, third): pixel rows v0 .. v0 + 13
    // take centre rows v - 10 .. v inside the tile
    if (tid < kI * 3 * 3) {
        const int u = tid % kI, m = (tid / kI) % 3, v0 = kVLen * (tid / (kI * 3));
        double acc[kVLen];
#pragma unroll
        for (int o = 0; o < kVLen; o++) acc[o] = 0.0;
#pragma unroll
        for (int ii = 0; ii < kVLen + kWin - 1; ii++) {
            const int i = v0 - 2 * kR + ii;
            const double v = (i >= 0 && i < kT) ? S.b.ht[m][i][u] : 0.0;
#pragma unroll
            for (int o = 0; o < kVLen; o++) {
                const int t = 2 * kR + o - ii;
                if (t >= 0 && t < kWin) acc[o] += w.g[t] * v;
            }
        }
#pragma unroll
        for (int o = 0; o < kVLen; o++) S.a.vt[m][v0 + o][u] = acc[o];
    }
    __syncthreads();
    // P6 the block's pixel partial A + 2 B x + C y over the region (pixel values re-read: L2)
    double* slot = part + (((size_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * (kI * kI);
    for (int k = tid; k < kI * kI; k += kLossThreads) {
        const int v = k / kI, u = k % kI;
        if (cx0 + u >= W || cy0 + v >= H) continue;
        const size_t off = ((size_t)(cy0 + v) * W + (cx0 + u)) * 3 + c;
        const double x = __ldg(render + off), y = __ldg(target + off);
        slot[k] = S.a.vt[0][v][u] + 2.0 * S.a.vt[1][v][u] * x + S.a.vt[2][v][u] * y;
    }
}

// one thread per pixel (all three channels), image rows over the grid's rows.  dL_q = (1 - lambda) sign(r - t) / (3 N)
//   - lambda / (3 Nv) (sum over the <= 2x2 centre tiles whose region holds q of their partial)
constexpr int kCombThreads = 128;  // pixels per combine block (1237 columns: 10 blocks, 3% idle)
__global__ void __launch_bounds__(kCombThreads) loss_combine_kernel(int W, int H, float lambda, const float* __restrict__ render,
                                                          const float* __restrict__ target,
                                                          const double* __restrict__ part, int gx, int gy,
                                                          float* __restrict__ dL, double* __restrict__ l1_part) {
    pdl_wait();
    __shared__ double red[kCombThreads / 32];
    const int tid = threadIdx.x;
    const int Wv = W - 2 * kR, Hv = H - 2 * kR;
    const bool ssim = lambda != 0.0f && Wv > 0 && Hv > 0;
    const double inv_n = 1.0 / (3.0 * (double)W * (double)H);
    const double k_ssim = ssim ? -(double)lambda / (3.0 * (double)Wv * (double)Hv) : 0.0;
    const int qx = blockIdx.x * kCombThreads + tid;
    double l1 = 0.0;
    for (int qy = blockIdx.y; qx < W && qy < H; qy += gridDim.y) {  // rows blockIdx.y + k gridDim.y
        const size_t q = (size_t)qy * W + qx;
        // tiles b with 0 <= q - 32 b < 42, ascending: (x1 - 1 when it reaches q,) x1; -1 = none
        const int x1 = min(qx / kT, gx - 1), y1 = min(qy / kT, gy - 1);
        const int bx[2] = {x1 >= 1 && qx - kT * (x1 - 1) < kI ? x1 - 1 : -1, x1};
        const int by[2] = {y1 >= 1 && qy - kT * (y1 - 1) < kI ? y1 - 1 : -1, y1};
        // every load in flight before the arithmetic: 3 + 3 pixel values, up to 3 x 4 partials
        // (tile k's slot offset for this pixel once; the channels are gx gy 42^2 apart)
        const size_t cstride = (size_t)gx * gy * (kI * kI);
        size_t toff[4];
        bool tok[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int ty = by[k >> 1], tx = bx[k & 1];
            tok[k] = ssim && ty >= 0 && tx >= 0;
            toff[k] = tok[k] ? (size_t)(ty * gx + tx) * (kI * kI) + (size_t)((qy - kT * ty) * kI + (qx - kT * tx)) : 0;
        }
        float xs[3], ys[3];
        double pv[3][4];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            xs[c] = __ldg(render + q * 3 + c);
            ys[c] = __ldg(target + q * 3 + c);
#pragma unroll
            for (int k = 0; k < 4; k++) pv[c][k] = tok[k] ? __ldg(part + toff[k] + c * cstride) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const double d = (double)xs[c] - (double)ys[c];
            l1 += fabs(d);
            double g = (1.0 - (double)lambda) * (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;
            if (ssim) g += k_ssim * (((pv[c][0] + pv[c][1]) + pv[c][2]) + pv[c][3]);  // tiles in fixed order
            dL[q * 3 + c] = (float)g;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) l1 += __shfl_xor_sync(VKS_FULL_MASK, l1, o);
    if ((tid & 31) == 0) red[tid >> 5] = l1;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int i = 0; i < kCombThreads / 32; i++) t += red[i];
        l1_part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kLossThreads) loss_finalize_kernel(int W, int H, float lambda, const double* __restrict__ s_part,
                                                                    int ns, const double* __restrict__ l1_part, int nl,
                                                                    float* __restrict__ loss) {
    pdl_wait();
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
    double *part, *s_part, *l1_part;
    int gx, gy, ncx, ncy, nl;
    size_t bytes;
};

LossWs carve_loss(void* base, int W, int H) {
    LossWs w{};
    const int Wv = W - 2 * kR > 0 ? W - 2 * kR : 0, Hv = H - 2 * kR > 0 ? H - 2 * kR : 0;
    w.gx = (Wv + kT - 1) / kT;
    w.gy = (Hv + kT - 1) / kT;
    const size_t nfwd = (size_t)3 * w.gx * w.gy;
    w.ncx = (W + kCombThreads - 1) / kCombThreads;
    w.ncy = H < 65535 ? H : 65535;  // grid rows (the kernel strides over the image rows)
    w.nl = w.ncx * w.ncy;
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t n) { double* p = b ? reinterpret_cast<double*>(b + off) : nullptr; off += (8 * n + 255) & ~(size_t)255; return p; };
    w.part = take(nfwd * kI * kI > 0 ? nfwd * kI * kI : 1);
    w.s_part = take(nfwd > 0 ? nfwd : 1);
    w.l1_part = take(w.nl > 0 ? (size_t)w.nl : 1);
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
    // shared memory beyond 48 KB: the attribute is set on every call (per-device state)
    if (cudaFuncSetAttribute(ssim_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FusedSmem)))
        return cuda_fail(cudaGetLastError(), "loss smem attribute");
    if (ssim) {
        const dim3 g(ws.gx, ws.gy, 3);
        launch_k(ssim_fused_kernel, g, kLossThreads, sizeof(FusedSmem), s, W, H, render, target, w, ws.part, ws.s_part);
        ns = (int)(g.x * g.y * g.z);
        if (int e = LaunchCheck::check()) return e;
    }
    if (ws.nl > 0) {
        launch_k(loss_combine_kernel, dim3(ws.ncx, ws.ncy), kCombThreads, 0, s, W, H, lambda, render, target, ws.part, ws.gx, ws.gy, dL,
                                                  ws.l1_part);
        if (int e = LaunchCheck::check()) return e;
    }
    if (loss) {
        launch_k(loss_finalize_kernel, 1, kLossThreads, 0, s, W, H, lambda, ws.s_part, ns, ws.l1_part, ws.nl, loss);
        return LaunchCheck::check();
    }
    return VKS_OK;
}

}  // namespace vks
