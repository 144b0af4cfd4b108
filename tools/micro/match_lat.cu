// microbenchmark: latency (dependent chain, 1 warp) and throughput (many warps) of
// __match_any_sync, __reduce_or_sync, __shfl_sync and a shared-memory load
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(unsigned* out, int iters, unsigned seed) {
    __shared__ unsigned sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 7 + 1;
    __syncthreads();
    unsigned v = threadIdx.x * seed;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (OP == 0) v = __match_any_sync(0xffffffffu, v & 7) + v;
        else if (OP == 1) v = __reduce_or_sync(0xffffffffu, v) + v;
        else if (OP == 2) v = __shfl_sync(0xffffffffu, v, v & 31) + 1;
        else if (OP == 3) v = sm[v & 1023] + v;
        else v = v * 3 + 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned)(t1 - t0);
    out[1 + blockIdx.x * blockDim.x + threadIdx.x] = v;
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 64 << 20);
    const char* names[] = {"match_any", "reduce_or", "shfl_idx", "lds", "imad"};
    const int iters = 4096;
    for (int op = 0; op < 5; op++) {
        unsigned h = 0;
        auto run = [&](int blocks, int threads) {
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            switch (op) {
                case 0: chain<0><<<blocks, threads>>>(d, iters, 3); break;
                case 1: chain<1><<<blocks, threads>>>(d, iters, 3); break;
                case 2: chain<2><<<blocks, threads>>>(d, iters, 3); break;
                case 3: chain<3><<<blocks, threads>>>(d, iters, 3); break;
                default: chain<4><<<blocks, threads>>>(d, iters, 3); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            return ms;
        };
        run(1, 32);
        run(1, 32);
        cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
        float ms = run(148 * 32, 256);  // 64 warps per SM
        double warp_ops = 148.0 * 32 * 8 * iters;
        printf("%-10s latency %.1f cyc/op (1 warp)   throughput %.2f warp-ops/cyc/SM (64 warps/SM, 1.9 GHz assumed)\n",
               names[op], (double)h / iters, warp_ops / (ms * 1e-3 * 1.9e9) / 148.0);
    }
    return 0;
}
