// DFMA throughput microbenchmark: many independent FMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8, threads = 256, iters = 20000;
    double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
    k<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"dfma_per_sm_per_clk_at_1965\": %.2f}\n",
           fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12, ms, sms, fmas / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}
