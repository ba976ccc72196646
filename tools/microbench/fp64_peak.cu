// FP64 (scalar DFMA pipe) peak of this GPU: every thread runs 16 independent
// fma chains; FLOP/s = 2 * fmas / time.  Build + run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/microbench/fp64_peak.cu && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; q++) acc[q] = threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < 16; q++) acc[q] = fma(acc[q], a, b);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) s += acc[q];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *d;
    cudaMalloc(&d, 8);
    const int iters = 1 << 14, blocks = sms * 8, threads = 256;
    k_dfma<<<blocks, threads>>>(d, 16, 0.999, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
    return 0;
}
