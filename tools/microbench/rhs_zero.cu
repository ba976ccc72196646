// Microbenchmark: cost of reading (and zeroing) int32 grids that the
// previous kernel accumulated with L2 atomics.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atomics(int *q, long long m, long long n, int stride) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        long long base = (i * 167) % (m - 8);
        atomicAdd(&q[base], 1); atomicAdd(&q[base + 1], 1);
        atomicAdd(&q[base + stride], 1); atomicAdd(&q[(base + stride + 1) % m], 1);
    }
}
__global__ void k_plainwrite(int *q, long long m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) q[i] = (int)i;
}
__global__ void k_read_zero(const float *c, int *q, long long m, float *rhs) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m; l += (long long)gridDim.x * blockDim.x) {
        int a = q[l], b = q[l + m]; q[l] = 0; q[l + m] = 0;
        rhs[l] = c[l] + (float)a * 0.5f - (float)b;
    }
}
__global__ void k_read_only(const float *c, const int *q, long long m, float *rhs) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m; l += (long long)gridDim.x * blockDim.x) {
        int a = q[l], b = q[l + m];
        rhs[l] = c[l] + (float)a * 0.5f - (float)b;
    }
}
__global__ void k_read_zero_dbl(const float *c, int *q, long long m, float *rhs) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m; l += (long long)gridDim.x * blockDim.x) {
        int a = q[l], b = q[l + m]; q[l] = 0; q[l + m] = 0;
        double r = __dadd_rn((double)c[l], __dmul_rn((double)a, 0.5)); r = __dsub_rn(r, (double)b);
        rhs[l] = (float)r;
    }
}
int main() {
    const long long m = 4096LL * 4096, n = 10000000;
    int *q; float *c, *rhs;
    cudaMalloc(&q, 2 * m * 4); cudaMalloc(&c, m * 4); cudaMalloc(&rhs, m * 4);
    cudaMemset(q, 0, 2 * m * 4); cudaMemset(c, 0, m * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    const char *names[] = {"read_zero", "read_only", "read_zero_dbl"};
    for (int variant = 0; variant < 3; variant++)
      for (int pre = 0; pre < 3; pre++) {
        for (int rep = 0; rep < 3; rep++) {
            if (pre == 0) k_atomics<<<148 * 8, 256>>>(q, 2 * m, n, 4096);
            else if (pre == 1) k_plainwrite<<<148 * 8, 256>>>(q, 2 * m);
            else cudaMemset(q, 0, 2 * m * 4);
            cudaEventRecord(a);
            if (variant == 0) k_read_zero<<<2368, 256>>>(c, q, m, rhs);
            else if (variant == 1) k_read_only<<<2368, 256>>>(c, q, m, rhs);
            else k_read_zero_dbl<<<2368, 256>>>(c, q, m, rhs);
            cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("%-14s after %-10s: %8.1f us\n", names[variant], pre == 0 ? "atomics" : pre == 1 ? "writes" : "memset", ms * 1e3);
      }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
