// Atomics whose targets lie within a moving band (the sorted-engine pattern):
// element i (processed in order) hits key(i) = base_row(i) + N(0, sigma) rows.
#include <cstdio>
#include <cuda_runtime.h>
#include <curand_kernel.h>
__global__ void k_keys(int *keys, long long n, int ncol, int nrow, float per_row, float sigma_rows, unsigned long long seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        curandStatePhilox4_32_10_t s; curand_init(seed, i, 0, &s);
        float2 g = curand_normal2(&s);
        int row = (int)(i / per_row) + (int)(g.x * sigma_rows);
        int col = (int)((i % (long long)per_row) * (ncol / per_row)) + (int)(g.y * sigma_rows);
        row = ((row % nrow) + nrow) % nrow; col = ((col % ncol) + ncol) % ncol;
        keys[i] = row * ncol + col;
    }
}
template <int MODE>
__global__ void k_atom(const int *keys, long long n, int *counts, int *ranks, const float4 *stream_in, float4 *stream_out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int k = keys[i];
        if (MODE == 0) ranks[i] = atomicAdd(&counts[k], 1);
        if (MODE == 1) atomicAdd(&counts[k], 1);
        if (MODE == 2) { ranks[i] = atomicAdd(&counts[k], 1); float4 v = __ldcs(stream_in + i); __stcs(stream_out + i, v); float4 v2 = __ldcs(stream_in + n + i); __stcs(stream_out + n + i, v2);}
        if (MODE == 3) { float4 v = __ldcs(stream_in + i); __stcs(stream_out + i, v); float4 v2 = __ldcs(stream_in + n + i); __stcs(stream_out + n + i, v2);}
    }
}
int main() {
    const long long n = 10000000; const int ncol = 4045, nrow = 4045; const long long m = (long long)ncol * nrow;
    int *keys, *counts, *ranks; float4 *si, *so;
    cudaMalloc(&keys, n * 4); cudaMalloc(&counts, m * 4); cudaMalloc(&ranks, n * 4);
    cudaMalloc(&si, 2 * n * 16); cudaMalloc(&so, 2 * n * 16); cudaMemset(si, 0, 2*n*16);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    float sig[] = {0.f, 2.f, 18.f, 54.f};
    for (int si_ = 0; si_ < 4; si_++) {
        k_keys<<<sms * 8, 256>>>(keys, n, ncol, nrow, n / (float)nrow, sig[si_], 1234);
        for (int mode = 0; mode < 4; mode++) for (int persist = 0; persist < 2; persist++) {
            int grid = persist ? sms * 8 : (int)((n + 255) / 256);
            for (int rep = 0; rep < 2; rep++) {
                cudaMemset(counts, 0, m * 4);
                cudaEventRecord(a);
                if (mode == 0) k_atom<0><<<grid, 256>>>(keys, n, counts, ranks, si, so);
                if (mode == 1) k_atom<1><<<grid, 256>>>(keys, n, counts, ranks, si, so);
                if (mode == 2) k_atom<2><<<grid, 256>>>(keys, n, counts, ranks, si, so);
                if (mode == 3) k_atom<3><<<grid, 256>>>(keys, n, counts, ranks, si, so);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            }
            printf("sigma %5.1f rows mode %d (%s) grid %s: %8.1f us\n", sig[si_], mode,
                   mode == 0 ? "atom+ret" : mode == 1 ? "red" : mode == 2 ? "atom+ret+stream 640MB" : "stream only",
                   persist ? "persistent" : "full", ms * 1e3);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
