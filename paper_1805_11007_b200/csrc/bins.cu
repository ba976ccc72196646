// bins.cu -- cell-list construction on the device.
//
// Reference: motion.py:170-199 (_soft_forces_fused binning sweep): flat cell
// f = cy * n0 + cx of cells of side size/n >= cutoff, counting sort into a
// stable `order` (ascending particle index within a cell) and CSR `starts`.
//
// Device pipeline (all int32; N and the cell count stay below 2^31):
//   k_bin_count    key[i] = f(pos[i]); counts[key]++           (atomics in L2)
//   k_scan         starts = exclusive_scan(counts)             (single pass,
//                  decoupled look-back; starts[nflat] = N)
//   k_bin_scatter  slot = starts[key] + (--counts[key]); order[slot] = i
//                  (the decrement leaves counts all-zero for the next step,
//                  so no memset pass over the cell table is ever needed)
//   k_seg_sort     restore ascending index inside each cell (cells hold a
//                  handful of particles, insertion sort is exact and cheap)
// The result is bit-identical to the reference's `order`/`starts`.
#include "common.cuh"

namespace cs {

template <class P>
__global__ void k_bin_count(const P *__restrict__ pos, long long n, BinGeom g,
                            int *__restrict__ keys, int *__restrict__ counts) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x, y;
        load2(pos, i, x, y);
        const int c0 = cell_axis(x, g.lo0, g.eff0, g.n0);
        const int c1 = cell_axis(y, g.lo1, g.eff1, g.n1);
        const int key = c1 * g.n0 + c0;
        keys[i] = key;
        atomicAdd(&counts[key], 1);
    }
}

__global__ void k_bin_scatter(const int *__restrict__ keys, long long n,
                              const int *__restrict__ starts, int *__restrict__ counts,
                              int *__restrict__ order, int *__restrict__ skeys) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int key = keys[i];
        const int slot = starts[key] + atomicSub(&counts[key], 1) - 1;
        order[slot] = (int)i;
        skeys[slot] = key;
    }
}

__global__ void k_seg_sort(int *__restrict__ order, const int *__restrict__ skeys, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int key = skeys[t];
        if (t > 0 && skeys[t - 1] == key) continue;
        long long end = t + 1;
        while (end < n && skeys[end] == key) end++;
        if (end - t < 2) continue;
        for (long long a = t + 1; a < end; a++) {
            const int v = order[a];
            long long b = a - 1;
            while (b >= t && order[b] > v) {
                order[b + 1] = order[b];
                b--;
            }
            order[b + 1] = v;
        }
    }
}

// ------------------------------------------------------------------ scan
// Single-pass exclusive scan with decoupled look-back.  Tile = BLOCK*ITEMS
// consecutive counts; each tile publishes (status, value) packed in one
// 64-bit word: status 1 = local aggregate, 2 = inclusive prefix.
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(SCAN_BLOCK)
k_scan(const int *__restrict__ in, int *__restrict__ out, long long n,
       unsigned long long *__restrict__ flags, unsigned int *__restrict__ tile_counter) {
    __shared__ unsigned int s_tile;
    __shared__ int s_warp[SCAN_BLOCK / 32];
    __shared__ int s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long base = tile * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int tsum = 0;
    if (base + SCAN_ITEMS <= n) {
        const int4 a = *reinterpret_cast<const int4 *>(in + base);
        const int4 b = *reinterpret_cast<const int4 *>(in + base + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) v[k] = (base + k < n) ? in[base + k] : 0;
    }
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) tsum += v[k];
    // block exclusive scan of thread sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < SCAN_BLOCK / 32 ? s_warp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < SCAN_BLOCK / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
        if (lane == SCAN_BLOCK / 32 - 1) {
            const int total = wi;
            // publish and look back (single thread)
            int prefix = 0;
            if (tile == 0) {
                st_release(&flags[0], (2ULL << 32) | (unsigned)total);
            } else {
                st_release(&flags[tile], (1ULL << 32) | (unsigned)total);
                long long j = tile - 1;
                while (true) {
                    const unsigned long long f = ld_acquire(&flags[j]);
                    const unsigned s = (unsigned)(f >> 32);
                    if (s == 0) continue;
                    prefix += (int)(unsigned)(f & 0xffffffffu);
                    if (s == 2) break;
                    j--;
                }
                st_release(&flags[tile], (2ULL << 32) | (unsigned)(prefix + total));
            }
            s_prefix = prefix;
        }
    }
    __syncthreads();
    int run = s_prefix + s_warp[warp] + (incl - tsum);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (base < n && base + SCAN_ITEMS >= n) out[n] = run;  // starts[nflat] = total
}

int exclusive_scan_i32(cs_ctx *ctx, const int *in, int *out, long long n) {
    const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    CS_TRY(ctx->tile_flags.ensure(sizeof(unsigned long long) * (tiles + 2)));
    unsigned long long *flags = ctx->tile_flags.as<unsigned long long>();
    CS_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * (tiles + 2), ctx->stream));
    unsigned int *counter = reinterpret_cast<unsigned int *>(flags + tiles + 1);
    if (n == 0) {
        CS_CUDA(cudaMemsetAsync(out, 0, sizeof(int), ctx->stream));
        return CS_OK;
    }
    k_scan<<<(unsigned)tiles, SCAN_BLOCK, 0, ctx->stream>>>(in, out, n, flags, counter);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// ------------------------------------------------------------------ driver
int bin_particles(cs_ctx *ctx, int prec, const void *pos, long long n, const BinGeom &g) {
    const long long nflat = (long long)g.n0 * g.n1;
    if (nflat >= (1LL << 31) - 1) {
        set_error("cell table too large (%lld cells)", nflat);
        return CS_ERR_PARAM;
    }
    const size_t nb = sizeof(int) * (size_t)(n > 0 ? n : 1);
    CS_TRY(ctx->keys.ensure(nb));
    CS_TRY(ctx->skeys.ensure(nb));
    CS_TRY(ctx->order.ensure(nb));
    CS_TRY(ctx->starts.ensure(sizeof(int) * (size_t)(nflat + 1)));
    const size_t cb = sizeof(int) * (size_t)nflat;
    if (ctx->counts.bytes < cb) {
        CS_TRY(ctx->counts.ensure(cb));
        CS_CUDA(cudaMemsetAsync(ctx->counts.p, 0, ctx->counts.bytes, ctx->stream));
    }
    int *keys = ctx->keys.as<int>(), *counts = ctx->counts.as<int>();
    int *starts = ctx->starts.as<int>(), *order = ctx->order.as<int>();
    const int B = 256;
    if (n > 0) {
        if (prec == CS_F64)
            k_bin_count<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const double *>(pos), n, g, keys, counts);
        else
            k_bin_count<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const float *>(pos), n, g, keys, counts);
        CS_LAUNCH_CHECK();
    }
    CS_TRY(exclusive_scan_i32(ctx, counts, starts, nflat));
    if (n > 0) {
        k_bin_scatter<<<grid_for(n, B), B, 0, ctx->stream>>>(keys, n, starts, counts, order,
                                                             ctx->skeys.as<int>());
        CS_LAUNCH_CHECK();
        k_seg_sort<<<grid_for(n, B), B, 0, ctx->stream>>>(order, ctx->skeys.as<int>(), n);
        CS_LAUNCH_CHECK();
    }
    ctx->launches += 3;
    return CS_OK;
}

}  // namespace cs
