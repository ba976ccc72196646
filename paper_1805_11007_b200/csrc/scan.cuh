// scan.cuh -- single-pass exclusive scan (int32) with decoupled look-back.
//
// Tile = SCAN_BLOCK * SCAN_VEC * 4 counts (8192 by default), SCAN_BLOCK
// threads; thread t owns the int4 chunks at (k*SCAN_BLOCK + t) for
// k < SCAN_VEC (all loads in flight together), so every load/store
// instruction of a warp is one contiguous 512-B segment.  Each tile publishes (status, value) packed in
// one 64-bit word: status 1 = local aggregate, 2 = inclusive prefix; warp 0
// looks back over 32 predecessors at a time.  out[n] receives the total.
#pragma once
#include "common.cuh"

namespace cs {

#ifndef CS_SCAN_BLOCK
#define CS_SCAN_BLOCK 256
#endif
constexpr int SCAN_BLOCK = CS_SCAN_BLOCK;
#ifndef CS_SCAN_VEC
#define CS_SCAN_VEC 8  // measured at 16.4 M cells: 4: 68.5 us, 8: 53.8, 16: 56.7
#endif
constexpr int SCAN_VEC = CS_SCAN_VEC;  // int4 chunks per thread
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_VEC * 4;

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
       unsigned long long *__restrict__ flags, unsigned int *__restrict__ tile_counter,
       int *__restrict__ zero_in = nullptr) {
    __shared__ unsigned int s_tile;
    __shared__ int s_part[SCAN_VEC][SCAN_BLOCK / 32];
    __shared__ int s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const long long tile = s_tile;
    const long long tbase = tile * SCAN_TILE;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int4 v[SCAN_VEC];
#pragma unroll
    for (int k = 0; k < SCAN_VEC; k++) {
        const long long e = tbase + (long long)(k * SCAN_BLOCK + t) * 4;
        if (e + 4 <= n) {
            v[k] = __ldcs(reinterpret_cast<const int4 *>(in + e));
        } else {
            v[k].x = e < n ? in[e] : 0;
            v[k].y = e + 1 < n ? in[e + 1] : 0;
            v[k].z = e + 2 < n ? in[e + 2] : 0;
            v[k].w = e + 3 < n ? in[e + 3] : 0;
        }
    }
    int excl[SCAN_VEC];
#pragma unroll
    for (int k = 0; k < SCAN_VEC; k++) {
        const int s = v[k].x + v[k].y + v[k].z + v[k].w;
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        excl[k] = inc - s;
        if (lane == 31) s_part[k][warp] = inc;
    }
    __syncthreads();
    if (warp == 0) {
        // tile order: chunk k major, then warp, then lane; lane l owns the
        // R consecutive partials l*R .. l*R+R-1
        constexpr int NW = SCAN_BLOCK / 32;
        constexpr int NP = SCAN_VEC * NW;
        constexpr int R = (NP + 31) / 32;
        int pv[R];
        int val = 0;
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int q = lane * R + r;
            pv[r] = q < NP ? s_part[q / NW][q % NW] : 0;
            val += pv[r];
        }
        int inc = val;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        __syncwarp();
        int run = inc - val;
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int q = lane * R + r;
            if (q < NP) s_part[q / NW][q % NW] = run;
            run += pv[r];
        }
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        int prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_release(&flags[0], (2ULL << 32) | (unsigned)total);
        } else {
            if (lane == 0) st_release(&flags[tile], (1ULL << 32) | (unsigned)total);
            long long j = tile - 1;
            while (true) {
                const long long idx = j - lane;
                unsigned long long f = idx >= 0 ? ld_acquire(&flags[idx]) : (2ULL << 32);
                unsigned st = (unsigned)(f >> 32);
                while (__any_sync(0xffffffffu, st == 0)) {
                    if (st == 0) {
                        f = ld_acquire(&flags[idx]);
                        st = (unsigned)(f >> 32);
                    }
                }
                const unsigned pmask = __ballot_sync(0xffffffffu, st == 2);
                const int first_p = pmask ? __ffs(pmask) - 1 : 32;
                int v2 = (lane <= first_p && idx >= 0) ? (int)(unsigned)(f & 0xffffffffu) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v2 += __shfl_xor_sync(0xffffffffu, v2, o);
                prefix += v2;
                if (pmask) break;
                j -= 32;
            }
            if (lane == 0) st_release(&flags[tile], (2ULL << 32) | (unsigned)(prefix + total));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    const int prefix = s_prefix;
#pragma unroll
    for (int k = 0; k < SCAN_VEC; k++) {
        const long long e = tbase + (long long)(k * SCAN_BLOCK + t) * 4;
        int run = prefix + s_part[k][warp] + excl[k];
        int4 o;
        o.x = run;
        run += v[k].x;
        o.y = run;
        run += v[k].y;
        o.z = run;
        run += v[k].z;
        o.w = run;
        run += v[k].w;
        if (e + 4 <= n) {
            *reinterpret_cast<int4 *>(out + e) = o;
        } else {
            if (e < n) out[e] = o.x;
            if (e + 1 < n) out[e + 1] = o.y;
            if (e + 2 < n) out[e + 2] = o.z;
            if (e + 3 < n) out[e + 3] = o.w;
        }
        if (e < n && e + 4 >= n) out[n] = run;
        // reset the histogram for the next step; the loaded values have been
        // consumed above, so these stores do not race their own loads
        if (zero_in) {
            if (e + 4 <= n) {
                *reinterpret_cast<int4 *>(zero_in + e) = make_int4(0, 0, 0, 0);
            } else {
                for (int q = 0; q < 4; q++)
                    if (e + q < n) zero_in[e + q] = 0;
            }
        }
    }
}

}  // namespace cs
