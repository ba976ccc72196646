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
//   k_bin_scatter  slot = starts[key] + (--counts[key]); slots[slot] = i
//                  (the decrement leaves counts all-zero for the next step,
//                  so no memset pass over the cell table is ever needed)
//   k_seg_rank     order[start + rank] = slots[t], rank = the number of the
//                  cell's particles with a smaller index (ascending index
//                  inside each cell, as the reference's stable sort)
// The result is bit-identical to the reference's `order`/`starts`.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "deposit.cuh"
#include "scan.cuh"

namespace cs {

// keys[i] = cell of particle i; with a DepBin also keys[n + i] = nflat +
// its deposit bin (-1: not depositing) -- one count array for both
template <class P, bool DEP>
__global__ void k_bin_count(const P *__restrict__ pos, long long n, BinGeom g,
                            int *__restrict__ keys, int *__restrict__ counts,
                            const uint8_t *__restrict__ type, DepBin dep) {
    const int nflat = g.n0 * g.n1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x, y;
        load2(pos, i, x, y);
        const int c0 = cell_axis(x, g.lo0, g.eff0, g.n0);
        const int c1 = cell_axis(y, g.lo1, g.eff1, g.n1);
        const int key = c1 * g.n0 + c0;
        keys[i] = key;
        atomicAdd(&counts[key], 1);
        if (DEP) {
            int dk = -1;
            if (route_bits(type, i, dep.route)) {
                const GridGeom &gg = dep.gg;
                const double u0 = ddiv(dsub(x, gg.lo0), gg.d0);
                const double u1 = ddiv(dsub(y, gg.lo1), gg.d1);
                if (fabs(u0) < 0x1p52 && fabs(u1) < 0x1p52) {
                    dk = nflat + dep_bin_axis(u1, dep.kind, gg.n, gg.per) * gg.n +
                         dep_bin_axis(u0, dep.kind, gg.n, gg.per);
                    atomicAdd(&counts[dk], 1);
                }
            }
            keys[n + i] = dk;
        }
    }
}

template <bool DEP>
__global__ void k_bin_scatter(const int *__restrict__ keys, long long n,
                              const int *__restrict__ starts, int *__restrict__ counts,
                              int *__restrict__ slots) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int key = keys[i];
        slots[starts[key] + atomicSub(&counts[key], 1) - 1] = (int)i;
        if (DEP) {
            const int dk = keys[n + i];
            if (dk >= 0) slots[starts[dk] + atomicSub(&counts[dk], 1) - 1] = (int)i;
        }
    }
}

// Stable placement: the particle in slot t (cell order, arbitrary inside a
// cell) goes to its cell start + the number of the cell's particles with a
// smaller index (O(m) reads of the cell's L1-resident slots per particle).
// Deposit slots (t >= n, with a DepBin) are ranked the same way inside
// their bin; the particle's position and (index, route) word are copied to
// dpos / dmeta at t - n.
template <class P, bool DEP>
__global__ void k_seg_rank(const int *__restrict__ slots, const int *__restrict__ keys,
                           const int *__restrict__ starts, long long n, int *__restrict__ order,
                           const P *__restrict__ pos, const uint8_t *__restrict__ type,
                           P *__restrict__ spos, uint8_t *__restrict__ stype, int nall,
                           P *__restrict__ dpos, unsigned *__restrict__ dmeta, Route route) {
    const long long total = DEP ? (long long)starts[nall] : n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = slots[t];
        const bool dep = DEP && t >= n;
        const int key = dep ? keys[n + v] : keys[v];
        const int s = starts[key], e = starts[key + 1];
        int rank = 0;
        for (int u = s; u < e; u++) rank += __ldg(slots + u) < v;
        if (dep) {
            const long long d = s + rank - n;
            reinterpret_cast<typename Vec2<P>::T *>(dpos)[d] =
                reinterpret_cast<const typename Vec2<P>::T *>(pos)[v];
            dmeta[d] = (unsigned)v | (route_bits(type, v, route) << 30);
            continue;
        }
        order[s + rank] = v;
        spos[2 * (s + rank)] = pos[2 * (long long)v];
        spos[2 * (s + rank) + 1] = pos[2 * (long long)v + 1];
        if (type) stype[s + rank] = type[v];
    }
}

// Mid-size systems (cfg1: 10^4 particles, 10^4 cells + 128^2 deposit bins;
// cfg2: 10^5 particles) are bound by the four dependent launches above, each
// a few microseconds of work: k_bin_coop runs the same four phases in ONE
// cooperative launch with grid-wide barriers between them.  The scan is two
// level: every block sums its contiguous segment of the counts, all blocks
// scan the block sums (at most a few hundred) and then their own segment.
// Same keys, starts, order and deposit lists as the multi-kernel path.
constexpr int BIN_COOP_THREADS = 256;

template <class P, bool DEP>
__global__ void __launch_bounds__(BIN_COOP_THREADS)
k_bin_coop(const P *__restrict__ pos, long long n, BinGeom g, int *__restrict__ keys,
           int *__restrict__ counts, int *__restrict__ starts, int *__restrict__ slots,
           int *__restrict__ order, const uint8_t *__restrict__ type, P *__restrict__ spos,
           uint8_t *__restrict__ stype, DepBin dep, int nall, P *__restrict__ dpos,
           unsigned *__restrict__ dmeta, int *__restrict__ block_sums) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int nflat = g.n0 * g.n1;
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gstride = (long long)gridDim.x * blockDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ int s_w[BIN_COOP_THREADS / 32];
    // segment of the count array each block scans
    const int seg = (nall + gridDim.x - 1) / gridDim.x;
    // ---- keys and counts (k_bin_count)
    for (long long i = gtid; i < n; i += gstride) {
        double x, y;
        load2(pos, i, x, y);
        const int key = cell_axis(y, g.lo1, g.eff1, g.n1) * g.n0 + cell_axis(x, g.lo0, g.eff0, g.n0);
        keys[i] = key;
        atomicAdd(&counts[key], 1);
        if (DEP) {
            int dk = -1;
            if (route_bits(type, i, dep.route)) {
                const GridGeom &gg = dep.gg;
                const double u0 = ddiv(dsub(x, gg.lo0), gg.d0);
                const double u1 = ddiv(dsub(y, gg.lo1), gg.d1);
                if (fabs(u0) < 0x1p52 && fabs(u1) < 0x1p52) {
                    dk = nflat + dep_bin_axis(u1, dep.kind, gg.n, gg.per) * gg.n +
                         dep_bin_axis(u0, dep.kind, gg.n, gg.per);
                    atomicAdd(&counts[dk], 1);
                }
            }
            keys[n + i] = dk;
        }
    }
    grid.sync();
    // ---- exclusive scan of counts[0, nall) -> starts (starts[nall] = total)
    const int s0 = min((int)blockIdx.x * seg, nall), s1 = min(s0 + seg, nall);
    auto block_sum = [&](int v) {  // sum of v over the block, in every thread
        __syncthreads();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_w[warp] = v;
        __syncthreads();
        int t = 0;
#pragma unroll
        for (int w = 0; w < BIN_COOP_THREADS / 32; w++) t += s_w[w];
        return t;
    };
    {
        int part = 0;
        for (int c = s0 + tid; c < s1; c += BIN_COOP_THREADS) part += counts[c];
        const int tot = block_sum(part);
        if (tid == 0) block_sums[blockIdx.x] = tot;
    }
    grid.sync();
    {
        int part = 0;  // counts of the segments before this block's
        for (int b = tid; b < (int)blockIdx.x; b += BIN_COOP_THREADS) part += block_sums[b];
        int carry = block_sum(part);
        if (blockIdx.x == gridDim.x - 1) {
            int all = 0;
            for (int b = tid; b < (int)gridDim.x; b += BIN_COOP_THREADS) all += block_sums[b];
            all = block_sum(all);
            if (tid == 0) starts[nall] = all;
        }
        for (int c0 = s0; c0 < s1; c0 += BIN_COOP_THREADS) {  // tiles of the segment, in order
            const int c = c0 + tid;
            const int v = c < s1 ? counts[c] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            __syncthreads();
            if (lane == 31) s_w[warp] = inc;
            __syncthreads();
            int wb = 0, tile = 0;
#pragma unroll
            for (int w = 0; w < BIN_COOP_THREADS / 32; w++) {
                wb += w < warp ? s_w[w] : 0;
                tile += s_w[w];
            }
            if (c < s1) starts[c] = carry + wb + inc - v;
            carry += tile;
        }
    }
    grid.sync();
    // ---- unordered placement into the cell / bin ranges (k_bin_scatter); the
    // countdown leaves counts all-zero for the next call
    for (long long i = gtid; i < n; i += gstride) {
        const int key = keys[i];
        slots[starts[key] + atomicSub(&counts[key], 1) - 1] = (int)i;
        if (DEP) {
            const int dk = keys[n + i];
            if (dk >= 0) slots[starts[dk] + atomicSub(&counts[dk], 1) - 1] = (int)i;
        }
    }
    grid.sync();
    // ---- stable order inside a cell / bin and the sorted copies (k_seg_rank)
    const long long total = DEP ? (long long)starts[nall] : n;
    for (long long t = gtid; t < total; t += gstride) {
        const int v = slots[t];
        const bool isdep = DEP && t >= n;
        const int key = isdep ? keys[n + v] : keys[v];
        const int sb = starts[key], se = starts[key + 1];
        int rank = 0;
        for (int u = sb; u < se; u++) rank += slots[u] < v;
        if (isdep) {
            const long long d = sb + rank - n;
            reinterpret_cast<typename Vec2<P>::T *>(dpos)[d] =
                reinterpret_cast<const typename Vec2<P>::T *>(pos)[v];
            dmeta[d] = (unsigned)v | (route_bits(type, v, dep.route) << 30);
            continue;
        }
        order[sb + rank] = v;
        spos[2 * (sb + rank)] = pos[2 * (long long)v];
        spos[2 * (sb + rank) + 1] = pos[2 * (long long)v + 1];
        if (type) stype[sb + rank] = type[v];
    }
}

// Small systems (cfg0: 10^3 particles, 10^4 cells) are launch-bound: one
// 1024-thread block does the whole sweep in shared memory -- keys and
// histogram, exclusive scan into `starts`, an unordered placement by
// shared-memory claims, then the stable order: each particle goes to its
// cell start + the number of the cell's particles with a smaller index
// (as k_seg_rank).  Same order / starts as the multi-kernel path.
constexpr int BIN_SMALL_THREADS = 1024;
constexpr int BIN_SMALL_MAX_CELLS = 12 * 1024;
constexpr long long BIN_SMALL_MAX_N = 4 * 1024;

template <class P>
__global__ void __launch_bounds__(BIN_SMALL_THREADS)
k_bin_small(const P *__restrict__ pos, int n, BinGeom g, int *__restrict__ starts,
            int *__restrict__ order, const uint8_t *__restrict__ type, P *__restrict__ spos,
            uint8_t *__restrict__ stype) {
    extern __shared__ int sm[];
    const int nflat = g.n0 * g.n1;
    int *cnt = sm;                 // nflat + 1: counts, then starts
    int *fill = cnt + nflat + 1;   // nflat: claim cursors
    int *keys = fill + nflat;      // n
    int *slots = keys + n;         // n: particle of each slot, unordered in a cell
    __shared__ int wsum[BIN_SMALL_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int c = tid; c <= nflat; c += BIN_SMALL_THREADS) cnt[c] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += BIN_SMALL_THREADS) {
        double x, y;
        load2(pos, i, x, y);
        const int key = cell_axis(y, g.lo1, g.eff1, g.n1) * g.n0 + cell_axis(x, g.lo0, g.eff0, g.n0);
        keys[i] = key;
        atomicAdd(&cnt[key], 1);
    }
    __syncthreads();
    // exclusive scan of cnt[0, nflat): per-thread run, block scan of the sums
    const int per = (nflat + BIN_SMALL_THREADS - 1) / BIN_SMALL_THREADS;
    const int c0 = tid * per, c1 = min(c0 + per, nflat);
    int run = 0;
    for (int c = c0; c < c1; c++) run += cnt[c];
    int inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    int acc = inc - run + (warp > 0 ? wsum[warp - 1] : 0);
    for (int c = c0; c < c1; c++) {
        const int v = cnt[c];
        cnt[c] = acc;
        fill[c] = acc;
        starts[c] = acc;
        acc += v;
    }
    if (tid == 0) {
        cnt[nflat] = n;
        starts[nflat] = n;
    }
    __syncthreads();
    for (int i = tid; i < n; i += BIN_SMALL_THREADS) slots[atomicAdd(&fill[keys[i]], 1)] = i;
    __syncthreads();
    for (int t = tid; t < n; t += BIN_SMALL_THREADS) {
        const int v = slots[t];
        const int key = keys[v];
        const int s0 = cnt[key], s1 = cnt[key + 1];
        int rank = 0;
        for (int u = s0; u < s1; u++) rank += slots[u] < v;
        order[s0 + rank] = v;
    }
    __syncthreads();  // the block's order writes are visible to the block
    for (int k = tid; k < n; k += BIN_SMALL_THREADS) {  // coalesced stores of the copies
        const int v = order[k];
        spos[2 * k] = pos[2 * (long long)v];
        spos[2 * k + 1] = pos[2 * (long long)v + 1];
        if (type) stype[k] = type[v];
    }
}

// ------------------------------------------------------------------ scan
int exclusive_scan_i32(cs_ctx *ctx, const int *in, int *out, long long n, int *zero_in) {
    const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    CS_TRY(ctx->tile_flags.ensure(sizeof(unsigned long long) * (tiles + 2)));
    unsigned long long *flags = ctx->tile_flags.as<unsigned long long>();
    CS_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned long long) * (tiles + 2), ctx->stream));
    unsigned int *counter = reinterpret_cast<unsigned int *>(flags + tiles + 1);
    if (n == 0) {
        CS_CUDA(cudaMemsetAsync(out, 0, sizeof(int), ctx->stream));
        return CS_OK;
    }
    k_scan<<<(unsigned)tiles, SCAN_BLOCK, 0, ctx->stream>>>(in, out, n, flags, counter, zero_in);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// ------------------------------------------------------------------ driver
template <class P, bool DEP>
static void bin_launch(cs_ctx *ctx, const P *pos, long long n, const BinGeom &g,
                       const uint8_t *type, const DepBin &dep, int nall, int phase) {
    const int B = 256;
    int *keys = ctx->keys.as<int>(), *counts = ctx->counts.as<int>();
    int *starts = ctx->starts.as<int>();
    if (phase == 0)
        k_bin_count<P, DEP><<<grid_for(n, B), B, 0, ctx->stream>>>(pos, n, g, keys, counts, type,
                                                                    dep);
    else if (phase == 1)
        k_bin_scatter<DEP><<<grid_for(n, B), B, 0, ctx->stream>>>(keys, n, starts, counts,
                                                                  ctx->skeys.as<int>());
    else
        k_seg_rank<P, DEP><<<grid_for(DEP ? 2 * n : n, B), B, 0, ctx->stream>>>(
            ctx->skeys.as<int>(), keys, starts, n, ctx->order.as<int>(), pos, type,
            ctx->spos.as<P>(), ctx->stype.as<uint8_t>(), nall, ctx->dep_pos.as<P>(),
            ctx->dep_meta.as<unsigned>(), dep.route);
}

int bin_particles(cs_ctx *ctx, int prec, const void *pos, long long n, const BinGeom &g,
                  const uint8_t *type, const DepBin *dep, bool *dep_done) {
    if (dep_done) *dep_done = false;
    const long long nflat = (long long)g.n0 * g.n1;
    const long long nb = dep ? (long long)dep->gg.n * dep->gg.n : 0;
    const long long nall = nflat + nb;
    if (nall >= (1LL << 31) - 1 || (dep && 2 * n >= (1LL << 31) - 1)) {
        set_error("cell table too large (%lld cells)", nall);
        return CS_ERR_PARAM;
    }
    const size_t np = (size_t)(n > 0 ? n : 1);
    CS_TRY(ctx->order.ensure(sizeof(int) * np));
    CS_TRY(ctx->spos.ensure((prec == CS_F64 ? 16 : 8) * np));
    CS_TRY(ctx->stype.ensure(np));
    uint8_t *stype = ctx->stype.as<uint8_t>();
    if (n <= BIN_SMALL_MAX_N && nflat <= BIN_SMALL_MAX_CELLS && !getenv("CS_BIN_MULTI")) {
        CS_TRY(ctx->starts.ensure(sizeof(int) * (size_t)(nflat + 1)));
        int *starts = ctx->starts.as<int>(), *order = ctx->order.as<int>();
        const size_t smem = sizeof(int) * (size_t)(2 * nflat + 1 + 2 * n);
        static size_t smem_set = 0;
        if (smem > smem_set) {
            CS_CUDA(cudaFuncSetAttribute(k_bin_small<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CS_CUDA(cudaFuncSetAttribute(k_bin_small<float>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            smem_set = smem;
        }
        if (prec == CS_F64)
            k_bin_small<double><<<1, BIN_SMALL_THREADS, smem, ctx->stream>>>(
                static_cast<const double *>(pos), (int)n, g, starts, order, type,
                ctx->spos.as<double>(), stype);
        else
            k_bin_small<float><<<1, BIN_SMALL_THREADS, smem, ctx->stream>>>(
                static_cast<const float *>(pos), (int)n, g, starts, order, type,
                ctx->spos.as<float>(), stype);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
        return CS_OK;
    }
    const size_t nk = dep ? 2 * np : np;
    CS_TRY(ctx->keys.ensure(sizeof(int) * nk));
    CS_TRY(ctx->skeys.ensure(sizeof(int) * nk));
    CS_TRY(ctx->starts.ensure(sizeof(int) * (size_t)(nall + 1)));
    if (dep) {
        CS_TRY(ctx->dep_pos.ensure((prec == CS_F64 ? 16 : 8) * np));
        CS_TRY(ctx->dep_meta.ensure(sizeof(unsigned) * np));
    }
    const size_t cb = sizeof(int) * (size_t)nall;
    if (ctx->counts.bytes < cb) {  // kept all-zero between calls (the scatter counts down)
        CS_TRY(ctx->counts.ensure(cb));
        CS_CUDA(cudaMemsetAsync(ctx->counts.p, 0, ctx->counts.bytes, ctx->stream));
    }
    const DepBin none{};
    const DepBin &d = dep ? *dep : none;
    if (n > 0 && n <= (1LL << 16) && !getenv("CS_BIN_MULTI")) {  // (10^5: no faster, measured)
        // one cooperative launch; every block resident (grid-wide barriers)
        static int coop_blocks = 0;
        if (!coop_blocks) {
            int dev = 0, sms = 0, coop = 0, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bin_coop<double, true>,
                                                          BIN_COOP_THREADS, 0);
            coop_blocks = coop && per > 0 ? sms * (per > 2 ? 2 : per) : -1;
        }
        if (coop_blocks > 0) {
            CS_TRY(ctx->coop_sums.ensure(sizeof(int) * (size_t)coop_blocks));  // segment totals
            int grid = grid_for(dep ? 2 * n : n, BIN_COOP_THREADS, coop_blocks);
            int *keys = ctx->keys.as<int>(), *counts = ctx->counts.as<int>();
            int *starts = ctx->starts.as<int>(), *slots = ctx->skeys.as<int>();
            int *order = ctx->order.as<int>(), *bsums = ctx->coop_sums.as<int>();
            int nall_i = (int)nall;
            long long nn = n;
            BinGeom gv = g;
            DepBin dv = d;
            const void *fn;
            void *spos = ctx->spos.p, *dpos = ctx->dep_pos.p;
            unsigned *dmeta = ctx->dep_meta.as<unsigned>();
            if (prec == CS_F64)
                fn = dep ? (const void *)k_bin_coop<double, true> : (const void *)k_bin_coop<double, false>;
            else
                fn = dep ? (const void *)k_bin_coop<float, true> : (const void *)k_bin_coop<float, false>;
            void *args[] = {(void *)&pos, &nn, &gv, &keys, &counts, &starts, &slots, &order,
                            (void *)&type, &spos, &stype, &dv, &nall_i, &dpos, &dmeta, &bsums};
            CS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BIN_COOP_THREADS), args, 0,
                                                ctx->stream));
            ctx->launches += 1;
            if (dep_done) *dep_done = dep != nullptr;
            return CS_OK;
        }
    }
    for (int phase = 0; phase < 3; phase++) {
        if (phase == 1) CS_TRY(exclusive_scan_i32(ctx, ctx->counts.as<int>(),
                                                  ctx->starts.as<int>(), nall));
        if (n == 0) continue;
        if (prec == CS_F64) {
            if (dep) bin_launch<double, true>(ctx, static_cast<const double *>(pos), n, g, type, d,
                                              (int)nall, phase);
            else bin_launch<double, false>(ctx, static_cast<const double *>(pos), n, g, type, d,
                                           (int)nall, phase);
        } else {
            if (dep) bin_launch<float, true>(ctx, static_cast<const float *>(pos), n, g, type, d,
                                             (int)nall, phase);
            else bin_launch<float, false>(ctx, static_cast<const float *>(pos), n, g, type, d,
                                          (int)nall, phase);
        }
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    if (dep_done) *dep_done = dep != nullptr;
    return CS_OK;
}

}  // namespace cs
