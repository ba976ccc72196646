// observe.cu -- a realisation's observables on the device, in numpy's
// arithmetic (engine.py:230-235 msd, :317-352 the recording; numpy's
// pairwise summation and histogram2d binning restated).
//
//   msd:   mean over particles of (0 + dx^2) + dy^2, dx = pos - anchor in
//          binary64 -- numpy's add.reduce over the contiguous squares is the
//          pairwise sum of loops_utils.h.src (< 8 terms in order from -0.0,
//          <= 128 in 8 interleaved accumulators, beyond that split at n / 2
//          rounded down to a multiple of 8).  The recursion tree is cut at
//          depth MSD_D: every subtree below is summed by one thread with the
//          same recursion, the top of the tree is re-walked by one thread
//          over those partial sums: the association is numpy's exactly.
//   hist:  numpy.histogram2d(x, y, bins, range) of one species: bin index =
//          searchsorted(edges, v, 'right') (edges = numpy's linspace, passed
//          in), a value on the last edge moved into the last bin, outliers
//          dropped; counts stored transposed ([y bin][x bin]) as engine.py's
//          h.T; per_sample > 0 bins the samples of a batched ensemble (sample
//          = index / per_sample) into consecutive b x b blocks.
#include "common.cuh"

namespace cs {

constexpr int MSD_D = 10;  // 1024 subtrees

__device__ double obs_pairwise(const double *v, long long n) {
    if (n < 8) {
        double res = -0.0;
        for (long long i = 0; i < n; i++) res = dadd(res, v[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int q = 0; q < 8; q++) r[q] = v[q];
        long long i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int q = 0; q < 8; q++) r[q] = dadd(r[q], v[i + q]);
        double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                          dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
        for (; i < n; i++) res = dadd(res, v[i]);
        return res;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    return dadd(obs_pairwise(v, n2), obs_pairwise(v + n2, n - n2));
}

template <class P>
__global__ void k_sq_disp(const P *__restrict__ pos, const P *__restrict__ anchor, long long n,
                          double *__restrict__ sq) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double d0 = dsub((double)pos[2 * i], (double)anchor[2 * i]);
        const double d1 = dsub((double)pos[2 * i + 1], (double)anchor[2 * i + 1]);
        sq[i] = dadd(dadd(-0.0, dmul(d0, d0)), dmul(d1, d1));
    }
}

// subtree k (the path bits of k from the root, MSD_D levels): its range, or
// a leaf reached earlier (computed only by the thread whose remaining bits
// are zero); partial[k] = its pairwise sum
__global__ void k_msd_subtrees(const double *__restrict__ sq, long long n,
                               double *__restrict__ partial) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (1 << MSD_D)) return;
    long long off = 0, len = n;
    for (int d = 0; d < MSD_D; d++) {
        if (len <= 128) {
            if (k & ((1 << (MSD_D - d)) - 1)) return;  // another thread's copy of this leaf
            break;
        }
        long long n2 = len / 2;
        n2 -= n2 % 8;
        if ((k >> (MSD_D - 1 - d)) & 1) {
            off += n2;
            len -= n2;
        } else {
            len = n2;
        }
    }
    partial[k] = obs_pairwise(sq + off, len);
}

__device__ double msd_top(const double *partial, long long len, int d, int path) {
    if (len <= 128 || d == MSD_D) return partial[path << (MSD_D - d)];
    long long n2 = len / 2;
    n2 -= n2 % 8;
    return dadd(msd_top(partial, n2, d + 1, path << 1),
                msd_top(partial, len - n2, d + 1, (path << 1) | 1));
}

__global__ void k_msd_finish(const double *__restrict__ partial, long long n, double *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    *out = ddiv(msd_top(partial, n, 0, 0), (double)n);
}

template <class P>
__global__ void k_hist2d(const P *__restrict__ pos, const uint8_t *__restrict__ type, long long n,
                         int sp, const double *__restrict__ ex, const double *__restrict__ ey,
                         int b, long long per, unsigned long long *__restrict__ counts) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (sp >= 0 && type[i] != sp) continue;
        const double x = (double)pos[2 * i], y = (double)pos[2 * i + 1];
        int ix = 0, iy = 0;  // searchsorted(edges, v, 'right') = #edges <= v
        for (int e = 0; e <= b; e++) {
            ix += ex[e] <= x;
            iy += ey[e] <= y;
        }
        if (x == ex[b]) ix -= 1;
        if (y == ey[b]) iy -= 1;
        if (ix < 1 || ix > b || iy < 1 || iy > b) continue;
        const long long smp = per > 0 ? i / per : 0;  // sample of a batched ensemble
        atomicAdd(&counts[(smp * b + (iy - 1)) * b + (ix - 1)], 1ull);
    }
}

}  // namespace cs

extern "C" {

int cs_msd(cs_ctx *ctx, int32_t prec, const void *pos, const void *anchor, int64_t n,
           double *out) {
    using namespace cs;
    if (n < 1) {
        set_error("msd of an empty population");
        return CS_ERR_PARAM;
    }
    if (prec != CS_F64 && prec != CS_F32) {
        set_error("prec must be CS_F64 or CS_F32");
        return CS_ERR_PARAM;
    }
    CS_TRY(ctx->obs.ensure(sizeof(double) * ((size_t)n + (1 << MSD_D))));
    double *sq = ctx->obs.as<double>();
    double *partial = sq + n;
    if (prec == CS_F64)
        k_sq_disp<double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const double *>(pos), static_cast<const double *>(anchor), n, sq);
    else
        k_sq_disp<float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const float *>(pos), static_cast<const float *>(anchor), n, sq);
    CS_LAUNCH_CHECK();
    k_msd_subtrees<<<(1 << MSD_D) / 128, 128, 0, ctx->stream>>>(sq, n, partial);
    CS_LAUNCH_CHECK();
    k_msd_finish<<<1, 32, 0, ctx->stream>>>(partial, n, out);
    CS_LAUNCH_CHECK();
    ctx->launches += 3;
    return CS_OK;
}

int cs_hist2d(cs_ctx *ctx, int32_t prec, const void *pos, const uint8_t *type, int64_t n,
              int32_t species, const double *edges_x, const double *edges_y, int32_t bins,
              int64_t per_sample, uint64_t *counts) {
    using namespace cs;
    if (bins < 1 || (species >= 0 && !type) || per_sample < 0) {
        set_error("cs_hist2d: bins must be positive (and the species array given)");
        return CS_ERR_PARAM;
    }
    const long long samples = per_sample > 0 ? (n + per_sample - 1) / per_sample : 1;
    CS_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * (size_t)bins * bins * samples,
                            ctx->stream));
    if (n == 0) return CS_OK;
    if (prec == CS_F64)
        k_hist2d<double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const double *>(pos), type, n, species, edges_x, edges_y, bins, per_sample,
            reinterpret_cast<unsigned long long *>(counts));
    else
        k_hist2d<float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const float *>(pos), type, n, species, edges_x, edges_y, bins, per_sample,
            reinterpret_cast<unsigned long long *>(counts));
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

}  // extern "C"
