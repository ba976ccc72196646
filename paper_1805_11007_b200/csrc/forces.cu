// forces.cu -- soft pair forces over the cell list.
//
// Reference: motion.py:200-245 (_soft_forces_fused pair loop).  Per
// particle i, the ring o1 in {-1,0,1} (y) is the outer loop and o0 the inner
// one, with the periodic de-duplication for 1- and 2-cell axes
// (motion.py:209-212, :219-222) and range checks on reflecting axes; within
// a cell j runs in ascending index; j == i is skipped; the displacement is
// minimum-imaged with round-half-even (rint); pairs with r2 > cut2 or
// r2 == 0 are skipped; otherwise f += -(exp(-r/eps) / (eps r)) * dx.
//
// Every floating-point operation is an explicitly rounded binary64 op in
// the reference order and exp is the glibc restatement (glibc_exp.h), so
// the force on each particle is bit-identical to the reference's.  fp32
// storage is widened to binary64 on load (the fp32 variants compute on the
// stored binary32 values exactly as the fp64 oracle would).
//
// One thread per sorted slot: consecutive threads handle particles of the
// same/adjacent cells, so neighbour reads are shared through L1/L2.
#include "common.cuh"

namespace cs {

template <class P>
__global__ void __launch_bounds__(256)
k_soft_forces(const P *__restrict__ pos, const uint8_t *__restrict__ type,
              const int *__restrict__ order, const int *__restrict__ starts, long long n,
              BinGeom g, PairTab pt, double *__restrict__ out, const DevStatus *st) {
    if (st && st->abort) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = order[t];
        double fx = 0.0, fy = 0.0;
        pair_loop(pos, type, order, starts, g, pt, i,
                  [&](int, double s, double dx0, double dx1) {
                      fx = dadd(fx, dmul(s, dx0));
                      fy = dadd(fy, dmul(s, dx1));
                  });
        reinterpret_cast<double2 *>(out)[i] = make_double2(fx, fy);
    }
}

template <class P>
__global__ void k_count_pairs(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                              const int *__restrict__ order, const int *__restrict__ starts,
                              long long n, BinGeom g, PairTab pt, int *__restrict__ cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int c = 0;
        pair_loop(pos, type, order, starts, g, pt, (int)i,
                  [&](int, double, double, double) { c++; });
        cnt[i] = c;
    }
}

template <class P>
__global__ void k_fill_pairs(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                             const int *__restrict__ order, const int *__restrict__ starts,
                             long long n, BinGeom g, PairTab pt, const int *__restrict__ off,
                             int64_t *__restrict__ pairs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long w = off[i];
        pair_loop(pos, type, order, starts, g, pt, (int)i,
                  [&](int j, double, double, double) {
                      pairs[2 * w] = i;
                      pairs[2 * w + 1] = j;
                      w++;
                  });
    }
}

int launch_soft_forces(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                       long long n, const BinGeom &g, const PairTab &pt, double *out,
                       const DevStatus *st) {
    if (n == 0) return CS_OK;
    const int B = 256;
    const int *order = ctx->order.as<int>(), *starts = ctx->starts.as<int>();
    if (prec == CS_F64)
        k_soft_forces<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const double *>(pos), type, order, starts, n, g, pt, out, st);
    else
        k_soft_forces<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const float *>(pos), type, order, starts, n, g, pt, out, st);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int run_soft_force_pairs(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                         long long n, const BinGeom &g, const PairTab &pt, int64_t *pairs,
                         int64_t cap, int64_t *count) {
    const int B = 256;
    CS_TRY(ctx->pair_counts.ensure(sizeof(int) * (size_t)(n + 1)));
    CS_TRY(ctx->pair_offsets.ensure(sizeof(int) * (size_t)(n + 1)));
    int *cnt = ctx->pair_counts.as<int>(), *off = ctx->pair_offsets.as<int>();
    const int *order = ctx->order.as<int>(), *starts = ctx->starts.as<int>();
    if (n > 0) {
        if (prec == CS_F64)
            k_count_pairs<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const double *>(pos), type, order, starts, n, g, pt, cnt);
        else
            k_count_pairs<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const float *>(pos), type, order, starts, n, g, pt, cnt);
        CS_LAUNCH_CHECK();
    }
    CS_TRY(exclusive_scan_i32(ctx, cnt, off, n));
    int total = 0;
    CS_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *count = total;
    if (total > cap || n == 0 || pairs == nullptr) return CS_OK;
    if (prec == CS_F64)
        k_fill_pairs<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const double *>(pos), type, order, starts, n, g, pt, off, pairs);
    else
        k_fill_pairs<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const float *>(pos), type, order, starts, n, g, pt, off, pairs);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

}  // namespace cs
