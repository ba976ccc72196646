// hard.cu -- the hard-sphere overlap correction (motion.py:301-352,
// resolve_hard_sphere), for the small systems the reference runs it on.
//
// One sweep over the proposals: the pairs (i < j) whose minimum-image
// distance is below epsilon at the start of the sweep (the reference's
// vectorised scan: d2 = (-0 + dx^2) + dy^2 < eps^2) are processed once, in
// ascending (i, j) order, against the current buffer: re-measured
// (sqrt of dx . dx, which numpy evaluates through BLAS ddot as
// fma(dy, dy, dx dx) on this host), skipped if already separated, else
// pushed apart by 2 (eps - d) along the centre line, split by the
// diffusivities.  The scan is parallel (O(N^2), one thread per i, then a
// scan of the per-i counts and an ordered fill); the sweep is inherently
// sequential and runs on one thread.  Coincident pairs take the reference's
// id-derived direction with the device cos/sin (not glibc's: the only
// non-bitwise case, a measure-zero event).
#include "common.cuh"

namespace cs {

int exclusive_scan_i32(cs_ctx *ctx, const int *in, int *out, long long n, int *zero_in);

struct HsArgs {
    long long n;
    cs_domain dom;
    double eps, eps2;
    double D[2];
};

template <class P>
__device__ __forceinline__ void hs_disp(const P *x, long long i, long long j, const HsArgs &a,
                                        double &d0, double &d1) {
    double xi, yi, xj, yj;
    load2(x, i, xi, yi);
    load2(x, j, xj, yj);
    d0 = dsub(xj, xi);
    d1 = dsub(yj, yi);
    const double s0 = dsub(a.dom.hi[0], a.dom.lo[0]), s1 = dsub(a.dom.hi[1], a.dom.lo[1]);
    if (a.dom.periodic[0]) d0 = dsub(d0, dmul(s0, rint(ddiv(d0, s0))));
    if (a.dom.periodic[1]) d1 = dsub(d1, dmul(s1, rint(ddiv(d1, s1))));
}

template <class P>
__global__ void k_hs_count(const P *__restrict__ x, HsArgs a, int *__restrict__ cnt,
                           const int *__restrict__ off, int2 *__restrict__ hits) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
         i += (long long)gridDim.x * blockDim.x) {
        int c = 0;
        for (long long j = i + 1; j < a.n; j++) {
            double d0, d1;
            hs_disp(x, i, j, a, d0, d1);
            const double d2 = dadd(dadd(-0.0, dmul(d0, d0)), dmul(d1, d1));
            if (d2 < a.eps2) {
                if (hits) hits[off[i] + c] = make_int2((int)i, (int)j);
                c++;
            }
        }
        if (!hits) cnt[i] = c;
    }
}

template <class P>
__global__ void k_hs_sweep(P *__restrict__ x, const uint8_t *__restrict__ type, HsArgs a,
                           const int *__restrict__ total, const int2 *__restrict__ hits) {
    const int nh = *total;
    for (int h = 0; h < nh; h++) {
        const int i = hits[h].x, j = hits[h].y;
        double d0, d1;
        hs_disp(x, i, j, a, d0, d1);
        const double d = dsqrt(fma(d1, d1, dmul(d0, d0)));  // BLAS ddot of (d0, d1)
        if (d >= a.eps) continue;
        double u0, u1;
        if (d == 0.0) {  // _tiebreak_direction (motion.py:304-307)
            const double G = 0.6180339887498949;
            const double th = dmul(2.0 * 3.141592653589793,
                                   fmod(dadd(dmul(G, (double)(i + 1)),
                                             dmul(dmul(G, G), (double)(j + 1))),
                                        1.0));
            u0 = cos(th);
            u1 = sin(th);
        } else {
            u0 = ddiv(d0, d);
            u1 = ddiv(d1, d);
        }
        const double dp = dsub(a.eps, d);
        const double Di = a.D[type ? (type[i] ? 1 : 0) : 0], Dj = a.D[type ? (type[j] ? 1 : 0) : 0];
        const double tot = dadd(Di, Dj);
        const double share = tot == 0.0 ? 0.5 : ddiv(Di, tot);
        const double mi = dmul(dmul(2.0, dp), share), mj = dmul(dmul(2.0, dp), dsub(1.0, share));
        double xi, yi, xj, yj;
        load2(x, i, xi, yi);
        load2(x, j, xj, yj);
        store2(x, i, dsub(xi, dmul(u0, mi)), dsub(yi, dmul(u1, mi)));
        store2(x, j, dadd(xj, dmul(u0, mj)), dadd(yj, dmul(u1, mj)));
    }
}

// prop (n, 2) in place; *n_hits = pairs found by the scan
int launch_hard_sphere(cs_ctx *ctx, int prec, void *prop, const uint8_t *type, long long n,
                       const cs_domain &dom, double eps, const double D[2], int *n_hits_dev) {
    if (n < 2) return CS_OK;
    HsArgs a;
    a.n = n;
    a.dom = dom;
    a.eps = eps;
    a.eps2 = eps * eps;
    a.D[0] = D[0];
    a.D[1] = D[1];
    CS_TRY(ctx->pair_counts.ensure(sizeof(int) * (size_t)(n + 1)));
    CS_TRY(ctx->pair_offsets.ensure(sizeof(int) * (size_t)(n + 1)));
    int *cnt = ctx->pair_counts.as<int>(), *off = ctx->pair_offsets.as<int>();
    const int B = 128;
    if (prec == CS_F64)
        k_hs_count<double><<<grid_for(n, B), B, 0, ctx->stream>>>((const double *)prop, a, cnt,
                                                                  nullptr, nullptr);
    else
        k_hs_count<float><<<grid_for(n, B), B, 0, ctx->stream>>>((const float *)prop, a, cnt,
                                                                 nullptr, nullptr);
    CS_LAUNCH_CHECK();
    CS_TRY(exclusive_scan_i32(ctx, cnt, off, n, nullptr));
    // the hit list: bounded by the scan total, read back to size the buffer
    int total = 0;
    CS_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_hits_dev) CS_CUDA(cudaMemcpyAsync(n_hits_dev, off + n, sizeof(int),
                                            cudaMemcpyDeviceToDevice, ctx->stream));
    if (total == 0) return CS_OK;
    CS_TRY(ctx->tmp.ensure(sizeof(int2) * (size_t)total));
    int2 *hits = ctx->tmp.as<int2>();
    if (prec == CS_F64)
        k_hs_count<double><<<grid_for(n, B), B, 0, ctx->stream>>>((const double *)prop, a, cnt,
                                                                  off, hits);
    else
        k_hs_count<float><<<grid_for(n, B), B, 0, ctx->stream>>>((const float *)prop, a, cnt,
                                                                 off, hits);
    CS_LAUNCH_CHECK();
    if (prec == CS_F64)
        k_hs_sweep<double><<<1, 1, 0, ctx->stream>>>((double *)prop, type, a, off + n, hits);
    else
        k_hs_sweep<float><<<1, 1, 0, ctx->stream>>>((float *)prop, type, a, off + n, hits);
    CS_LAUNCH_CHECK();
    ctx->launches += 4;
    return CS_OK;
}

}  // namespace cs

extern "C" int cs_resolve_hard_sphere(cs_ctx *ctx, int32_t prec, void *prop,
                                      const uint8_t *type, int64_t n, const cs_domain *dom,
                                      double eps, double d_alpha, double d_beta) {
    if (prec != CS_F64 && prec != CS_F32) {
        cs::set_error("unknown precision %d", prec);
        return CS_ERR_PARAM;
    }
    const double D[2] = {d_alpha, d_beta};
    return cs::launch_hard_sphere(ctx, prec, prop, type, n, *dom, eps, D, nullptr);
}
