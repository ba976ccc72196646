// motion.cu -- Euler-Maruyama proposal and boundary resolution.
//
// Reference: motion.py:268-282 (em_step: ((x + amp xi) + drift dt) + force dt
// with amp = sqrt((2 D) dt), numpy left to right, no contraction) and
// motion.py:355-402 (_boundaries_kernel: non-finite pass, then per axis
// periodic wrap with anchor shift or reflection; status 1/2/3).
//
// The standalone kernels here back the function-level seams; the fused
// per-step version lives in sim.cu (k_update), which applies the same
// arithmetic in one pass with the bilinear drift refresh.
#include "common.cuh"

namespace cs {

template <class P>
__global__ void k_em_step(const P *__restrict__ pos, const double *__restrict__ D,
                          const double *__restrict__ drift, const double *__restrict__ force,
                          const P *__restrict__ xi, double dt, long long n, P *__restrict__ out,
                          int tamed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double amp = dsqrt(dmul(dmul(2.0, D[i]), dt));
        double x, y, x0, x1;
        load2(pos, i, x, y);
        load2(xi, i, x0, x1);
        const double d0 = drift ? drift[2 * i] : 0.0, d1 = drift ? drift[2 * i + 1] : 0.0;
        const double f0 = force ? force[2 * i] : 0.0, f1 = force ? force[2 * i + 1] : 0.0;
        double i0, i1;
        force_increment(f0, f1, dt, tamed, i0, i1);
        const double nx = dadd(dadd(dadd(x, dmul(amp, x0)), dmul(d0, dt)), i0);
        const double ny = dadd(dadd(dadd(y, dmul(amp, x1)), dmul(d1, dt)), i1);
        store2(out, i, nx, ny);
    }
}

template <class P>
__global__ void k_boundaries(P *__restrict__ x, P *__restrict__ anchor, long long n,
                             cs_domain d, DevStatus *st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double v[2], a[2];
        load2(x, i, v[0], v[1]);
        load2(anchor, i, a[0], a[1]);
        if (!(isfinite(v[0]) && isfinite(v[1]))) {
            atomicMin(&st->key, err_key(0, i, CS_NONFINITE));
            continue;
        }
        bool ok = true;
        for (int ax = 0; ax < 2 && ok; ax++) {
            const int code = boundary_axis(v[ax], a[ax], d.lo[ax], d.hi[ax], d.periodic[ax]);
            if (code) {
                atomicMin(&st->key, err_key(1 + ax, i, code));
                ok = false;
            }
        }
        if (!ok) continue;
        store2(x, i, v[0], v[1]);
        store2(anchor, i, a[0], a[1]);
    }
}

int launch_em_step(cs_ctx *ctx, int prec, const void *pos, const double *D, const double *drift,
                   const double *force, const void *xi, double dt, long long n, void *out,
                   int tamed) {
    if (n == 0) return CS_OK;
    const int B = 256;
    if (prec == CS_F64)
        k_em_step<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
            (const double *)pos, D, drift, force, (const double *)xi, dt, n, (double *)out,
            tamed);
    else
        k_em_step<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
            (const float *)pos, D, drift, force, (const float *)xi, dt, n, (float *)out, tamed);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

int launch_boundaries(cs_ctx *ctx, int prec, void *x, void *anchor, long long n,
                      const cs_domain &d, DevStatus *st) {
    if (n == 0) return CS_OK;
    const int B = 256;
    if (prec == CS_F64)
        k_boundaries<double><<<grid_for(n, B), B, 0, ctx->stream>>>((double *)x, (double *)anchor,
                                                                    n, d, st);
    else
        k_boundaries<float><<<grid_for(n, B), B, 0, ctx->stream>>>((float *)x, (float *)anchor, n,
                                                                   d, st);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

}  // namespace cs
