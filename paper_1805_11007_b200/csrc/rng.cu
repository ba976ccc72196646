// rng.cu -- numpy's Generator(PCG64) on the device.
//
// The reference draws every realisation's Brownian increments and reaction
// uniforms from numpy generators seeded SeedSequence(seed_base + N s)
// .spawn(3) (engine.py:272-275; one (N, 2) standard_normal block per step,
// motion.py:277; one random(N) block per step, reactions.py:57).  The batched
// ensemble engine draws them here instead of on the host, bit for bit:
//   PCG64      128-bit LCG, numpy's default multiplier, XSL-RR output, step
//              then output (numpy/random/src/pcg64/pcg64.h)
//   random     (u64 >> 11) * 2^-53
//   normal     the 256-layer ziggurat of distributions.c
//              (random_standard_normal) with numpy's own tables
//              (ziggurat_tables.h, tools/ziggurat_tables.py); the wedge test
//              uses the glibc-exact exp (glibc_exp.h), the tail the
//              glibc-exact log1p below.
// The host's generator states (bit_generator.state) seed the device streams;
// tests/test_gpu_rng.py checks the draws against numpy bit for bit.
#include <math_constants.h>

#include "common.cuh"
#include "ziggurat_tables.h"

namespace cs {

// glibc 2.39's log1p on an FMA host (the x86_64 FMA variant of the fdlibm
// algorithm, Estrin-evaluated polynomial): the operations below are the ones
// its compiled code performs, each fused multiply-add where it fuses.
// Verified bit for bit against the host libm (tests/test_gpu_rng.py).
__device__ __noinline__ double log1p_glibc(double x) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
                 Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                 Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                 Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    const int hx = __double2hiint(x);
    const int ax = hx & 0x7fffffff;
    int k = 1, hu = 0;
    double f = 0.0, c = 0.0, u;
    if (hx < 0x3FDA827A) {
        if (ax >= 0x3ff00000) {
            if (x == -1.0) return -CUDART_INF;
            return CUDART_NAN;
        }
        if (ax < 0x3e200000) {
            if (ax < 0x3c900000) return x;
            return fma(-dmul(x, x), 0.5, x);
        }
        if (hx > 0 || hx <= (int)0xbfd2bec4) {
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return dadd(x, x);
    }
    if (k != 0) {
        if (hx < 0x43400000) {
            u = dadd(1.0, x);
            hu = __double2hiint(u);
            k = (hu >> 20) - 1023;
            c = k > 0 ? dsub(1.0, dsub(u, x)) : dsub(x, dsub(u, 1.0));
            c = ddiv(c, u);
        } else {
            u = x;
            hu = __double2hiint(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
        } else {
            k += 1;
            u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
            hu = (0x00100000 - hu) >> 2;
        }
        f = dsub(u, 1.0);
    }
    const double hfsq = dmul(dmul(0.5, f), f);
    const double dk = (double)k;
    if (hu == 0) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = fma(dk, ln2_lo, c);
            return fma(dk, ln2_hi, c);
        }
        const double R = dmul(fma(-f, 0.66666666666666666, 1.0), hfsq);
        if (k == 0) return dsub(f, R);
        return fma(dk, ln2_hi, -dsub(dsub(R, fma(dk, ln2_lo, c)), f));
    }
    const double s = ddiv(f, dadd(2.0, f));
    const double z = dmul(s, s);
    const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
    const double z2 = dmul(z, z), z4 = dmul(z2, z2), z6 = dmul(z4, z2);
    const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, dmul(z2, R2))));
    const double t = dmul(s, dadd(hfsq, R));
    if (k == 0) return dsub(f, dsub(hfsq, t));
    return fma(dk, ln2_hi, -dsub(dsub(hfsq, dadd(t, fma(dk, ln2_lo, c))), f));
}

// the ziggurat tables are indexed by a random byte per lane: read from
// shared memory (constant memory would serialise the 32 lanes' addresses)
struct ZigTables {
    unsigned long long ki[256];
    double wi[256], fi[256];
};

struct Pcg64 {
    unsigned long long hi, lo, ihi, ilo;  // state, increment (128-bit)
    const ZigTables *zt;
    __device__ __forceinline__ unsigned long long next64() {
        constexpr unsigned long long MH = 0x2360ED051FC65DA4ull, ML = 0x4385DF649FCCF645ull;
        // state = state * M + inc (mod 2^128)
        const unsigned long long p_lo = lo * ML;
        const unsigned long long p_hi = __umul64hi(lo, ML) + lo * MH + hi * ML;
        lo = p_lo + ilo;
        hi = p_hi + ihi + (lo < p_lo ? 1ull : 0ull);
        const unsigned rot = (unsigned)(hi >> 58);
        const unsigned long long v = hi ^ lo;
        return (v >> rot) | (v << ((64u - rot) & 63u));
    }
    __device__ __forceinline__ double next_double() {
        return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
    }
    __device__ double standard_normal() {
        constexpr double ZR = 3.6541528853610087963519472518;
        constexpr double ZIR = 0.27366123732975827203338247596;
        for (;;) {
            unsigned long long r = next64();
            const int idx = (int)(r & 0xff);
            r >>= 8;
            const int sign = (int)(r & 1);
            const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
            double x = dmul((double)rabs, zt->wi[idx]);
            if (sign) x = -x;
            if (rabs < zt->ki[idx]) return x;
            if (idx == 0) {
                for (;;) {
                    const double xx = dmul(-ZIR, log1p_glibc(-next_double()));
                    const double yy = -log1p_glibc(-next_double());
                    if (dadd(yy, yy) > dmul(xx, xx))
                        return ((rabs >> 8) & 1) ? -dadd(ZR, xx) : dadd(ZR, xx);
                }
            } else {
                const double f0 = zt->fi[idx - 1];
                const double f1 = zt->fi[idx];
                if (dadd(dmul(dsub(f0, f1), next_double()), f1) <
                    cs_exp(dmul(dmul(-0.5, x), x)))
                    return x;
            }
        }
    }
};

// out[(k * S + s) * m + j] = the (k * m + j)-th draw of stream s; state
// (S, 4) = {state_hi, state_lo, inc_hi, inc_lo}, advanced in place
__global__ void __launch_bounds__(64)
k_rng_fill(unsigned long long *__restrict__ state, int S, int kind, int k, long long m,
           double *__restrict__ out) {
    __shared__ ZigTables zt;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        zt.ki[i] = ZIG_KI[i];
        zt.wi[i] = __longlong_as_double((long long)ZIG_WI[i]);
        zt.fi[i] = __longlong_as_double((long long)ZIG_FI[i]);
    }
    __syncthreads();
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    Pcg64 g{state[4 * s], state[4 * s + 1], state[4 * s + 2], state[4 * s + 3], &zt};
    for (int kk = 0; kk < k; kk++) {
        double *o = out + ((long long)kk * S + s) * m;
        if (kind == 0)
            for (long long j = 0; j < m; j++) o[j] = g.standard_normal();
        else
            for (long long j = 0; j < m; j++) o[j] = g.next_double();
    }
    state[4 * s] = g.hi;
    state[4 * s + 1] = g.lo;
}

__global__ void k_log1p(const double *x, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = log1p_glibc(x[i]);
}

}  // namespace cs

extern "C" {

int cs_rng_fill(cs_ctx *ctx, uint64_t *state, int32_t n_streams, int32_t kind, int32_t k,
                int64_t m, double *out) {
    if (n_streams < 0 || k < 0 || m < 0 || (kind != 0 && kind != 1)) {
        cs::set_error("cs_rng_fill: bad arguments");
        return CS_ERR_PARAM;
    }
    if (n_streams == 0 || k == 0 || m == 0) return CS_OK;
    cs::k_rng_fill<<<(n_streams + 63) / 64, 64, 0, ctx->stream>>>(
        reinterpret_cast<unsigned long long *>(state), n_streams, kind, k, m, out);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int cs_log1p_batch(cs_ctx *ctx, const double *x, double *y, int64_t n) {
    if (n == 0) return CS_OK;
    cs::k_log1p<<<cs::grid_for(n, 256), 256, 0, ctx->stream>>>(x, y, n);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

}  // extern "C"
