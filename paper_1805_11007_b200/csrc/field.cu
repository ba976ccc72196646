#include <stdlib.h>
// field.cu -- grid side of the hot path: deposits, the semi-implicit field
// step, the gradient stencil and bilinear sampling.
//
// References (chemosim/):
//   rhs            field.py:220-227    c(1 - dt g) + (dt ka) ra - (rb c)(dt kb)
//   solve          field.py:162-201    (I - dt d_c L) c' = rhs
//                  neumann: DCT-I modal solve, 4 dense GEMMs through the
//                  cosine basis (here: fp64 tiled GEMM kernels, same basis);
//                  periodic: the reference factors the sparse system with
//                  SuperLU; the same circulant system is diagonalised here by
//                  a 2-D real FFT (cuFFT D2Z/Z2D or R2C/C2R), which is exact
//                  up to rounding and the only feasible route at 4096^2+.
//   checks         field.py:229-238    non-finite -> FloatingPointError,
//                  negative weighted mass < -1e-12 -> warning
//   gradient       field.py:128-137, 242-245  CSR rows in column order
//   bilinear       coupling.py:216-262
// Deposits: deposit.cu (node gathers in the reference's summation order).
#include <cufft.h>
#include <math.h>

#include <vector>

#include "common.cuh"

namespace cs {

// ------------------------------------------------------------------ bilinear
template <class P, class G>
__global__ void k_bilinear(const P *__restrict__ pts, long long np, const G *__restrict__ vals,
                           int m, GridGeom gg, G *__restrict__ out,
                           unsigned long long *__restrict__ clamped) {
    int local = 0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < np;
         p += (long long)gridDim.x * blockDim.x) {
        double x, y;
        load2(pts, p, x, y);
        Bilin b;
        local += bilinear_stencil(x, y, gg, b);
        for (int k = 0; k < m; k++) out[p * m + k] = (G)bilinear_apply(b, vals, m, k);
    }
    if (local) atomicAdd(clamped, (unsigned long long)local);
}

int launch_bilinear(cs_ctx *ctx, int prec, const void *pts, long long np, const void *vals, int m,
                    const GridGeom &gg, void *out, unsigned long long *clamped) {
    if (np == 0) return CS_OK;
    const int B = 256;
    if (prec == CS_F64)
        k_bilinear<double, double><<<grid_for(np, B), B, 0, ctx->stream>>>(
            (const double *)pts, np, (const double *)vals, m, gg, (double *)out, clamped);
    else
        k_bilinear<float, float><<<grid_for(np, B), B, 0, ctx->stream>>>(
            (const float *)pts, np, (const float *)vals, m, gg, (float *)out, clamped);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

// ------------------------------------------------------------------ gradient
D1Coef make_d1(double h) {
    const double two_h = 2.0 * h;
    D1Coef c;
    c.m1 = -1.0 / two_h;
    c.p1 = 1.0 / two_h;
    c.l0 = -3.0 / two_h;
    c.l1 = 4.0 / two_h;
    c.l2 = -1.0 / two_h;
    c.r0 = 1.0 / two_h;
    c.r1 = -4.0 / two_h;
    c.r2 = 3.0 / two_h;
    return c;
}

// grad = (d1x c, d1y c); when st != NULL also the step_field post-checks on
// c: any non-finite node and the weighted mass of the negative nodes.
// Serial epilogue of the field checks of one step (after every block's
// atomics): a non-finite node stops the run, a negative weighted mass is
// counted.
__device__ __forceinline__ void field_finish_body(DevStatus *st, int step) {
    volatile DevStatus *v = st;
    if (v->abort) return;
    if (v->field_bad) {
        st->key = err_key(0, 0, CS_FIELD_NONFINITE);
        st->abort = 1;
        st->step = step;
    }
    if (v->neg_flag && v->neg_mass < -1e-12) {
        if (v->neg_steps == 0) st->first_neg = v->neg_mass;
        st->neg_steps = v->neg_steps + 1;
    }
    st->neg_flag = 0;
    st->neg_mass = 0.0;
}

// thread 0 of every block of a gradient launch, after its block's atomics:
// the last block to arrive runs the epilogue (step >= 0) and re-arms the
// counter
__device__ __forceinline__ void field_checks_arrive(DevStatus *st, int step) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    if (prev + 1 == gridDim.x) {
        __threadfence();
        if (step >= 0) field_finish_body(st, step);
        st->blocks_done = 0;
    }
}

template <class G>
__global__ void __launch_bounds__(256)
k_gradient(const G *__restrict__ c, int n, int per, D1Coef kx, D1Coef ky, double wcell,
           G *__restrict__ grad, DevStatus *st, int *__restrict__ zero_q, int step) {
    const bool dead = st && st->abort;
    const long long m = (long long)n * n;
    double neg = 0.0;
    int bad = 0, anyneg = 0;
    // rows j = blockIdx.x + k gridDim.x; threads stride along the row
    if (!dead)
    for (int j = blockIdx.x; j < n; j += gridDim.x)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const long long l = (long long)j * n + i;
        const double gx = d1_at(c, (long long)j * n, 1, i, n, per, kx);
        const double gy = d1_at(c, (long long)i, n, j, n, per, ky);
        store2(grad, l, gx, gy);
        if (zero_q) {  // sorted engine: clear the deposit grids (no load of them here)
            zero_q[l] = 0;
            zero_q[l + m] = 0;
        }
        if (st) {
            const double v = (double)c[l];
            if (!isfinite(v)) bad = 1;
            if (v < 0.0) {
                double w = wcell;
                if (!per) {
                    const double wi = (i == 0 || i == n - 1) ? 0.5 : 1.0;
                    const double wj = (j == 0 || j == n - 1) ? 0.5 : 1.0;
                    w = (wj * wi) * wcell;
                }
                neg += w * v;
                anyneg = 1;
            }
        }
    }
    if (!st) return;
    // block reduction of the negative mass, one atomic per block
    __shared__ double s_neg[8];
    __shared__ int s_flags[8];
    for (int o = 16; o > 0; o >>= 1) {
        neg += __shfl_xor_sync(0xffffffffu, neg, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        anyneg |= __shfl_xor_sync(0xffffffffu, anyneg, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_neg[warp] = neg;
        s_flags[warp] = bad | (anyneg << 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int f = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            t += s_neg[w];
            f |= s_flags[w];
        }
        if (f & 1) atomicExch(&st->field_bad, 1);
        if (f & 2) {
            atomicAdd(&st->neg_mass, t);
            atomicExch(&st->neg_flag, 1);
        }
        field_checks_arrive(st, step);
    }
}

// Periodic binary32 grid, n % 4 == 0: the same gradient, checks and deposit
// grid reset as k_gradient with 16-byte accesses -- a thread owns nodes
// i0 .. i0+3 of row j (row j, j-1, j+1 as float4 plus the two scalar
// x-neighbours).  Each derivative is the periodic CSR row of d1 summed in
// column order (d1_at): interior (0 + m1 c[i-1]) + p1 c[i+1], the wrapped
// ends (0 + p1 c[i+1]) + m1 c[i-1].
__device__ __forceinline__ double d1_per(double cm, double cp, bool wrapped, const D1Coef &k) {
    const double am = dmul(k.m1, cm), ap = dmul(k.p1, cp);
    return wrapped ? dadd(dadd(0.0, ap), am) : dadd(dadd(0.0, am), ap);
}

// A block owns strips of R consecutive rows x 1024 columns and slides down
// them with rows j-1, j, j+1 of its four columns in registers: one new
// 16-byte load per row instead of three (R = 1: a row per strip).
__global__ void __launch_bounds__(256)
k_gradient_per4(const float *__restrict__ c, int n, D1Coef kx, D1Coef ky, double wcell,
                float *__restrict__ grad, DevStatus *st, int *__restrict__ zero_q, int step,
                int R, int jbase = 0, int jrows = -1, int own0 = 0, int own1 = 1 << 30) {
    // (slab mode: the rows jbase .. jbase + jrows - 1 (mod n); the field checks
    // count the own rows [own0, own1) only)
    const bool dead = st->abort != 0;
    const long long m = (long long)n * n;
    const int n4 = n >> 2;
    double neg = 0.0;
    int bad = 0, anyneg = 0;
    if (jrows < 0) jrows = n;
    if (dead) jrows = 0;
    const int nchunk = (n4 + 255) >> 8, ngroups = (jrows + R - 1) / R;
    for (int sidx = blockIdx.x; sidx < ngroups * nchunk; sidx += gridDim.x) {
        const int rg = sidx / nchunk, t = (sidx - rg * nchunk) * 256 + threadIdx.x;
        if (t >= n4) continue;
        const int jj0 = rg * R, jj1 = jj0 + R < jrows ? jj0 + R : jrows;
        int j = (jbase + jj0) % n;
        if (j < 0) j += n;
        const int i0 = 4 * t;
        const int il = i0 == 0 ? n - 1 : i0 - 1, ir = i0 + 4 == n ? 0 : i0 + 4;
        const float4 *c4 = reinterpret_cast<const float4 *>(c);
        float4 dn = c4[(long long)(j == 0 ? n - 1 : j - 1) * n4 + t];
        float4 v = c4[(long long)j * n4 + t];
        for (int jj = jj0; jj < jj1; jj++) {
            const int jp = j == n - 1 ? 0 : j + 1;
            const float4 up = c4[(long long)jp * n4 + t];
            const float left = c[(long long)j * n + il];
            const float right = c[(long long)j * n + ir];
            const bool check = j >= own0 && j < own1;
            const float cv[6] = {left, v.x, v.y, v.z, v.w, right};
            const float dv[4] = {dn.x, dn.y, dn.z, dn.w}, uv[4] = {up.x, up.y, up.z, up.w};
            double gx[4], gy[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int i = i0 + q;
                gx[q] = d1_per((double)cv[q], (double)cv[q + 2], i == 0 || i == n - 1, kx);
                gy[q] = d1_per((double)dv[q], (double)uv[q], j == 0 || j == n - 1, ky);
                const double x = (double)cv[q + 1];
                if (check && !isfinite(x)) bad = 1;
                if (check && x < 0.0) {
                    neg += wcell * x;
                    anyneg = 1;
                }
            }
            const long long l = (long long)j * n + i0;
            float4 *g4 = reinterpret_cast<float4 *>(grad + 2 * l);
            g4[0] = make_float4((float)gx[0], (float)gy[0], (float)gx[1], (float)gy[1]);
            g4[1] = make_float4((float)gx[2], (float)gy[2], (float)gx[3], (float)gy[3]);
            if (zero_q) {
                *reinterpret_cast<int4 *>(zero_q + l) = make_int4(0, 0, 0, 0);
                *reinterpret_cast<int4 *>(zero_q + l + m) = make_int4(0, 0, 0, 0);
            }
            dn = v;
            v = up;
            j = jp;
        }
    }
    __shared__ double s_neg[8];
    __shared__ int s_flags[8];
    for (int o = 16; o > 0; o >>= 1) {
        neg += __shfl_xor_sync(0xffffffffu, neg, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        anyneg |= __shfl_xor_sync(0xffffffffu, anyneg, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        s_neg[warp] = neg;
        s_flags[warp] = bad | (anyneg << 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tsum = 0.0;
        int f = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            tsum += s_neg[w];
            f |= s_flags[w];
        }
        if (f & 1) atomicExch(&st->field_bad, 1);
        if (f & 2) {
            atomicAdd(&st->neg_mass, tsum);
            atomicExch(&st->neg_flag, 1);
        }
        field_checks_arrive(st, step);
    }
}


// rows per strip and grid of k_gradient_per4: strips of up to 8 rows, but at
// least about two blocks per resident slot (8 blocks of 256 threads per SM);
// measured at 4096^2 (CS_GRAD_ROWS): 1 row 61.7, 4: 53.6, 8: 53.8, 13: 60.3,
// 16: 56.1 us
static void gradient_per4_shape(int n, int jrows, int *R, int *grid) {
    const int nchunk = ((n >> 2) + 255) >> 8, slots = 148 * 8;
    int r = (int)((long long)jrows * nchunk / (2 * slots));
    if (const char *e = getenv("CS_GRAD_ROWS")) r = atoi(e);
    r = r < 1 ? 1 : (r > 8 && !getenv("CS_GRAD_ROWS") ? 8 : (r > 16 ? 16 : r));
    const long long strips = (long long)((jrows + r - 1) / r) * nchunk;
    *R = r;
    *grid = (int)(strips < 1 ? 1 : (strips < slots ? strips : slots));
}

// slab mode (periodic binary32 grids): the gradient of the grid rows
// jbase .. jbase + jrows - 1 (mod n) from c rows one wider on either side;
// the field checks of the own rows [own0, own1)
int launch_gradient_rows(cs_ctx *ctx, const float *c, const GridGeom &gg, float *grad,
                         DevStatus *st, int step, int jbase, int jrows, int own0, int own1) {
    if (!(gg.per && gg.n % 4 == 0 && gg.n >= 8)) {
        set_error("slab gradient: periodic grid with n_c a multiple of 4");
        return CS_ERR_PARAM;
    }
    const D1Coef kx = make_d1(gg.d0), ky = make_d1(gg.d1);
    int R, g2;
    gradient_per4_shape(gg.n, jrows, &R, &g2);
    k_gradient_per4<<<g2, 256, 0, ctx->stream>>>(c, gg.n, kx, ky, gg.d0 * gg.d1, grad, st,
                                                 nullptr, step, R, jbase, jrows, own0, own1);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int launch_gradient(cs_ctx *ctx, int prec, const void *c, const GridGeom &gg, void *grad,
                    DevStatus *st, int step, int *zero_q) {
    const long long m = (long long)gg.n * gg.n;
    const D1Coef kx = make_d1(gg.d0), ky = make_d1(gg.d1);
    const double wcell = gg.d0 * gg.d1;
    const int B = 256;
    const int g2 = gg.n < 148 * 8 ? gg.n : 148 * 8;
    // (the field-check epilogue runs in the launch's last block, step >= 0)
    if (prec == CS_F64)
        k_gradient<double><<<g2, B, 0, ctx->stream>>>(
            (const double *)c, gg.n, gg.per, kx, ky, wcell, (double *)grad, st, zero_q, step);
    else if (gg.per && st && gg.n % 4 == 0 && gg.n >= 8 && !getenv("CS_GRAD_GENERIC")) {
        int R, g4;
        gradient_per4_shape(gg.n, gg.n, &R, &g4);
        k_gradient_per4<<<g4, B, 0, ctx->stream>>>((const float *)c, gg.n, kx, ky, wcell,
                                                  (float *)grad, st, zero_q, step, R);
    } else {
        k_gradient<float><<<g2, B, 0, ctx->stream>>>(
            (const float *)c, gg.n, gg.per, kx, ky, wcell, (float *)grad, st, zero_q, step);
    }
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// ------------------------------------------------------------------ rhs
RhsCoef make_rhs_coef(double dt, double ka, double kb, double gamma) {
    RhsCoef k;
    k.has_g = gamma != 0.0;
    k.has_a = ka != 0.0;
    k.has_b = kb != 0.0;
    k.one_m_dtg = 1.0 - dt * gamma;
    k.dka = dt * ka;
    k.dkb = dt * kb;
    return k;
}

template <class G, class R>
__global__ void k_rhs(const G *__restrict__ c, const G *__restrict__ ra, const G *__restrict__ rb,
                      long long m, RhsCoef k, R *__restrict__ rhs, const DevStatus *st) {
    if (st && st->abort) return;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const double cv = (double)c[l];
        double r = k.has_g ? dmul(cv, k.one_m_dtg) : cv;
        if (k.has_a) r = dadd(r, dmul(k.dka, (double)ra[l]));
        if (k.has_b) r = dsub(r, dmul(dmul((double)rb[l], cv), k.dkb));
        rhs[l] = (R)r;
    }
}

// ------------------------------------------------------------------ gather
// deposit_gather (coupling.py:190-213): node l (x fastest, field.py:62-66)
// against every selected particle in index order; d = node - p, minimum
// image on a periodic grid, r2 = d0^2 + d1^2, out += inv_norm *
// exp(-r2 / (2 h^2)) when r2 <= cutoff^2 (the reference's numpy exp is its
// SIMD variant: 1-ulp differences from the glibc exp used here).
template <class P>
__global__ void k_deposit_gather(const P *__restrict__ pos, long long np, GridGeom gg,
                                 double spanx, double spany, double h, double cutoff,
                                 double inv_norm, double *__restrict__ out) {
    const long long m = (long long)gg.n * gg.n;
    const double c2 = dmul(cutoff, cutoff);
    const double den = dmul(2.0, dmul(h, h));
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(l % gg.n), j = (int)(l / gg.n);
        const double nx = dadd(gg.lo0, dmul((double)i, gg.d0));
        const double ny = dadd(gg.lo1, dmul((double)j, gg.d1));
        double acc = 0.0;
        for (long long p = 0; p < np; p++) {
            double px, py;
            load2(pos, p, px, py);
            double d0 = dsub(nx, px), d1 = dsub(ny, py);
            if (gg.per) {
                d0 = dsub(d0, dmul(spanx, rint(ddiv(d0, spanx))));
                d1 = dsub(d1, dmul(spany, rint(ddiv(d1, spany))));
            }
            const double r2 = dadd(dmul(d0, d0), dmul(d1, d1));
            if (r2 <= c2) acc = dadd(acc, dmul(inv_norm, cs_exp(ddiv(-r2, den))));
        }
        out[l] = acc;
    }
}

int launch_deposit_gather(cs_ctx *ctx, int prec, const void *pos, long long np,
                          const GridGeom &gg, double spanx, double spany, double h, double cutoff,
                          double inv_norm, double *out) {
    const long long m = (long long)gg.n * gg.n;
    if (prec == CS_F64)
        k_deposit_gather<double><<<grid_for(m, 128), 128, 0, ctx->stream>>>(
            static_cast<const double *>(pos), np, gg, spanx, spany, h, cutoff, inv_norm, out);
    else
        k_deposit_gather<float><<<grid_for(m, 128), 128, 0, ctx->stream>>>(
            static_cast<const float *>(pos), np, gg, spanx, spany, h, cutoff, inv_norm, out);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// ------------------------------------------------------------------ GEMM
// C = A * op(B) (row-major n x n fp64), op = transpose when TB; optional
// element-wise scale by E; output to O.  64x64 tiles, 256 threads, 4x4 per
// thread, K-step 16 staged through shared memory.
template <bool TB, class O>
__global__ void __launch_bounds__(256)
k_gemm(const double *__restrict__ A, const double *__restrict__ B, const double *__restrict__ E,
       O *__restrict__ C, int n) {
    __shared__ double As[16][64 + 1];
    __shared__ double Bs[16][64 + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < n; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int kk = e & 15, r = e >> 4;
            const int gr = row0 + r, gk = k0 + kk;
            As[kk][r] = (gr < n && gk < n) ? A[(long long)gr * n + gk] : 0.0;
            const int gc = col0 + r;
            double bv = 0.0;
            if (gc < n && gk < n) bv = TB ? B[(long long)gc * n + gk] : B[(long long)gk * n + gc];
            Bs[kk][r] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; kk++) {
            double a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                a[u] = As[kk][ty + 16 * u];
                b[u] = Bs[kk][tx + 16 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int v = 0; v < 4; v++) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const int r = row0 + ty + 16 * u, cc = col0 + tx + 16 * v;
            if (r < n && cc < n) {
                double val = acc[u][v];
                if (E) val *= E[(long long)r * n + cc];
                C[(long long)r * n + cc] = (O)val;
            }
        }
}

// Small grids (n <= 256): 16x16 output tiles, one output per thread, so that
// a 128^2 solve spreads over 64 SMs instead of 4.  Same k-ordered fma chain
// per output as k_gemm (bitwise equal).
template <bool TB, class O>
__global__ void __launch_bounds__(256)
k_gemm16(const double *__restrict__ A, const double *__restrict__ B, const double *__restrict__ E,
         O *__restrict__ C, int n) {
    __shared__ double As[16][17];
    __shared__ double Bs[16][17];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int r = blockIdx.y * 16 + ty, cc = blockIdx.x * 16 + tx;
    double acc = 0.0;
    for (int k0 = 0; k0 < n; k0 += 16) {
        const int ra = blockIdx.y * 16 + ty, ka = k0 + tx;
        As[ty][tx] = (ra < n && ka < n) ? A[(long long)ra * n + ka] : 0.0;
        const int kb = k0 + ty, cb = blockIdx.x * 16 + tx;
        double bv = 0.0;
        if (kb < n && cb < n) bv = TB ? B[(long long)cb * n + kb] : B[(long long)kb * n + cb];
        Bs[ty][tx] = bv;
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; kk++) acc = fma(As[ty][kk], Bs[kk][tx], acc);  // zero padding as k_gemm
        __syncthreads();
    }
    if (r < n && cc < n) {
        double val = acc;
        if (E) val *= E[(long long)r * n + cc];
        C[(long long)r * n + cc] = (O)val;
    }
}

// Grids up to 128^2: two GEMMs of the modal solve per launch.  A block owns
// ROWS2 rows r: P_r = L_r M (M staged whole in shared memory), then
// out_r = (P_r N^T) * E_r with N^T = NT staged in the same buffer.  Each
// output is the k-ordered fma chain from +0.0 of k_gemm / k_gemm16 (without
// their zero padding), so the solve is unchanged; half the launches, and
// no round trip of the intermediate through memory.
constexpr int ROWS2 = 2;
constexpr int ROWS2_MAX_N = 128;

// one bulk copy (TMA engine) of `bytes` into shared memory, completing on
// the mbarrier at `bar` (phase `ph`)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes,
                                          unsigned long long *bar) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(d), "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long *bar, unsigned ph) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W;\n}" ::"r"(b), "r"(ph)
        : "memory");
}

template <class O>
__global__ void __launch_bounds__(128)
k_gemm_rows2(const double *__restrict__ L, const double *__restrict__ M,
             const double *__restrict__ NT, const double *__restrict__ E, O *__restrict__ out,
             int n) {
    extern __shared__ __align__(16) double sm2[];
    // one single-use barrier per half of M and of N^T: the first half of
    // each phase runs while the second half lands, and N^T's first half
    // streams into M's rows once every thread is past them
    __shared__ unsigned long long bar[4];
    double *Ms = sm2;                       // n * n
    double *lrow = Ms + (size_t)n * n;      // [k][ROWS2]
    double *prow = lrow + ROWS2 * n;        // [k][ROWS2]
    const int r0 = blockIdx.x * ROWS2, c = threadIdx.x;
    const int h = n / 2;
    const unsigned hb = (unsigned)(sizeof(double) * h * n);
    const unsigned tb = (unsigned)(sizeof(double) * (n - h) * n);
    if (threadIdx.x == 0) {
        for (int b = 0; b < 4; b++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&bar[b]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        bulk_load(Ms, M, hb, &bar[0]);
        bulk_load(Ms + (size_t)h * n, M + (size_t)h * n, tb, &bar[1]);
    }
    for (int i = threadIdx.x; i < ROWS2 * n; i += blockDim.x) {
        const int u = i / n, k = i - u * n, r = r0 + u;
        lrow[k * ROWS2 + u] = r < n ? __ldg(L + (size_t)r * n + k) : 0.0;
    }
    __syncthreads();
    double acc[ROWS2];
#pragma unroll
    for (int u = 0; u < ROWS2; u++) acc[u] = 0.0;
    const bool on = c < n;
    bar_wait(&bar[0], 0);
    if (on) {
#pragma unroll 4
        for (int k = 0; k < h; k++) {
            const double m = Ms[k * n + c];
#pragma unroll
            for (int u = 0; u < ROWS2; u++) acc[u] = fma(lrow[k * ROWS2 + u], m, acc[u]);
        }
    }
    __syncthreads();  // M's first half consumed: N^T's first half goes there
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_load(Ms, NT, hb, &bar[2]);
    }
    bar_wait(&bar[1], 0);
    if (on) {
#pragma unroll 4
        for (int k = h; k < n; k++) {
            const double m = Ms[k * n + c];
#pragma unroll
            for (int u = 0; u < ROWS2; u++) acc[u] = fma(lrow[k * ROWS2 + u], m, acc[u]);
        }
#pragma unroll
        for (int u = 0; u < ROWS2; u++) prow[c * ROWS2 + u] = acc[u];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bulk_load(Ms + (size_t)h * n, NT + (size_t)h * n, tb, &bar[3]);
    }
#pragma unroll
    for (int u = 0; u < ROWS2; u++) acc[u] = 0.0;
    bar_wait(&bar[2], 0);
    if (on) {
#pragma unroll 4
        for (int k = 0; k < h; k++) {
            const double m = Ms[k * n + c];
#pragma unroll
            for (int u = 0; u < ROWS2; u++) acc[u] = fma(prow[k * ROWS2 + u], m, acc[u]);
        }
    }
    bar_wait(&bar[3], 0);
    if (on) {
#pragma unroll 4
        for (int k = h; k < n; k++) {
            const double m = Ms[k * n + c];
#pragma unroll
            for (int u = 0; u < ROWS2; u++) acc[u] = fma(prow[k * ROWS2 + u], m, acc[u]);
        }
#pragma unroll
        for (int u = 0; u < ROWS2; u++) {
            const int r = r0 + u;
            if (r < n) {
                double val = acc[u];
                if (E) val *= E[(size_t)r * n + c];
                out[(size_t)r * n + c] = (O)val;
            }
        }
    }
}

template <class O>
static int gemm_rows2(cs_ctx *ctx, const double *L, const double *M, const double *NT,
                      const double *E, O *out, int n) {
    const size_t smem = sizeof(double) * ((size_t)n * n + 2 * ROWS2 * (size_t)n);
    static size_t set = 0;
    if (smem > set) {
        CS_CUDA(cudaFuncSetAttribute(k_gemm_rows2<double>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CS_CUDA(cudaFuncSetAttribute(k_gemm_rows2<float>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        set = smem;
    }
    const int threads = (n + 31) / 32 * 32;
    k_gemm_rows2<O><<<(n + ROWS2 - 1) / ROWS2, threads, smem, ctx->stream>>>(L, M, NT, E, out, n);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

template <class O>
int gemm(cs_ctx *ctx, const double *A, const double *B, bool tb, const double *E, O *C, int n) {
    if (n <= 256) {
        dim3 grid16((n + 15) / 16, (n + 15) / 16);
        if (tb) k_gemm16<true, O><<<grid16, 256, 0, ctx->stream>>>(A, B, E, C, n);
        else k_gemm16<false, O><<<grid16, 256, 0, ctx->stream>>>(A, B, E, C, n);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
        return CS_OK;
    }
    dim3 grid((n + 63) / 64, (n + 63) / 64);
    if (tb) k_gemm<true, O><<<grid, 256, 0, ctx->stream>>>(A, B, E, C, n);
    else k_gemm<false, O><<<grid, 256, 0, ctx->stream>>>(A, B, E, C, n);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// ------------------------------------------------------------------ FFT
// spectrum row ky (blockIdx.y), modes kx along x: multiply by
// 1 / (n^2 (1 - dt d_c (lambda_y + lambda_x)))
template <class CT>
__global__ void __launch_bounds__(256)
k_mode_scale(CT *__restrict__ spec, int n, const double *__restrict__ lx,
             const double *__restrict__ ly, double dtdc, double inv_nn) {
    const int nh = n / 2 + 1;
    constexpr int U = 8;  // loads in flight per thread
    for (int ky = blockIdx.x; ky < n; ky += gridDim.x) {
        const double lyv = __ldg(ly + ky);
        CT *row = spec + (long long)ky * nh;
        for (int k0 = threadIdx.x; k0 < nh; k0 += U * blockDim.x) {
            CT v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int kx = k0 + u * blockDim.x;
                if (kx < nh) v[u] = row[kx];
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int kx = k0 + u * blockDim.x;
                if (kx < nh) {
                    const double s = inv_nn / (1.0 - dtdc * (lyv + __ldg(lx + kx)));
                    v[u].x = v[u].x * s;
                    v[u].y = v[u].y * s;
                    row[kx] = v[u];
                }
            }
        }
    }
}

}  // namespace cs

namespace cs {

static int cufft_check(cufftResult r, const char *what) {
    if (r != CUFFT_SUCCESS) {
        set_error("cuFFT %s failed (%d)", what, (int)r);
        return CS_ERR_CUFFT;
    }
    return CS_OK;
}

int field_ops_create(cs_ctx *ctx, int prec, const cs_grid *g, double d_c, double dt,
                     cs_field_ops **out) {
    if (!(dt > 0)) {
        set_error("dt must be positive");
        return CS_ERR_PARAM;
    }
    if (g->n_c < 3) {
        set_error("n_c must be at least 3");
        return CS_ERR_PARAM;
    }
    auto *ops = new cs_field_ops();
    ops->ctx = ctx;
    ops->prec = prec;
    ops->gg = make_grid_geom(*g);
    ops->dt = dt;
    ops->d_c = d_c;
    const int n = g->n_c;
    const size_t m = (size_t)n * n;
    const size_t es = prec == CS_F64 ? 8 : 4;
    *out = ops;
    if (d_c * dt == 0.0) {
        ops->kind = 0;
        CS_CUDA(cudaMalloc(&ops->rhs, m * es));
        return CS_OK;
    }
    if (!g->periodic) {
        // DCT-I basis (field.py:190-196): F[k][j] = w_j cos(pi k j / (n-1)),
        // w = 1 at the ends and 2 inside (scipy dct type 1 of the identity);
        // its inverse is F / (2 (n-1)).
        ops->kind = 1;
        std::vector<double> F(m), Inv(m), E(m), lam_x(n), lam_y(n);
        const long long period = 2LL * (n - 1);
        for (int k = 0; k < n; k++)
            for (int j = 0; j < n; j++) {
                const long long kj = ((long long)k * j) % period;
                const double c = cos(M_PI * (double)kj / (double)(n - 1));
                const double w = (j == 0 || j == n - 1) ? 1.0 : 2.0;
                F[(size_t)k * n + j] = w * c;
                Inv[(size_t)k * n + j] = w * c / (double)period;
            }
        for (int k = 0; k < n; k++) {
            lam_x[k] = (2.0 * cos(M_PI * k / (n - 1)) - 2.0) / (ops->gg.d0 * ops->gg.d0);
            lam_y[k] = (2.0 * cos(M_PI * k / (n - 1)) - 2.0) / (ops->gg.d1 * ops->gg.d1);
        }
        for (int ky = 0; ky < n; ky++)
            for (int kx = 0; kx < n; kx++)
                E[(size_t)ky * n + kx] = 1.0 / (1.0 - dt * d_c * (lam_y[ky] + lam_x[kx]));
        CS_CUDA(cudaMalloc(&ops->F, m * 8));
        CS_CUDA(cudaMalloc(&ops->Inv, m * 8));
        CS_CUDA(cudaMalloc(&ops->E, m * 8));
        CS_CUDA(cudaMalloc(&ops->T1, m * 8));
        CS_CUDA(cudaMalloc(&ops->T2, m * 8));
        CS_CUDA(cudaMalloc(&ops->rhs, m * 8));
        CS_CUDA(cudaMemcpy(ops->F, F.data(), m * 8, cudaMemcpyHostToDevice));
        CS_CUDA(cudaMemcpy(ops->Inv, Inv.data(), m * 8, cudaMemcpyHostToDevice));
        CS_CUDA(cudaMemcpy(ops->E, E.data(), m * 8, cudaMemcpyHostToDevice));
        if (n <= ROWS2_MAX_N) {  // transposed copies for k_gemm_rows2
            std::vector<double> FT(m), InvT(m);
            for (int k = 0; k < n; k++)
                for (int j = 0; j < n; j++) {
                    FT[(size_t)j * n + k] = F[(size_t)k * n + j];
                    InvT[(size_t)j * n + k] = Inv[(size_t)k * n + j];
                }
            CS_CUDA(cudaMalloc(&ops->FT, m * 8));
            CS_CUDA(cudaMalloc(&ops->InvT, m * 8));
            CS_CUDA(cudaMemcpy(ops->FT, FT.data(), m * 8, cudaMemcpyHostToDevice));
            CS_CUDA(cudaMemcpy(ops->InvT, InvT.data(), m * 8, cudaMemcpyHostToDevice));
        }
        return CS_OK;
    }
    // periodic: eigenvalues (2 cos(2 pi k / n) - 2) / h^2 of the circulant
    // 1-D Laplacians of field.py:114-125.
    ops->kind = 2;
    std::vector<double> lx(n), ly(n);
    for (int k = 0; k < n; k++) {
        lx[k] = (2.0 * cos(2.0 * M_PI * k / n) - 2.0) / (ops->gg.d0 * ops->gg.d0);
        ly[k] = (2.0 * cos(2.0 * M_PI * k / n) - 2.0) / (ops->gg.d1 * ops->gg.d1);
    }
    CS_CUDA(cudaMalloc(&ops->lx, n * 8));
    CS_CUDA(cudaMalloc(&ops->ly, n * 8));
    CS_CUDA(cudaMemcpy(ops->lx, lx.data(), n * 8, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(ops->ly, ly.data(), n * 8, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMalloc(&ops->rhs, m * es));
    if (spectral_on(ops)) return CS_OK;  // spectral.cu allocates its own buffers
    const size_t nh = (size_t)n / 2 + 1;
    CS_CUDA(cudaMalloc(&ops->spec, (size_t)n * nh * 2 * es));
    CS_TRY(cufft_check(cufftPlan2d(&ops->pf, n, n, prec == CS_F64 ? CUFFT_D2Z : CUFFT_R2C),
                       "plan fwd"));
    CS_TRY(cufft_check(cufftPlan2d(&ops->pi, n, n, prec == CS_F64 ? CUFFT_Z2D : CUFFT_C2R),
                       "plan inv"));
    ops->have_plans = true;
    return CS_OK;
}

void field_ops_destroy(cs_field_ops *ops) {
    if (!ops) return;
    if (ops->have_plans) {
        cufftDestroy(ops->pf);
        cufftDestroy(ops->pi);
    }
    for (void *p : {(void *)ops->F, (void *)ops->Inv, (void *)ops->FT, (void *)ops->InvT,
                    (void *)ops->E, (void *)ops->T1,
                    (void *)ops->T2, (void *)ops->lx, (void *)ops->ly, ops->rhs, ops->spec,
                    ops->specT, ops->tw})
        if (p) cudaFree(p);
    delete ops;
}

// out = solve(ops->rhs) for the prepared system.  out has the grid dtype.
int field_solve_rhs(cs_field_ops *ops, void *out) {
    cs_ctx *ctx = ops->ctx;
    const int n = ops->gg.n;
    const size_t m = (size_t)n * n;
    const size_t es = ops->prec == CS_F64 ? 8 : 4;
    if (ops->kind == 0) {
        if (out != ops->rhs)
            CS_CUDA(cudaMemcpyAsync(out, ops->rhs, m * es, cudaMemcpyDeviceToDevice, ctx->stream));
        return CS_OK;
    }
    if (ops->kind == 1) {
        // modal = E * (F X F^T); out = Inv modal Inv^T (field.py:166-167)
        const double *X = (const double *)ops->rhs;
        if (ops->FT && n % 2 == 0 && !getenv("CS_GEMM16")) {
            CS_TRY(gemm_rows2<double>(ctx, ops->F, X, ops->FT, ops->E, ops->T2, n));
            if (ops->prec == CS_F64)
                return gemm_rows2<double>(ctx, ops->Inv, ops->T2, ops->InvT, nullptr,
                                          (double *)out, n);
            return gemm_rows2<float>(ctx, ops->Inv, ops->T2, ops->InvT, nullptr, (float *)out, n);
        }
        CS_TRY(gemm<double>(ctx, ops->F, X, false, nullptr, ops->T1, n));
        CS_TRY(gemm<double>(ctx, ops->T1, ops->F, true, ops->E, ops->T2, n));
        CS_TRY(gemm<double>(ctx, ops->Inv, ops->T2, false, nullptr, ops->T1, n));
        if (ops->prec == CS_F64)
            CS_TRY(gemm<double>(ctx, ops->T1, ops->Inv, true, nullptr, (double *)out, n));
        else
            CS_TRY(gemm<float>(ctx, ops->T1, ops->Inv, true, nullptr, (float *)out, n));
        return CS_OK;
    }
    if (spectral_on(ops)) return spectral_solve(ops, ops->rhs, out);
    if (!ops->have_plans) {
        set_error("periodic solve: no cuFFT plans (CS_CUFFT set after the operator was built)");
        return CS_ERR_PARAM;
    }
    CS_TRY(cufft_check(cufftSetStream(ops->pf, ctx->stream), "stream"));
    CS_TRY(cufft_check(cufftSetStream(ops->pi, ctx->stream), "stream"));
    const double dtdc = ops->dt * ops->d_c;
    const double inv_nn = 1.0 / ((double)n * (double)n);
    const int B = 256;
    const long long ms = (long long)n * (n / 2 + 1);
    if (ops->prec == CS_F64) {
        CS_TRY(cufft_check(cufftExecD2Z(ops->pf, (cufftDoubleReal *)ops->rhs,
                                        (cufftDoubleComplex *)ops->spec),
                           "D2Z"));
        k_mode_scale<double2><<<(n < 148 * 8 ? n : 148 * 8), B, 0, ctx->stream>>>(
            (double2 *)ops->spec, n, ops->lx, ops->ly, dtdc, inv_nn);
        CS_LAUNCH_CHECK();
        CS_TRY(cufft_check(cufftExecZ2D(ops->pi, (cufftDoubleComplex *)ops->spec,
                                        (cufftDoubleReal *)out),
                           "Z2D"));
    } else {
        CS_TRY(cufft_check(cufftExecR2C(ops->pf, (cufftReal *)ops->rhs, (cufftComplex *)ops->spec),
                           "R2C"));
        k_mode_scale<float2><<<(n < 148 * 8 ? n : 148 * 8), B, 0, ctx->stream>>>(
            (float2 *)ops->spec, n, ops->lx, ops->ly, dtdc, inv_nn);
        CS_LAUNCH_CHECK();
        CS_TRY(cufft_check(cufftExecC2R(ops->pi, (cufftComplex *)ops->spec, (cufftReal *)out),
                           "C2R"));
    }
    ctx->launches += 1;  // k_mode_scale (cuFFT's own kernels not counted)
    return CS_OK;
}

int field_rhs(cs_field_ops *ops, const void *c, const void *ra, const void *rb, double ka,
              double kb, double gamma, const DevStatus *st) {
    cs_ctx *ctx = ops->ctx;
    const double dt = ops->dt;
    const RhsCoef k = make_rhs_coef(dt, ka, kb, gamma);
    const long long m = (long long)ops->gg.n * ops->gg.n;
    const int B = 256;
    const int G = grid_for(m, B, 148 * 16);
    if (ops->prec == CS_F64) {
        k_rhs<double, double><<<G, B, 0, ctx->stream>>>((const double *)c, (const double *)ra,
                                                        (const double *)rb, m, k,
                                                        (double *)ops->rhs, st);
    } else if (ops->kind == 1) {
        k_rhs<float, double><<<G, B, 0, ctx->stream>>>((const float *)c, (const float *)ra,
                                                       (const float *)rb, m, k,
                                                       (double *)ops->rhs, st);
    } else {
        k_rhs<float, float><<<G, B, 0, ctx->stream>>>((const float *)c, (const float *)ra,
                                                      (const float *)rb, m, k,
                                                      (float *)ops->rhs, st);
    }
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// copy an external rhs (grid dtype) into the ops' rhs slot (solve seam)
int field_load_rhs(cs_field_ops *ops, const void *rhs) {
    cs_ctx *ctx = ops->ctx;
    const long long m = (long long)ops->gg.n * ops->gg.n;
    if (ops->kind == 1 && ops->prec == CS_F32) {
        RhsCoef k{};  // identity: rhs = c
        k_rhs<float, double><<<grid_for(m, 256, 148 * 16), 256, 0, ctx->stream>>>(
            (const float *)rhs, nullptr, nullptr, m, k, (double *)ops->rhs, nullptr);
        CS_LAUNCH_CHECK();
        return CS_OK;
    }
    const size_t es = ops->prec == CS_F64 ? 8 : 4;
    CS_CUDA(cudaMemcpyAsync(ops->rhs, rhs, (size_t)m * es, cudaMemcpyDeviceToDevice, ctx->stream));
    return CS_OK;
}

}  // namespace cs
