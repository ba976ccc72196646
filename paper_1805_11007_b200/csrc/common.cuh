// common.cuh -- shared device helpers, context and scratch management.
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "../../include/chemo_b200.h"
#include "glibc_exp.h"

namespace cs {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);

#define CS_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) {                                             \
            ::cs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,       \
                            cudaGetErrorString(e_));                         \
            return CS_ERR_CUDA;                                              \
        }                                                                    \
    } while (0)

#define CS_LAUNCH_CHECK()                                                    \
    do {                                                                     \
        cudaError_t e_ = cudaGetLastError();                                 \
        if (e_ != cudaSuccess) {                                             \
            ::cs::set_error("%s:%d launch: %s", __FILE__, __LINE__,          \
                            cudaGetErrorString(e_));                         \
            return CS_ERR_CUDA;                                              \
        }                                                                    \
    } while (0)

#define CS_TRY(expr)                                                         \
    do {                                                                     \
        int rc_ = (expr);                                                    \
        if (rc_ != CS_OK) return rc_;                                        \
    } while (0)

// ---------------------------------------------------------------- scratch
struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
    int ensure(size_t need);  // grow-only, contents not preserved
    void release();
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// Device status word shared by every kernel of a fused step: kernels return
// immediately once `abort` is set (a later step must not run on a state the
// reference would have refused).
struct DevStatus {
    unsigned long long key;   // min over (rank, particle, code), ~0 = ok
    int abort;
    int step;
    int field_bad;
    unsigned blocks_done;     // gradient launches: blocks past their field checks
    long long clamped;
    long long neg_steps;
    double first_neg;
    double neg_mass;          // scratch: this step's negative weighted mass
    int neg_flag;             // scratch: this step saw a negative node
    int pad2;
    unsigned long long react_flips[2];  // Alpha -> Beta, Beta -> Alpha
    unsigned long long react_high_n;    // particle-steps with a flip probability > 1
    unsigned long long react_high_bits; // max such probability (binary64 bits; > 0)
};

// error key: rank 0 = non-finite (lowest index wins), rank 1 + ax = axis
// error; within a rank the lowest particle index wins.
__host__ __device__ inline unsigned long long err_key(int rank, long long i, int code) {
    return ((unsigned long long)rank << 60) | ((unsigned long long)i << 3) |
           (unsigned long long)code;
}

}  // namespace cs

struct cs_fast;

struct cs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cs::Buf keys, skeys, counts, starts, order, force, tile_flags, tmp, status, zpar, obs, spos,
        coop_sums,
        stype,
        pair_counts, pair_offsets, host_scratch,
        // ordered deposit (deposit.cu): bin keys / counts / starts, slots, sorted copies
        dep_keys, dep_counts, dep_starts, dep_slots, dep_pos, dep_meta;
    cs::DevStatus *dstat() { return status.as<cs::DevStatus>(); }
    int64_t launches = 0;
};

namespace cs {

// ---------------------------------------------------------------- math
// Explicitly rounded binary64 arithmetic: the reference (numba/numpy) never
// contracts a*b+c, so neither may the parity-critical kernels.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

__host__ __device__ __forceinline__ long long pymod(long long a, long long n) {
    long long r = a % n;
    return r < 0 ? r + n : r;
}

template <class P> struct Vec2;
template <> struct Vec2<double> { using T = double2; };
template <> struct Vec2<float> { using T = float2; };

template <class P>
__device__ __forceinline__ void load2(const P *__restrict__ a, long long i, double &x, double &y) {
    auto v = reinterpret_cast<const typename Vec2<P>::T *>(a)[i];
    x = (double)v.x;
    y = (double)v.y;
}
template <class P>
__device__ __forceinline__ void store2(P *__restrict__ a, long long i, double x, double y) {
    typename Vec2<P>::T v;
    v.x = (P)x;
    v.y = (P)y;
    reinterpret_cast<typename Vec2<P>::T *>(a)[i] = v;
}

// Cell geometry of the reference binning (motion.py:171-174).
struct BinGeom {
    int n0, n1;
    double lo0, lo1, size0, size1, eff0, eff1;
    int per0, per1;
};

BinGeom make_geom(const cs_domain &d, double cell_cutoff);

__device__ __forceinline__ int cell_axis(double v, double lo, double eff, int n) {
    double f = floor(ddiv(dsub(v, lo), eff));
    if (!(f >= 0.0)) return 0;  // also NaN -> 0
    if (f >= (double)n) return n - 1;
    return (int)f;
}

// fl(a / b) and floor(fl(a / b)) without a division in the common case.
// When b is a power of two a * (1/b) is exact.  Otherwise q = a * fl(1/b)
// is within 3 ulp of fl(a/b), so floor(q) == floor(fl(a/b)) unless q lies
// within a (generous) 2^-49 relative band of an integer, where the exact
// quotient is recomputed.
struct ExactDiv {
    double b, inv;
    int pow2;
};
ExactDiv make_exact_div(double b);
__device__ __forceinline__ double ediv(double a, const ExactDiv &d) {
    return d.pow2 ? dmul(a, d.inv) : ddiv(a, d.b);
}
static __device__ __noinline__ double floor_ddiv(double a, double b) { return floor(ddiv(a, b)); }
__device__ __forceinline__ double floor_div(double a, const ExactDiv &d) {
    const double q = dmul(a, d.inv);
    double f = floor(q);
    if (!d.pow2) {
        const double tol = fabs(q) * 0x1p-49 + 0x1p-1022;
        if (dsub(q, f) < tol || dsub(dadd(f, 1.0), q) < tol) f = floor_ddiv(a, d.b);
    }
    return f;
}
__device__ __forceinline__ int cell_axis_fast(double v, double lo, const ExactDiv &eff, int n) {
    const double f = floor_div(dsub(v, lo), eff);
    if (!(f >= 0.0)) return 0;
    if (f >= (double)n) return n - 1;
    return (int)f;
}

struct PairTab {
    double eps[4];
    double cut2[4];
};
PairTab make_pairtab(const cs_pair_params &pp);

// Grid geometry (field.py:33-66) for coupling kernels.
struct GridGeom {
    int n;
    int per;
    double lo0, lo1, d0, d1;
};
GridGeom make_grid_geom(const cs_grid &g);

// Bilinear stencil of coupling.py:216-258 (_bilinear): corner node indices
// and weights in the reference arithmetic; returns the number of clamped
// coordinates (neumann hull clamp).
struct Bilin {
    long long r00, r10, r01, r11;
    double w00, w10, w01, w11;
};
__device__ __forceinline__ int bilinear_stencil(double px, double py, const GridGeom &gg,
                                                Bilin &b) {
    int clamped = 0;
    double u0 = ddiv(dsub(px, gg.lo0), gg.d0);
    double u1 = ddiv(dsub(py, gg.lo1), gg.d1);
    long long b0, b1, c0, c1;
    double f0, f1;
    const int n = gg.n;
    if (gg.per) {
        const double f0f = floor(u0), f1f = floor(u1);
        b0 = pymod((long long)f0f, n);
        b1 = pymod((long long)f1f, n);
        f0 = dsub(u0, f0f);
        f1 = dsub(u1, f1f);
        c0 = (b0 + 1) % n;
        c1 = (b1 + 1) % n;
    } else {
        const double nm1 = (double)(n - 1);
        if (u0 < 0.0) { u0 = 0.0; clamped++; }
        else if (u0 > nm1) { u0 = nm1; clamped++; }
        if (u1 < 0.0) { u1 = 0.0; clamped++; }
        else if (u1 > nm1) { u1 = nm1; clamped++; }
        b0 = (long long)floor(u0);
        if (b0 > n - 2) b0 = n - 2;
        b1 = (long long)floor(u1);
        if (b1 > n - 2) b1 = n - 2;
        f0 = dsub(u0, (double)b0);
        f1 = dsub(u1, (double)b1);
        c0 = b0 + 1;
        c1 = b1 + 1;
    }
    b.w00 = dmul(dsub(1.0, f0), dsub(1.0, f1));
    b.w10 = dmul(f0, dsub(1.0, f1));
    b.w01 = dmul(dsub(1.0, f0), f1);
    b.w11 = dmul(f0, f1);
    b.r00 = b1 * n + b0;
    b.r10 = b1 * n + c0;
    b.r01 = c1 * n + b0;
    b.r11 = c1 * n + c0;
    return clamped;
}

// sum in the reference order: ((w00 v00 + w10 v10) + w01 v01) + w11 v11
template <class G>
__device__ __forceinline__ double bilinear_apply(const Bilin &b, const G *__restrict__ v, int m,
                                                 int k) {
    const double a = dmul(b.w00, (double)v[b.r00 * m + k]);
    const double c = dmul(b.w10, (double)v[b.r10 * m + k]);
    const double d = dmul(b.w01, (double)v[b.r01 * m + k]);
    const double e = dmul(b.w11, (double)v[b.r11 * m + k]);
    return dadd(dadd(dadd(a, c), d), e);
}

// The interaction increment of the proposal: force dt (em_step,
// motion.py:281-282) or, tamed (tamed_step, motion.py:283-298),
// (force dt) / (1 + ||force|| dt) with ||force|| = sqrt((-0 + f0^2) + f1^2)
// (numpy's pairwise row sum).
__device__ __forceinline__ void force_increment(double f0, double f1, double dt, int tamed,
                                                double &i0, double &i1) {
    if (!tamed) {
        i0 = dmul(f0, dt);
        i1 = dmul(f1, dt);
        return;
    }
    const double fn = dsqrt(dadd(dadd(-0.0, dmul(f0, f0)), dmul(f1, f1)));
    const double den = dadd(1.0, dmul(fn, dt));
    i0 = ddiv(dmul(f0, dt), den);
    i1 = ddiv(dmul(f1, dt), den);
}

// One axis of _boundaries_kernel (motion.py:363-401).  Returns 0, 2 or 3.
__device__ __forceinline__ int boundary_axis(double &v, double &a, double lo, double hi,
                                             int per) {
    const double size = dsub(hi, lo);
    if (per) {
        const double k = floor(ddiv(dsub(v, lo), size));
        if (k != 0.0) {
            const double shift = dmul(k, size);
            v = dsub(v, shift);
            a = dsub(a, shift);
        }
        for (int it = 0; it < 2; it++) {
            if (v >= hi) {
                v = dsub(v, size);
                a = dsub(a, size);
            } else if (v < lo) {
                v = dadd(v, size);
                a = dadd(a, size);
            } else {
                break;
            }
        }
        return 0;
    }
    if (v > dadd(hi, size) || v < dsub(lo, size)) return 2;
    for (int it = 0; it < 4; it++) {
        if (v > hi) v = dsub(dmul(2.0, hi), v);
        else if (v < lo) v = dsub(dmul(2.0, lo), v);
        else return 0;
    }
    return 3;
}

inline int grid_for(long long n, int block, int max_blocks = 148 * 64) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

// ---------------------------------------------------------------- launchers
// bins.cu
// order / starts of the reference's cell list, and positions (and types, if
// given) copied into that order in ctx->spos / ctx->stype for the force walk
struct DepBin;
// With `dep`, the same pass also bins the depositing particles for the
// ordered deposit (deposit.cu): their bins follow the cells in ctx->counts /
// ctx->starts (starts[nflat + b], slots numbered from n), the positions and
// (index, route) words in bin order go to ctx->dep_pos / ctx->dep_meta.
// *dep_done tells whether it did (the single-block small path does not).
int bin_particles(cs_ctx *ctx, int prec, const void *pos, long long n, const BinGeom &g,
                  const uint8_t *type = nullptr, const DepBin *dep = nullptr,
                  bool *dep_done = nullptr);
// the implicit solve's right-hand side c (1 - dt gamma) + dt ka rho_a -
// dt kb rho_b c (field.py:226-232), fused into the deposit gather of a
// DCT-solved grid (rhs in binary64)
struct RhsCoef {
    double one_m_dtg, dka, dkb;
    int has_g, has_a, has_b;
};
RhsCoef make_rhs_coef(double dt, double ka, double kb, double gamma);
struct RhsFuse {
    const void *c;  // grid dtype
    RhsCoef k;
    double *rhs;
};
int launch_deposit_binned(cs_ctx *ctx, int prec, const GridGeom &gg, int kind, double h,
                          double cutoff, const int *starts, int off, void *ra, void *rb,
                          const DevStatus *st,
                          const RhsFuse *rf = nullptr);
int exclusive_scan_i32(cs_ctx *ctx, const int *in, int *out, long long n,
                       int *zero_in = nullptr);
// forces.cu
int launch_soft_forces(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                       long long n, const BinGeom &g, const PairTab &pt, double *out,
                       const DevStatus *st);
int launch_cell_xy(cs_ctx *ctx, int prec, const void *pos, long long n, const BinGeom &g,
                   int *out);
int launch_index_forces(cs_ctx *ctx, int prec, const void *pos, long long n, const int *cxy,
                        const int *order, const int *starts, int ncx, int ncy, double effx,
                        double effy, int perx, int pery, double lx, double ly, double eps,
                        double cutoff, double *out);
// field.cu
int launch_deposit_gather(cs_ctx *ctx, int prec, const void *pos, long long np,
                          const GridGeom &gg, double spanx, double spany, double h, double cutoff,
                          double inv_norm, double *out);
// motion.cu / field.cu / sim.cu
int record_error(cs_ctx *ctx);
int run_soft_force_pairs(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                         long long n, const BinGeom &g, const PairTab &pt,
                         int64_t *pairs, int64_t cap, int64_t *count);


// ---- shared with ensemble.cu (definitions of the host helpers in field.cu)
struct Route {
    unsigned char bits[3];  // indexed by min(type, 2): bit0 -> rho_a, bit1 -> rho_b
};

__device__ __forceinline__ unsigned route_bits(const uint8_t *type, long long p, const Route &r) {
    const unsigned t = type ? (unsigned)type[p] : 0u;
    return r.bits[t < 2u ? t : 2u];
}

struct GaussParams {
    double inv_norm, two_h2, cut2;
    int w0, w1;
};

// Deposit bins built together with the cell list (bins.cu / deposit.cu).
struct DepBin {
    GridGeom gg;
    int kind;  // CS_CIC / CS_GAUSSIAN
    Route route;
};

GaussParams make_gauss(const GridGeom &gg, double h, double cutoff);

// d1 coefficients (field.py:128-137), each entry value / (2 h) as the
// reference's lil / scalar division produces them.
struct D1Coef {
    double m1, p1;        // interior / periodic: -1/(2h), +1/(2h)
    double l0, l1, l2;    // neumann row 0: -3, 4, -1 over 2h
    double r0, r1, r2;    // neumann row n-1 (cols n-3, n-2, n-1): 1, -4, 3 over 2h
};
D1Coef make_d1(double h);

template <class G>
__device__ __forceinline__ double d1_at(const G *__restrict__ c, long long base, long long stride,
                                        int i, int n, int per, const D1Coef &k) {
    if (per) {
        const int im = i == 0 ? n - 1 : i - 1, ip = i == n - 1 ? 0 : i + 1;
        const double am = dmul(k.m1, (double)c[base + im * stride]);
        const double ap = dmul(k.p1, (double)c[base + ip * stride]);
        return im < ip ? dadd(dadd(0.0, am), ap) : dadd(dadd(0.0, ap), am);
    }
    if (i == 0)
        return dadd(dadd(dadd(0.0, dmul(k.l0, (double)c[base])),
                         dmul(k.l1, (double)c[base + stride])),
                    dmul(k.l2, (double)c[base + 2 * stride]));
    if (i == n - 1)
        return dadd(dadd(dadd(0.0, dmul(k.r0, (double)c[base + (long long)(n - 3) * stride])),
                         dmul(k.r1, (double)c[base + (long long)(n - 2) * stride])),
                    dmul(k.r2, (double)c[base + (long long)(n - 1) * stride]));
    return dadd(dadd(0.0, dmul(k.m1, (double)c[base + (long long)(i - 1) * stride])),
                dmul(k.p1, (double)c[base + (long long)(i + 1) * stride]));
}


// The reference pair loop of one particle (motion.py:200-245); used by
// forces.cu and ensemble.cu.
template <class P, class Visit>
__device__ __forceinline__ void pair_loop(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                                          const int *__restrict__ order,
                                          const int *__restrict__ starts, const BinGeom &g,
                                          const PairTab &pt, int i, Visit visit) {
    double xi, yi;
    load2(pos, i, xi, yi);
    const int cx = cell_axis(xi, g.lo0, g.eff0, g.n0);
    const int cy = cell_axis(yi, g.lo1, g.eff1, g.n1);
    const int ti = type ? (int)type[i] : 0;
    for (int o1 = -1; o1 <= 1; o1++) {
        int g1 = cy + o1;
        if (g.per1) {
            if (g.n1 == 1 && o1 != 0) continue;
            if (g.n1 == 2 && o1 == 1) continue;
            g1 = (int)pymod(g1, g.n1);
        } else if (g1 < 0 || g1 >= g.n1) {
            continue;
        }
        for (int o0 = -1; o0 <= 1; o0++) {
            int g0 = cx + o0;
            if (g.per0) {
                if (g.n0 == 1 && o0 != 0) continue;
                if (g.n0 == 2 && o0 == 1) continue;
                g0 = (int)pymod(g0, g.n0);
            } else if (g0 < 0 || g0 >= g.n0) {
                continue;
            }
            const int f = g1 * g.n0 + g0;
            const int kend = starts[f + 1];
            for (int k = starts[f]; k < kend; k++) {
                const int j = order[k];
                if (j == i) continue;
                double xj, yj;
                load2(pos, j, xj, yj);
                double dx0 = dsub(xj, xi);
                double dx1 = dsub(yj, yi);
                if (g.per0) dx0 = dsub(dx0, dmul(g.size0, rint(ddiv(dx0, g.size0))));
                if (g.per1) dx1 = dsub(dx1, dmul(g.size1, rint(ddiv(dx1, g.size1))));
                const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                const int t = ti * 2 + (type ? (int)type[j] : 0);
                if (r2 > pt.cut2[t] || r2 == 0.0) continue;
                const double eps = pt.eps[t];
                const double r = dsqrt(r2);
                const double s = -ddiv(cs_exp(-ddiv(r, eps)), dmul(eps, r));
                visit(j, s, dx0, dx1);
            }
        }
    }
}

}  // namespace cs

// ------------------------------------------------------------------ ops
struct cs_field_ops {
    cs_ctx *ctx = nullptr;
    int prec = CS_F64;
    cs::GridGeom gg{};
    int kind = 0;  // 0 identity, 1 dct, 2 fft
    double dt = 0, d_c = 0;
    double *F = nullptr, *Inv = nullptr, *E = nullptr, *T1 = nullptr, *T2 = nullptr;
    double *FT = nullptr, *InvT = nullptr;  // transposes (grids <= 128^2: k_gemm_rows2)
    double *lx = nullptr, *ly = nullptr;
    void *rhs = nullptr;   // G (fft / identity) or double (dct)
    void *spec = nullptr;  // complex n x (n/2+1) (cuFFT path)
    cufftHandle pf = 0, pi = 0;
    bool have_plans = false;
    void *specT = nullptr, *tw = nullptr;  // spectral.cu: transposed half spectrum, twiddles
};

namespace cs {
// spectral.cu: the periodic solve as three fused passes (n = 2^k, 16..8192);
// CS_CUFFT=1 selects the cuFFT path instead (comparisons)
int spectral_supported(int n);
inline bool spectral_on(const cs_field_ops *ops) {
    return ops->kind == 2 && spectral_supported(ops->gg.n) && !getenv("CS_CUFFT");
}
int spectral_step_q(cs_field_ops *ops, float *c, const int *q, double gamma, double ka,
                    double kb, double scale, const DevStatus *st);
int spectral_step_g(cs_field_ops *ops, void *c, const void *ra, const void *rb, double gamma,
                    double ka, double kb, const DevStatus *st);
int spectral_solve(cs_field_ops *ops, const void *rhs, void *out);
}  // namespace cs

