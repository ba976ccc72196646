// deposit.cuh -- per-particle deposit arithmetic shared by the direct
// engine's ordered deposit (deposit.cu) and the ensemble engine (ensemble.cu).
#pragma once
#include "common.cuh"

namespace cs {

constexpr unsigned DEP_ID_MASK = (1u << 30) - 1u;

// The particle's deposit bin.  CIC: the base cell floor(u) (periodic:
// wrapped; neumann: clipped to [0, n-2], coupling.py:124-131); gaussian: the
// nearest node floor(u + 0.5) (periodic: wrapped; neumann: clamped to
// [0, n-1] -- a clamped particle keeps its true offsets for the stamp test).
__device__ __forceinline__ int dep_bin_axis(double u, int kind, int n, int per) {
    double b = floor(kind == CS_CIC ? u : dadd(u, 0.5));
    if (per) return (int)pymod((long long)b, n);  // |b| < 2^52 (checked by the caller)
    const double top = (double)(kind == CS_CIC ? n - 2 : n - 1);
    b = b < 0.0 ? 0.0 : (b > top ? top : b);
    return (int)b;
}

// CIC weights of one particle (coupling.py:120-137): corner q = 00, 10, 01, 11
__device__ __forceinline__ double cic_weight(double x, double y, const GridGeom &gg, double unit,
                                             int q) {
    const double u0 = ddiv(dsub(x, gg.lo0), gg.d0);
    const double u1 = ddiv(dsub(y, gg.lo1), gg.d1);
    double f0, f1;
    if (gg.per) {
        f0 = dsub(u0, floor(u0));
        f1 = dsub(u1, floor(u1));
    } else {
        const double top = (double)(gg.n - 2);
        double b0 = floor(u0), b1 = floor(u1);
        b0 = b0 < 0.0 ? 0.0 : (b0 > top ? top : b0);
        b1 = b1 < 0.0 ? 0.0 : (b1 > top ? top : b1);
        f0 = dsub(u0, b0);
        f1 = dsub(u1, b1);
    }
    const double wx = (q & 1) ? f0 : dsub(1.0, f0);
    const double wy = (q & 2) ? f1 : dsub(1.0, f1);
    return dmul(dmul(wx, wy), unit);
}

// The stamp value particle (x, y) leaves on node (i, j) (coupling.py:95-110):
// false if the node is outside its stamp or beyond the cutoff.
__device__ __forceinline__ bool gauss_term_u(double u0, double u1, int i, int j,
                                             const GridGeom &gg, const GaussParams &gp,
                                             double &v) {
    const long long b0 = (long long)floor(dadd(u0, 0.5));
    const long long b1 = (long long)floor(dadd(u1, 0.5));
    long long o0 = (long long)i - b0, o1 = (long long)j - b1;
    if (gg.per) {
        o0 = pymod(o0, gg.n);
        if (o0 > gp.w0) o0 -= gg.n;
        o1 = pymod(o1, gg.n);
        if (o1 > gp.w1) o1 -= gg.n;
    }
    if (o0 < -gp.w0 || o0 > gp.w0 || o1 < -gp.w1 || o1 > gp.w1) return false;
    const double dy = dmul(dsub(u1, (double)(b1 + o1)), gg.d1);
    const double dy2 = dmul(dy, dy);
    const double dxp = dmul(dsub(u0, (double)(b0 + o0)), gg.d0);
    const double r2 = dadd(dmul(dxp, dxp), dy2);
    if (!(r2 <= gp.cut2)) return false;
    v = dmul(gp.inv_norm, cs_exp(-ddiv(r2, gp.two_h2)));
    return true;
}
__device__ __forceinline__ bool gauss_term(double x, double y, int i, int j, const GridGeom &gg,
                                           const GaussParams &gp, double &v) {
    return gauss_term_u(ddiv(dsub(x, gg.lo0), gg.d0), ddiv(dsub(y, gg.lo1), gg.d1), i, j, gg,
                        gp, v);
}

}  // namespace cs
