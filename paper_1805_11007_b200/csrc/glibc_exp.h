/*
 * glibc_exp.h -- binary64 exp that reproduces the host glibc (>= 2.28,
 * x86-64 FMA code path) bit for bit, for host and device.
 *
 * Why: the reference's pair force calls exp() through numba, which lowers
 * to the host libm (numba np.exp == glibc exp on 10^6 inputs).
 * CUDA's exp() is a different (<= 1 ulp) implementation, so bitwise force
 * parity needs the same algorithm on the device.
 *
 * Algorithm (the published design of glibc's exp, from ARM
 * optimized-routines): k = round(x * N / ln2), r = x - k ln2/N (two-part
 * constant), exp(x) = 2^(k/N) * (1 + tmp) with
 *   tmp = tail + r + r^2 (C2 + r C3) + r^4 (C4 + r C5)
 * evaluated with the fused multiply-adds the FMA build of glibc uses, and a
 * rescaled path for |x| >= 512.  The 2^(i/N) table is generated from first
 * principles by tools/exp_table.py.  Verified bitwise against the host libm
 * on 2e8 inputs over [-740, 740] (tests/test_oracle_golden.py re-checks a
 * sample on every run; tests/test_gpu_parity.py checks the device copy).
 */
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define CS_HD __device__ __forceinline__
/* plain global memory (L1-resident, 2 KB): lanes index it divergently, which
 * the constant cache would serialise */
#define CS_EXP_TABLE_ATTR __device__ static
#else
#define CS_HD static inline
#define CS_EXP_TABLE_ATTR static
#endif

#include "glibc_exp_table.h"

#ifdef __CUDACC__
#define CS_AS_U64(x) ((uint64_t)__double_as_longlong(x))
#define CS_AS_F64(u) __longlong_as_double((long long)(u))
#define CS_FMA(a, b, c) __fma_rn((a), (b), (c))
#define CS_MUL(a, b) __dmul_rn((a), (b))
#define CS_ADD(a, b) __dadd_rn((a), (b))
#define CS_SUB(a, b) __dsub_rn((a), (b))
#else
static inline uint64_t cs_as_u64_(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double cs_as_f64_(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define CS_AS_U64(x) cs_as_u64_(x)
#define CS_AS_F64(u) cs_as_f64_(u)
#define CS_FMA(a, b, c) fma((a), (b), (c))
#define CS_MUL(a, b) ((a) * (b))
#define CS_ADD(a, b) ((a) + (b))
#define CS_SUB(a, b) ((a) - (b))
#endif

#ifdef __CUDACC__
#define CS_EXP_TAB(i) __ldg(&cs_exp_tab[i])
#else
#define CS_EXP_TAB(i) cs_exp_tab[i]
#endif

CS_HD double cs_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    double scale, y;
    if ((ki & 0x80000000ULL) == 0) {
        /* k > 0: the scale exponent may have overflowed by <= 460 */
        sbits -= 1009ULL << 52;
        scale = CS_AS_F64(sbits);
        return CS_MUL(0x1p1009, CS_FMA(scale, tmp, scale));
    }
    /* k < 0: careful rounding into the subnormal range */
    sbits += 1022ULL << 52;
    scale = CS_AS_F64(sbits);
    y = CS_ADD(scale, CS_MUL(scale, tmp));
    if (y < 1.0) {
        double lo = CS_ADD(CS_SUB(scale, y), CS_MUL(scale, tmp));
        double hi = CS_ADD(1.0, y);
        lo = CS_ADD(CS_ADD(CS_SUB(1.0, hi), y), lo);
        y = CS_SUB(CS_ADD(hi, lo), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return CS_MUL(0x1p-1022, y);
}

CS_HD double cs_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep0 * CS_EXP_N;
    const double Shift = 0x1.8p52;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8;
    const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = (uint32_t)(CS_AS_U64(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if (abstop - 0x3c9u >= 0x80000000u) return CS_ADD(1.0, x); /* tiny */
        if (abstop >= 0x409u) {                                      /* |x| >= 1024 */
            if (CS_AS_U64(x) == CS_AS_U64(-INFINITY)) return 0.0;
            if (abstop >= 0x7ffu) return CS_ADD(1.0, x);
            return (CS_AS_U64(x) >> 63) ? 0.0 : INFINITY;
        }
        abstop = 0; /* 512 <= |x| < 1024 */
    }
    double kd = CS_FMA(InvLn2N, x, Shift);
    const uint64_t ki = CS_AS_U64(kd);
    kd = CS_SUB(kd, Shift);
    const double r = CS_FMA(kd, NegLn2loN, CS_FMA(kd, NegLn2hiN, x));
    const uint64_t idx = 2 * (ki % CS_EXP_N);
    const uint64_t top = ki << (52 - CS_EXP_TABLE_BITS);
    const double tail = CS_AS_F64(CS_EXP_TAB(idx));
    const uint64_t sbits = CS_EXP_TAB(idx + 1) + top;
    const double r2 = CS_MUL(r, r);
    const double tmp = CS_FMA(CS_MUL(r2, r2), CS_FMA(r, C5, C4),
                              CS_FMA(r2, CS_FMA(r, C3, C2), CS_ADD(tail, r)));
    if (abstop == 0) return cs_exp_specialcase(tmp, sbits, ki);
    const double scale = CS_AS_F64(sbits);
    return CS_FMA(scale, tmp, scale);
}
