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

// ---------------------------------------------------------------------------
// One numpy stream drawn by the whole GPU (bit-identical to numpy's
// sequential Generator(PCG64).standard_normal / .random of the same state).
//
// The raw 64-bit outputs of PCG64 are addressable (jump-ahead of the LCG), but
// a ziggurat normal consumes a variable number of them (1 on the fast path,
// ~1.3 % take 2+: the wedge test draws a uniform and may restart, the tail
// loops on pairs of uniforms).  The stream is cut into chunks of ZC raw
// positions; a normal belongs to the chunk holding the position of its
// accepting attempt.  Per raw position p the attempt starting there has an
// advance adv(p) (raws consumed) and a flag final(p) (returns a value or
// restarts at p + adv).
//   k_zpar_scan:   a warp per chunk evaluates every position's attempt, walks
//                  the attempt chain from entry offset 0 (32 positions at a
//                  time: a ballot finds the next multi-raw attempt) and, for
//                  entry offsets 1..31, the short prefix until it joins that
//                  chain: table[chunk][e] = (normals, exit offset into the
//                  next chunk);
//   k_zpar_group / k_zpar_top / k_zpar_resolve: the chunk tables are
//                  composed per group of ZG chunks, the groups walked from
//                  entry 0, then every chunk's entry offset and first output
//                  index resolved;
//   k_zpar_emit:   a warp per chunk re-evaluates its positions and writes the
//                  normals of its chain from its entry offset.
// The last normal's end is the number of raws consumed; the stream state is
// advanced by exactly that (k_zpar_state).
constexpr int ZC = 2048;       // raw positions per chunk
constexpr int ZG = 128;        // chunks per group
constexpr int ZE = 32;         // entry offsets tabulated per chunk
constexpr int ZW = 4;          // warps (chunks) per block
typedef unsigned __int128 u128;

struct ZparState {
    unsigned long long s_hi, s_lo, i_hi, i_lo;  // stream state and increment at draw start
    long long m;                                // values wanted
    int kind;                                   // 0 normal, 1 uniform
    int f32;                                    // write binary32
};

__device__ __forceinline__ u128 mk128(unsigned long long hi, unsigned long long lo) {
    return ((u128)hi << 64) | lo;
}
constexpr unsigned long long PCG_MH = 0x2360ED051FC65DA4ull, PCG_ML = 0x4385DF649FCCF645ull;

// (A, C) with S_{k+d} = A S_k + C for the LCG S' = M S + inc
__device__ void lcg_jump(u128 inc, unsigned long long d, u128 &A, u128 &C) {
    u128 cm = mk128(PCG_MH, PCG_ML), cp = inc, am = 1, ap = 0;
    while (d) {
        if (d & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        d >>= 1;
    }
    A = am;
    C = ap;
}

__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
    const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
    const unsigned rot = (unsigned)(hi >> 58);
    const unsigned long long v = hi ^ lo;
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

// attempt at a raw position: state s = S_{p+1} (its output is raw p).
// returns adv | final << 7 (adv <= 127, else 0 = unsupported) and the value
__device__ int zig_attempt(u128 s, u128 inc, const ZigTables &zt, double &val) {
    constexpr double ZR = 3.6541528853610087963519472518;
    constexpr double ZIR = 0.27366123732975827203338247596;
    const u128 M = mk128(PCG_MH, PCG_ML);
    unsigned long long r = pcg_out(s);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = dmul((double)rabs, zt.wi[idx]);
    if (sign) x = -x;
    val = x;
    if (rabs < zt.ki[idx]) return 1 | 128;
    auto next_double = [&]() {
        s = s * M + inc;
        return (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    };
    if (idx == 0) {
        for (int tries = 1; tries <= 63; tries++) {
            const double xx = dmul(-ZIR, log1p_glibc(-next_double()));
            const double yy = -log1p_glibc(-next_double());
            if (dadd(yy, yy) > dmul(xx, xx)) {
                val = ((rabs >> 8) & 1) ? -dadd(ZR, xx) : dadd(ZR, xx);
                return (1 + 2 * tries) | 128;
            }
        }
        return 0;
    }
    const double f0 = zt.fi[idx - 1], f1 = zt.fi[idx];
    if (dadd(dmul(dsub(f0, f1), next_double()), f1) < cs_exp(dmul(dmul(-0.5, x), x))) return 2 | 128;
    return 2;  // rejected: the normal restarts at p + 2
}

__device__ __forceinline__ void zig_tables_load(ZigTables &zt) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        zt.ki[i] = ZIG_KI[i];
        zt.wi[i] = __longlong_as_double((long long)ZIG_WI[i]);
        zt.fi[i] = __longlong_as_double((long long)ZIG_FI[i]);
    }
}

// the attempt codes (and values) of the chunk's ZC positions into shared memory
__device__ void zpar_eval(const ZparState &z, long long chunk, const ZigTables &zt,
                          unsigned char *code, double *vals, int *bad) {
    const int lane = threadIdx.x & 31;
    const u128 inc = mk128(z.i_hi, z.i_lo);
    u128 A, C, A32, C32;
    lcg_jump(inc, (unsigned long long)(chunk * ZC + lane + 1), A, C);
    u128 s = A * mk128(z.s_hi, z.s_lo) + C;
    lcg_jump(inc, 32, A32, C32);
    for (int q = lane; q < ZC; q += 32) {
        double v;
        const int c = zig_attempt(s, inc, zt, v);
        if (!c) *bad = 1;
        code[q] = (unsigned char)c;
        if (vals) vals[q] = v;
        s = A32 * s + C32;
    }
}

// chain walk over the chunk from entry e0 (warp-uniform); visit(q0, f) is
// called for each run of f consecutive single-raw final attempts at q0..,
// single(q) for each multi-raw attempt; returns the exit position (>= ZC)
template <class Run, class One>
__device__ int zpar_walk(const unsigned char *code, int e0, Run run, One one) {
    const int lane = threadIdx.x & 31;
    int q = e0;
    while (q < ZC) {
        const int p = q + lane;
        const bool simple = p >= ZC || code[p] == (1 | 128);
        const unsigned m = __ballot_sync(0xffffffffu, !simple);
        const int f0 = m ? __ffs(m) - 1 : 32;
        const int f = min(f0, ZC - q);
        if (f > 0) run(q, f);
        q += f;
        if (q >= ZC || f0 == 32) continue;
        one(q);
        q += code[q] & 127;
    }
    return q;
}

__global__ void __launch_bounds__(32 * ZW)
k_zpar_scan(ZparState z, long long nchunks, unsigned *__restrict__ table, int *bad) {
    __shared__ ZigTables zt;
    __shared__ unsigned char code_s[ZW][ZC];
    __shared__ unsigned short cb_s[ZW][ZC];     // walk-0 normals before a visited position
    __shared__ unsigned vis_s[ZW][ZC / 32];     // walk-0 attempt starts
    zig_tables_load(zt);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long chunk = (long long)blockIdx.x * ZW + warp;
    if (chunk >= nchunks) return;
    unsigned char *code = code_s[warp];
    unsigned short *cb = cb_s[warp];
    unsigned *vis = vis_s[warp];
    for (int w = lane; w < ZC / 32; w += 32) vis[w] = 0u;
    zpar_eval(z, chunk, zt, code, nullptr, bad);
    __syncwarp();
    int cnt = 0;
    const int exit0 = zpar_walk(
        code, 0,
        [&](int q, int f) {
            if (lane < f) {
                const int p = q + lane;
                atomicOr(&vis[p >> 5], 1u << (p & 31));
                cb[p] = (unsigned short)(cnt + lane);
            }
            cnt += f;
        },
        [&](int q) {
            if (lane == 0) {
                atomicOr(&vis[q >> 5], 1u << (q & 31));
                cb[q] = (unsigned short)cnt;
            }
            cnt += code[q] >> 7;
        });
    __syncwarp();
    // entries 1..ZE-1: walk until the chain joins walk 0 (or leaves the chunk)
    int e = lane, c = 0, q = lane;
    if (lane > 0) {
        while (q < ZC && !((vis[q >> 5] >> (q & 31)) & 1u)) {
            c += code[q] >> 7;
            q += code[q] & 127;
        }
    }
    int ex, ce;
    if (lane == 0) {
        ex = exit0 - ZC;
        ce = cnt;
    } else if (q >= ZC) {
        ex = q - ZC;
        ce = c;
    } else {
        ex = exit0 - ZC;
        ce = c + (cnt - cb[q]);
    }
    if (ex >= ZE) *bad = 1;
    table[chunk * ZE + e] = ((unsigned)ce << 8) | (unsigned)(ex & 0xff);
}

// group table: gt[g][e] = (normals, exit entry) of chunks g*ZG .. composed
__global__ void __launch_bounds__(32) k_zpar_group(const unsigned *__restrict__ table,
                                                   long long nchunks, unsigned long long *gt) {
    __shared__ unsigned t[ZG * ZE];
    const long long c0 = (long long)blockIdx.x * ZG;
    const int nc = (int)min((long long)ZG, nchunks - c0);
    for (int i = threadIdx.x; i < nc * ZE; i += 32) t[i] = table[c0 * ZE + i];
    __syncwarp();
    int e = threadIdx.x;
    unsigned long long total = 0;
    for (int c = 0; c < nc; c++) {
        const unsigned v = t[c * ZE + e];
        total += v >> 8;
        e = (int)(v & 0xff);
        if (e >= ZE) e = ZE - 1;  // flagged by the scan
    }
    gt[(long long)blockIdx.x * ZE + threadIdx.x] = (total << 8) | (unsigned long long)e;
}

// groups walked from entry 0: each group's entry and first output index
// (the group tables staged in shared memory when they fit)
constexpr int ZTOP_MAX = 160;  // groups staged: 160 * 32 * 8 B = 40 KB
__global__ void __launch_bounds__(256) k_zpar_top(const unsigned long long *gt, long long ngroups,
                                                  long long *gentry_off) {
    __shared__ unsigned long long t[ZTOP_MAX * ZE];
    const bool stage = ngroups <= ZTOP_MAX;
    if (stage)
        for (int i = threadIdx.x; i < ngroups * ZE; i += blockDim.x) t[i] = gt[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned long long *src = stage ? t : gt;
    int e = 0;
    long long off = 0;
    for (long long g = 0; g < ngroups; g++) {
        gentry_off[2 * g] = e;
        gentry_off[2 * g + 1] = off;
        const unsigned long long v = src[g * ZE + e];
        off += (long long)(v >> 8);
        e = (int)(v & 0xff);
    }
    gentry_off[2 * ngroups] = e;
    gentry_off[2 * ngroups + 1] = off;  // normals available
}

// every chunk's entry and first output index
__global__ void __launch_bounds__(32) k_zpar_resolve(const unsigned *__restrict__ table,
                                                     long long nchunks,
                                                     const long long *gentry_off,
                                                     long long *centry_off) {
    __shared__ unsigned t[ZG * ZE];
    const long long c0 = (long long)blockIdx.x * ZG;
    const int nc = (int)min((long long)ZG, nchunks - c0);
    for (int i = threadIdx.x; i < nc * ZE; i += 32) t[i] = table[c0 * ZE + i];
    __syncwarp();
    if (threadIdx.x != 0) return;
    int e = (int)gentry_off[2 * blockIdx.x];
    long long off = gentry_off[2 * blockIdx.x + 1];
    for (int c = 0; c < nc; c++) {
        centry_off[2 * (c0 + c)] = e;
        centry_off[2 * (c0 + c) + 1] = off;
        const unsigned v = t[c * ZE + e];
        off += v >> 8;
        e = (int)(v & 0xff);
        if (e >= ZE) e = ZE - 1;
    }
}

__global__ void __launch_bounds__(32 * ZW)
k_zpar_emit(ZparState z, long long nchunks, const long long *centry_off, void *out,
            long long *raws_used, int *bad) {
    __shared__ ZigTables zt;
    __shared__ unsigned char code_s[ZW][ZC];
    __shared__ unsigned short oidx_s[ZW][ZC];  // output index (+1) of an attempt's value, 0: none
    zig_tables_load(zt);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long chunk = (long long)blockIdx.x * ZW + warp;
    if (chunk >= nchunks) return;
    const long long base = centry_off[2 * chunk + 1];
    if (base >= z.m) return;
    unsigned char *code = code_s[warp];
    unsigned short *oidx = oidx_s[warp];
    for (int q = lane; q < ZC; q += 32) oidx[q] = 0;
    zpar_eval(z, chunk, zt, code, nullptr, bad);
    __syncwarp();
    int o = 0;  // normals of this chunk so far
    zpar_walk(
        code, (int)centry_off[2 * chunk],
        [&](int q, int f) {
            if (lane < f) oidx[q + lane] = (unsigned short)(o + lane + 1);
            o += f;
        },
        [&](int q) {
            if (code[q] >> 7) {
                if (lane == 0) oidx[q] = (unsigned short)(o + 1);
                o += 1;
            }
        });
    __syncwarp();
    // second pass over the positions (same lane order as zpar_eval): values
    const u128 inc = mk128(z.i_hi, z.i_lo);
    u128 A, C, A32, C32;
    lcg_jump(inc, (unsigned long long)(chunk * ZC + lane + 1), A, C);
    u128 st = A * mk128(z.s_hi, z.s_lo) + C;
    lcg_jump(inc, 32, A32, C32);
    for (int q = lane; q < ZC; q += 32) {
        const int k = (int)oidx[q] - 1;
        if (k >= 0 && base + k < z.m) {
            double v;
            const int c = zig_attempt(st, inc, zt, v);
            const long long i = base + k;
            if (z.f32) static_cast<float *>(out)[i] = (float)v;
            else static_cast<double *>(out)[i] = v;
            if (i == z.m - 1) *raws_used = chunk * ZC + q + (c & 127);
        }
        st = A32 * st + C32;
    }
}

// uniforms: one raw per value, (u64 >> 11) * 2^-53
__global__ void k_zpar_uniform(ZparState z, void *out) {
    const u128 inc = mk128(z.i_hi, z.i_lo);
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t0 >= z.m) return;
    u128 A, C, As, Cs;
    lcg_jump(inc, (unsigned long long)(t0 + 1), A, C);
    u128 s = A * mk128(z.s_hi, z.s_lo) + C;
    lcg_jump(inc, (unsigned long long)stride, As, Cs);
    for (long long i = t0; i < z.m; i += stride) {
        const double v = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
        if (z.f32) static_cast<float *>(out)[i] = (float)v;
        else static_cast<double *>(out)[i] = v;
        s = As * s + Cs;
    }
}

// state advanced by the raws consumed
__global__ void k_zpar_state(ZparState z, const long long *raws_used, unsigned long long *state) {
    if (threadIdx.x != 0) return;
    u128 A, C;
    const u128 inc = mk128(z.i_hi, z.i_lo);
    const long long r = z.kind == 1 ? z.m : *raws_used;
    lcg_jump(inc, (unsigned long long)r, A, C);
    const u128 s = A * mk128(z.s_hi, z.s_lo) + C;
    state[0] = (unsigned long long)(s >> 64);
    state[1] = (unsigned long long)s;
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

int cs_rng_fill_stream(cs_ctx *ctx, uint64_t *state, int32_t kind, int64_t m, int32_t f32,
                       void *out) {
    using namespace cs;
    if ((kind != 0 && kind != 1) || m < 0 || !state) {
        set_error("cs_rng_fill_stream: bad arguments");
        return CS_ERR_PARAM;
    }
    if (m == 0) return CS_OK;
    ZparState z;
    z.s_hi = state[0];
    z.s_lo = state[1];
    z.i_hi = state[2];
    z.i_lo = state[3];
    z.m = m;
    z.kind = kind;
    z.f32 = f32 ? 1 : 0;
    CS_TRY(ctx->tmp.ensure(64));  // raws_used, bad, new state
    long long *raws_used = ctx->tmp.as<long long>();
    int *bad = reinterpret_cast<int *>(raws_used + 1);
    unsigned long long *nstate = reinterpret_cast<unsigned long long *>(raws_used + 2);
    CS_CUDA(cudaMemsetAsync(ctx->tmp.p, 0, 16, ctx->stream));
    long long avail = m;
    if (kind == 1) {
        k_zpar_uniform<<<grid_for(m, 256), 256, 0, ctx->stream>>>(z, out);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    } else {
        // raws: ~1.013 per normal; chunks for 5 % more plus two spare
        const long long nchunks = (long long)((double)m * 1.05 / ZC) + 2;
        const long long ngroups = (nchunks + ZG - 1) / ZG;
        CS_TRY(ctx->zpar.ensure(sizeof(unsigned) * (size_t)nchunks * ZE +
                                sizeof(unsigned long long) * (size_t)ngroups * ZE +
                                sizeof(long long) * (size_t)(2 * ngroups + 2) +
                                sizeof(long long) * (size_t)(2 * nchunks)));
        unsigned *table = ctx->zpar.as<unsigned>();
        unsigned long long *gt = reinterpret_cast<unsigned long long *>(table + nchunks * ZE);
        long long *goff = reinterpret_cast<long long *>(gt + ngroups * ZE);
        long long *coff = goff + 2 * ngroups + 2;
        const unsigned blocks = (unsigned)((nchunks + ZW - 1) / ZW);
        k_zpar_scan<<<blocks, 32 * ZW, 0, ctx->stream>>>(z, nchunks, table, bad);
        CS_LAUNCH_CHECK();
        k_zpar_group<<<(unsigned)ngroups, 32, 0, ctx->stream>>>(table, nchunks, gt);
        CS_LAUNCH_CHECK();
        k_zpar_top<<<1, 256, 0, ctx->stream>>>(gt, ngroups, goff);
        CS_LAUNCH_CHECK();
        k_zpar_resolve<<<(unsigned)ngroups, 32, 0, ctx->stream>>>(table, nchunks, goff, coff);
        CS_LAUNCH_CHECK();
        k_zpar_emit<<<blocks, 32 * ZW, 0, ctx->stream>>>(z, nchunks, coff, out, raws_used, bad);
        CS_LAUNCH_CHECK();
        ctx->launches += 5;
        CS_CUDA(cudaMemcpyAsync(&avail, goff + 2 * ngroups + 1, sizeof(long long),
                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    k_zpar_state<<<1, 1, 0, ctx->stream>>>(z, raws_used, nstate);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    int badh = 0;
    unsigned long long ns[2];
    CS_CUDA(cudaMemcpyAsync(&badh, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(ns, nstate, sizeof(ns), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (badh || avail < m) {
        set_error("cs_rng_fill_stream: %s", badh ? "an attempt outside the tabulated range"
                                                 : "too few raw draws scanned");
        return CS_ERR_PARAM;
    }
    state[0] = ns[0];
    state[1] = ns[1];
    return CS_OK;
}

int cs_log1p_batch(cs_ctx *ctx, const double *x, double *y, int64_t n) {
    if (n == 0) return CS_OK;
    cs::k_log1p<<<cs::grid_for(n, 256), 256, 0, ctx->stream>>>(x, y, n);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

}  // extern "C"
