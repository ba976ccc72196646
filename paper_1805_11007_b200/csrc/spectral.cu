// spectral.cu -- the periodic implicit field step as three fused passes.
//
// The semi-implicit field step on a periodic grid (field.py:209-239 with the
// operator of build_operators, field.py:173-201; the reference factors the
// sparse system with SuperLU) is diagonal in Fourier space:
//     c' = IDFT2( DFT2(rhs) / (1 - dt d_c (lx[kx] + ly[ky])) ),
// lx, ly the eigenvalues of the circulant 1-D Laplacians (field.py:114-125).
// Any n = 2^k (16 .. 8192), binary32 or binary64, in three passes over the
// grid instead of the seven of a library R2C -> scale -> C2R:
//
//   k_spec_rows_fwd  the rhs of two grid rows, fused (field.py:220-227:
//                    c (1 - dt g) + (dt ka) ra - (rb c)(dt kb); from the
//                    sorted engine's fixed-point deposits, the direct
//                    engine's density arrays, or a given rhs), packed as one
//                    complex row, one n-point FFT, split into the two half
//                    spectra (the two-real-rows-in-one trick), stored
//                    TRANSPOSED: specT[kx][ky], 2 x GPB consecutive ky per kx;
//   k_spec_cols      per spectrum column (contiguous in specT): forward FFT,
//                    the mode scale, inverse FFT -- the column never leaves
//                    shared memory between the two;
//   k_spec_rows_inv  the two half spectra of a row pair recombined into one
//                    complex row (Hermitian extension), one inverse FFT, the
//                    two real rows written to c.
//
// FFTs: Stockham passes of radix 16 (the 16 values of a butterfly in
// registers, the row in shared memory: read all, barrier, write all -- every
// pass in place), then one pass of radix 2, 4 or 8 for the rest of n; n / 16
// threads per transform.  Twiddles from a table of exp(-2 pi i k / n)
// computed in binary64 on the host (binary32 radix-16 passes: four loads,
// w, w^2, w^4, w^8, and products at most three deep; otherwise one load per
// twiddle).  Arithmetic in the grid's precision, like cuFFT's R2C/C2R and
// D2Z/Z2D; the mode scale is a binary64 factor applied to the stored values.
#include <math.h>

#include <vector>

#include "common.cuh"

#ifndef CS_SPEC_SECTOR
#define CS_SPEC_SECTOR 0  // rows blocks wide enough for 32-byte transposed stores (8192: slower)
#endif
// resident blocks per SM asked of the compiler (binary32, >= 4096 points);
// measured: cols 4096: 1 -> 256, 2 -> 233, 3 -> 223 us/solve; 8192: 2 best
template <int N> constexpr int cols_minb() { return N >= 8192 ? 2 : 3; }
#ifndef CS_SPEC_ROWS_MINB
#define CS_SPEC_ROWS_MINB 2  // measured: 4096: 1 -> 243, 2 -> 224, 3 -> 252 us; 8192: 2 best
#endif

namespace cs {

template <class T> struct Cplx;
template <> struct Cplx<float> { using V = float2; };
template <> struct Cplx<double> { using V = double2; };

__device__ __forceinline__ float2 mk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
template <class V> __device__ __forceinline__ V cadd(V a, V b) { return mk(a.x + b.x, a.y + b.y); }
template <class V> __device__ __forceinline__ V csub(V a, V b) { return mk(a.x - b.x, a.y - b.y); }
template <class V> __device__ __forceinline__ V cmul(V a, V b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <class V> __device__ __forceinline__ V mul_mi(V a) { return mk(a.y, -a.x); }  // * -i

// two consecutive complex values with one 16-byte access where that is one
// (binary32), else two
__device__ __forceinline__ void ld2(const float2 *p, float2 &a, float2 &b) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    a = make_float2(v.x, v.y);
    b = make_float2(v.z, v.w);
}
__device__ __forceinline__ void ld2(const double2 *p, double2 &a, double2 &b) {
    a = p[0];
    b = p[1];
}
__device__ __forceinline__ void st2(float2 *p, float2 a, float2 b) {
    *reinterpret_cast<float4 *>(p) = make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st2(double2 *p, double2 a, double2 b) {
    p[0] = a;
    p[1] = b;
}

// shared-memory index: one padding slot per 16 elements (the radix-16
// stores of 16 consecutive elements per thread do not hit one bank)
__host__ __device__ constexpr int sp(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int pad_len(int n) { return n + n / 16; }

template <class V> __device__ __forceinline__ void dft2(V &a0, V &a1) {
    const V s = cadd(a0, a1);
    a1 = csub(a0, a1);
    a0 = s;
}

// forward 4-point DFT in place (W4 = -i)
template <class V> __device__ __forceinline__ void dft4(V &a0, V &a1, V &a2, V &a3) {
    const V s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const V s13 = cadd(a1, a3), d13 = csub(a1, a3);
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = mk(d02.x + d13.y, d02.y - d13.x);  // d02 - i d13
    a3 = mk(d02.x - d13.y, d02.y + d13.x);  // d02 + i d13
}

// forward 8-point DFT, natural order: r = r1 + 2 r2, k = k1 + 4 k2;
// DFT4 over r2, twiddle W8^(r1 k1), DFT2 over r1
template <class V> __device__ __forceinline__ void dft8(V *v) {
    using S = decltype(v[0].x);
    const S h = (S)0.70710678118654752440;
    dft4(v[0], v[2], v[4], v[6]);
    dft4(v[1], v[3], v[5], v[7]);
    const V y1 = v[1], y3 = cmul(v[3], mk(h, -h)), y5 = mul_mi(v[5]), y7 = cmul(v[7], mk(-h, -h));
    const V x0 = v[0], x2 = v[2], x4 = v[4], x6 = v[6];
    v[0] = cadd(x0, y1);
    v[4] = csub(x0, y1);
    v[1] = cadd(x2, y3);
    v[5] = csub(x2, y3);
    v[2] = cadd(x4, y5);
    v[6] = csub(x4, y5);
    v[3] = cadd(x6, y7);
    v[7] = csub(x6, y7);
}

// forward 16-point DFT, natural order: r = r1 + 4 r2, k = k1 + 4 k2;
// DFT4 over r2, twiddle W16^(r1 k1), DFT4 over r1
template <class V> __device__ __forceinline__ void dft16(V *v) {
    using S = decltype(v[0].x);
#pragma unroll
    for (int r1 = 0; r1 < 4; r1++) dft4(v[r1], v[r1 + 4], v[r1 + 8], v[r1 + 12]);
    const S c1 = (S)0.92387953251128675613, s1 = (S)0.38268343236508977173,
            h = (S)0.70710678118654752440;
    v[5] = cmul(v[5], mk(c1, -s1));    // W^1
    v[6] = cmul(v[6], mk(h, -h));      // W^2
    v[7] = cmul(v[7], mk(s1, -c1));    // W^3
    v[9] = cmul(v[9], mk(h, -h));      // W^2
    v[10] = mul_mi(v[10]);             // W^4 = -i
    v[11] = cmul(v[11], mk(-h, -h));   // W^6
    v[13] = cmul(v[13], mk(s1, -c1));  // W^3
    v[14] = cmul(v[14], mk(-h, -h));   // W^6
    v[15] = cmul(v[15], mk(-c1, s1));  // W^9
#pragma unroll
    for (int k1 = 0; k1 < 4; k1++) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    V t[16];  // X[k1 + 4 k2] sits at v[k2 + 4 k1]
#pragma unroll
    for (int k1 = 0; k1 < 4; k1++)
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++) t[k1 + 4 * k2] = v[k2 + 4 * k1];
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = t[i];
}

template <int R, class V> __device__ __forceinline__ void dft_r(V *v) {
    if constexpr (R == 16) dft16(v);
    else if constexpr (R == 8) dft8(v);
    else if constexpr (R == 4) dft4(v[0], v[1], v[2], v[3]);
    else dft2(v[0], v[1]);
}

// One Stockham radix-R pass (stride Ns: the product of the earlier radices)
// of the forward N-point FFT of buf (shared memory, in place) by the N / 16
// threads j of one group; 16 / R butterflies per thread; block-wide barriers.
template <class V, int N, int R, int Ns>
__device__ __forceinline__ void fft_pass(V *buf, int j, const V *__restrict__ tw) {
    constexpr int NT = N / 16, B = 16 / R;
    V v[B][R];
#pragma unroll
    for (int b = 0; b < B; b++)
#pragma unroll
        for (int r = 0; r < R; r++) v[b][r] = buf[sp(j + b * NT + r * (N / R))];
    if constexpr (Ns > 1) {
#pragma unroll
        for (int b = 0; b < B; b++) {
            const int jj = j + b * NT;
            const int e = (jj % Ns) * (N / (R * Ns));  // W_{R Ns}^(r jm) = tw[r e]
            if constexpr (R == 16 && sizeof(V) == 8) {
                // binary32: w, w^2, w^4, w^8 loaded, products at most three deep
                const V w1 = tw[e], w2 = tw[2 * e], w4 = tw[4 * e], w8 = tw[8 * e];
                const V w3 = cmul(w1, w2), w5 = cmul(w4, w1), w6 = cmul(w4, w2),
                        w7 = cmul(w4, w3);
                const V w[16] = {w1, w1, w2, w3, w4, w5, w6, w7, w8, cmul(w8, w1), cmul(w8, w2),
                                 cmul(w8, w3), cmul(w8, w4), cmul(w8, w5), cmul(w8, w6),
                                 cmul(w8, w7)};
#pragma unroll
                for (int r = 1; r < 16; r++) v[b][r] = cmul(v[b][r], w[r]);
            } else {
#pragma unroll
                for (int r = 1; r < R; r++) v[b][r] = cmul(v[b][r], tw[r * e]);
            }
        }
    }
#pragma unroll
    for (int b = 0; b < B; b++) dft_r<R>(v[b]);
    __syncthreads();
#pragma unroll
    for (int b = 0; b < B; b++) {
        const int jj = j + b * NT;
        const int d = (jj / Ns) * Ns * R + (jj % Ns);
#pragma unroll
        for (int r = 0; r < R; r++) buf[sp(d + r * Ns)] = v[b][r];
    }
    __syncthreads();
}

template <class V, int N, int Ns = 1>
__device__ __forceinline__ void fft(V *buf, int j, const V *__restrict__ tw) {
    if constexpr (Ns * 16 <= N) {
        fft_pass<V, N, 16, Ns>(buf, j, tw);
        fft<V, N, Ns * 16>(buf, j, tw);
    } else if constexpr (Ns < N) {
        fft_pass<V, N, N / Ns, Ns>(buf, j, tw);
    }
}

// ---------------------------------------------------------------- rhs sources
struct SpecRhs {
    double one_m_dtg, dka, dkb, scale;
    int has_g, has_a, has_b;
};

// the sorted engine: binary32 c and int32 fixed-point deposits q (a | b)
struct SrcQ {
    const float *c;
    const int *q;
    long long m;
    SpecRhs k;
    __device__ __forceinline__ float operator()(long long l) const {
        const double cv = (double)c[l];
        double r = k.has_g ? dmul(cv, k.one_m_dtg) : cv;
        if (k.has_a) r = dadd(r, dmul(k.dka, dmul((double)q[l], k.scale)));
        if (k.has_b) r = dsub(r, dmul(dmul(dmul((double)q[l + m], k.scale), cv), k.dkb));
        return (float)r;
    }
    // elements l .. l+3 (l a multiple of 4): 16-byte loads
    __device__ __forceinline__ void load4(long long l, float (&o)[4]) const {
        const float4 cv = *reinterpret_cast<const float4 *>(c + l);
        const int4 qa = k.has_a ? *reinterpret_cast<const int4 *>(q + l) : make_int4(0, 0, 0, 0);
        const int4 qb = k.has_b ? *reinterpret_cast<const int4 *>(q + m + l) : make_int4(0, 0, 0, 0);
        const float cs[4] = {cv.x, cv.y, cv.z, cv.w};
        const int as[4] = {qa.x, qa.y, qa.z, qa.w}, bs[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const double c_ = (double)cs[i];
            double r = k.has_g ? dmul(c_, k.one_m_dtg) : c_;
            if (k.has_a) r = dadd(r, dmul(k.dka, dmul((double)as[i], k.scale)));
            if (k.has_b) r = dsub(r, dmul(dmul(dmul((double)bs[i], k.scale), c_), k.dkb));
            o[i] = (float)r;
        }
    }
};

// the direct engine: c, rho_a, rho_b in the grid dtype (field.cu k_rhs)
template <class G> struct SrcG {
    const G *c, *ra, *rb;
    SpecRhs k;
    __device__ __forceinline__ G operator()(long long l) const {
        const double cv = (double)c[l];
        double r = k.has_g ? dmul(cv, k.one_m_dtg) : cv;
        if (k.has_a) r = dadd(r, dmul(k.dka, (double)ra[l]));
        if (k.has_b) r = dsub(r, dmul(dmul((double)rb[l], cv), k.dkb));
        return (G)r;
    }
    __device__ __forceinline__ void load4(long long l, G (&o)[4]) const {
#pragma unroll
        for (int i = 0; i < 4; i++) o[i] = (*this)(l + i);
    }
};

// a given rhs (Operators.solve)
template <class G> struct SrcPlain {
    const G *r;
    __device__ __forceinline__ G operator()(long long l) const { return r[l]; }
    __device__ __forceinline__ void load4(long long l, G (&o)[4]) const {
#pragma unroll
        for (int i = 0; i < 4; i++) o[i] = r[l + i];
    }
};

// Which part of the transform a launch does: the single-domain solve is
// {0, N, 0, NH, 0}.  A y-slab rank (slabs.py) transforms its own grid rows
// [row0, row0 + rows) into a half spectrum laid out [kx][ld = rows], and the
// columns kx0 .. kx0 + ncols of the all-to-all transposed spectrum, whose
// element (kx, ky) sits at [ky / rp][kx - kx0][ky % rp] (rp grid rows per rank).
struct SpecPart {
    int row0, ld, kx0, ncols, rp;
};

// groups (complex row pairs, N/16 threads each) per rows block: up to ~512
// threads and 150 KB of shared rows, but at least ~2 blocks per SM (small
// grids are latency-bound: more, smaller blocks)
template <class T, int N> constexpr int rows_gpb() {
    int g = 512 / (N / 16);
    if (g > 8) g = 8;
    while (g > 1 && N / (2 * g) < 296) g /= 2;
    constexpr size_t row = sizeof(typename Cplx<T>::V) * pad_len(N);
    while (g > 1 && g * row > 150 * 1024) g /= 2;
    if (g < 1) g = 1;
    // the transposed stores of a kx: 2 g complex values, at least one 32-byte sector
    if (CS_SPEC_SECTOR && 2 * g * sizeof(typename Cplx<T>::V) < 32 && 2 * g * row <= 150 * 1024 &&
        2 * g * (N / 16) <= 1024 && N / (4 * g) >= 148)
        g *= 2;
    return g;
}
// columns per cols block: up to ~256 threads, at least ~2 blocks per SM
template <int N> constexpr int cols_cpb() {
    int g = 256 / (N / 16);
    while (g > 1 && (N / 2 + 1) / g < 296) g /= 2;
    return g < 1 ? 1 : g;
}

// Forward rows: a block owns 2 GPB grid rows (GPB complex FFTs, one per group
// of N/16 threads) and writes their half spectra transposed, specT[kx][ky].
template <class T, int N, int GPB, class Src>
__global__ void __launch_bounds__(GPB *(N / 16), (N >= 4096 && sizeof(T) == 4) ? CS_SPEC_ROWS_MINB : 1)
k_spec_rows_fwd(Src src, typename Cplx<T>::V *__restrict__ specT,
                const typename Cplx<T>::V *__restrict__ tw, const DevStatus *st, SpecPart pt) {
    using V = typename Cplx<T>::V;
    constexpr int NT = N / 16, NH = N / 2 + 1, PAD = pad_len(N);
    extern __shared__ __align__(16) unsigned char s_raw[];
    V *bufs = reinterpret_cast<V *>(s_raw);
    if (st && st->abort) return;
    const int T_ = threadIdx.x, g = T_ / NT, j = T_ % NT;
    const int y0 = pt.row0 + 2 * GPB * blockIdx.x;
    V *buf = bufs + g * PAD;
    const long long r0 = (long long)(y0 + 2 * g) * N, r1 = r0 + N;
#pragma unroll 2
    for (int e = j; e < N / 4; e += NT) {  // four consecutive elements per access
        T a[4], b[4];
        src.load4(r0 + 4 * e, a);
        src.load4(r1 + 4 * e, b);
#pragma unroll
        for (int i = 0; i < 4; i++) buf[sp(4 * e + i)] = mk(a[i], b[i]);
    }
    __syncthreads();
    fft<V, N>(buf, j, tw);
    // split Z of each pair: Xa = (Z[k] + conj Z[-k]) / 2, Xb = (Z[k] - conj Z[-k]) / 2i
    const T half = (T)0.5;
    for (int kx = T_; kx < NH; kx += GPB * NT) {
        const int kn = (N - kx) & (N - 1);
        V *o = specT + (long long)kx * pt.ld + (y0 - pt.row0);
#pragma unroll
        for (int q = 0; q < GPB; q++) {
            const V z = bufs[q * PAD + sp(kx)], w = bufs[q * PAD + sp(kn)];
            st2(o + 2 * q, mk(half * (z.x + w.x), half * (z.y - w.y)),
                mk(half * (z.y + w.y), half * (w.x - z.x)));
        }
    }
}

// CPB spectrum columns (contiguous in specT) per block: forward FFT along
// ky, the mode scale, inverse FFT, all in shared memory.
template <class T, int N, int CPB>
__global__ void __launch_bounds__(CPB *(N / 16), (N >= 4096 && sizeof(T) == 4) ? cols_minb<N>() : 1)
k_spec_cols(typename Cplx<T>::V *__restrict__ specT, const double *__restrict__ lx,
            const double *__restrict__ ly, double dtdc, double inv_nn,
            const typename Cplx<T>::V *__restrict__ tw, const DevStatus *st, SpecPart pt) {
    using V = typename Cplx<T>::V;
    constexpr int NT = N / 16, PAD = pad_len(N);
    extern __shared__ __align__(16) unsigned char s_raw[];
    if (st && st->abort) return;
    const int g = threadIdx.x / NT, j = threadIdx.x % NT;
    const int kl = blockIdx.x * CPB + g;  // column of this launch
    const bool live = kl < pt.ncols;     // every thread stays for the barriers
    V *col = reinterpret_cast<V *>(s_raw) + g * PAD;
    // element ky of the column: contiguous, or gathered from the rank blocks
    auto at = [&](int ky) -> V * {
        if (!pt.rp) return specT + (long long)(live ? kl : 0) * N + ky;
        return specT + (long long)(ky / pt.rp) * pt.ncols * pt.rp +
               (long long)(live ? kl : 0) * pt.rp + ky % pt.rp;
    };
#pragma unroll 4
    for (int e = j; e < N / 2; e += NT) {  // two complex values per access (rp is even)
        V a = mk((T)0, (T)0), b = a;
        if (live) ld2(at(2 * e), a, b);
        col[sp(2 * e)] = a;
        col[sp(2 * e + 1)] = b;
    }
    __syncthreads();
    fft<V, N>(col, j, tw);
    const double lxv = live ? __ldg(lx + pt.kx0 + kl) : 0.0;
#pragma unroll 4
    for (int ky = j; ky < N; ky += NT) {
        const double s = inv_nn / (1.0 - dtdc * (__ldg(ly + ky) + lxv));
        const V v = col[sp(ky)];
        col[sp(ky)] = mk((T)(v.x * s), (T)(-(v.y * s)));  // conjugated: IDFT = conj DFT conj
    }
    __syncthreads();
    fft<V, N>(col, j, tw);
    if (live) {
#pragma unroll 4
        for (int e = j; e < N / 2; e += NT) {
            const V p = col[sp(2 * e)], q = col[sp(2 * e + 1)];
            st2(at(2 * e), mk(p.x, -p.y), mk(q.x, -q.y));
        }
    }
}

// Inverse rows: a block owns 2 GPB grid rows; every kx's (Xa, Xb) pairs
// recombined into Z = A + iB over the full row (Hermitian extension; the
// imaginary parts of the DC and Nyquist terms dropped, as by a C2R
// transform), one inverse FFT per pair.
template <class T, int N, int GPB, class G>
__global__ void __launch_bounds__(GPB *(N / 16), (N >= 4096 && sizeof(T) == 4) ? CS_SPEC_ROWS_MINB : 1)
k_spec_rows_inv(const typename Cplx<T>::V *__restrict__ specT, G *__restrict__ c,
                const typename Cplx<T>::V *__restrict__ tw, const DevStatus *st, SpecPart pt) {
    using V = typename Cplx<T>::V;
    constexpr int NT = N / 16, NH = N / 2 + 1, PAD = pad_len(N);
    extern __shared__ __align__(16) unsigned char s_raw[];
    V *bufs = reinterpret_cast<V *>(s_raw);
    if (st && st->abort) return;
    const int T_ = threadIdx.x, g = T_ / NT, j = T_ % NT;
    const int y0 = pt.row0 + 2 * GPB * blockIdx.x;
    for (int kx = T_; kx < NH; kx += GPB * NT) {
        const V *in = specT + (long long)kx * pt.ld + (y0 - pt.row0);
#pragma unroll
        for (int q = 0; q < GPB; q++) {
            V a, b;
            ld2(in + 2 * q, a, b);
            if (kx == 0 || kx == N / 2) {
                a.y = (T)0;
                b.y = (T)0;
            }
            // Z[kx] = A + iB, stored conjugated for IDFT(Z) = conj(DFT(conj Z))
            bufs[q * PAD + sp(kx)] = mk(a.x - b.y, -(a.y + b.x));
            if (kx > 0 && kx < N / 2)  // Z[N - kx] = conj(A) + i conj(B)
                bufs[q * PAD + sp(N - kx)] = mk(a.x + b.y, -(b.x - a.y));
        }
    }
    __syncthreads();
    V *buf = bufs + g * PAD;
    fft<V, N>(buf, j, tw);
    G *c0 = c + (long long)(y0 + 2 * g) * N, *c1 = c0 + N;
#pragma unroll 4
    for (int x = j; x < N; x += NT) {
        const V z = buf[sp(x)];
        c0[x] = (G)z.x;     // Re conj(DFT(conj Z)) = Re DFT(conj Z)
        c1[x] = (G)(-z.y);  // Im conj(...)
    }
}

// ---------------------------------------------------------------- host side
int spectral_supported(int n) {
    return n >= 16 && n <= 8192 && (n & (n - 1)) == 0;
}

// which passes: 1 rows forward, 2 columns, 4 rows inverse (7: the whole solve)
template <class T, int N, class Src, class G>
static int spec_run(cs_ctx *ctx, cs_field_ops *ops, const Src &src, G *out, const DevStatus *st,
                    int passes = 7, SpecPart pt = SpecPart{0, N, 0, N / 2 + 1, 0},
                    int rows = N, void *spec = nullptr) {
    using V = typename Cplx<T>::V;
    constexpr int GPB = rows_gpb<T, N>(), CPB = cols_cpb<N>(), NH = N / 2 + 1;
    constexpr int rows_smem = GPB * pad_len(N) * (int)sizeof(V);
    constexpr int cols_smem = CPB * pad_len(N) * (int)sizeof(V);
    static bool attr = false;  // per instantiation
    if (!attr) {
        CS_CUDA(cudaFuncSetAttribute(k_spec_rows_fwd<T, N, GPB, Src>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, rows_smem));
        CS_CUDA(cudaFuncSetAttribute(k_spec_rows_inv<T, N, GPB, G>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, rows_smem));
        CS_CUDA(cudaFuncSetAttribute(k_spec_cols<T, N, CPB>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, cols_smem));
        attr = true;
    }
    V *specT = static_cast<V *>(spec ? spec : ops->specT);
    const V *tw = static_cast<const V *>(ops->tw);
    if ((passes & 5) && rows % (2 * GPB)) {
        set_error("spectral solve: %d grid rows per rank is not a multiple of %d", rows, 2 * GPB);
        return CS_ERR_PARAM;
    }
    (void)NH;
    if (passes & 1) {
        k_spec_rows_fwd<T, N, GPB, Src><<<rows / (2 * GPB), GPB * (N / 16), rows_smem,
                                          ctx->stream>>>(src, specT, tw, st, pt);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    if (passes & 2) {
        const double inv_nn = 1.0 / ((double)N * (double)N);
        k_spec_cols<T, N, CPB><<<(pt.ncols + CPB - 1) / CPB, CPB * (N / 16), cols_smem,
                                 ctx->stream>>>(specT, ops->lx, ops->ly, ops->dt * ops->d_c,
                                                inv_nn, tw, st, pt);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    if (passes & 4) {
        k_spec_rows_inv<T, N, GPB, G><<<rows / (2 * GPB), GPB * (N / 16), rows_smem,
                                        ctx->stream>>>(specT, out, tw, st, pt);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    return CS_OK;
}

template <class T, class Src, class G>
static int spec_dispatch(cs_ctx *ctx, cs_field_ops *ops, const Src &src, G *out,
                         const DevStatus *st, int passes = 7, const SpecPart *pt = nullptr,
                         int rows = 0, void *spec = nullptr) {
#define CS_SPEC_CASE(NN)                                                                      \
    case NN:                                                                                  \
        return pt ? spec_run<T, NN>(ctx, ops, src, out, st, passes, *pt, rows, spec)          \
                  : spec_run<T, NN>(ctx, ops, src, out, st);
    switch (ops->gg.n) {
        CS_SPEC_CASE(16)
        CS_SPEC_CASE(32)
        CS_SPEC_CASE(64)
        CS_SPEC_CASE(128)
        CS_SPEC_CASE(256)
        CS_SPEC_CASE(512)
        CS_SPEC_CASE(1024)
        CS_SPEC_CASE(2048)
        CS_SPEC_CASE(4096)
        CS_SPEC_CASE(8192)
    }
#undef CS_SPEC_CASE
    set_error("spectral solve: n = %d is not a power of two in [16, 8192]", ops->gg.n);
    return CS_ERR_PARAM;
}

// the transposed spectrum and the twiddle table of this operator
static int spec_prepare(cs_field_ops *ops) {
    if (ops->specT) return CS_OK;
    const int n = ops->gg.n;
    const size_t es = ops->prec == CS_F64 ? 16 : 8;  // complex element
    CS_CUDA(cudaMalloc(&ops->specT, es * (size_t)(n / 2 + 1) * n));
    CS_CUDA(cudaMalloc(&ops->tw, es * (size_t)n));
    std::vector<double> w(2 * (size_t)n);
    for (int k = 0; k < n; k++) {
        const double a = -2.0 * M_PI * (double)k / (double)n;
        w[2 * k] = cos(a);
        w[2 * k + 1] = sin(a);
    }
    if (ops->prec == CS_F64) {
        CS_CUDA(cudaMemcpy(ops->tw, w.data(), es * n, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> wf(w.begin(), w.end());
        CS_CUDA(cudaMemcpy(ops->tw, wf.data(), es * n, cudaMemcpyHostToDevice));
    }
    return CS_OK;
}

static SpecRhs spec_rhs(double dt, double gamma, double ka, double kb, double scale) {
    SpecRhs k;
    k.one_m_dtg = 1.0 - dt * gamma;
    k.dka = dt * ka;
    k.dkb = dt * kb;
    k.scale = scale;
    k.has_g = gamma != 0.0;
    k.has_a = ka != 0.0;
    k.has_b = kb != 0.0;
    return k;
}

// sorted engine: c (binary32, in place) from c and the fixed-point deposits q
int spectral_step_q(cs_field_ops *ops, float *c, const int *q, double gamma, double ka,
                    double kb, double scale, const DevStatus *st) {
    CS_TRY(spec_prepare(ops));
    const long long m = (long long)ops->gg.n * ops->gg.n;
    SrcQ src{c, q, m, spec_rhs(ops->dt, gamma, ka, kb, scale)};
    return spec_dispatch<float>(ops->ctx, ops, src, c, st);
}

// direct engine: c (grid dtype, in place) from c, rho_a, rho_b
int spectral_step_g(cs_field_ops *ops, void *c, const void *ra, const void *rb, double gamma,
                    double ka, double kb, const DevStatus *st) {
    CS_TRY(spec_prepare(ops));
    const SpecRhs k = spec_rhs(ops->dt, gamma, ka, kb, 1.0);
    if (ops->prec == CS_F64) {
        SrcG<double> src{(const double *)c, (const double *)ra, (const double *)rb, k};
        return spec_dispatch<double>(ops->ctx, ops, src, (double *)c, st);
    }
    SrcG<float> src{(const float *)c, (const float *)ra, (const float *)rb, k};
    return spec_dispatch<float>(ops->ctx, ops, src, (float *)c, st);
}

// y-slab pieces (binary32, the sorted engine's slab mode): rows forward of
// the own grid rows [row0, row0 + rows) into spec [NH][rows]; the columns
// kx0 .. kx0 + ncols of the transposed blocks [rank][ncols][rp]; rows inverse.
int spectral_slab_rows(cs_field_ops *ops, float *c, const int *q, double gamma, double ka,
                       double kb, double scale, int row0, int rows, void *spec, int inverse,
                       const DevStatus *st) {
    CS_TRY(spec_prepare(ops));
    const long long m = (long long)ops->gg.n * ops->gg.n;
    const int NH = ops->gg.n / 2 + 1;
    SpecPart pt{row0, rows, 0, NH, 0};
    SrcQ src{c, q, m, spec_rhs(ops->dt, gamma, ka, kb, scale)};
    return spec_dispatch<float>(ops->ctx, ops, src, c, st, inverse ? 4 : 1, &pt, rows, spec);
}

int spectral_slab_cols(cs_field_ops *ops, void *blocks, int kx0, int ncols, int rp,
                       const DevStatus *st) {
    CS_TRY(spec_prepare(ops));
    if (rp % 2) {
        set_error("spectral slab columns: rows per rank must be even");
        return CS_ERR_PARAM;
    }
    SpecPart pt{0, 0, kx0, ncols, rp};
    SrcPlain<float> none{nullptr};
    return spec_dispatch<float>(ops->ctx, ops, none, (float *)nullptr, st, 2, &pt, 0, blocks);
}

// out = solve(rhs), both in the grid dtype
int spectral_solve(cs_field_ops *ops, const void *rhs, void *out) {
    CS_TRY(spec_prepare(ops));
    if (ops->prec == CS_F64)
        return spec_dispatch<double>(ops->ctx, ops, SrcPlain<double>{(const double *)rhs},
                                     (double *)out, nullptr);
    return spec_dispatch<float>(ops->ctx, ops, SrcPlain<float>{(const float *)rhs}, (float *)out,
                                nullptr);
}

}  // namespace cs
