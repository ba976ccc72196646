// spectral.cu -- fused periodic solve for the sorted engine's binary32 grid.
//
// The semi-implicit field step on a periodic grid (field.py:209-239 with the
// operator of build_operators, field.py:173-201) is diagonal in Fourier
// space: c' = IDFT2( DFT2(rhs) / (1 - dt d_c (lx[kx] + ly[ky])) ), which the
// generic path evaluates as k_fast_rhs -> cuFFT R2C (row pass + two column
// passes) -> k_mode_scale -> cuFFT C2R (two column passes + row pass): seven
// full passes over the spectrum.  Here the same transform is three passes:
//
//   k_spec_rows_fwd  rhs of grid rows (fused: c, fixed-point deposits), two
//                    rows packed as one complex row, one 4096-point FFT, split
//                    into the two half spectra (the two-real-rows-in-one
//                    trick), stored transposed: specT[kx][ky];
//   k_spec_cols      per spectrum column (contiguous in specT): forward FFT,
//                    the mode scale of k_mode_scale, inverse FFT -- the
//                    column never leaves shared memory between the two;
//   k_spec_rows_inv  the two half spectra of a row pair recombined into one
//                    complex row (Hermitian extension), one inverse FFT, the
//                    two real rows written to c.
//
// FFTs: 4096 = 16^3, Stockham radix-16 with the 16 values of a butterfly in
// registers and the row in shared memory (read all, barrier, write all, so
// every pass is in place), twiddles from a table of exp(-2 pi i k / 4096)
// rounded from binary64 (per pass four loads, w, w^2, w^4, w^8, and products
// at most three deep).  Arithmetic is binary32 like cuFFT's single
// precision path; the mode scale is computed exactly as k_mode_scale
// (binary64 factor applied to the binary32 values).  The row kernels own 4
// grid rows per block, so each transposed spectrum access (4 consecutive ky
// of one kx) is one aligned 32-byte sector.
#include "common.cuh"

namespace cs {

constexpr int SP_N = 4096;
constexpr int SP_NH = SP_N / 2 + 1;  // 2049 spectrum columns
constexpr int SP_T = 256;            // threads per 4096-point FFT (16 values each)

constexpr int SP_PAD = SP_N + SP_N / 16;  // padded shared row (one slot per 16)

__device__ float2 g_w4096[SP_N];  // exp(-2 pi i k / 4096)

// shared-memory index of element i: one padding slot per 16 elements, so the
// first Stockham pass's stores (16 consecutive elements per thread) do not
// all land in one bank
__device__ __forceinline__ int sp(int i) { return i + (i >> 4); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// forward 4-point DFT in place (W4 = -i)
__device__ __forceinline__ void dft4(float2 &a0, float2 &a1, float2 &a2, float2 &a3) {
    const float2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const float2 s13 = cadd(a1, a3), d13 = csub(a1, a3);
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = make_float2(d02.x + d13.y, d02.y - d13.x);  // d02 - i d13
    a3 = make_float2(d02.x - d13.y, d02.y + d13.x);  // d02 + i d13
}

// forward 16-point DFT of v (natural order in, natural order out):
// r = r1 + 4 r2, k = k1 + 4 k2; DFT4 over r2, twiddle W16^(r1 k1), DFT4 over r1
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
#pragma unroll
    for (int r1 = 0; r1 < 4; r1++) dft4(v[r1], v[r1 + 4], v[r1 + 8], v[r1 + 12]);
    // v[r1 + 4 k1] *= W16^(r1 k1)
    const float c1 = 0.92387953251128674f, s1 = 0.38268343236508977f, h = 0.70710678118654752f;
    v[5] = cmul(v[5], make_float2(c1, -s1));    // W^1
    v[6] = cmul(v[6], make_float2(h, -h));      // W^2
    v[7] = cmul(v[7], make_float2(s1, -c1));    // W^3
    v[9] = cmul(v[9], make_float2(h, -h));      // W^2
    v[10] = make_float2(v[10].y, -v[10].x);     // W^4 = -i
    v[11] = cmul(v[11], make_float2(-h, -h));   // W^6
    v[13] = cmul(v[13], make_float2(s1, -c1));  // W^3
    v[14] = cmul(v[14], make_float2(-h, -h));   // W^6
    v[15] = cmul(v[15], make_float2(-c1, s1));  // W^9
#pragma unroll
    for (int k1 = 0; k1 < 4; k1++) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // X[k1 + 4 k2] sits at v[k2 + 4 k1]: transpose the 4x4 index
    float2 t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; k1++)
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++) t[k1 + 4 * k2] = v[k2 + 4 * k1];
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = t[i];
}

// One Stockham radix-16 pass (Ns compile-time, so every index is shifts and
// masks) of the forward 4096-point FFT of buf (shared memory, in place) by the
// SP_T threads j = 0..255 of one group; the barriers are block-wide.
template <int Ns>
__device__ __forceinline__ void fft_pass(float2 *buf, int j) {
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = buf[sp(j + r * SP_T)];
    if (Ns > 1) {
        // exp(-2 pi i r jm / (16 Ns)) = w^r with w = W4096^(jm N / (16 Ns)): four
        // table loads (w, w^2, w^4, w^8) and products at most three deep
        const int e = (j % Ns) * (SP_N / (Ns * 16));
        const float2 w1 = g_w4096[e], w2 = g_w4096[2 * e], w4 = g_w4096[4 * e],
                     w8 = g_w4096[8 * e];
        const float2 w3 = cmul(w1, w2), w5 = cmul(w4, w1), w6 = cmul(w4, w2), w7 = cmul(w4, w3);
        v[1] = cmul(v[1], w1);
        v[2] = cmul(v[2], w2);
        v[3] = cmul(v[3], w3);
        v[4] = cmul(v[4], w4);
        v[5] = cmul(v[5], w5);
        v[6] = cmul(v[6], w6);
        v[7] = cmul(v[7], w7);
        v[8] = cmul(v[8], w8);
        v[9] = cmul(v[9], cmul(w8, w1));
        v[10] = cmul(v[10], cmul(w8, w2));
        v[11] = cmul(v[11], cmul(w8, w3));
        v[12] = cmul(v[12], cmul(w8, w4));
        v[13] = cmul(v[13], cmul(w8, w5));
        v[14] = cmul(v[14], cmul(w8, w6));
        v[15] = cmul(v[15], cmul(w8, w7));
    }
    dft16(v);
    __syncthreads();
    const int d = (j / Ns) * Ns * 16 + (j % Ns);
#pragma unroll
    for (int r = 0; r < 16; r++) buf[sp(d + r * Ns)] = v[r];
    __syncthreads();
}

__device__ __forceinline__ void fft4096(float2 *buf, int j) {
    fft_pass<1>(buf, j);
    fft_pass<16>(buf, j);
    fft_pass<256>(buf, j);
}

struct SpecRhs {
    double one_m_dtg, dka, dkb, scale;
    int has_g, has_a, has_b;
};

// rhs of row l (binary64 as k_fast_rhs, stored binary32 as the rhs buffer)
__device__ __forceinline__ float spec_rhs(const float *c, const int *q, long long l, long long m,
                                          const SpecRhs &k) {
    const double cv = (double)c[l];
    double r = k.has_g ? dmul(cv, k.one_m_dtg) : cv;
    if (k.has_a) r = dadd(r, dmul(k.dka, dmul((double)q[l], k.scale)));
    if (k.has_b) r = dsub(r, dmul(dmul(dmul((double)q[l + m], k.scale), cv), k.dkb));
    return (float)r;
}

// Forward rows: a block owns 4 grid rows (two complex FFTs, one per 256-thread
// group) and writes their half spectra TRANSPOSED, specT[kx][ky], four
// consecutive ky per kx = one 32-byte sector per store.
// rhs from loaded values (the same operations as spec_rhs)
__device__ __forceinline__ float spec_rhs_v(float c, int qa, int qb, const SpecRhs &k) {
    const double cv = (double)c;
    double r = k.has_g ? dmul(cv, k.one_m_dtg) : cv;
    if (k.has_a) r = dadd(r, dmul(k.dka, dmul((double)qa, k.scale)));
    if (k.has_b) r = dsub(r, dmul(dmul(dmul((double)qb, k.scale), cv), k.dkb));
    return (float)r;
}

__global__ void __launch_bounds__(2 * SP_T)
k_spec_rows_fwd(const float *__restrict__ c, const int *__restrict__ q, SpecRhs k,
                float2 *__restrict__ specT, const DevStatus *st) {
    extern __shared__ float2 sbuf[];  // [2][SP_PAD]
    float2 (*bufs)[SP_PAD] = reinterpret_cast<float2 (*)[SP_PAD]>(sbuf);
    if (st->abort) return;
    const int T = threadIdx.x, g = T / SP_T, j = T % SP_T;
    const long long m = (long long)SP_N * SP_N;
    const int y0 = 4 * blockIdx.x;  // rows y0 .. y0+3; group g packs rows y0+2g, y0+2g+1
    float2 *buf = bufs[g];
    const long long r0 = (long long)(y0 + 2 * g) * SP_N, r1 = r0 + SP_N;
    // 16-byte loads: thread j takes elements 4e .. 4e+3, e = j + 256 u
    const float4 *c0 = reinterpret_cast<const float4 *>(c + r0);
    const float4 *c1 = reinterpret_cast<const float4 *>(c + r1);
    const int4 *qa0 = reinterpret_cast<const int4 *>(q + r0);
    const int4 *qa1 = reinterpret_cast<const int4 *>(q + r1);
    const int4 *qb0 = reinterpret_cast<const int4 *>(q + m + r0);
    const int4 *qb1 = reinterpret_cast<const int4 *>(q + m + r1);
#pragma unroll 2
    for (int u = 0; u < 4; u++) {
        const int e = j + u * SP_T;
        const float4 ca = c0[e], cb = c1[e];
        const int4 pa = k.has_a ? qa0[e] : make_int4(0, 0, 0, 0);
        const int4 pb = k.has_a ? qa1[e] : make_int4(0, 0, 0, 0);
        const int4 sa4 = k.has_b ? qb0[e] : make_int4(0, 0, 0, 0);
        const int4 sb4 = k.has_b ? qb1[e] : make_int4(0, 0, 0, 0);
        const float cav[4] = {ca.x, ca.y, ca.z, ca.w}, cbv[4] = {cb.x, cb.y, cb.z, cb.w};
        const int pav[4] = {pa.x, pa.y, pa.z, pa.w}, pbv[4] = {pb.x, pb.y, pb.z, pb.w};
        const int sav[4] = {sa4.x, sa4.y, sa4.z, sa4.w}, sbv[4] = {sb4.x, sb4.y, sb4.z, sb4.w};
#pragma unroll
        for (int i = 0; i < 4; i++)
            buf[sp(4 * e + i)] = make_float2(spec_rhs_v(cav[i], pav[i], sav[i], k),
                                             spec_rhs_v(cbv[i], pbv[i], sbv[i], k));
    }
    __syncthreads();
    fft4096(buf, j);
    // split Z of each pair: Xa = (Z[k] + conj Z[-k]) / 2, Xb = (Z[k] - conj Z[-k]) / 2i;
    // store (Xa0, Xb0, Xa1, Xb1) of kx as one 32-byte sector
    for (int kx = T; kx < SP_NH; kx += 2 * SP_T) {
        const int kn = (SP_N - kx) & (SP_N - 1);
        const float2 z0 = bufs[0][sp(kx)], w0 = bufs[0][sp(kn)];
        const float2 z1 = bufs[1][sp(kx)], w1 = bufs[1][sp(kn)];
        float4 *o = reinterpret_cast<float4 *>(specT + (long long)kx * SP_N + y0);
        o[0] = make_float4(0.5f * (z0.x + w0.x), 0.5f * (z0.y - w0.y), 0.5f * (z0.y + w0.y),
                           0.5f * (w0.x - z0.x));
        o[1] = make_float4(0.5f * (z1.x + w1.x), 0.5f * (z1.y - w1.y), 0.5f * (z1.y + w1.y),
                           0.5f * (w1.x - z1.x));
    }
}

// One spectrum column (contiguous in specT) per block: forward FFT along ky,
// the mode scale of k_mode_scale, inverse FFT, all in shared memory.
#ifndef CS_SPEC_COLS_MINB
#define CS_SPEC_COLS_MINB 4
#endif
__global__ void __launch_bounds__(SP_T, CS_SPEC_COLS_MINB)
k_spec_cols(float2 *__restrict__ specT, const double *__restrict__ lx,
            const double *__restrict__ ly, double dtdc, double inv_nn, const DevStatus *st) {
    __shared__ float2 col[SP_PAD];
    if (st->abort) return;
    const int j = threadIdx.x;
    const int kx = blockIdx.x;
    float4 *gcol = reinterpret_cast<float4 *>(specT + (long long)kx * SP_N);
#pragma unroll
    for (int u = 0; u < 8; u++) {  // 2 elements per float4, coalesced
        const int e = j + u * SP_T;
        const float4 a = gcol[e];
        col[sp(2 * e)] = make_float2(a.x, a.y);
        col[sp(2 * e + 1)] = make_float2(a.z, a.w);
    }
    __syncthreads();
    fft4096(col, j);
    const double lxv = __ldg(lx + kx);
#pragma unroll 4
    for (int u = 0; u < 16; u++) {
        const int ky = j + u * SP_T;
        const double s = inv_nn / (1.0 - dtdc * (__ldg(ly + ky) + lxv));
        float2 v = col[sp(ky)];
        v.x = v.x * s;
        v.y = v.y * s;
        col[sp(ky)] = make_float2(v.x, -v.y);  // conjugated: IDFT(v) = conj(DFT(conj v))
    }
    __syncthreads();
    fft4096(col, j);
#pragma unroll
    for (int u = 0; u < 8; u++) {
        const int e = j + u * SP_T;
        const float2 p0 = col[sp(2 * e)], p1 = col[sp(2 * e + 1)];
        gcol[e] = make_float4(p0.x, -p0.y, p1.x, -p1.y);
    }
}

// Inverse rows: a block owns 4 grid rows; reads (Xa0, Xb0, Xa1, Xb1) of every
// kx as one 32-byte sector, recombines each pair into Z = A + iB over the
// full row (Hermitian extension; the imaginary parts of the DC and Nyquist
// terms are ignored, as by a C2R transform), one inverse FFT per pair.
__global__ void __launch_bounds__(2 * SP_T)
k_spec_rows_inv(const float2 *__restrict__ specT, float *__restrict__ c, const DevStatus *st) {
    extern __shared__ float2 sbuf[];  // [2][SP_PAD]
    float2 (*bufs)[SP_PAD] = reinterpret_cast<float2 (*)[SP_PAD]>(sbuf);
    if (st->abort) return;
    const int T = threadIdx.x, g = T / SP_T, j = T % SP_T;
    const int y0 = 4 * blockIdx.x;
    for (int kx = T; kx < SP_NH; kx += 2 * SP_T) {
        const float4 *i4 = reinterpret_cast<const float4 *>(specT + (long long)kx * SP_N + y0);
        const float4 p = i4[0], q = i4[1];
        float2 a0 = make_float2(p.x, p.y), b0 = make_float2(p.z, p.w);
        float2 a1 = make_float2(q.x, q.y), b1 = make_float2(q.z, q.w);
        if (kx == 0 || kx == SP_N / 2) {
            a0.y = b0.y = a1.y = b1.y = 0.f;
        }
        // Z[kx] = A + iB, stored conjugated for IDFT(Z) = conj(DFT(conj Z))
        bufs[0][sp(kx)] = make_float2(a0.x - b0.y, -(a0.y + b0.x));
        bufs[1][sp(kx)] = make_float2(a1.x - b1.y, -(a1.y + b1.x));
        if (kx > 0 && kx < SP_N / 2) {  // Z[N - kx] = conj(A) + i conj(B)
            bufs[0][sp(SP_N - kx)] = make_float2(a0.x + b0.y, -(b0.x - a0.y));
            bufs[1][sp(SP_N - kx)] = make_float2(a1.x + b1.y, -(b1.x - a1.y));
        }
    }
    __syncthreads();
    float2 *buf = bufs[g];
    fft4096(buf, j);
    float *c0 = c + (long long)(y0 + 2 * g) * SP_N, *c1 = c0 + SP_N;
#pragma unroll 4
    for (int u = 0; u < 16; u++) {
        const int x = j + u * SP_T;
        const float2 z = buf[sp(x)];
        c0[x] = z.x;   // Re conj(DFT(conj Z)) = Re DFT(conj Z)
        c1[x] = -z.y;  // Im conj(...)
    }
}

static bool g_tw_ready = false;

int spectral_supported(int n) { return n == SP_N; }

size_t spectral_spec_bytes() { return sizeof(float2) * (size_t)SP_NH * SP_N; }

// One periodic field step on the sorted engine's binary32 grid: c (in place)
// from c and the fixed-point deposits q (2 x n^2).
int spectral_step(cs_ctx *ctx, float *c, const int *q, double one_m_dtg, double dka, double dkb,
                  int has_g, int has_a, int has_b, double scale, const double *lx,
                  const double *ly, double dtdc, float2 *spec, const DevStatus *st) {
    if (!g_tw_ready) {
        static float2 h[SP_N];
        for (int k = 0; k < SP_N; k++) {
            const double a = -2.0 * 3.14159265358979323846 * (double)k / (double)SP_N;
            h[k] = make_float2((float)cos(a), (float)sin(a));
        }
        CS_CUDA(cudaMemcpyToSymbol(g_w4096, h, sizeof(h)));
        const int rows_smem = (int)(2 * SP_PAD * sizeof(float2));
        CS_CUDA(cudaFuncSetAttribute(k_spec_rows_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     rows_smem));
        CS_CUDA(cudaFuncSetAttribute(k_spec_rows_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     rows_smem));
        g_tw_ready = true;
    }
    SpecRhs k{one_m_dtg, dka, dkb, scale, has_g, has_a, has_b};
    const size_t rows_smem = 2 * SP_PAD * sizeof(float2);
    k_spec_rows_fwd<<<SP_N / 4, 2 * SP_T, rows_smem, ctx->stream>>>(c, q, k, spec, st);
    CS_LAUNCH_CHECK();
    const double inv_nn = 1.0 / ((double)SP_N * (double)SP_N);
    k_spec_cols<<<SP_NH, SP_T, 0, ctx->stream>>>(spec, lx, ly, dtdc, inv_nn, st);
    CS_LAUNCH_CHECK();
    k_spec_rows_inv<<<SP_N / 4, 2 * SP_T, rows_smem, ctx->stream>>>(spec, c, st);
    CS_LAUNCH_CHECK();
    ctx->launches += 3;
    return CS_OK;
}

}  // namespace cs
