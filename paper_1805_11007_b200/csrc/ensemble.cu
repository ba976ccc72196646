// ensemble.cu -- many small realisations per GPU.
//
// The paper's workload is an ensemble of small systems (fig1: N = 200
// particles on a 52^2 Neumann grid, thousands of seeded realisations,
// engine.py:455-484), which the reference parallelises only across
// processes.  Here one 256-thread CTA owns one realisation for a block of
// K steps: particles, cell list and grid live in shared memory, and every
// stage of Realisation._step_inner (engine.py:369-393) runs in the CTA
// between barriers, in the reference's order and arithmetic:
//   deposit (coupling.py:77-110 gaussian / :113-138 CIC) -> rhs
//   (field.py:224-229) -> DCT-I modal solve (field.py:162-167, the same
//   k-ordered fma GEMMs as field.cu's k_gemm) -> field checks
//   (field.py:229-238) -> refresh (coupling.py:302-325, the gradient
//   stencil of field.py:128-137 evaluated at the four corner nodes) ->
//   cell list + pair forces (motion.py:170-245, csrc/common.cuh pair_loop)
//   -> Euler-Maruyama + boundaries (motion.py:268-282, :355-430) ->
//   fixed-step reactions (reactions.py:43-81).
// The Brownian increments and reaction uniforms of every realisation come
// from its own generator streams on the host (the reference's RNG
// contract), K steps at a time.  Deposits are node gathers in the
// reference's particle order (bit-identical; see ens_deposit).
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "deposit.cuh"

namespace cs {

struct EnsArgs {
    int n, nc, ncell, k_steps, step0;
    double *pos, *anchor, *drift, *local_c;  // [S][n][2], [S][n]
    uint8_t *type;                           // [S][n]
    double *c;                               // [S][nc^2]
    const double *xi;                        // step k, realisation s: xi + k xs + 2 n s
    long long xs;
    const double *u;                         // reaction uniforms: u + k us + n s
    long long us;
    const double *F, *Inv, *E;               // DCT-I operators (field.cu)
    DevStatus *st;                           // [S]
    cs_domain dom;
    BinGeom g;
    PairTab pt;
    int interact, refresh, field, deposit_kind, solve;
    double amp[2], dt, chi[2];
    int chi_pinned[2];
    GaussParams gp;
    GridGeom gg;
    Route route;
    double one_m_dtg, dka, dkb;
    int has_g, has_a, has_b;
    D1Coef kx, ky;
    double wcell;
    int react;
    double p_ab, r_beta;
    int qper;  // doubles of pair queue per warp (in the grid scratch ra/rb)
    int tamed;
    int thread_forces;  // a thread per particle instead of a warp (sparse systems)
    int scratch;        // doubles of grid scratch (ra, rb / pair queues) after c
    int pbits_words;    // u64 words of the gaussian deposit's particle bitsets (0: binned path)
};

// C = A op(B) (E *) for n <= 64 inside one CTA: T = ceil(n / 4) and thread
// (ty, tx) < (T, T) owns rows ty + T u, columns tx + T v (u, v < 4) -- no
// wasted products for n = 4T; the k loop is sequential fma, the
// accumulation order of field.cu's k_gemm.
template <bool BT>
__device__ __forceinline__ void cta_gemm(const double *A, const double *B, const double *E,
                                         double *C, int n) {
    const int T = (n + 3) >> 2;
    const int tid = threadIdx.x;
    if (tid >= T * T) return;
    const int ty = tid / T, tx = tid - ty * T;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
        for (int v = 0; v < 4; v++) acc[u][v] = 0.0;
    int rr[4], cc[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        rr[u] = min(ty + T * u, n - 1);
        cc[u] = min(tx + T * u, n - 1);
    }
    for (int k = 0; k < n; k++) {
        double a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            a[u] = A[rr[u] * n + k];
            b[u] = BT ? B[cc[u] * n + k] : B[k * n + cc[u]];
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int v = 0; v < 4; v++) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
        for (int v = 0; v < 4; v++) {
            const int r = ty + T * u, col = tx + T * v;
            if (r < n && col < n) {
                double val = acc[u][v];
                if (E) val *= E[r * n + col];
                C[r * n + col] = val;
            }
        }
}

__device__ __forceinline__ double grad_bilinear(const Bilin &b, const double *c, int n, int per,
                                                const D1Coef &k, int axis) {
    const long long r[4] = {b.r00, b.r10, b.r01, b.r11};
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int j = (int)(r[q] / n), i = (int)(r[q] - (long long)j * n);
        v[q] = axis == 0 ? d1_at(c, (long long)j * n, 1, i, n, per, k)
                         : d1_at(c, (long long)i, n, j, n, per, k);
    }
    return dadd(dadd(dadd(dmul(b.w00, v[0]), dmul(b.w10, v[1])), dmul(b.w01, v[2])),
                dmul(b.w11, v[3]));
}

__device__ __forceinline__ void set_status(DevStatus *st, int *s_abort, unsigned long long key,
                                           int step) {
    atomicMin(&st->key, key);
    st->abort = 1;
    st->step = step;
    *s_abort = 1;
}

constexpr int ENS_THREADS = 256;

constexpr int ENS_DEP_BUF = 16;
constexpr int ENS_PBITS_MAX = 1024;  // particles per realisation for the bitset deposit  // stamps per node sorted in a thread's buffer (more: selection)

// deposit_both inside the CTA in the reference's summation order (the
// algorithm of deposit.cu, in shared memory; the grid is neumann, nc <= 64):
// depositing particles binned by their deposit bin (CIC: base cell,
// gaussian: nearest node), ascending index inside a bin; then one thread per
// node sums its stamps in particle order.  key[p] = the bin (-1: not
// depositing); bend[k] = the end of bin k's range in order[] (its start is
// bend[k - 1]); uu (the force scratch, free until the pair forces) keeps
// each particle's grid coordinates u = (x - lo) / d; slots (the local
// concentration rows, rewritten by the refresh) the unordered claims; a
// 64-bit mask per row marks the occupied bins, so that a node visits only
// the non-empty bins of its stamp window.  Gaussian stamps of up to
// ENS_PBITS_MAX particles skip the bins: per grid row and per grid column a
// bitset over the particle indices (pbits) marks the particles binned
// there, and a node's candidates are (OR of its window rows) AND (OR of its
// window columns) -- visited in ascending index with no sorting.
__device__ __noinline__ void ens_deposit(const EnsArgs &a, const double *pos, const uint8_t *type,
                                         int *key, int *order, int *bend, int *slots,
                                         double *uu, unsigned long long *pbits, double *ra,
                                         double *rb, int tid) {
    __shared__ unsigned long long s_rowmask[64];
    __shared__ int s_wsum[32];
    const int NTH = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const GridGeom &gg = a.gg;
    const int nc = gg.n, m = nc * nc, n = a.n;
    const int kind = a.deposit_kind;
    const int W = (n + 63) >> 6;  // bitset words per grid row / column
    const bool use_bits = kind == CS_GAUSSIAN && pbits != nullptr;
    for (int k = tid; k < m; k += NTH) bend[k] = 0;
    for (int r = tid; r < 64; r += NTH) s_rowmask[r] = 0ULL;
    if (use_bits)
        for (int w = tid; w < 2 * nc * W; w += NTH) pbits[w] = 0ULL;
    __syncthreads();
    for (int p = tid; p < n; p += NTH) {
        int k = -1;
        if (route_bits(type, p, a.route)) {
            const double u0 = ddiv(dsub(pos[2 * p], gg.lo0), gg.d0);
            const double u1 = ddiv(dsub(pos[2 * p + 1], gg.lo1), gg.d1);
            uu[2 * p] = u0;
            uu[2 * p + 1] = u1;
            if (fabs(u0) < 0x1p52 && fabs(u1) < 0x1p52) {
                const int r = dep_bin_axis(u1, kind, nc, 0), c = dep_bin_axis(u0, kind, nc, 0);
                k = r * nc + c;
                atomicOr(&s_rowmask[r], 1ULL << c);
                if (use_bits) {
                    atomicOr(&pbits[r * W + (p >> 6)], 1ULL << (p & 63));
                    atomicOr(&pbits[(nc + c) * W + (p >> 6)], 1ULL << (p & 63));
                } else {
                    atomicAdd(&bend[k], 1);
                }
            }
        }
        key[p] = k;
    }
    __syncthreads();
    if (use_bits) {
        const GaussParams &gp = a.gp;
        for (int l = tid; l < m; l += NTH) {
            const int j = l / nc, i = l - j * nc;
            const int r0 = max(j - gp.w1, 0), r1 = min(j + gp.w1, nc - 1);
            const int cl = max(i - gp.w0, 0), ch = min(i + gp.w0, nc - 1);
            const unsigned long long cmask =
                ch - cl >= 63 ? ~0ULL : (((1ULL << (ch - cl + 1)) - 1ULL) << cl);
            unsigned long long any = 0ULL;
            for (int r = r0; r <= r1; r++) any |= s_rowmask[r];
            double sa = 0.0, sb = 0.0;
            if (any & cmask) {
                for (int w = 0; w < W; w++) {
                    unsigned long long mr = 0ULL, mc = 0ULL;
                    for (int r = r0; r <= r1; r++) mr |= pbits[r * W + w];
                    if (!mr) continue;
                    for (int c = cl; c <= ch; c++) mc |= pbits[(nc + c) * W + w];
                    unsigned long long mm = mr & mc;
                    while (mm) {
                        const int p = (w << 6) + __ffsll((long long)mm) - 1;
                        mm &= mm - 1ULL;
                        double v;
                        if (!gauss_term_u(uu[2 * p], uu[2 * p + 1], i, j, gg, gp, v)) continue;
                        const unsigned bits = route_bits(type, p, a.route);
                        if (bits & 1u) sa = dadd(sa, v);
                        if (bits & 2u) sb = dadd(sb, v);
                    }
                }
            }
            ra[l] = sa;
            rb[l] = sb;
        }
        return;
    }
    {  // exclusive scan of the counts in place: a run of bins per thread
        const int per = (m + NTH - 1) / NTH;
        const int k0 = tid * per, k1 = min(k0 + per, m);
        int run = 0;
        for (int k = k0; k < k1; k++) run += bend[k];
        int inc = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += y;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            int w = lane < NTH / 32 ? s_wsum[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            if (lane < NTH / 32) s_wsum[lane] = w;
        }
        __syncthreads();
        int acc = inc - run + (warp > 0 ? s_wsum[warp - 1] : 0);
        for (int k = k0; k < k1; k++) {
            const int v = bend[k];
            bend[k] = acc;
            acc += v;
        }
    }
    __syncthreads();
    // unordered claims (bend[k]: start -> end of bin k), then every particle
    // at its bin start + the number of the bin's particles with a smaller index
    for (int p = tid; p < n; p += NTH)
        if (key[p] >= 0) slots[atomicAdd(&bend[key[p]], 1)] = p;
    __syncthreads();
    const int total = bend[m - 1];
    for (int t = tid; t < total; t += NTH) {
        const int v = slots[t];
        const int k = key[v];
        const int s0 = k ? bend[k - 1] : 0, s1 = bend[k];
        int rank = 0;
        for (int u = s0; u < s1; u++) rank += slots[u] < v;
        order[s0 + rank] = v;
    }
    __syncthreads();
    if (kind == CS_CIC) {
        const double unit = ddiv(1.0, dmul(gg.d0, gg.d1));
        for (int l = tid; l < m; l += NTH) {
            const int j = l / nc, i = l - j * nc;
            double sa = 0.0, sb = 0.0;
            for (int q = 0; q < 4; q++) {
                const int bx = i - (q & 1), by = j - (q >> 1);
                if (bx < 0 || by < 0 || bx > nc - 2 || by > nc - 2) continue;
                if (!((s_rowmask[by] >> bx) & 1ULL)) continue;  // an empty base cell
                const int k = by * nc + bx;
                double ca = 0.0, cb = 0.0;
                for (int t = k ? bend[k - 1] : 0; t < bend[k]; t++) {
                    const int p = order[t];
                    const double w = cic_weight(pos[2 * p], pos[2 * p + 1], gg, unit, q);
                    const unsigned bits = route_bits(type, p, a.route);
                    if (bits & 1u) ca = dadd(ca, w);
                    if (bits & 2u) cb = dadd(cb, w);
                }
                sa = dadd(sa, ca);
                sb = dadd(sb, cb);
            }
            ra[l] = sa;
            rb[l] = sb;
        }
        return;
    }
    const GaussParams &gp = a.gp;
    for (int l = tid; l < m; l += NTH) {
        const int j = l / nc, i = l - j * nc;
        const int r0 = max(j - gp.w1, 0), r1 = min(j + gp.w1, nc - 1);
        const int cl = max(i - gp.w0, 0), ch = min(i + gp.w0, nc - 1);
        const unsigned long long cmask =
            ch - cl >= 63 ? ~0ULL : (((1ULL << (ch - cl + 1)) - 1ULL) << cl);
        // the stamps on this node in batches of the ENS_DEP_BUF smallest
        // particle indices above the previous batch's, each sorted and summed
        unsigned idb[ENS_DEP_BUF];
        double vb[ENS_DEP_BUF];
        double sa = 0.0, sb = 0.0;
        int last = -1;
        bool more = true;
        while (more) {
            int cnt = 0;
            more = false;
            for (int r = r0; r <= r1; r++) {
                unsigned long long bits = s_rowmask[r] & cmask;
                while (bits) {
                    const int c = __ffsll((long long)bits) - 1;
                    bits &= bits - 1ULL;
                    const int k = r * nc + c;
                    for (int t = k ? bend[k - 1] : 0; t < bend[k]; t++) {
                        const int p = order[t];
                        if (p <= last) continue;
                        if (cnt == ENS_DEP_BUF && p > (int)idb[ENS_DEP_BUF - 1]) {
                            more = true;
                            break;  // the rest of this bin is larger still
                        }
                        double v;
                        if (!gauss_term_u(uu[2 * p], uu[2 * p + 1], i, j, gg, gp, v)) continue;
                        int q = cnt;
                        if (cnt == ENS_DEP_BUF) {
                            more = true;
                            q = ENS_DEP_BUF - 1;
                        } else {
                            cnt++;
                        }
                        while (q > 0 && (int)idb[q - 1] > p) {
                            idb[q] = idb[q - 1];
                            vb[q] = vb[q - 1];
                            q--;
                        }
                        idb[q] = (unsigned)p;
                        vb[q] = v;
                    }
                }
            }
            for (int q = 0; q < cnt; q++) {
                const unsigned bits = route_bits(type, (int)idb[q], a.route);
                if (bits & 1u) sa = dadd(sa, vb[q]);
                if (bits & 2u) sb = dadd(sb, vb[q]);
            }
            if (cnt) last = (int)idb[cnt - 1];
        }
        ra[l] = sa;
        rb[l] = sb;
    }
}

// the reference pair loop of one particle (rare: a particle with more accepted
// partners than the lane-dense path keeps)
__device__ __forceinline__ double2 ens_forces_plain(const double *pos, const uint8_t *type,
                                                 const int *order, const int *starts,
                                                 const BinGeom &g, const PairTab &pt, int i) {
    double fx = 0.0, fy = 0.0;
    pair_loop(pos, type, order, starts, g, pt, i, [&](int, double sc, double dx0, double dx1) {
        fx = dadd(fx, dmul(sc, dx0));
        fy = dadd(fy, dmul(sc, dx1));
    });
    return make_double2(fx, fy);
}

// LEAN: the instantiation for a field-free, reaction-free realisation with
// thread-per-particle forces (cfg0 on the CTA engine).  The general kernel is
// ~290 KB of code; a step of such a system jumps over most of it, and the
// instruction fetches of every jump target cost more than the work between
// them -- this instantiation compiles the unused stages out.
template <int NT, bool LEAN = false>
__global__ void __launch_bounds__(NT)
k_ensemble(const __grid_constant__ EnsArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_abort;
    __shared__ double s_red[NT / 32];
    __shared__ int s_flag[NT / 32];
    const int n = a.n, m = a.nc * a.nc, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const long long s = blockIdx.x;
    double *pos = sm, *anc = pos + 2 * n, *drift = anc + 2 * n, *frc = drift + 2 * n;
    double *lc = frc + 2 * n, *c = lc + n, *ra = c + m, *rb = ra + m;
    int *order = reinterpret_cast<int *>(ra + a.scratch);
    int *starts = order + n, *cur = starts + a.ncell + 1, *key = cur + a.ncell;
    int *dbend = key + n;  // deposit bins: the end of each bin's range (nc^2)
    unsigned long long *pbits =  // per grid row / column particle bitsets (gaussian deposit)
        reinterpret_cast<unsigned long long *>(ra + a.scratch - a.pbits_words);
    uint8_t *type = reinterpret_cast<uint8_t *>(dbend + a.nc * a.nc);
    DevStatus *st = a.st + s;
    for (int i = tid; i < 2 * n; i += NT) {
        pos[i] = a.pos[2 * n * s + i];
        anc[i] = a.anchor[2 * n * s + i];
        drift[i] = a.drift[2 * n * s + i];
    }
    for (int i = tid; i < n; i += NT) {
        lc[i] = a.local_c[n * s + i];
        type[i] = a.type[n * s + i];
    }
    if (!LEAN && (a.field || a.refresh))
        for (int l = tid; l < m; l += NT) c[l] = a.c[(long long)m * s + l];
    if (tid == 0) s_abort = st->abort;
    if (a.interact)
        for (int f = tid; f <= a.ncell; f += NT) starts[f] = 0;
    long long clamped = 0;
    unsigned long long high_n = 0;
    double high = 0.0;
    __syncthreads();
#ifdef CS_CTA_TIMING
    __shared__ long long s_t[12];
    long long t_last = clock64();
    if (tid == 0) for (int q = 0; q < 12; q++) s_t[q] = 0;
#define CS_TICK(i) do { if (tid == 0) { const long long now_ = clock64(); s_t[i] += now_ - t_last; t_last = now_; } } while (0)
#else
#define CS_TICK(i) do { } while (0)
#endif
    for (int kk = 0; kk < a.k_steps; kk++) {
        if (s_abort) break;
        const int step = a.step0 + kk;
        CS_TICK(0);
        // this thread's first increment of the step, requested before the
        // step's other phases (one global-memory latency off the EM phase)
        const double *xk = a.xi + (long long)kk * a.xs + 2LL * n * s;
        double2 xpre = make_double2(0.0, 0.0);
        if (tid < n) xpre = *reinterpret_cast<const double2 *>(xk + 2 * tid);
        const GridGeom &gg = a.gg;
        const int nc = gg.n;
        if (!LEAN && a.field) {
            // ---- deposit_both (coupling.py:77-110, 113-138), every node summed
            // in the reference's particle order (see deposit.cu): depositing
            // particles binned by deposit row (CIC: base row, gaussian: nearest
            // row), ascending index inside a row; then one thread per node
            ens_deposit(a, pos, type, key, order, dbend, reinterpret_cast<int *>(lc), frc,
                        a.pbits_words ? pbits : nullptr, ra, rb, tid);
            __syncthreads();
            // ---- rhs (field.py:224-229), in place into ra
            for (int l = tid; l < m; l += NT) {
                const double cv = c[l];
                double r = a.has_g ? dmul(cv, a.one_m_dtg) : cv;
                if (a.has_a) r = dadd(r, dmul(a.dka, ra[l]));
                if (a.has_b) r = dsub(r, dmul(dmul(rb[l], cv), a.dkb));
                ra[l] = r;
            }
            __syncthreads();
            // ---- implicit solve (field.py:162-170)
            if (a.solve) {
                cta_gemm<false>(a.F, ra, nullptr, rb, nc);  // T1 = F X
                __syncthreads();
                cta_gemm<true>(rb, a.F, a.E, ra, nc);       // T2 = E * (T1 F^T)
                __syncthreads();
                cta_gemm<false>(a.Inv, ra, nullptr, rb, nc);  // U = Inv T2
                __syncthreads();
                cta_gemm<true>(rb, a.Inv, nullptr, c, nc);    // c = U Inv^T
            } else {
                for (int l = tid; l < m; l += NT) c[l] = ra[l];
            }
            __syncthreads();
            // ---- post-checks (field.py:229-238): non-finite, negative mass
            double neg = 0.0;
            int flags = 0;
            for (int l = tid; l < m; l += NT) {
                const double v = c[l];
                if (!isfinite(v)) flags |= 1;
                if (v < 0.0) {
                    const int j = l / nc, i = l - j * nc;
                    const double wi = (i == 0 || i == nc - 1) ? 0.5 : 1.0;
                    const double wj = (j == 0 || j == nc - 1) ? 0.5 : 1.0;
                    neg += ((wj * wi) * a.wcell) * v;
                    flags |= 2;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                neg += __shfl_xor_sync(0xffffffffu, neg, o);
                flags |= __shfl_xor_sync(0xffffffffu, flags, o);
            }
            if (lane == 0) {
                s_red[warp] = neg;
                s_flag[warp] = flags;
            }
            __syncthreads();
            if (tid == 0) {
                double t = 0.0;
                int f = 0;
                for (int w = 0; w < NT / 32; w++) {
                    t += s_red[w];
                    f |= s_flag[w];
                }
                if (f & 1) set_status(st, &s_abort, err_key(0, 0, CS_FIELD_NONFINITE), step);
                if ((f & 2) && t < -1e-12) {
                    if (st->neg_steps == 0) st->first_neg = t;
                    st->neg_steps += 1;
                }
            }
            __syncthreads();
            if (s_abort) break;
        }
        // ---- refresh (coupling.py:302-325)
        if (!LEAN && a.refresh) {
            for (int p = tid; p < n; p += NT) {
                Bilin b;
                clamped += 2 * bilinear_stencil(pos[2 * p], pos[2 * p + 1], gg, b);
                lc[p] = bilinear_apply(b, c, 1, 0);
                const int t = type[p] ? 1 : 0;
                double d0 = grad_bilinear(b, c, nc, gg.per, a.kx, 0);
                double d1 = grad_bilinear(b, c, nc, gg.per, a.ky, 1);
                if (a.chi_pinned[t]) {
                    d0 = 0.0;
                    d1 = 0.0;
                } else if (a.chi[t] != 1.0) {
                    d0 = dmul(d0, a.chi[t]);
                    d1 = dmul(d1, a.chi[t]);
                }
                drift[2 * p] = d0;
                drift[2 * p + 1] = d1;
            }
        }
        // ---- cell list + pair forces (motion.py:170-245)
        if (a.interact) {
            // (the cell counts were cleared before the first step and by the
            // previous step's EM phase, which does not read the cell table)
            CS_TICK(1);
#pragma unroll 1
            for (int p = tid; p < n; p += NT) {
                const double2 xp = reinterpret_cast<const double2 *>(pos)[p];
                const int k = cell_axis(xp.y, a.g.lo1, a.g.eff1, a.g.n1) * a.g.n0 +
                              cell_axis(xp.x, a.g.lo0, a.g.eff0, a.g.n0);
                key[p] = k;
                atomicAdd(&starts[k + 1], 1);
            }
            __syncthreads();
            CS_TICK(2);
            {  // inclusive scan of starts[1..ncell] (the counts): a run of cells
               // per thread, then the block's run totals
                // (an odd run length: the threads' runs start on distinct banks)
                const int per = ((a.ncell + NT - 1) / NT) | 1;
                const int f0 = min(1 + tid * per, a.ncell + 1), f1 = min(f0 + per, a.ncell + 1);
                int run = 0;
                for (int f = f0; f < f1; f++) run += starts[f];
                int inc = run;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += y;
                }
                if (lane == 31) s_flag[warp] = inc;
                __syncthreads();
                if (warp == 0) {
                    int w = lane < NT / 32 ? s_flag[lane] : 0;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, w, d);
                        if (lane >= d) w += y;
                    }
                    if (lane < NT / 32) s_flag[lane] = w;
                }
                __syncthreads();
                int acc = inc - run + (warp > 0 ? s_flag[warp - 1] : 0);
                for (int f = f0; f < f1; f++) {  // starts[f] = first slot of cell f
                    acc += starts[f];
                    starts[f] = acc;
                    if (f < a.ncell) cur[f] = acc;  // and its claim cursor
                }
                if (tid == 0) cur[0] = 0;
                __syncthreads();
                CS_TICK(3);
            }
            {
                // stable placement (ascending index inside a cell,
                // motion.py:195-199): unordered claims into the cell ranges
                // (the force scratch holds the slots), then every particle at
                // its cell start + the number of the cell's particles with a
                // smaller index
                int *slots = reinterpret_cast<int *>(frc);
#pragma unroll 1
                for (int p = tid; p < n; p += NT) slots[atomicAdd(&cur[key[p]], 1)] = p;
                __syncthreads();
                CS_TICK(4);
#pragma unroll 1
                for (int t = tid; t < n; t += NT) {
                    const int v = slots[t];
                    const int k = key[v];
                    const int s0 = starts[k], s1 = starts[k + 1];
                    int rank = 0;
                    for (int u = s0; u < s1; u++) rank += slots[u] < v;
                    order[s0 + rank] = v;
                }
            }
            __syncthreads();
            CS_TICK(5);
            if (LEAN || a.thread_forces) {
                // sparse systems (<= 2 particles per cell; the single-
                // realisation CTA engine): a lane per particle walks its ring in
                // the reference order (as common.cuh pair_loop) with the exact
                // test only, keeping up to four accepted partners; the warp's
                // accepted pairs are then evaluated one per lane (the binary64
                // sqrt / exp / divisions on dense lanes instead of once per
                // lane that happens to hold a pair) and every owner adds its
                // terms in walk order.  All exchange is by shuffles.
                const BinGeom &g = a.g;
                const unsigned ltm = (1u << lane) - 1u;
                for (int ib = warp * 32; ib < n; ib += NT) {
                    const int i = ib + lane;
                    const bool live = i < n;
                    double xi = 0.0, yi = 0.0;
                    int ti = 0, nacc = 0, pj0 = 0, pj1 = 0, pj2 = 0, pj3 = 0;
                    if (live) {
                        const double2 pi = reinterpret_cast<const double2 *>(pos)[i];
                        xi = pi.x;
                        yi = pi.y;
                        ti = type[i] ? 1 : 0;
                        const int cy = key[i] / g.n0, cx = key[i] - cy * g.n0;  // binned above
                        auto candidate = [&](int k) {
                            const int j = order[k];
                            if (j == i) return;
                            const double2 pj = reinterpret_cast<const double2 *>(pos)[j];
                            double dx0 = dsub(pj.x, xi);
                            double dx1 = dsub(pj.y, yi);
                            if (g.per0) dx0 = dsub(dx0, dmul(g.size0, rint(ddiv(dx0, g.size0))));
                            if (g.per1) dx1 = dsub(dx1, dmul(g.size1, rint(ddiv(dx1, g.size1))));
                            const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                            const int t = ti * 2 + (type[j] ? 1 : 0);
                            if (r2 > a.pt.cut2[t] || r2 == 0.0) return;
                            if (nacc == 0) pj0 = j;
                            else if (nacc == 1) pj1 = j;
                            else if (nacc == 2) pj2 = j;
                            else if (nacc == 3) pj3 = j;
                            nacc++;
                        };
                        // the ring's cells of one row are consecutive in the
                        // cell table unless the row wraps around a periodic
                        // axis: one slot range per row, in the reference's
                        // order (o0 ascending, ascending index inside a cell)
                        const bool rows = !g.per0 || (g.n0 >= 3 && cx >= 1 && cx + 1 < g.n0);
                        const int c0 = cx >= 1 ? cx - 1 : 0, c1 = cx + 1 < g.n0 ? cx + 1 : g.n0 - 1;
                        for (int o1 = -1; o1 <= 1; o1++) {
                            int g1 = cy + o1;
                            if (g.per1) {
                                if (g.n1 == 1 && o1 != 0) continue;
                                if (g.n1 == 2 && o1 == 1) continue;
                                g1 = (int)pymod(g1, g.n1);
                            } else if (g1 < 0 || g1 >= g.n1) {
                                continue;
                            }
                            if (rows) {
                                const int kend = starts[g1 * g.n0 + c1 + 1];
                                for (int k = starts[g1 * g.n0 + c0]; k < kend; k++) candidate(k);
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
                                for (int k = starts[f]; k < kend; k++) candidate(k);
                            }
                        }
                    }
                    CS_TICK(8);
                    const int nq = nacc < 4 ? nacc : 4;
                    // entries level by level: (lane, s) -> b_s + its rank in level s
                    const unsigned m0 = __ballot_sync(0xffffffffu, nq > 0);
                    const unsigned m1 = __ballot_sync(0xffffffffu, nq > 1);
                    const unsigned m2 = __ballot_sync(0xffffffffu, nq > 2);
                    const unsigned m3 = __ballot_sync(0xffffffffu, nq > 3);
                    const int b1 = __popc(m0), b2 = b1 + __popc(m1), b3 = b2 + __popc(m2);
                    const int total = b3 + __popc(m3);
                    double fx = 0.0, fy = 0.0;
                    for (int r0 = 0; r0 < total; r0 += 32) {
                        const int e = r0 + lane;
                        const int lv = e >= b3 ? 3 : (e >= b2 ? 2 : (e >= b1 ? 1 : 0));
                        const unsigned ml = lv == 3 ? m3 : (lv == 2 ? m2 : (lv == 1 ? m1 : m0));
                        const int bl = lv == 3 ? b3 : (lv == 2 ? b2 : (lv == 1 ? b1 : 0));
                        const int ow = e < total ? (int)__fns(ml, 0, e - bl + 1) : lane;
                        const int q0 = __shfl_sync(0xffffffffu, pj0, ow);
                        const int q1 = __shfl_sync(0xffffffffu, pj1, ow);
                        const int q2 = __shfl_sync(0xffffffffu, pj2, ow);
                        const int q3 = __shfl_sync(0xffffffffu, pj3, ow);
                        const double xo = __shfl_sync(0xffffffffu, xi, ow);
                        const double yo = __shfl_sync(0xffffffffu, yi, ow);
                        const int to = __shfl_sync(0xffffffffu, ti, ow);
                        double tx = 0.0, ty = 0.0;
                        if (e < total) {
                            const int j = lv == 3 ? q3 : (lv == 2 ? q2 : (lv == 1 ? q1 : q0));
                            const double2 pj = reinterpret_cast<const double2 *>(pos)[j];
                            double dx0 = dsub(pj.x, xo);
                            double dx1 = dsub(pj.y, yo);
                            if (g.per0) dx0 = dsub(dx0, dmul(g.size0, rint(ddiv(dx0, g.size0))));
                            if (g.per1) dx1 = dsub(dx1, dmul(g.size1, rint(ddiv(dx1, g.size1))));
                            const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                            const double eps = a.pt.eps[to * 2 + (type[j] ? 1 : 0)];
                            const double rr = dsqrt(r2);
                            const double sc = -ddiv(cs_exp(-ddiv(rr, eps)), dmul(eps, rr));
                            tx = dmul(sc, dx0);
                            ty = dmul(sc, dx1);
                        }
                        // owners take their terms in level (= walk) order
#pragma unroll
                        for (int s2 = 0; s2 < 4; s2++) {
                            if ((s2 == 1 && !m1) || (s2 == 2 && !m2) || (s2 == 3 && !m3)) break;
                            const unsigned mm = s2 == 3 ? m3 : (s2 == 2 ? m2 : (s2 == 1 ? m1 : m0));
                            const int bb = s2 == 3 ? b3 : (s2 == 2 ? b2 : (s2 == 1 ? b1 : 0));
                            const int src = bb + __popc(mm & ltm) - r0;
                            const bool mine = s2 < nq && src >= 0 && src < 32;
                            const double vx = __shfl_sync(0xffffffffu, tx, mine ? src : 0);
                            const double vy = __shfl_sync(0xffffffffu, ty, mine ? src : 0);
                            if (mine) {
                                fx = dadd(fx, vx);
                                fy = dadd(fy, vy);
                            }
                        }
                    }
                    CS_TICK(9);
                    if (live) {
                        if (nacc > 4) {  // more partners than kept: the plain loop
                            const double2 ff = ens_forces_plain(pos, type, order, starts, a.g,
                                                                a.pt, i);
                            fx = ff.x;
                            fy = ff.y;
                        }
                        frc[2 * i] = fx;
                        frc[2 * i + 1] = fy;
                    }
                }
            } else {
            // one warp per particle: the lanes test its ring candidates 32 at
            // a time in ring order (cells o1-major, ascending index inside a
            // cell) and evaluate the accepted pair terms in parallel; the
            // terms are then added in candidate order (motion.py:240-243)
            const BinGeom &g = a.g;
            double *wq = ra + (long long)warp * a.qper;  // this warp's pair queue
            const int qcap = a.qper / 4;
            for (int i = warp; i < n; i += NT / 32) {
                const double xi = pos[2 * i], yi = pos[2 * i + 1];
                const int cx = cell_axis(xi, g.lo0, g.eff0, g.n0);
                const int cy = cell_axis(yi, g.lo1, g.eff1, g.n1);
                const int ti = type[i] ? 1 : 0;
                int rs = 0, rl = 0;
                if (lane < 9) {
                    const int o1 = lane / 3 - 1, o0 = lane % 3 - 1;
                    int g1 = cy + o1, g0 = cx + o0;
                    bool ok = true;
                    if (g.per1) {
                        if ((g.n1 == 1 && o1 != 0) || (g.n1 == 2 && o1 == 1)) ok = false;
                        g1 = (int)pymod(g1, g.n1);
                    } else if (g1 < 0 || g1 >= g.n1) {
                        ok = false;
                    }
                    if (g.per0) {
                        if ((g.n0 == 1 && o0 != 0) || (g.n0 == 2 && o0 == 1)) ok = false;
                        g0 = (int)pymod(g0, g.n0);
                    } else if (g0 < 0 || g0 >= g.n0) {
                        ok = false;
                    }
                    if (ok) {
                        const int f = g1 * g.n0 + g0;
                        rs = starts[f];
                        rl = starts[f + 1] - rs;
                    }
                }
                int incl = rl;
#pragma unroll
                for (int d = 1; d < 16; d <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 8);
                int pre[9], cs_[9];
#pragma unroll
                for (int r = 0; r < 9; r++) {
                    pre[r] = __shfl_sync(0xffffffffu, incl - rl, r);
                    cs_[r] = __shfl_sync(0xffffffffu, rs, r);
                }
                // accepted pairs are queued (ballot-compacted, candidate
                // order) in the warp's slice of the grid scratch, their terms
                // evaluated 32 at a time, then added in order by lane 0
                double fx = 0.0, fy = 0.0;
                int nq = 0;
                auto flush = [&]() {
                    __syncwarp();
                    for (int e = lane; e < nq; e += 32) {
                        double *qe = wq + 4 * e;
                        const double eps = qe[3], rr = dsqrt(qe[2]);
                        const double sc = -ddiv(cs_exp(-ddiv(rr, eps)), dmul(eps, rr));
                        qe[0] = dmul(sc, qe[0]);
                        qe[1] = dmul(sc, qe[1]);
                    }
                    __syncwarp();
                    if (lane == 0)
                        for (int e = 0; e < nq; e++) {
                            fx = dadd(fx, wq[4 * e]);
                            fy = dadd(fy, wq[4 * e + 1]);
                        }
                    __syncwarp();
                    nq = 0;
                };
                for (int k0 = 0; k0 < total; k0 += 32) {
                    if (nq + 32 > qcap) flush();
                    const int k = k0 + lane;
                    double dx0 = 0.0, dx1 = 0.0, r2 = 0.0, eps = 0.0;
                    bool acc = false;
                    if (k < total) {
                        int r = 0;
#pragma unroll
                        for (int q = 1; q < 9; q++) r = k >= pre[q] ? q : r;
                        int base = cs_[0] - pre[0];
#pragma unroll
                        for (int q = 1; q < 9; q++) base = r == q ? cs_[q] - pre[q] : base;
                        const int j = order[base + k];
                        if (j != i) {
                            dx0 = dsub(pos[2 * j], xi);
                            dx1 = dsub(pos[2 * j + 1], yi);
                            if (g.per0) dx0 = dsub(dx0, dmul(g.size0, rint(ddiv(dx0, g.size0))));
                            if (g.per1) dx1 = dsub(dx1, dmul(g.size1, rint(ddiv(dx1, g.size1))));
                            r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                            const int t = ti * 2 + (type[j] ? 1 : 0);
                            acc = !(r2 > a.pt.cut2[t] || r2 == 0.0);
                            eps = a.pt.eps[t];
                        }
                    }
                    const unsigned msk = __ballot_sync(0xffffffffu, acc);
                    if (acc) {
                        double *qe = wq + 4 * (nq + __popc(msk & ((1u << lane) - 1u)));
                        qe[0] = dx0;
                        qe[1] = dx1;
                        qe[2] = r2;
                        qe[3] = eps;
                    }
                    nq += __popc(msk);
                }
                flush();
                if (lane == 0) {
                    frc[2 * i] = fx;
                    frc[2 * i + 1] = fy;
                }
            }
            }
        }
        __syncthreads();
        CS_TICK(6);
        // ---- Euler-Maruyama + boundaries (motion.py:268-282, 355-430)
        if (a.interact)  // the next step's cell counts
            for (int f = tid; f <= a.ncell; f += NT) starts[f] = 0;
#pragma unroll 1
        for (int p = tid; p < n; p += NT) {
            const int t = type[p] ? 1 : 0;
            const double amp = a.amp[t];
            const double z0 = p == tid ? xpre.x : xk[2 * p], z1 = p == tid ? xpre.y : xk[2 * p + 1];
            double2 *pos2 = reinterpret_cast<double2 *>(pos), *anc2 = reinterpret_cast<double2 *>(anc);
            const double2 fp = a.interact ? reinterpret_cast<const double2 *>(frc)[p]
                                          : make_double2(0.0, 0.0);
            const double2 xp = pos2[p], dp = reinterpret_cast<const double2 *>(drift)[p];
            double i0, i1;
            force_increment(fp.x, fp.y, a.dt, a.tamed, i0, i1);
            double v[2];
            v[0] = dadd(dadd(dadd(xp.x, dmul(amp, z0)), dmul(dp.x, a.dt)), i0);
            v[1] = dadd(dadd(dadd(xp.y, dmul(amp, z1)), dmul(dp.y, a.dt)), i1);
            const double raw0 = v[0], raw1 = v[1];
            bool ok = isfinite(v[0]) && isfinite(v[1]);
            if (!ok) set_status(st, &s_abort, err_key(0, p, CS_NONFINITE), step);
            const double2 ap = anc2[p];
            double an[2] = {ap.x, ap.y};
            for (int ax = 0; ok && ax < 2; ax++) {
                const int code = boundary_axis(v[ax], an[ax], a.dom.lo[ax], a.dom.hi[ax],
                                               a.dom.periodic[ax]);
                if (code) {
                    set_status(st, &s_abort, err_key(1 + ax, p, code), step);
                    ok = false;
                }
            }
            if (!ok) {  // the raw proposal stays visible for the host's message
                pos2[p] = make_double2(raw0, raw1);
                continue;
            }
            pos2[p] = make_double2(v[0], v[1]);
            anc2[p] = make_double2(an[0], an[1]);
        }
        __syncthreads();
        CS_TICK(7);
        if (s_abort) break;
        // ---- fixed-step reactions (reactions.py:43-81)
        if (!LEAN && a.react) {
            const double *uk = a.u + (long long)kk * a.us + (long long)n * s;
            for (int p = tid; p < n; p += NT) {
                const double ui = uk[p];
                if (type[p] == 0) {
                    if (a.p_ab > 1.0) {
                        high_n++;
                        high = fmax(high, a.p_ab);
                    }
                    if (ui < a.p_ab) type[p] = 1;
                } else if (a.r_beta != 0.0) {
                    const double cv = lc[p];
                    const double conc = cv > 0.0 || cv != cv ? cv : 0.0;
                    const double pb = dmul(dmul(a.r_beta, conc), a.dt);
                    if (pb > 1.0) {
                        high_n++;
                        high = fmax(high, pb);
                    }
                    if (ui < pb) {
                        type[p] = 0;
                        drift[2 * p] = 0.0;
                        drift[2 * p + 1] = 0.0;
                    }
                }
            }
            __syncthreads();
        }
    }
    __syncthreads();
#ifdef CS_CTA_TIMING
    if (tid == 0 && blockIdx.x == 0)
        printf("cta timing (cycles/step): top %lld zero %lld count %lld scan %lld claim %lld rank %lld force %lld (walk %lld eval %lld) em %lld\n",
               s_t[0] / a.k_steps, s_t[1] / a.k_steps, s_t[2] / a.k_steps, s_t[3] / a.k_steps,
               s_t[4] / a.k_steps, s_t[5] / a.k_steps, s_t[6] / a.k_steps, s_t[8] / a.k_steps,
               s_t[9] / a.k_steps, s_t[7] / a.k_steps);
#endif
    for (int i = tid; i < 2 * n; i += NT) {
        a.pos[2 * n * s + i] = pos[i];
        a.anchor[2 * n * s + i] = anc[i];
        a.drift[2 * n * s + i] = drift[i];
    }
    for (int i = tid; i < n; i += NT) {
        a.local_c[n * s + i] = lc[i];
        a.type[n * s + i] = type[i];
    }
    if (!LEAN && a.field)
        for (int l = tid; l < m; l += NT) a.c[(long long)m * s + l] = c[l];
    if (clamped) atomicAdd((unsigned long long *)&st->clamped, (unsigned long long)clamped);
    if (high_n) {
        atomicAdd(&st->react_high_n, high_n);
        atomicMax(&st->react_high_bits, (unsigned long long)__double_as_longlong(high));
    }
}

}  // namespace cs

namespace cs {

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// DOUBLE_pairwise_sum): < 8 terms in order from -0.0; <= 128 terms in 8
// interleaved accumulators folded ((r0 + r1) + (r2 + r3)) + ((r4 + r5) +
// (r6 + r7)) plus the tail in order; beyond, split at n / 2 rounded down to
// a multiple of 8.  Used for the per-sample mean squared displacement.
__device__ double np_pairwise_sum(const double *v, int n) {
    if (n < 8) {
        double res = -0.0;
        for (int i = 0; i < n; i++) res = dadd(res, v[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int q = 0; q < 8; q++) r[q] = v[q];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int q = 0; q < 8; q++) r[q] = dadd(r[q], v[i + q]);
        double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                          dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
        for (; i < n; i++) res = dadd(res, v[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return dadd(np_pairwise_sum(v, n2), np_pairwise_sum(v + n2, n - n2));
}

// per sample: Alpha count and msd = mean over particles of
// (0 + dx^2) + dy^2 (engine.py:230-235 in numpy's reduction order); one
// block per sample, the squared displacements staged in shared memory
__global__ void __launch_bounds__(256)
k_ens_observe(const double *__restrict__ pos, const double *__restrict__ anchor,
              const uint8_t *__restrict__ type, int n, long long *__restrict__ n_alpha,
              double *__restrict__ msd) {
    extern __shared__ double sq[];
    __shared__ int s_cnt;
    const long long s = blockIdx.x;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int c = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double d0 = dsub(pos[2 * n * s + 2 * i], anchor[2 * n * s + 2 * i]);
        const double d1 = dsub(pos[2 * n * s + 2 * i + 1], anchor[2 * n * s + 2 * i + 1]);
        sq[i] = dadd(dadd(-0.0, dmul(d0, d0)), dmul(d1, d1));
        c += type[(long long)n * s + i] == 0 ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, c);
    __syncthreads();
    if (threadIdx.x == 0) {
        n_alpha[s] = s_cnt;
        msd[s] = ddiv(np_pairwise_sum(sq, n), (double)n);
    }
}

}  // namespace cs

// ---------------------------------------------------------------- host side
namespace cs {
int field_ops_create(cs_ctx *ctx, int prec, const cs_grid *g, double d_c, double dt,
                     cs_field_ops **out);
void field_ops_destroy(cs_field_ops *ops);
}  // namespace cs

struct cs_ens {
    cs_ctx *ctx = nullptr;
    cs_sim_params p{};
    int n_real = 0;
    int steps_done = 0;
    cs::EnsArgs a{};
    cs_field_ops *ops = nullptr;
    cs::Buf status;  // DevStatus[n_real]
    size_t smem = 0;
    int threads = 256;
};

namespace cs {

// scratch doubles after c: ra and rb of the field stage, reused as the warps'
// pair queues by the force stage (at least 64 entries of 4 doubles per warp)
// pbits: u64 words of the gaussian deposit's bitsets (2 nc ceil(n/64)),
// after ra and rb (the pair queues reuse the whole region later)
static size_t ens_scratch(int nc, int warps, size_t pbits = 0) {
    const size_t m = (size_t)nc * nc;
    const size_t q = (size_t)warps * 4 * 64;
    return 2 * m + pbits > q ? 2 * m + pbits : q;
}

static size_t ens_pbits_words(const cs_sim_params *p, int nc) {
    if (!p->field_active || p->deposit_kind != CS_GAUSSIAN || p->n > ENS_PBITS_MAX) return 0;
    return 2 * (size_t)nc * (size_t)((p->n + 63) / 64);
}

static size_t ens_smem(int n, int nc, int ncell, int warps, size_t pbits) {
    const size_t m = (size_t)nc * nc;
    return sizeof(double) * (9 * (size_t)n + m + ens_scratch(nc, warps, pbits)) +
           sizeof(int) * (2 * (size_t)n + 2 * (size_t)ncell + 1 + m) + (size_t)n + 16;
}

int ens_create(cs_ctx *ctx, const cs_sim_params *p, int n_real, cs_ens **out) {
    *out = nullptr;
    if (p->prec != CS_F64) {
        set_error("the ensemble engine runs in binary64 (prec must be CS_F64)");
        return CS_ERR_PARAM;
    }
    if (p->n < 1 || p->n > 4096 || n_real < 1) {
        set_error("ensemble: 1 <= n <= 4096 particles per realisation and >= 1 realisation");
        return CS_ERR_PARAM;
    }
    const bool grid = p->field_active || p->refresh_active;
    if (grid && (p->grid.periodic || p->grid.n_c < 3 || p->grid.n_c > 64)) {
        set_error("ensemble: the grid must be neumann with 3 <= n_c <= 64 "
                  "(periodic grids run through cs_sim)");
        return CS_ERR_PARAM;
    }
    auto *e = new cs_ens();
    *out = e;
    e->ctx = ctx;
    e->p = *p;
    e->n_real = n_real;
    EnsArgs &a = e->a;
    a.n = (int)p->n;
    a.nc = grid ? p->grid.n_c : 0;
    a.dom = p->domain;
    a.interact = p->interaction == 1;
    a.ncell = 0;
    if (a.interact) {
        a.g = make_geom(p->domain, p->pairs.cell_cutoff);
        a.pt = make_pairtab(p->pairs);
        a.ncell = a.g.n0 * a.g.n1;
    }
    a.refresh = p->refresh_active;
    a.field = p->field_active;
    for (int t = 0; t < 2; t++) {
        a.amp[t] = p->amp[t];
        a.chi[t] = p->chi[t];
        a.chi_pinned[t] = p->chi_pinned[t];
        a.route.bits[t] = (unsigned char)((p->secretes[t] ? 1 : 0) | (p->consumes[t] ? 2 : 0));
    }
    a.route.bits[2] = 0;
    a.dt = p->dt;
    if (grid) {
        a.gg = make_grid_geom(p->grid);
        a.kx = make_d1(a.gg.d0);
        a.ky = make_d1(a.gg.d1);
        a.wcell = a.gg.d0 * a.gg.d1;
    }
    if (a.field) {
        a.deposit_kind = p->deposit_kind;
        a.gp = make_gauss(a.gg, p->kernel_h, p->kernel_cutoff);
        a.has_g = p->gamma != 0.0;
        a.has_a = p->k_alpha != 0.0;
        a.has_b = p->k_beta != 0.0;
        a.one_m_dtg = 1.0 - p->dt * p->gamma;
        a.dka = p->dt * p->k_alpha;
        a.dkb = p->dt * p->k_beta;
        CS_TRY(field_ops_create(ctx, CS_F64, &p->grid, p->d_c, p->dt, &e->ops));
        a.solve = e->ops->kind == 1;
        a.F = e->ops->F;
        a.Inv = e->ops->Inv;
        a.E = e->ops->E;
    }
    a.tamed = p->integrator == 1;
    a.react = p->react;
    a.p_ab = p->react_p_ab;
    a.r_beta = p->react_r_beta;
    // one realisation (the CTA engine of cs_sim): 1024 threads, and a thread
    // per particle for the pair forces when the system is sparse
    // (cfg0, 1000 particles: 512 threads 19.5 us/step, 1024 threads 15.6)
    e->threads = n_real == 1 ? (getenv("CS_CTA_THREADS") ? atoi(getenv("CS_CTA_THREADS"))
                                                         : (p->n >= 768 ? 1024 : 512))
                             : ENS_THREADS;
    a.thread_forces = n_real == 1 && a.interact && (double)a.n <= 2.0 * (double)a.ncell;
    const size_t pw = ens_pbits_words(p, a.nc);
    a.pbits_words = (int)pw;
    const int qwarps = a.thread_forces ? 0 : e->threads / 32;  // warps with a pair queue
    a.scratch = (int)ens_scratch(a.nc, qwarps, pw);
    a.qper = qwarps ? a.scratch / qwarps : 0;
    e->smem = ens_smem(a.n, a.nc, a.ncell, qwarps, pw);
    int dev_max = 0;
    CS_CUDA(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                   ctx->device));
    if (e->smem + 2048 > (size_t)dev_max) {
        set_error("ensemble: a realisation needs %zu B of shared memory (> %d)", e->smem,
                  dev_max);
        return CS_ERR_PARAM;
    }
    CS_CUDA(cudaFuncSetAttribute(k_ensemble<ENS_THREADS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->smem));
    CS_CUDA(cudaFuncSetAttribute(k_ensemble<1024, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->smem));
    CS_CUDA(cudaFuncSetAttribute(k_ensemble<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)e->smem));
    CS_CUDA(cudaFuncSetAttribute(k_ensemble<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)e->smem));
    CS_CUDA(cudaFuncSetAttribute(k_ensemble<768>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)e->smem));
    CS_TRY(e->status.ensure(sizeof(DevStatus) * (size_t)n_real));
    std::vector<DevStatus> init((size_t)n_real);
    for (auto &d : init) {
        d = DevStatus{};
        d.key = ~0ULL;
        d.step = -1;
    }
    CS_CUDA(cudaMemcpy(e->status.p, init.data(), sizeof(DevStatus) * (size_t)n_real,
                       cudaMemcpyHostToDevice));
    return CS_OK;
}

void ens_destroy(cs_ens *e) {
    if (!e) return;
    field_ops_destroy(e->ops);
    e->status.release();
    delete e;
}

int ens_step(cs_ens *e, const cs_ens_state *s, const double *xi, const double *u, int k) {
    if (k <= 0) return CS_OK;
    if (e->p.react && !u) {
        set_error("params.react is set: the ensemble step needs the reaction uniforms");
        return CS_ERR_PARAM;
    }
    if (!s->pos || !s->anchor || !s->drift || !s->local_c || !s->type ||
        ((e->a.field || e->a.refresh) && !s->c)) {
        set_error("ensemble state: pos, anchor, drift, local_c, type (and c) are required");
        return CS_ERR_PARAM;
    }
    EnsArgs a = e->a;
    a.pos = s->pos;
    a.anchor = s->anchor;
    a.drift = s->drift;
    a.local_c = s->local_c;
    a.type = s->type;
    a.c = s->c;
    a.xi = xi;
    a.xs = 2LL * a.n * e->n_real;
    a.u = u;
    a.us = (long long)a.n * e->n_real;
    a.st = e->status.as<DevStatus>();
    a.k_steps = k;
    a.step0 = e->steps_done;
    if (e->threads == 1024 && a.thread_forces && !a.field && !a.refresh && !a.react)
        k_ensemble<1024, true><<<e->n_real, 1024, e->smem, e->ctx->stream>>>(a);
    else if (e->threads == 1024)
        k_ensemble<1024><<<e->n_real, 1024, e->smem, e->ctx->stream>>>(a);
    else if (e->threads == 768)
        k_ensemble<768><<<e->n_real, 768, e->smem, e->ctx->stream>>>(a);
    else if (e->threads == 512)
        k_ensemble<512><<<e->n_real, 512, e->smem, e->ctx->stream>>>(a);
    else
        k_ensemble<ENS_THREADS><<<e->n_real, ENS_THREADS, e->smem, e->ctx->stream>>>(a);
    CS_LAUNCH_CHECK();
    e->ctx->launches += 1;
    e->steps_done += k;
    return CS_OK;
}

int ens_reset_status(cs_ens *e) {
    std::vector<DevStatus> init((size_t)e->n_real);
    for (auto &d : init) {
        d = DevStatus{};
        d.key = ~0ULL;
        d.step = -1;
    }
    CS_CUDA(cudaMemcpyAsync(e->status.p, init.data(), sizeof(DevStatus) * init.size(),
                            cudaMemcpyHostToDevice, e->ctx->stream));
    CS_CUDA(cudaStreamSynchronize(e->ctx->stream));
    e->steps_done = 0;
    return CS_OK;
}

int ens_observe(cs_ens *e, const cs_ens_state *s, int64_t *n_alpha, double *msd) {
    k_ens_observe<<<e->n_real, 256, sizeof(double) * (size_t)e->a.n, e->ctx->stream>>>(
        s->pos, s->anchor, s->type, e->a.n, reinterpret_cast<long long *>(n_alpha), msd);
    CS_LAUNCH_CHECK();
    e->ctx->launches += 1;
    return CS_OK;
}

int ens_status(cs_ens *e, cs_status *out) {
    std::vector<DevStatus> d((size_t)e->n_real);
    CS_CUDA(cudaMemcpyAsync(d.data(), e->status.p, sizeof(DevStatus) * d.size(),
                            cudaMemcpyDeviceToHost, e->ctx->stream));
    CS_CUDA(cudaStreamSynchronize(e->ctx->stream));
    for (int r = 0; r < e->n_real; r++) {
        cs_status &o = out[r];
        const DevStatus &x = d[(size_t)r];
        o = cs_status{};
        o.code = CS_OK;
        o.step = -1;
        o.particle = -1;
        o.axis = -1;
        if (x.key != ~0ULL) {
            const int rank = (int)(x.key >> 60);
            o.code = (int)(x.key & 7ULL);
            o.particle = (long long)((x.key >> 3) & ((1ULL << 57) - 1));
            o.axis = rank >= 1 ? rank - 1 : 0;
            o.step = x.step;
            if (o.code == CS_FIELD_NONFINITE) {
                o.particle = -1;
                o.axis = -1;
            }
        }
        o.clamped = x.clamped;
        o.neg_mass_steps = x.neg_steps;
        o.first_neg_mass = x.first_neg;
        o.steps_done = e->steps_done;
        o.react_high_count = (int64_t)x.react_high_n;
        o.react_high_max = 0.0;
        if (x.react_high_n) memcpy(&o.react_high_max, &x.react_high_bits, sizeof(double));
    }
    return CS_OK;
}

}  // namespace cs

extern "C" {

int cs_ens_create(cs_ctx *ctx, const cs_sim_params *p, int32_t n_real, cs_ens **out) {
    const int rc = cs::ens_create(ctx, p, n_real, out);
    if (rc != CS_OK) {
        cs::ens_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

int cs_ens_destroy(cs_ens *e) {
    cs::ens_destroy(e);
    return CS_OK;
}

int cs_ens_step(cs_ens *e, const cs_ens_state *st, const double *xi, const double *u,
                int32_t k_steps) {
    return cs::ens_step(e, st, xi, u, k_steps);
}

int cs_ens_status(cs_ens *e, cs_status *out) { return cs::ens_status(e, out); }

int cs_ens_observe(cs_ens *e, const cs_ens_state *st, int64_t *n_alpha, double *msd) {
    return cs::ens_observe(e, st, n_alpha, msd);
}

}  // extern "C"
