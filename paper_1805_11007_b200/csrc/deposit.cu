// deposit.cu -- nodal number densities in the reference's summation order.
//
// References (chemosim/):
//   CIC        coupling.py:113-138  four np.bincount passes (corners 00, 10,
//              01, 11), each summing its weights in ascending particle
//              index, added to the zeroed grid one pass after the other
//   gaussian   coupling.py:45-110   one serial sweep in particle order; each
//              particle adds its stamp node by node (no node twice: a
//              periodic stamp wider than the grid is rejected, :156-157)
// So every node value is a fixed sequence of binary64 adds.  Reproducing it
// needs each node's contributions in ascending particle index -- a gather,
// not a scatter with atomics (whose order changes from run to run):
//   k_dep_keys    deposit bin of each depositing particle (CIC: its base
//                 cell, gaussian: its nearest node) and per-bin counts
//   scan          bin starts
//   k_dep_scatter unordered placement into the bin ranges (counts -> 0)
//   k_dep_rank    stable placement: bin start + the number of the bin's
//                 particles with a smaller index; the positions and
//                 (index, route) words copied into bin order
//   k_dep_gather_cic / _gauss   one thread per node: CIC sums corner q of
//                 the one bin that owns it, q = 0..3, then adds the four
//                 partial sums in the reference's order; gaussian collects
//                 the stamps of the bins in its window, orders them by
//                 particle index (batches of DEP_BUF) and adds them in that
//                 order.
// The result is bit-identical to the reference and run-to-run
// deterministic.  Binary32 grids (fp32 mode) sum in binary64 in the same
// order and round once.
#include <math.h>

#include "deposit.cuh"

namespace cs {

template <class P>
__global__ void k_dep_keys(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                           long long n, GridGeom gg, int kind, Route route,
                           int *__restrict__ keys, int *__restrict__ counts,
                           const DevStatus *st) {
    if (st && st->abort) return;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        int key = -1;
        if (route_bits(type, p, route)) {
            double x, y;
            load2(pos, p, x, y);
            const double u0 = ddiv(dsub(x, gg.lo0), gg.d0);
            const double u1 = ddiv(dsub(y, gg.lo1), gg.d1);
            if (fabs(u0) < 0x1p52 && fabs(u1) < 0x1p52) {  // also false for NaN
                key = dep_bin_axis(u1, kind, gg.n, gg.per) * gg.n +
                      dep_bin_axis(u0, kind, gg.n, gg.per);
                atomicAdd(&counts[key], 1);
            }
        }
        keys[p] = key;
    }
}

__global__ void k_dep_scatter(const int *__restrict__ keys, long long n,
                              const int *__restrict__ starts, int *__restrict__ counts,
                              int *__restrict__ slots, const DevStatus *st) {
    if (st && st->abort) return;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const int key = keys[p];
        if (key < 0) continue;
        slots[starts[key] + atomicSub(&counts[key], 1) - 1] = (int)p;
    }
}

template <class P>
__global__ void k_dep_rank(const int *__restrict__ slots, const int *__restrict__ keys,
                           const int *__restrict__ starts, int nb, const P *__restrict__ pos,
                           const uint8_t *__restrict__ type, Route route, P *__restrict__ spos,
                           unsigned *__restrict__ meta, const DevStatus *st) {
    if (st && st->abort) return;
    const long long total = starts[nb];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = slots[t];
        const int key = keys[v];
        const int s = starts[key], e = starts[key + 1];
        int rank = 0;
        for (int u = s; u < e; u++) rank += __ldg(slots + u) < v;
        reinterpret_cast<typename Vec2<P>::T *>(spos)[s + rank] =
            reinterpret_cast<const typename Vec2<P>::T *>(pos)[v];
        meta[s + rank] = (unsigned)v | (route_bits(type, v, route) << 30);
    }
}

template <class P, class G>
__global__ void __launch_bounds__(256)
k_dep_gather_cic(const int *__restrict__ starts, int off, const P *__restrict__ spos,
                 const unsigned *__restrict__ meta, GridGeom gg, G *__restrict__ ra,
                 G *__restrict__ rb, const DevStatus *st) {
    if (st && st->abort) return;
    const int n = gg.n;
    const long long m = (long long)n * n;
    const double unit = ddiv(1.0, dmul(gg.d0, gg.d1));
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(l / n), i = (int)(l - (long long)j * n);
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            int bx = i - (q & 1), by = j - (q >> 1);
            if (gg.per) {
                bx = bx < 0 ? bx + n : bx;
                by = by < 0 ? by + n : by;
            } else if (bx < 0 || by < 0 || bx > n - 2 || by > n - 2) {
                continue;  // the pass's bincount is 0 here; x + 0.0 == x
            }
            const int key = by * n + bx;
            double ca = 0.0, cb = 0.0;
            const int e = starts[key + 1] - off;
            for (int t = starts[key] - off; t < e; t++) {
                double x, y;
                load2(spos, t, x, y);
                const double w = cic_weight(x, y, gg, unit, q);
                const unsigned bits = meta[t] >> 30;
                if (bits & 1u) ca = dadd(ca, w);
                if (bits & 2u) cb = dadd(cb, w);
            }
            sa = dadd(sa, ca);
            sb = dadd(sb, cb);
        }
        ra[l] = (G)sa;
        rb[l] = (G)sb;
    }
}

// The same sums with four lanes per node, lane q summing corner pass q of
// its node; the node's first lane then adds the passes in order 0..3 (as
// k_dep_gather_cic): 4x the threads, a quarter of the serial chain each.
// RHS: the node's rhs of the implicit solve as well (k_rhs's arithmetic on
// the stored densities).
template <class P, class G, bool RHS>
__global__ void __launch_bounds__(128)
k_dep_gather_cic4(const int *__restrict__ starts, int off, const P *__restrict__ spos,
                  const unsigned *__restrict__ meta, GridGeom gg, G *__restrict__ ra,
                  G *__restrict__ rb, const DevStatus *st, const G *__restrict__ c,
                  RhsCoef rk, double *__restrict__ rhs) {
    if (st && st->abort) return;
    const int n = gg.n;
    const long long m4 = 4LL * n * n;
    const double unit = ddiv(1.0, dmul(gg.d0, gg.d1));
    const int lane = threadIdx.x & 31, lead = lane & ~3;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); base < m4;
         base += stride) {
        const long long g = base + lane;
        const long long l = g >> 2;
        const int q = (int)(g & 3);
        double ca = 0.0, cb = 0.0;
        bool has = false;
        if (g < m4) {
            const int j = (int)(l / n), i = (int)(l - (long long)j * n);
            int bx = i - (q & 1), by = j - (q >> 1);
            if (gg.per) {
                bx = bx < 0 ? bx + n : bx;
                by = by < 0 ? by + n : by;
                has = true;
            } else {
                has = !(bx < 0 || by < 0 || bx > n - 2 || by > n - 2);
            }
            if (has) {
                const int key = by * n + bx;
                const int e = starts[key + 1] - off;
                for (int t = starts[key] - off; t < e; t++) {
                    double x, y;
                    load2(spos, t, x, y);
                    const double w = cic_weight(x, y, gg, unit, q);
                    const unsigned bits = meta[t] >> 30;
                    if (bits & 1u) ca = dadd(ca, w);
                    if (bits & 2u) cb = dadd(cb, w);
                }
            }
        }
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const double va = __shfl_sync(0xffffffffu, ca, lead + u);
            const double vb = __shfl_sync(0xffffffffu, cb, lead + u);
            const bool h = __shfl_sync(0xffffffffu, has, lead + u);
            if (h) {  // a pass outside a reflecting grid's cells adds nothing
                sa = dadd(sa, va);
                sb = dadd(sb, vb);
            }
        }
        if (q == 0 && g < m4) {
            const G ga = (G)sa, gb = (G)sb;
            ra[l] = ga;
            rb[l] = gb;
            if (RHS) {
                const double cv = (double)c[l];
                double r = rk.has_g ? dmul(cv, rk.one_m_dtg) : cv;
                if (rk.has_a) r = dadd(r, dmul(rk.dka, (double)ga));
                if (rk.has_b) r = dsub(r, dmul(dmul((double)gb, cv), rk.dkb));
                rhs[l] = r;
            }
        }
    }
}

// Window of node (i, j): rows j-w1..j+w1, and per row the bins of columns
// i-w0..i+w0 as at most two contiguous key ranges (a periodic wrap splits it).
template <class Visit>
__device__ __forceinline__ void gauss_window(int i, int j, const GridGeom &gg,
                                             const GaussParams &gp,
                                             const int *__restrict__ starts, int off,
                                             Visit visit) {
    const int n = gg.n;
    for (int o1 = -gp.w1; o1 <= gp.w1; o1++) {
        int jj = j + o1;
        if (gg.per) jj = jj < 0 ? jj + n : (jj >= n ? jj - n : jj);
        else if (jj < 0 || jj >= n) continue;
        int a0 = i - gp.w0, a1 = i + gp.w0;
        int seg[2][2], ns = 0;
        if (gg.per) {
            if (a0 < 0) {
                seg[ns][0] = a0 + n; seg[ns][1] = n - 1; ns++;
                seg[ns][0] = 0; seg[ns][1] = a1; ns++;
            } else if (a1 >= n) {
                seg[ns][0] = a0; seg[ns][1] = n - 1; ns++;
                seg[ns][0] = 0; seg[ns][1] = a1 - n; ns++;
            } else {
                seg[ns][0] = a0; seg[ns][1] = a1; ns++;
            }
        } else {
            seg[0][0] = a0 < 0 ? 0 : a0;
            seg[0][1] = a1 > n - 1 ? n - 1 : a1;
            ns = seg[0][0] <= seg[0][1] ? 1 : 0;
        }
        for (int k = 0; k < ns; k++) {
            const int t0 = starts[jj * n + seg[k][0]] - off;
            const int t1 = starts[jj * n + seg[k][1] + 1] - off;
            for (int t = t0; t < t1; t++) visit(t);
        }
    }
}

constexpr int DEP_BUF = 48;

template <class P, class G>
__global__ void __launch_bounds__(128)
k_dep_gather_gauss(const int *__restrict__ starts, int off, const P *__restrict__ spos,
                   const unsigned *__restrict__ meta, GridGeom gg, GaussParams gp,
                   G *__restrict__ ra, G *__restrict__ rb, const DevStatus *st) {
    if (st && st->abort) return;
    const int n = gg.n;
    const long long m = (long long)n * n;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(l / n), i = (int)(l - (long long)j * n);
        // this node's stamps in batches of the DEP_BUF smallest particle
        // indices above the previous batch's, each kept sorted and summed
        unsigned key[DEP_BUF];
        double val[DEP_BUF];
        double sa = 0.0, sb = 0.0;
        long long last = -1;
        bool more = true;
        while (more) {
            int cnt = 0;
            more = false;
            gauss_window(i, j, gg, gp, starts, off, [&](int t) {
                const unsigned mk = meta[t];
                const unsigned id = mk & DEP_ID_MASK;
                if ((long long)id <= last) return;
                if (cnt == DEP_BUF && id > (key[DEP_BUF - 1] & DEP_ID_MASK)) {
                    more = true;  // beyond this batch
                    return;
                }
                double x, y, v;
                load2(spos, t, x, y);
                if (!gauss_term(x, y, i, j, gg, gp, v)) return;
                int k = cnt;
                if (cnt == DEP_BUF) {
                    more = true;  // the batch's largest index drops out
                    k = DEP_BUF - 1;
                } else {
                    cnt++;
                }
                while (k > 0 && (key[k - 1] & DEP_ID_MASK) > id) {
                    key[k] = key[k - 1];
                    val[k] = val[k - 1];
                    k--;
                }
                key[k] = mk;
                val[k] = v;
            });
            for (int k = 0; k < cnt; k++) {
                const unsigned bits = key[k] >> 30;
                if (bits & 1u) sa = dadd(sa, val[k]);
                if (bits & 2u) sb = dadd(sb, val[k]);
            }
            if (cnt) last = key[cnt - 1] & DEP_ID_MASK;
        }
        ra[l] = (G)sa;
        rb[l] = (G)sb;
    }
}

GaussParams make_gauss(const GridGeom &gg, double h, double cutoff) {
    GaussParams gp;
    gp.inv_norm = 1.0 / (2.0 * M_PI * h * h);
    gp.two_h2 = 2.0 * h * h;
    gp.cut2 = cutoff * cutoff;
    gp.w0 = (int)floor(cutoff / gg.d0 + 0.5);
    gp.w1 = (int)floor(cutoff / gg.d1 + 0.5);
    return gp;
}

bool gauss_too_wide(const GridGeom &gg, double cutoff) {
    const double dmin = gg.d0 < gg.d1 ? gg.d0 : gg.d1;
    return gg.per && ((int)floor(cutoff / dmin + 0.5)) * 2 + 1 > gg.n;
}

template <class P, class G>
static int dep_gather_t(cs_ctx *ctx, const int *starts, int off, const P *spos,
                        const unsigned *meta, const GridGeom &gg, int kind, double h,
                        double cutoff, G *ra, G *rb, const DevStatus *st,
                        const RhsFuse *rf = nullptr) {
    const long long nb = (long long)gg.n * gg.n;
    if (kind == CS_CIC) {
        if (rf)
            k_dep_gather_cic4<P, G, true><<<grid_for(4 * nb, 128), 128, 0, ctx->stream>>>(
                starts, off, spos, meta, gg, ra, rb, st, (const G *)rf->c, rf->k, rf->rhs);
        else if (getenv("CS_DEP_GATHER1"))
            k_dep_gather_cic<P, G><<<grid_for(nb, 256), 256, 0, ctx->stream>>>(
                starts, off, spos, meta, gg, ra, rb, st);
        else
            k_dep_gather_cic4<P, G, false><<<grid_for(4 * nb, 128), 128, 0, ctx->stream>>>(
                starts, off, spos, meta, gg, ra, rb, st, nullptr, RhsCoef{}, nullptr);
    } else {
        const GaussParams gp = make_gauss(gg, h, cutoff);
        k_dep_gather_gauss<P, G><<<grid_for(nb, 128), 128, 0, ctx->stream>>>(
            starts, off, spos, meta, gg, gp, ra, rb, st);
    }
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

// The gather alone, over bins built by bin_particles(..., DepBin) together
// with the cell list: the deposit bins' starts are starts[nflat ..] and
// their slots are numbered from n (off = n).
int launch_deposit_binned(cs_ctx *ctx, int prec, const GridGeom &gg, int kind, double h,
                          double cutoff, const int *starts, int off, void *ra, void *rb,
                          const DevStatus *st, const RhsFuse *rf) {
    if (prec == CS_F64)
        return dep_gather_t<double, double>(ctx, starts, off, ctx->dep_pos.as<double>(),
                                            ctx->dep_meta.as<unsigned>(), gg, kind, h, cutoff,
                                            (double *)ra, (double *)rb, st, rf);
    return dep_gather_t<float, float>(ctx, starts, off, ctx->dep_pos.as<float>(),
                                      ctx->dep_meta.as<unsigned>(), gg, kind, h, cutoff,
                                      (float *)ra, (float *)rb, st, rf);
}

template <class P, class G>
static int deposit_t(cs_ctx *ctx, const P *pos, const uint8_t *type, long long n,
                     const GridGeom &gg, int kind, double h, double cutoff, const Route &r,
                     G *ra, G *rb, const DevStatus *st) {
    const long long nb = (long long)gg.n * gg.n;
    if (kind == CS_GAUSSIAN) {
        const GaussParams gp = make_gauss(gg, h, cutoff);
        if (gp.w0 > 64 || gp.w1 > 64) {
            set_error("deposit: gaussian stamp wider than 129 nodes");
            return CS_ERR_PARAM;
        }
    }
    if (nb >= (1LL << 31) - 1 || n > (long long)DEP_ID_MASK) {
        set_error("deposit: grid or particle count too large");
        return CS_ERR_PARAM;
    }
    const size_t pn = (size_t)(n > 0 ? n : 1);
    CS_TRY(ctx->dep_keys.ensure(sizeof(int) * pn));
    CS_TRY(ctx->dep_slots.ensure(sizeof(int) * pn));
    CS_TRY(ctx->dep_meta.ensure(sizeof(unsigned) * pn));
    CS_TRY(ctx->dep_pos.ensure(2 * sizeof(P) * pn));
    CS_TRY(ctx->dep_starts.ensure(sizeof(int) * (size_t)(nb + 1)));
    if (ctx->dep_counts.bytes < sizeof(int) * (size_t)nb) {  // kept all-zero between calls
        CS_TRY(ctx->dep_counts.ensure(sizeof(int) * (size_t)nb));
        CS_CUDA(cudaMemsetAsync(ctx->dep_counts.p, 0, ctx->dep_counts.bytes, ctx->stream));
    }
    int *keys = ctx->dep_keys.as<int>(), *counts = ctx->dep_counts.as<int>();
    int *starts = ctx->dep_starts.as<int>(), *slots = ctx->dep_slots.as<int>();
    unsigned *meta = ctx->dep_meta.as<unsigned>();
    P *spos = ctx->dep_pos.as<P>();
    const int B = 256;
    if (n > 0) {
        k_dep_keys<P><<<grid_for(n, B), B, 0, ctx->stream>>>(pos, type, n, gg, kind, r, keys,
                                                             counts, st);
        CS_LAUNCH_CHECK();
    }
    CS_TRY(exclusive_scan_i32(ctx, counts, starts, nb));
    if (n > 0) {
        k_dep_scatter<<<grid_for(n, B), B, 0, ctx->stream>>>(keys, n, starts, counts, slots, st);
        CS_LAUNCH_CHECK();
        k_dep_rank<P><<<grid_for(n, B), B, 0, ctx->stream>>>(slots, keys, starts, (int)nb, pos,
                                                             type, r, spos, meta, st);
        CS_LAUNCH_CHECK();
        ctx->launches += 3;
    }
    return dep_gather_t<P, G>(ctx, starts, 0, spos, meta, gg, kind, h, cutoff, ra, rb, st);
}

int launch_deposit(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type, long long n,
                   const GridGeom &gg, int kind, double h, double cutoff,
                   const unsigned char bits[3], void *ra, void *rb, const DevStatus *st) {
    Route r;
    r.bits[0] = bits[0];
    r.bits[1] = bits[1];
    r.bits[2] = bits[2];
    if (prec == CS_F64)
        return deposit_t<double, double>(ctx, (const double *)pos, type, n, gg, kind, h, cutoff,
                                         r, (double *)ra, (double *)rb, st);
    return deposit_t<float, float>(ctx, (const float *)pos, type, n, gg, kind, h, cutoff, r,
                                   (float *)ra, (float *)rb, st);
}

}  // namespace cs
