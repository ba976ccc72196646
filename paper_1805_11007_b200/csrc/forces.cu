// forces.cu -- soft pair forces over the cell list.
//
// Reference: motion.py:200-245 (_soft_forces_fused pair loop).  Per
// particle i, the ring o1 in {-1,0,1} (y) is the outer loop and o0 the inner
// one, with the periodic de-duplication for 1- and 2-cell axes
// (motion.py:209-212, :219-222) and range checks on reflecting axes; within
// a cell j runs in ascending index; j == i is skipped; the displacement is
// minimum-imaged with round-half-even (rint); pairs with r2 > cut2 or
// r2 == 0 are skipped; otherwise f += -(exp(-r/eps) / (eps r)) * dx.
//
// Every floating-point operation is an explicitly rounded binary64 op in
// the reference order and exp is the glibc restatement (glibc_exp.h), so
// the force on each particle is bit-identical to the reference's.  fp32
// storage is widened to binary64 on load (the fp32 variants compute on the
// stored binary32 values exactly as the fp64 oracle would).
//
// One lane per sorted slot: consecutive lanes handle particles of the
// same/adjacent cells, so neighbour reads are shared through L1/L2.
#include "common.cuh"

namespace cs {

// Direct-engine pair forces, warp-compacted.  Lane = owner particle (slot
// t of the cell order).  The lane's ring is flattened into one candidate
// sequence in the reference order (o1 outer, o0 inner with the periodic
// de-duplication, ascending index in a cell) and the warp walks it with a
// uniform trip count; an accepted pair stores (dx0, dx1, r2, pair type) in the
// lane's shared-memory buffer.  Whenever a lane's buffer is full (and at the
// end), the warp evaluates all buffered pairs together, one per lane (the
// binary64 sqrt / exp / divisions run on full warps instead of on the ~20 %
// of lanes that accept in a given step), and each owner then adds its terms
// in buffer order = candidate order.  Same arithmetic as pair_loop: bitwise
// equal to the reference.  The minimum image skips the division when
// |dx| <= L/2 (then rint(dx / L) = +-0 and dx - L * (+-0) == dx).
constexpr int DF_WARPS = 4;
constexpr int DF_BUF = 8;

struct DfBuf {
    double dx[32 * DF_BUF], dy[32 * DF_BUF], r2[32 * DF_BUF];
    unsigned char tt[32 * DF_BUF];
    int base[33];
};

__device__ __forceinline__ double df_min_image(double dx, double size) {
    if (fabs(dx) <= 0.5 * size) return dx;
    return dsub(dx, dmul(size, rint(ddiv(dx, size))));
}

// evaluate every buffered pair of the warp, then each owner adds its terms
__device__ __forceinline__ void df_flush(DfBuf &B, const PairTab &pt, int lane, int &pend,
                                         double &fx, double &fy) {
    // exclusive prefix of the lanes' counts
    int inc = pend;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    B.base[lane] = inc - pend;
    if (lane == 31) B.base[32] = inc;
    __syncwarp();
    const int total = B.base[32];
    for (int e = lane; e < total; e += 32) {
        int lo = 0, hi = 31;  // owner: the last lane with base <= e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (B.base[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        const int q = lo * DF_BUF + (e - B.base[lo]);
        const double r2 = B.r2[q];
        const double eps = pt.eps[B.tt[q]];
        const double r = dsqrt(r2);
        const double sc = -ddiv(cs_exp(-ddiv(r, eps)), dmul(eps, r));
        B.dx[q] = dmul(sc, B.dx[q]);
        B.dy[q] = dmul(sc, B.dy[q]);
    }
    __syncwarp();
    for (int u = 0; u < pend; u++) {
        fx = dadd(fx, B.dx[lane * DF_BUF + u]);
        fy = dadd(fy, B.dy[lane * DF_BUF + u]);
    }
    pend = 0;
    __syncwarp();
}

template <class P>
__global__ void __launch_bounds__(32 * DF_WARPS)
k_soft_forces(const P *__restrict__ pos, const uint8_t *__restrict__ type,
              const int *__restrict__ order, const int *__restrict__ starts, long long n,
              BinGeom g, PairTab pt, double *__restrict__ out, const DevStatus *st,
              const P *__restrict__ spos, const uint8_t *__restrict__ stype) {
    if (st && st->abort) return;
    __shared__ DfBuf bufs[DF_WARPS];
    DfBuf &B = bufs[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const long long wstride = (long long)gridDim.x * blockDim.x;
    for (long long base = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); base < n;
         base += wstride) {
        const long long t = base + lane;
        const bool live = t < n;
        int i = 0, ti = 0, cx = 0, cy = 0, tot = 0;
        double xi = 0.0, yi = 0.0;
        // the lane's valid ring cells in reference order, as (start, end)
        int cs_[9], ce_[9], nc = 0;
        if (live) {
            i = order[t];
            load2(pos, i, xi, yi);
            cx = cell_axis(xi, g.lo0, g.eff0, g.n0);
            cy = cell_axis(yi, g.lo1, g.eff1, g.n1);
            ti = type ? (int)type[i] : 0;
#pragma unroll
            for (int c9 = 0; c9 < 9; c9++) {
                const int o1 = c9 / 3 - 1, o0 = c9 % 3 - 1;
                int g1 = cy + o1, g0 = cx + o0;
                bool ok = true;
                if (g.per1) {
                    if ((g.n1 == 1 && o1 != 0) || (g.n1 == 2 && o1 == 1)) ok = false;
                    g1 = g1 < 0 ? g1 + g.n1 : (g1 >= g.n1 ? g1 - g.n1 : g1);
                } else if (g1 < 0 || g1 >= g.n1) {
                    ok = false;
                }
                if (g.per0) {
                    if ((g.n0 == 1 && o0 != 0) || (g.n0 == 2 && o0 == 1)) ok = false;
                    g0 = g0 < 0 ? g0 + g.n0 : (g0 >= g.n0 ? g0 - g.n0 : g0);
                } else if (g0 < 0 || g0 >= g.n0) {
                    ok = false;
                }
                cs_[c9] = 0;
                ce_[c9] = 0;
                if (ok) {
                    const int f = g1 * g.n0 + g0;
                    cs_[c9] = starts[f];
                    ce_[c9] = starts[f + 1];
                    tot += ce_[c9] - cs_[c9];
                }
            }
        }
        (void)nc;
        const int totmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)tot);
        double fx = 0.0, fy = 0.0;
        int pend = 0;
        int c9 = 0, k = cs_[0], kend = ce_[0];
#pragma unroll 1
        for (int jj = 0; jj < totmax; jj++) {
            bool acc = false;
            if (jj < tot) {
                while (k == kend) {  // next non-empty ring cell
                    c9++;
                    k = c9 == 1 ? cs_[1] : c9 == 2 ? cs_[2] : c9 == 3 ? cs_[3] : c9 == 4 ? cs_[4]
                      : c9 == 5 ? cs_[5] : c9 == 6 ? cs_[6] : c9 == 7 ? cs_[7] : cs_[8];
                    kend = c9 == 1 ? ce_[1] : c9 == 2 ? ce_[2] : c9 == 3 ? ce_[3] : c9 == 4 ? ce_[4]
                         : c9 == 5 ? ce_[5] : c9 == 6 ? ce_[6] : c9 == 7 ? ce_[7] : ce_[8];
                }
                const int kk = k++;  // slot of the candidate (cell order, ascending id in a cell)
                if (kk != (int)t) {
                    double xj, yj;
                    load2(spos, kk, xj, yj);  // positions copied into slot order
                    double dx0 = dsub(xj, xi);
                    double dx1 = dsub(yj, yi);
                    if (g.per0) dx0 = df_min_image(dx0, g.size0);
                    if (g.per1) dx1 = df_min_image(dx1, g.size1);
                    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                    const int tt = ti * 2 + (stype ? (int)stype[kk] : 0);
                    if (!(r2 > pt.cut2[tt] || r2 == 0.0)) {
                        const int q = lane * DF_BUF + pend;
                        B.dx[q] = dx0;
                        B.dy[q] = dx1;
                        B.r2[q] = r2;
                        B.tt[q] = (unsigned char)tt;
                        pend++;
                        acc = true;
                    }
                }
            }
            (void)acc;
            if (__any_sync(0xffffffffu, pend == DF_BUF)) df_flush(B, pt, lane, pend, fx, fy);
        }
        if (__any_sync(0xffffffffu, pend > 0)) df_flush(B, pt, lane, pend, fx, fy);
        if (live) reinterpret_cast<double2 *>(out)[i] = make_double2(fx, fy);
    }
}

// Dense rings (cfg2: ~360 candidates and ~75 accepted pairs per owner).  A
// lane per owner leaves a 10^5-particle system with 3125 warps, ~5 per
// scheduler, and every trip is one dependent load -> distance -> test chain
// (ncu: no eligible warp 53 % of the cycles, 8 % of the FP64 roof).  Here a
// WARP owns a particle: the lanes test 32 consecutive candidates of the
// flattened ring at a time (coalesced reads of the cell-ordered copies),
// accepted pairs are appended to the warp's queue in candidate order
// (ballot / popc), the queue is evaluated one pair per lane, and lanes 0 / 1
// add the x / y terms in queue order = candidate order = the reference's.
// Same arithmetic as k_soft_forces, term for term: bitwise equal results.
constexpr int WF_WARPS = 8;
constexpr int WF_Q = 192;

struct WfBuf {
    double dx[WF_Q], dy[WF_Q], r2[WF_Q];
    unsigned char tt[WF_Q];
};

template <class P>
__global__ void __launch_bounds__(32 * WF_WARPS)
k_soft_forces_warp(const int *__restrict__ order, const int *__restrict__ starts, long long n,
                   BinGeom g, PairTab pt, double *__restrict__ out, const DevStatus *st,
                   const P *__restrict__ spos, const uint8_t *__restrict__ stype) {
    if (st && st->abort) return;
    __shared__ WfBuf bufs[WF_WARPS];
    WfBuf &B = bufs[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long wstride = (long long)gridDim.x * WF_WARPS;
    for (long long t = blockIdx.x * (long long)WF_WARPS + (threadIdx.x >> 5); t < n; t += wstride) {
        double xi, yi;
        load2(spos, t, xi, yi);
        const int ti = stype ? (int)stype[t] : 0;
        const int cx = cell_axis(xi, g.lo0, g.eff0, g.n0);
        const int cy = cell_axis(yi, g.lo1, g.eff1, g.n1);
        double fsum = 0.0;  // lane 0: the x sum, lane 1: the y sum
        int nq = 0;
        auto flush = [&]() {
            __syncwarp();
            for (int e = lane; e < nq; e += 32) {
                const double eps = pt.eps[B.tt[e]];
                const double r = dsqrt(B.r2[e]);
                const double sc = -ddiv(cs_exp(-ddiv(r, eps)), dmul(eps, r));
                B.dx[e] = dmul(sc, B.dx[e]);
                B.dy[e] = dmul(sc, B.dy[e]);
            }
            __syncwarp();
            if (lane < 2) {
                const double *src = lane ? B.dy : B.dx;
                for (int e = 0; e < nq; e++) fsum = dadd(fsum, src[e]);
            }
            __syncwarp();
            nq = 0;
        };
        // the slots [s, e) of consecutive ring cells, 64 candidates per trip:
        // both groups' position loads are in flight before either distance
        // test (a trip is otherwise one dependent load -> subtract -> test chain)
        auto segment = [&](int s, int e) {
            for (int k0 = s; k0 < e; k0 += 64) {
                if (nq + 64 > WF_Q) flush();
                int slot[2];
                bool live2[2];
                double xj[2], yj[2];
                int tj[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int k = k0 + 32 * h + lane;
                    live2[h] = k < e;
                    slot[h] = live2[h] ? k : (int)t;  // idle lanes re-read the owner
                    load2(spos, slot[h], xj[h], yj[h]);
                    tj[h] = stype ? (int)stype[slot[h]] : 0;
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    double dx0 = dsub(xj[h], xi);
                    double dx1 = dsub(yj[h], yi);
                    if (g.per0) dx0 = df_min_image(dx0, g.size0);
                    if (g.per1) dx1 = df_min_image(dx1, g.size1);
                    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                    const int tt = ti * 2 + tj[h];
                    const bool acc =
                        live2[h] && slot[h] != (int)t && !(r2 > pt.cut2[tt] || r2 == 0.0);
                    const unsigned msk = __ballot_sync(0xffffffffu, acc);
                    if (acc) {
                        const int q = nq + __popc(msk & lt);
                        B.dx[q] = dx0;
                        B.dy[q] = dx1;
                        B.r2[q] = r2;
                        B.tt[q] = (unsigned char)tt;
                    }
                    nq += __popc(msk);
                }
            }
        };
        // ring rows in reference order (o1 outer; the periodic de-duplication
        // and wall skips of motion.py:206-222).  The cells of a ring row are
        // consecutive in the cell table unless the row wraps around a periodic
        // x axis: then one slot range per row, else cell by cell (o0 inner).
        const bool xrow = !g.per0 || (g.n0 >= 3 && cx >= 1 && cx + 1 < g.n0);
        const int c0 = cx >= 1 ? cx - 1 : 0, c1 = cx + 1 < g.n0 ? cx + 1 : g.n0 - 1;
        for (int o1 = -1; o1 <= 1; o1++) {
            int g1 = cy + o1;
            if (g.per1) {
                if ((g.n1 == 1 && o1 != 0) || (g.n1 == 2 && o1 == 1)) continue;
                g1 = g1 < 0 ? g1 + g.n1 : (g1 >= g.n1 ? g1 - g.n1 : g1);
            } else if (g1 < 0 || g1 >= g.n1) {
                continue;
            }
            if (xrow) {
                segment(starts[g1 * g.n0 + c0], starts[g1 * g.n0 + c1 + 1]);
                continue;
            }
            for (int o0 = -1; o0 <= 1; o0++) {
                int g0 = cx + o0;
                if ((g.n0 == 1 && o0 != 0) || (g.n0 == 2 && o0 == 1)) continue;
                g0 = g0 < 0 ? g0 + g.n0 : (g0 >= g.n0 ? g0 - g.n0 : g0);
                const int f = g1 * g.n0 + g0;
                segment(starts[f], starts[f + 1]);
            }
        }
        flush();
        const double fx = __shfl_sync(0xffffffffu, fsum, 0);
        const double fy = __shfl_sync(0xffffffffu, fsum, 1);
        if (lane == 0) reinterpret_cast<double2 *>(out)[order[t]] = make_double2(fx, fy);
    }
}

// the reference pair loop of one particle, summed (the rare fallback)
template <class P>
__device__ __noinline__ double2 pair_loop_sum(const P *__restrict__ pos,
                                              const uint8_t *__restrict__ type,
                                              const int *__restrict__ order,
                                              const int *__restrict__ starts, BinGeom g,
                                              PairTab pt, int i) {
    double fx = 0.0, fy = 0.0;
    pair_loop(pos, type, order, starts, g, pt, i, [&](int, double s, double dx0, double dx1) {
        fx = dadd(fx, dmul(s, dx0));
        fy = dadd(fy, dmul(s, dx1));
    });
    return make_double2(fx, fy);
}

// Small systems (cfg1: 10^4 particles) are latency-bound in k_soft_forces:
// ~80 blocks, one lane per owner walking ~17 candidates in series.  Here
// nine lanes share an owner, lane c9 walking ring cell c9 (three owners per
// warp) and buffering its accepted pairs; the warp then evaluates all
// buffered pair terms together, one per lane, and the owner's first lane
// adds them cell by cell: candidate order, bitwise equal to k_soft_forces.
// A cell with more than RING_K accepted pairs sends the owner through
// pair_loop.
constexpr int RING_K = 6;
constexpr int RING_WARPS = 4;
constexpr long long RING_MAX_N = 1 << 16;

struct RingBuf {
    double dx[27 * RING_K], dy[27 * RING_K], r2[27 * RING_K];  // lane-major: lane * RING_K + u
    unsigned char tt[27 * RING_K];
    unsigned char nt[32];
    short base[33];  // exclusive prefix of nt over the lanes
};

template <class P>
__global__ void __launch_bounds__(32 * RING_WARPS)
k_soft_forces_ring(const int *__restrict__ order, const int *__restrict__ starts, long long n,
                   BinGeom g, PairTab pt, double *__restrict__ out, const DevStatus *st,
                   const P *__restrict__ spos, const uint8_t *__restrict__ stype,
                   const P *__restrict__ pos, const uint8_t *__restrict__ type) {
    if (st && st->abort) return;
    __shared__ RingBuf bufs[RING_WARPS];
    RingBuf &B = bufs[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int grp = lane / 9, c9 = lane - 9 * grp;  // grp 3: lanes 27-31, idle
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; 3 * w < n;
         w += warps) {
        const long long t = 3 * w + grp;
        const bool live = grp < 3 && t < n;
        int nt = 0;
        bool over = false;
        if (live) {
            double xi, yi;
            load2(spos, t, xi, yi);
            const int ti = stype ? (int)stype[t] : 0;
            const int cx = cell_axis(xi, g.lo0, g.eff0, g.n0);
            const int cy = cell_axis(yi, g.lo1, g.eff1, g.n1);
            const int o1 = c9 / 3 - 1, o0 = c9 % 3 - 1;
            int g1 = cy + o1, g0 = cx + o0;
            bool ok = true;
            if (g.per1) {
                if ((g.n1 == 1 && o1 != 0) || (g.n1 == 2 && o1 == 1)) ok = false;
                g1 = g1 < 0 ? g1 + g.n1 : (g1 >= g.n1 ? g1 - g.n1 : g1);
            } else if (g1 < 0 || g1 >= g.n1) {
                ok = false;
            }
            if (g.per0) {
                if ((g.n0 == 1 && o0 != 0) || (g.n0 == 2 && o0 == 1)) ok = false;
                g0 = g0 < 0 ? g0 + g.n0 : (g0 >= g.n0 ? g0 - g.n0 : g0);
            } else if (g0 < 0 || g0 >= g.n0) {
                ok = false;
            }
            if (ok) {
                const int f = g1 * g.n0 + g0;
                const int kb = starts[f], ke = starts[f + 1];
                for (int k = kb; k < ke; k++) {
                    if (k == (int)t) continue;
                    double xj, yj;
                    load2(spos, k, xj, yj);
                    double dx0 = dsub(xj, xi);
                    double dx1 = dsub(yj, yi);
                    if (g.per0) dx0 = df_min_image(dx0, g.size0);
                    if (g.per1) dx1 = df_min_image(dx1, g.size1);
                    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                    const int tt = ti * 2 + (stype ? (int)stype[k] : 0);
                    if (r2 > pt.cut2[tt] || r2 == 0.0) continue;
                    if (nt == RING_K) {
                        over = true;
                        break;
                    }
                    const int q = lane * RING_K + nt;
                    B.dx[q] = dx0;
                    B.dy[q] = dx1;
                    B.r2[q] = r2;
                    B.tt[q] = (unsigned char)tt;
                    nt++;
                }
            }
        }
        // exclusive prefix of the lanes' counts; the pairs are then evaluated
        // one per lane (term written back over the lane's dx / dy slot)
        int inc = nt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        B.nt[lane] = (unsigned char)nt;
        B.base[lane] = (short)(inc - nt);
        if (lane == 31) B.base[32] = (short)inc;
        __syncwarp();
        const int total = B.base[32];
        for (int e = lane; e < total; e += 32) {
            int lo = 0, hi = 26;  // the last lane with base <= e
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (B.base[mid] <= e) lo = mid;
                else hi = mid - 1;
            }
            const int q = lo * RING_K + (e - B.base[lo]);
            const double r2 = B.r2[q];
            const double eps = pt.eps[B.tt[q]];
            const double r = dsqrt(r2);
            const double sc = -ddiv(cs_exp(-ddiv(r, eps)), dmul(eps, r));
            B.dx[q] = dmul(sc, B.dx[q]);
            B.dy[q] = dmul(sc, B.dy[q]);
        }
        const unsigned gmask = grp < 3 ? 0x1ffu << (9 * grp) : 0u;
        const bool gover = (__ballot_sync(0xffffffffu, over) & gmask) != 0;
        __syncwarp();
        if (live && c9 == 0) {
            const int i = order[t];
            double fx = 0.0, fy = 0.0;
            if (gover) {
                const double2 f = pair_loop_sum(pos, type, order, starts, g, pt, i);
                fx = f.x;
                fy = f.y;
            } else {
                for (int c = 0; c < 9; c++) {
                    const int m = B.nt[lane + c];
                    for (int u = 0; u < m; u++) {
                        fx = dadd(fx, B.dx[(lane + c) * RING_K + u]);
                        fy = dadd(fy, B.dy[(lane + c) * RING_K + u]);
                    }
                }
            }
            reinterpret_cast<double2 *>(out)[i] = make_double2(fx, fy);
        }
        __syncwarp();
    }
}

template <class P>
__global__ void k_count_pairs(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                              const int *__restrict__ order, const int *__restrict__ starts,
                              long long n, BinGeom g, PairTab pt, int *__restrict__ cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int c = 0;
        pair_loop(pos, type, order, starts, g, pt, (int)i,
                  [&](int, double, double, double) { c++; });
        cnt[i] = c;
    }
}

template <class P>
__global__ void k_fill_pairs(const P *__restrict__ pos, const uint8_t *__restrict__ type,
                             const int *__restrict__ order, const int *__restrict__ starts,
                             long long n, BinGeom g, PairTab pt, const int *__restrict__ off,
                             int64_t *__restrict__ pairs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        long long w = off[i];
        pair_loop(pos, type, order, starts, g, pt, (int)i,
                  [&](int j, double, double, double) {
                      pairs[2 * w] = i;
                      pairs[2 * w + 1] = j;
                      w++;
                  });
    }
}

// ---------------------------------------------------------------- CellIndex
// cell_xy of every particle (spatial_index.py:113-115: floor((p - lo) / eff),
// clipped to the closed upper edge) -- the binning bins.cu does, exported
template <class P>
__global__ void k_cell_xy(const P *__restrict__ pos, long long n, BinGeom g, int *__restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x, y;
        load2(pos, i, x, y);
        out[2 * i] = cell_axis(x, g.lo0, g.eff0, g.n0);
        out[2 * i + 1] = cell_axis(y, g.lo1, g.eff1, g.n1);
    }
}

// accumulate_forces / _soft_forces (motion.py:107-143): per particle, the
// axis cells of _axis_cells (motion.py:91-104) -- reach r = ceil(cutoff /
// eff); a periodic axis with 2 r + 1 >= n is visited once, 0 .. n-1;
// otherwise centre - r .. centre + r, wrapped (periodic) or clipped -- y
// outer, x inner, members in index order; reference arithmetic throughout.
template <class P>
__global__ void k_index_forces(const P *__restrict__ pos, long long n, const int *__restrict__ cxy,
                               const int *__restrict__ order, const int *__restrict__ starts,
                               int ncx, int ncy, double effx, double effy, int perx, int pery,
                               double lx, double ly, double eps, double cutoff,
                               double *__restrict__ out) {
    const double cut2 = dmul(cutoff, cutoff);
    const int rx = (int)ceil(ddiv(cutoff, effx)), ry = (int)ceil(ddiv(cutoff, effy));
    const bool allx = perx && 2 * rx + 1 >= ncx, ally = pery && 2 * ry + 1 >= ncy;
    const int nx_it = allx ? ncx : 2 * rx + 1, ny_it = ally ? ncy : 2 * ry + 1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double xi, yi;
        load2(pos, i, xi, yi);
        const int cxi = cxy[2 * i], cyi = cxy[2 * i + 1];
        double fx = 0.0, fy = 0.0;
        for (int a = 0; a < ny_it; a++) {
            int gy = a;
            if (!ally) {
                gy = cyi - ry + a;
                if (pery) gy = (int)pymod(gy, ncy);
                else if (gy < 0 || gy >= ncy) continue;
            }
            for (int b = 0; b < nx_it; b++) {
                int gx = b;
                if (!allx) {
                    gx = cxi - rx + b;
                    if (perx) gx = (int)pymod(gx, ncx);
                    else if (gx < 0 || gx >= ncx) continue;
                }
                const int f = gy * ncx + gx;
                for (int k = starts[f]; k < starts[f + 1]; k++) {
                    const int j = order[k];
                    if (j == i) continue;
                    double xj, yj;
                    load2(pos, j, xj, yj);
                    double dx0 = dsub(xj, xi), dx1 = dsub(yj, yi);
                    if (perx) dx0 = dsub(dx0, dmul(lx, rint(ddiv(dx0, lx))));
                    if (pery) dx1 = dsub(dx1, dmul(ly, rint(ddiv(dx1, ly))));
                    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
                    if (r2 > cut2 || r2 == 0.0) continue;
                    const double r = dsqrt(r2);
                    const double sc = -ddiv(cs_exp(-ddiv(r, eps)), dmul(eps, r));
                    fx = dadd(fx, dmul(sc, dx0));
                    fy = dadd(fy, dmul(sc, dx1));
                }
            }
        }
        reinterpret_cast<double2 *>(out)[i] = make_double2(fx, fy);
    }
}

int launch_cell_xy(cs_ctx *ctx, int prec, const void *pos, long long n, const BinGeom &g,
                   int *out) {
    if (n == 0) return CS_OK;
    if (prec == CS_F64)
        k_cell_xy<double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const double *>(pos), n, g, out);
    else
        k_cell_xy<float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            static_cast<const float *>(pos), n, g, out);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int launch_index_forces(cs_ctx *ctx, int prec, const void *pos, long long n, const int *cxy,
                        const int *order, const int *starts, int ncx, int ncy, double effx,
                        double effy, int perx, int pery, double lx, double ly, double eps,
                        double cutoff, double *out) {
    if (n == 0) return CS_OK;
    if (prec == CS_F64)
        k_index_forces<double><<<grid_for(n, 128), 128, 0, ctx->stream>>>(
            static_cast<const double *>(pos), n, cxy, order, starts, ncx, ncy, effx, effy, perx,
            pery, lx, ly, eps, cutoff, out);
    else
        k_index_forces<float><<<grid_for(n, 128), 128, 0, ctx->stream>>>(
            static_cast<const float *>(pos), n, cxy, order, starts, ncx, ncy, effx, effy, perx,
            pery, lx, ly, eps, cutoff, out);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int launch_soft_forces(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                       long long n, const BinGeom &g, const PairTab &pt, double *out,
                       const DevStatus *st) {
    if (n == 0) return CS_OK;
    const int B = 32 * DF_WARPS;
    const int *order = ctx->order.as<int>(), *starts = ctx->starts.as<int>();
    // bin_particles left the positions (and types) in cell order in ctx->spos / stype
    uint8_t *stype = type ? ctx->stype.as<uint8_t>() : nullptr;
    // dense rings (>= 48 candidates per owner on average): a warp per owner
    // (CS_WARP_FORCES=0/1 overrides, read per call: tests run every kernel on the same inputs)
    const char *we = getenv("CS_WARP_FORCES");
    const double cand = 9.0 * (double)n / ((double)g.n0 * (double)g.n1);
    if (we ? atoi(we) != 0 : cand >= 48.0) {
        const int blocks = grid_for(n, WF_WARPS, 148 * 64);
        if (prec == CS_F64)
            k_soft_forces_warp<double><<<blocks, 32 * WF_WARPS, 0, ctx->stream>>>(
                order, starts, n, g, pt, out, st, ctx->spos.as<double>(), stype);
        else
            k_soft_forces_warp<float><<<blocks, 32 * WF_WARPS, 0, ctx->stream>>>(
                order, starts, n, g, pt, out, st, ctx->spos.as<float>(), stype);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
        return CS_OK;
    }
    static const int ring_env = getenv("CS_RING_FORCES") ? atoi(getenv("CS_RING_FORCES")) : -1;
    const bool ring = ring_env >= 0 ? ring_env != 0 : n <= RING_MAX_N;
    if (ring) {
        const long long warps = (n + 2) / 3;
        const int blocks = (int)((warps + RING_WARPS - 1) / RING_WARPS);
        if (prec == CS_F64)
            k_soft_forces_ring<double><<<blocks, 32 * RING_WARPS, 0, ctx->stream>>>(
                order, starts, n, g, pt, out, st, ctx->spos.as<double>(), stype,
                static_cast<const double *>(pos), type);
        else
            k_soft_forces_ring<float><<<blocks, 32 * RING_WARPS, 0, ctx->stream>>>(
                order, starts, n, g, pt, out, st, ctx->spos.as<float>(), stype,
                static_cast<const float *>(pos), type);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
        return CS_OK;
    }
    if (prec == CS_F64)
        k_soft_forces<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const double *>(pos), type, order, starts, n, g, pt, out, st,
            ctx->spos.as<double>(), stype);
    else
        k_soft_forces<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const float *>(pos), type, order, starts, n, g, pt, out, st,
            ctx->spos.as<float>(), stype);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int run_soft_force_pairs(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type,
                         long long n, const BinGeom &g, const PairTab &pt, int64_t *pairs,
                         int64_t cap, int64_t *count) {
    const int B = 256;
    CS_TRY(ctx->pair_counts.ensure(sizeof(int) * (size_t)(n + 1)));
    CS_TRY(ctx->pair_offsets.ensure(sizeof(int) * (size_t)(n + 1)));
    int *cnt = ctx->pair_counts.as<int>(), *off = ctx->pair_offsets.as<int>();
    const int *order = ctx->order.as<int>(), *starts = ctx->starts.as<int>();
    if (n > 0) {
        if (prec == CS_F64)
            k_count_pairs<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const double *>(pos), type, order, starts, n, g, pt, cnt);
        else
            k_count_pairs<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
                static_cast<const float *>(pos), type, order, starts, n, g, pt, cnt);
        CS_LAUNCH_CHECK();
    }
    CS_TRY(exclusive_scan_i32(ctx, cnt, off, n));
    int total = 0;
    CS_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *count = total;
    if (total > cap || n == 0 || pairs == nullptr) return CS_OK;
    if (prec == CS_F64)
        k_fill_pairs<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const double *>(pos), type, order, starts, n, g, pt, off, pairs);
    else
        k_fill_pairs<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
            static_cast<const float *>(pos), type, order, starts, n, g, pt, off, pairs);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

}  // namespace cs
