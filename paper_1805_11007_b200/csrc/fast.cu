// fast.cu -- the large-N engine: cell-sorted particle records.
//
// The direct engine (sim.cu) keeps the reference layout (rows in id order,
// motion.py / particles.py:1-7) and reaches neighbours through `order[]`:
// every neighbour read, force write and grid sample is a random 8-32 B
// access.  This engine keeps the particles physically sorted by cell in
// 16-byte records
//     { float x, y; uint32 id | type << 31; int16 wrap_x, wrap_y }
// (the periodic anchor is start_anchor - wraps * L, exact in binary64) and
// rebuilds the order every step with one counting-sort pass, so all
// per-particle traffic is coalesced and neighbour cells are contiguous.
//
// Per step (after the field step of sim.cu):
//   k_fast_step    one thread per sorted slot: pair forces over the 3x3
//                  reference ring, bilinear drift, EM proposal with
//                  xi[id], boundaries with wrap counting, new cell key +
//                  histogram atomic, CIC deposit of the new position for
//                  the next step's field (integer atomics, deterministic)
//   k_scan         exclusive scan of the histogram -> next cell table
//   k_fast_scatter counting-sort scatter of the new records
//
// Force summation order.  Inside a cell the records are in arbitrary
// (atomic-arrival) order, so the kernel does not rely on storage order:
// per ring cell it sums the accepted pairs in ascending particle id --
// exactly the reference's order (motion.py:206-243) -- by a single pass
// when a cell contributes at most one pair (the common case) and an
// id-ordered selection pass otherwise.  The force on every particle is
// therefore bit-identical to the reference arithmetic on the stored
// binary32 coordinates.
//
// Deposits accumulate w * 2^22 (w = CIC corner weight) in int32 per node:
// integer addition is associative, so the field is run-to-run
// deterministic; resolution 2.4e-7 of a particle mass per contribution.
#include <utility>

#include "common.cuh"


namespace cs {

struct __align__(16) Rec {
    float x, y;
    unsigned int meta;  // id | type << 31
    short wx, wy;
};

constexpr double Q_SCALE = 4194304.0;  // 2^22
constexpr unsigned ID_MASK = 0x7fffffffu;

struct FastArgs {
    const Rec *rec;
    const int *starts;
    Rec *tmp;
    int *keys;
    int *counts;
    const float *xi;    // this step's (N, 2) increments, indexed by id
    const float *grad;  // (n_c^2, 2)
    int *rho_q;         // 2 * m fixed-point deposits (a | b)
    long long n;
    BinGeom g;
    PairTab pt;
    GridGeom gg;
    double amp[2], dt, chi[2];
    int chi_pinned[2];
    int refresh, deposit, interact;
    unsigned bits[2];
    double half0, half1;
    cs_domain dom;
};

// minimum image with the |dx| <= L/2 shortcut: round(dx/L) is then +-0 and
// dx - L*(+-0) == dx exactly (dx is never -0.0: x - x = +0 under RN)
__device__ __forceinline__ double min_image(double dx, double size, double half) {
    if (fabs(dx) <= half) return dx;
    return dsub(dx, dmul(size, rint(ddiv(dx, size))));
}

__device__ __forceinline__ bool pair_term(const Rec &r, double xi, double yi, int ti,
                                          const FastArgs &a, double &tx, double &ty,
                                          bool want_term) {
    double dx0 = dsub((double)r.x, xi);
    double dx1 = dsub((double)r.y, yi);
    if (a.g.per0) dx0 = min_image(dx0, a.g.size0, a.half0);
    if (a.g.per1) dx1 = min_image(dx1, a.g.size1, a.half1);
    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
    const int t = ti * 2 + (int)(r.meta >> 31);
    if (r2 > a.pt.cut2[t] || r2 == 0.0) return false;
    if (want_term) {
        const double eps = a.pt.eps[t];
        const double rr = dsqrt(r2);
        const double s = -ddiv(cs_exp(-ddiv(rr, eps)), dmul(eps, rr));
        tx = dmul(s, dx0);
        ty = dmul(s, dx1);
    }
    return true;
}

__device__ __forceinline__ int boundary_axis_wraps(double &v, int &w, double lo, double hi,
                                                   int per) {
    const double size = dsub(hi, lo);
    if (per) {
        const double k = floor(ddiv(dsub(v, lo), size));
        if (k != 0.0) {
            v = dsub(v, dmul(k, size));
            w += (int)k;
        }
        for (int it = 0; it < 2; it++) {
            if (v >= hi) {
                v = dsub(v, size);
                w += 1;
            } else if (v < lo) {
                v = dadd(v, size);
                w -= 1;
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

__device__ __forceinline__ void cic_deposit_q(double x, double y, const GridGeom &gg,
                                              int *__restrict__ out) {
    const int nc = gg.n;
    const double u0 = ddiv(dsub(x, gg.lo0), gg.d0);
    const double u1 = ddiv(dsub(y, gg.lo1), gg.d1);
    long long b0, b1, c0, c1;
    double f0, f1;
    if (gg.per) {
        const double base0 = floor(u0), base1 = floor(u1);
        f0 = dsub(u0, base0);
        f1 = dsub(u1, base1);
        b0 = pymod((long long)base0, nc);
        b1 = pymod((long long)base1, nc);
        c0 = (b0 + 1) % nc;
        c1 = (b1 + 1) % nc;
    } else {
        b0 = (long long)floor(u0);
        b1 = (long long)floor(u1);
        b0 = b0 < 0 ? 0 : (b0 > nc - 2 ? nc - 2 : b0);
        b1 = b1 < 0 ? 0 : (b1 > nc - 2 ? nc - 2 : b1);
        f0 = dsub(u0, (double)b0);
        f1 = dsub(u1, (double)b1);
        c0 = b0 + 1;
        c1 = b1 + 1;
    }
    const double g0 = dsub(1.0, f0), g1 = dsub(1.0, f1);
    atomicAdd(&out[b1 * nc + b0], __double2int_rn(dmul(dmul(g0, g1), Q_SCALE)));
    atomicAdd(&out[b1 * nc + c0], __double2int_rn(dmul(dmul(f0, g1), Q_SCALE)));
    atomicAdd(&out[c1 * nc + b0], __double2int_rn(dmul(dmul(g0, f1), Q_SCALE)));
    atomicAdd(&out[c1 * nc + c0], __double2int_rn(dmul(dmul(f0, f1), Q_SCALE)));
}

__global__ void __launch_bounds__(256)
k_fast_step(FastArgs a, DevStatus *st, int step) {
    const bool dead = st->abort != 0;
    const int m = a.gg.n * a.gg.n;
    int clamped = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.n;
         t += (long long)gridDim.x * blockDim.x) {
        const Rec me = a.rec[t];
        const double x = (double)me.x, y = (double)me.y;
        const int ti = (int)(me.meta >> 31);
        const unsigned id = me.meta & ID_MASK;
        // ---- pair forces over the reference ring, canonical order
        double fx = 0.0, fy = 0.0;
        if (!dead && a.interact) {
            const int cx = cell_axis(x, a.g.lo0, a.g.eff0, a.g.n0);
            const int cy = cell_axis(y, a.g.lo1, a.g.eff1, a.g.n1);
            for (int o1 = -1; o1 <= 1; o1++) {
                int g1 = cy + o1;
                if (a.g.per1) {
                    if (a.g.n1 == 1 && o1 != 0) continue;
                    if (a.g.n1 == 2 && o1 == 1) continue;
                    g1 = g1 < 0 ? g1 + a.g.n1 : (g1 >= a.g.n1 ? g1 - a.g.n1 : g1);
                } else if (g1 < 0 || g1 >= a.g.n1) {
                    continue;
                }
                for (int o0 = -1; o0 <= 1; o0++) {
                    int g0 = cx + o0;
                    if (a.g.per0) {
                        if (a.g.n0 == 1 && o0 != 0) continue;
                        if (a.g.n0 == 2 && o0 == 1) continue;
                        g0 = g0 < 0 ? g0 + a.g.n0 : (g0 >= a.g.n0 ? g0 - a.g.n0 : g0);
                    } else if (g0 < 0 || g0 >= a.g.n0) {
                        continue;
                    }
                    const int f = g1 * a.g.n0 + g0;
                    const int kb = a.starts[f], ke = a.starts[f + 1];
                    int nacc = 0;
                    double tx1 = 0.0, ty1 = 0.0;
                    for (int k = kb; k < ke; k++) {
                        if (k == t) continue;
                        double tx, ty;
                        if (pair_term(a.rec[k], x, y, ti, a, tx, ty, nacc == 0)) {
                            if (nacc == 0) {
                                tx1 = tx;
                                ty1 = ty;
                            }
                            nacc++;
                        }
                    }
                    if (nacc == 1) {
                        fx = dadd(fx, tx1);
                        fy = dadd(fy, ty1);
                    } else if (nacc > 1) {
                        // ascending id among the accepted members
                        long long last = -1;
                        for (int r = 0; r < nacc; r++) {
                            unsigned best = 0xffffffffu;
                            int bk = -1;
                            for (int k = kb; k < ke; k++) {
                                if (k == t) continue;
                                const Rec rk = a.rec[k];
                                const unsigned idk = rk.meta & ID_MASK;
                                if ((long long)idk <= last || idk >= best) continue;
                                double tx, ty;
                                if (pair_term(rk, x, y, ti, a, tx, ty, false)) {
                                    best = idk;
                                    bk = k;
                                }
                            }
                            double tx, ty;
                            pair_term(a.rec[bk], x, y, ti, a, tx, ty, true);
                            fx = dadd(fx, tx);
                            fy = dadd(fy, ty);
                            last = best;
                        }
                    }
                }
            }
        }
        // ---- drift refresh at the start-of-step position
        double dr0 = 0.0, dr1 = 0.0;
        if (a.refresh && !dead) {
            Bilin b;
            clamped += 2 * bilinear_stencil(x, y, a.gg, b);
            dr0 = bilinear_apply(b, a.grad, 2, 0);
            dr1 = bilinear_apply(b, a.grad, 2, 1);
            if (a.chi_pinned[ti]) {
                dr0 = 0.0;
                dr1 = 0.0;
            } else if (a.chi[ti] != 1.0) {
                dr0 = dmul(dr0, a.chi[ti]);
                dr1 = dmul(dr1, a.chi[ti]);
            }
        }
        // ---- EM proposal (motion.py:281-282)
        const float2 z = __ldg(reinterpret_cast<const float2 *>(a.xi) + id);
        const double amp = a.amp[ti];
        double v[2];
        v[0] = dadd(dadd(dadd(x, dmul(amp, (double)z.x)), dmul(dr0, a.dt)), dmul(fx, a.dt));
        v[1] = dadd(dadd(dadd(y, dmul(amp, (double)z.y)), dmul(dr1, a.dt)), dmul(fy, a.dt));
        int w[2] = {me.wx, me.wy};
        bool ok = !dead;
        if (ok && !(isfinite(v[0]) && isfinite(v[1]))) {
            atomicMin(&st->key, err_key(0, id, CS_NONFINITE));
            st->abort = 1;
            st->step = step;
            ok = false;
        }
        if (ok) {
            for (int ax = 0; ax < 2; ax++) {
                const double raw = v[ax];
                const int code = boundary_axis_wraps(v[ax], w[ax], a.dom.lo[ax], a.dom.hi[ax],
                                                     a.dom.periodic[ax]);
                if (code) {
                    atomicMin(&st->key, err_key(1 + ax, id, code));
                    st->abort = 1;
                    st->step = step;
                    v[ax] = raw;  // the raw proposal stays visible for the message
                    ok = false;
                    break;
                }
            }
        }
        Rec out;
        if (dead) {
            out = me;
        } else {
            out.x = (float)v[0];
            out.y = (float)v[1];
            out.meta = me.meta;
            out.wx = (short)w[0];
            out.wy = (short)w[1];
        }
        // ---- bin the stored (binary32) coordinate for the next step
        const double nx = (double)out.x, ny = (double)out.y;
        const int key = cell_axis(ny, a.g.lo1, a.g.eff1, a.g.n1) * a.g.n0 +
                        cell_axis(nx, a.g.lo0, a.g.eff0, a.g.n0);
        a.tmp[t] = out;
        a.keys[t] = key;
        atomicAdd(&a.counts[key], 1);
        if (a.deposit && ok) {
            const unsigned bits = a.bits[ti];
            if (bits & 1u) cic_deposit_q(nx, ny, a.gg, a.rho_q);
            if (bits & 2u) cic_deposit_q(nx, ny, a.gg, a.rho_q + m);
        }
    }
    if (clamped) atomicAdd((unsigned long long *)&st->clamped, (unsigned long long)clamped);
}

__global__ void __launch_bounds__(256)
k_fast_scatter(const Rec *__restrict__ tmp, const int *__restrict__ keys, long long n,
               const int *__restrict__ starts, int *__restrict__ counts, Rec *__restrict__ out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int key = keys[t];
        const int slot = starts[key] + atomicSub(&counts[key], 1) - 1;
        out[slot] = tmp[t];
    }
}

// caller arrays (id order) -> records (id order) + keys + histogram
__global__ void k_fast_import(const float *__restrict__ pos, const float *__restrict__ anchor,
                              const uint8_t *__restrict__ type, long long n, BinGeom g,
                              Rec *__restrict__ tmp, int *__restrict__ keys,
                              int *__restrict__ counts, float *__restrict__ anchor0) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 p = reinterpret_cast<const float2 *>(pos)[i];
        Rec r;
        r.x = p.x;
        r.y = p.y;
        r.meta = (unsigned)i | ((type && type[i]) ? 0x80000000u : 0u);
        r.wx = 0;
        r.wy = 0;
        tmp[i] = r;
        reinterpret_cast<float2 *>(anchor0)[i] = reinterpret_cast<const float2 *>(anchor)[i];
        const int key = cell_axis((double)p.y, g.lo1, g.eff1, g.n1) * g.n0 +
                        cell_axis((double)p.x, g.lo0, g.eff0, g.n0);
        keys[i] = key;
        atomicAdd(&counts[key], 1);
    }
}

__global__ void k_fast_deposit(const Rec *__restrict__ rec, long long n, GridGeom gg,
                               unsigned bits0, unsigned bits1, int *__restrict__ rho_q) {
    const int m = gg.n * gg.n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const Rec r = rec[t];
        const unsigned bits = (r.meta >> 31) ? bits1 : bits0;
        if (bits & 1u) cic_deposit_q((double)r.x, (double)r.y, gg, rho_q);
        if (bits & 2u) cic_deposit_q((double)r.x, (double)r.y, gg, rho_q + m);
    }
}

// records (sorted) -> caller arrays (id order); anchor = anchor0 - wraps * L
__global__ void k_fast_export(const Rec *__restrict__ rec, long long n,
                              const float *__restrict__ anchor0, double size0, double size1,
                              float *__restrict__ pos, float *__restrict__ anchor) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const Rec r = rec[t];
        const unsigned id = r.meta & ID_MASK;
        reinterpret_cast<float2 *>(pos)[id] = make_float2(r.x, r.y);
        const float2 a0 = reinterpret_cast<const float2 *>(anchor0)[id];
        const float ax = (float)dsub((double)a0.x, dmul((double)r.wx, size0));
        const float ay = (float)dsub((double)a0.y, dmul((double)r.wy, size1));
        reinterpret_cast<float2 *>(anchor)[id] = make_float2(ax, ay);
    }
}

// fixed-point deposits -> caller rho arrays (float densities)
__global__ void k_fast_rho_export(const int *__restrict__ q, long long m2, double scale,
                                  float *__restrict__ ra, float *__restrict__ rb, long long m) {
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m2;
         l += (long long)gridDim.x * blockDim.x) {
        const float v = (float)((double)q[l] * scale);
        if (l < m) ra[l] = v;
        else rb[l - m] = v;
    }
}

// explicit part of step_field on fixed-point densities; zeroes them for the
// deposits of the coming update
template <class R>
__global__ void __launch_bounds__(256)
k_fast_rhs(const float *__restrict__ c, int *__restrict__ q, long long m, double one_m_dtg,
           double dka, double dkb, int has_g, int has_a, int has_b, double scale,
           R *__restrict__ rhs, const DevStatus *st) {
    if (st->abort) return;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const double cv = (double)c[l];
        const int qa = q[l], qb = q[l + m];
        q[l] = 0;
        q[l + m] = 0;
        double r = has_g ? dmul(cv, one_m_dtg) : cv;
        if (has_a) r = dadd(r, dmul(dka, dmul((double)qa, scale)));
        if (has_b) r = dsub(r, dmul(dmul(dmul((double)qb, scale), cv), dkb));
        rhs[l] = (R)r;
    }
}

}  // namespace cs

// ---------------------------------------------------------------------------
struct cs_fast {
    cs::Buf rec[2], tmp, keys, counts, starts[2], anchor0, rho_q;
    int cur = 0;
    bool imported = false;
    long long nflat = 0;
};

namespace cs {

int field_solve_rhs(cs_field_ops *ops, void *out);
int launch_gradient(cs_ctx *ctx, int prec, const void *c, const GridGeom &gg, void *grad,
                    DevStatus *st, int step);

int fast_create(cs_fast **out, long long n, const BinGeom &g, const GridGeom *gg) {
    auto *f = new cs_fast();
    *out = f;
    f->nflat = (long long)g.n0 * g.n1;
    const size_t nr = sizeof(Rec) * (size_t)(n > 0 ? n : 1);
    CS_TRY(f->rec[0].ensure(nr));
    CS_TRY(f->rec[1].ensure(nr));
    CS_TRY(f->tmp.ensure(nr));
    CS_TRY(f->keys.ensure(sizeof(int) * (size_t)(n > 0 ? n : 1)));
    CS_TRY(f->counts.ensure(sizeof(int) * (size_t)f->nflat));
    CS_CUDA(cudaMemset(f->counts.p, 0, f->counts.bytes));
    CS_TRY(f->starts[0].ensure(sizeof(int) * (size_t)(f->nflat + 1)));
    CS_TRY(f->starts[1].ensure(sizeof(int) * (size_t)(f->nflat + 1)));
    CS_TRY(f->anchor0.ensure(sizeof(float) * 2 * (size_t)(n > 0 ? n : 1)));
    if (gg) {
        CS_TRY(f->rho_q.ensure(sizeof(int) * 2 * (size_t)gg->n * gg->n));
        CS_CUDA(cudaMemset(f->rho_q.p, 0, f->rho_q.bytes));
    }
    return CS_OK;
}

void fast_destroy(cs_fast *f) {
    if (!f) return;
    for (Buf *b : {&f->rec[0], &f->rec[1], &f->tmp, &f->keys, &f->counts, &f->starts[0],
                   &f->starts[1], &f->anchor0, &f->rho_q})
        b->release();
    delete f;
}

static int fast_sort(cs_ctx *ctx, cs_fast *f, long long n, int nxt) {
    CS_TRY(exclusive_scan_i32(ctx, f->counts.as<int>(), f->starts[nxt].as<int>(), f->nflat));
    if (n > 0) {
        k_fast_scatter<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            f->tmp.as<Rec>(), f->keys.as<int>(), n, f->starts[nxt].as<int>(),
            f->counts.as<int>(), f->rec[nxt].as<Rec>());
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    f->cur = nxt;
    return CS_OK;
}

int fast_import(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                const BinGeom &g, const GridGeom &gg, const unsigned char bits[3]) {
    const long long n = p.n;
    if (n > 0) {
        k_fast_import<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            (const float *)s->pos, (const float *)s->anchor, s->type, n, g, f->tmp.as<Rec>(),
            f->keys.as<int>(), f->counts.as<int>(), f->anchor0.as<float>());
        CS_LAUNCH_CHECK();
    }
    CS_TRY(fast_sort(ctx, f, n, 0));
    if (p.field_active) {
        CS_CUDA(cudaMemsetAsync(f->rho_q.p, 0, f->rho_q.bytes, ctx->stream));
        if (n > 0) {
            k_fast_deposit<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
                f->rec[0].as<Rec>(), n, gg, bits[0], bits[1], f->rho_q.as<int>());
            CS_LAUNCH_CHECK();
        }
    }
    f->imported = true;
    return CS_OK;
}

int fast_export(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                const GridGeom &gg) {
    const long long n = p.n;
    if (!f->imported) return CS_OK;
    if (n > 0) {
        k_fast_export<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            f->rec[f->cur].as<Rec>(), n, f->anchor0.as<float>(), p.domain.hi[0] - p.domain.lo[0],
            p.domain.hi[1] - p.domain.lo[1], (float *)s->pos, (float *)s->anchor);
        CS_LAUNCH_CHECK();
    }
    if (p.field_active && s->rho_a && s->rho_b) {
        const long long m = (long long)gg.n * gg.n;
        const double scale = (1.0 / Q_SCALE) * (1.0 / (gg.d0 * gg.d1));
        k_fast_rho_export<<<grid_for(2 * m, 256), 256, 0, ctx->stream>>>(
            f->rho_q.as<int>(), 2 * m, scale, (float *)s->rho_a, (float *)s->rho_b, m);
        CS_LAUNCH_CHECK();
    }
    return CS_OK;
}

struct FastStepCfg {
    const cs_sim_params *p;
    BinGeom g;
    PairTab pt;
    GridGeom gg;
    cs_field_ops *ops;
    unsigned char bits[3];
};

int fast_field(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
               DevStatus *st, int step) {
    const cs_sim_params &p = *c.p;
    const long long m = (long long)c.gg.n * c.gg.n;
    const double dt = p.dt;
    const double scale = (1.0 / Q_SCALE) * (1.0 / (c.gg.d0 * c.gg.d1));
    if (c.ops->kind == 1)  // neumann DCT path solves in binary64
        k_fast_rhs<double><<<grid_for(m, 256, 148 * 16), 256, 0, ctx->stream>>>(
            (const float *)s->c, f->rho_q.as<int>(), m, 1.0 - dt * p.gamma, dt * p.k_alpha,
            dt * p.k_beta, p.gamma != 0.0, p.k_alpha != 0.0, p.k_beta != 0.0, scale,
            (double *)c.ops->rhs, st);
    else
        k_fast_rhs<float><<<grid_for(m, 256, 148 * 16), 256, 0, ctx->stream>>>(
            (const float *)s->c, f->rho_q.as<int>(), m, 1.0 - dt * p.gamma, dt * p.k_alpha,
            dt * p.k_beta, p.gamma != 0.0, p.k_alpha != 0.0, p.k_beta != 0.0, scale,
            (float *)c.ops->rhs, st);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    CS_TRY(field_solve_rhs(c.ops, s->c));
    return CS_OK;
}

int fast_particles(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
                   const void *xi, DevStatus *st, int step) {
    const cs_sim_params &p = *c.p;
    const long long n = p.n;
    FastArgs a;
    a.rec = f->rec[f->cur].as<Rec>();
    a.starts = f->starts[f->cur].as<int>();
    a.tmp = f->tmp.as<Rec>();
    a.keys = f->keys.as<int>();
    a.counts = f->counts.as<int>();
    a.xi = (const float *)xi;
    a.grad = (const float *)s->grad;
    a.rho_q = f->rho_q.as<int>();
    a.n = n;
    a.g = c.g;
    a.pt = c.pt;
    a.interact = p.interaction == 1;
    a.gg = c.gg;
    for (int t = 0; t < 2; t++) {
        a.amp[t] = p.amp[t];
        a.chi[t] = p.chi[t];
        a.chi_pinned[t] = p.chi_pinned[t];
        a.bits[t] = c.bits[t];
    }
    a.dt = p.dt;
    a.refresh = p.refresh_active;
    a.deposit = p.field_active;
    a.half0 = 0.5 * c.g.size0;
    a.half1 = 0.5 * c.g.size1;
    a.dom = p.domain;
    if (n > 0) {
        k_fast_step<<<grid_for(n, 256), 256, 0, ctx->stream>>>(a, st, step);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    return CS_OK;
}

int fast_resort(cs_ctx *ctx, cs_fast *f, long long n) { return fast_sort(ctx, f, n, 1 - f->cur); }

bool fast_imported(const cs_fast *f) { return f && f->imported; }

}  // namespace cs
