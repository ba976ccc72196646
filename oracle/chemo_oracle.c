/*
 * chemo_oracle.c -- CPU restatement of the reference (chemosim) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: it is loaded by
 * tests/, by __graft_entry__.smoke() as the checker, and by bench.py's
 * cpu_baseline / --impl reference leg.  The product path
 * (paper_1805_11007_b200) never links, loads or calls it.
 *
 * Every function restates one reference routine (paths relative to the
 * reference package root, /root/reference/pkg/src/chemosim):
 *
 *   or_soft_forces     motion.py:165-245  (_soft_forces_fused), generalised to
 *                      a per-type-pair (eps, cutoff) table; with a single type
 *                      and table entries (epsilon, cutoff) it is the
 *                      reference arithmetic operation for operation.
 *   or_em_step         motion.py:268-282  (em_step, numpy left-to-right)
 *   or_boundaries      motion.py:355-402  (_boundaries_kernel)
 *   or_cic_scatter     coupling.py:113-138 (_cic_scatter, 4 bincount passes)
 *   or_gauss_scatter   coupling.py:77-110 (_gauss_scatter_pair)
 *   or_bilinear        coupling.py:216-262 (_bilinear)
 *   or_gradient        field.py:128-137 + 242-245 (CSR d1x/d1y matvecs)
 *   or_field_rhs       field.py:220-227 (explicit part of step_field)
 *
 * Arithmetic is IEEE binary64 with no contraction (-ffp-contract=off); exp
 * is the host libm exp, which is what numba's np.exp lowers to (survey
 * 8c).  The implicit solve (field.py:162-201) lives in oracle/field.py on
 * numpy/scipy exactly as the reference calls them.
 *
 * Parity of this file against the reference itself is pinned by
 * tests/test_oracle_golden.py on fixtures produced by
 * tests/golden/make_golden.py (which imports the reference read-only).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline int64_t pymod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* np.round: round half to even (numba lowers it to rint under the default
 * rounding mode). */
static inline double np_round(double x) { return nearbyint(x); }

/* ------------------------------------------------------------------ */
/* binning: motion.py:170-199                                          */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n0, n1, nflat;
    double eff0, eff1;
    int64_t *cx, *cy, *starts, *order;
} or_bins;

static int bins_build(or_bins *b, const double *pos, int64_t n, double lo0,
                      double lo1, double size0, double size1,
                      double cell_cutoff) {
    int64_t n0 = (int64_t)(size0 / cell_cutoff);
    int64_t n1 = (int64_t)(size1 / cell_cutoff);
    if (n0 < 1) n0 = 1;
    if (n1 < 1) n1 = 1;
    b->n0 = n0;
    b->n1 = n1;
    b->nflat = n0 * n1;
    b->eff0 = size0 / (double)n0;
    b->eff1 = size1 / (double)n1;
    b->cx = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    b->cy = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    b->order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    b->starts = (int64_t *)calloc((size_t)(b->nflat + 1), sizeof(int64_t));
    if (!b->cx || !b->cy || !b->order || !b->starts) return -1;
    int64_t *counts = b->starts; /* counts[f+1]++ then cumsum in place */
    for (int64_t i = 0; i < n; i++) {
        int64_t c0 = (int64_t)floor((pos[2 * i] - lo0) / b->eff0);
        if (c0 < 0) c0 = 0;
        else if (c0 >= n0) c0 = n0 - 1;
        int64_t c1 = (int64_t)floor((pos[2 * i + 1] - lo1) / b->eff1);
        if (c1 < 0) c1 = 0;
        else if (c1 >= n1) c1 = n1 - 1;
        b->cx[i] = c0;
        b->cy[i] = c1;
        counts[c1 * n0 + c0 + 1] += 1;
    }
    for (int64_t f = 0; f < b->nflat; f++) counts[f + 1] += counts[f];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)b->nflat);
    if (!cursor) return -1;
    memcpy(cursor, b->starts, sizeof(int64_t) * (size_t)b->nflat);
    for (int64_t i = 0; i < n; i++) {
        int64_t f = b->cy[i] * n0 + b->cx[i];
        b->order[cursor[f]++] = i;
    }
    free(cursor);
    return 0;
}

static void bins_free(or_bins *b) {
    free(b->cx);
    free(b->cy);
    free(b->order);
    free(b->starts);
}

int or_bin_cells(const double *pos, int64_t n, double lo0, double lo1,
                 double size0, double size1, double cell_cutoff,
                 int64_t *n0_out, int64_t *n1_out, int64_t *starts_out,
                 int64_t starts_cap, int64_t *order_out) {
    or_bins b;
    if (bins_build(&b, pos, n, lo0, lo1, size0, size1, cell_cutoff)) return -1;
    *n0_out = b.n0;
    *n1_out = b.n1;
    int rc = 0;
    if (starts_out) {
        if (starts_cap < b.nflat + 1) rc = -2;
        else memcpy(starts_out, b.starts, sizeof(int64_t) * (size_t)(b.nflat + 1));
    }
    if (order_out && rc == 0) memcpy(order_out, b.order, sizeof(int64_t) * (size_t)n);
    bins_free(&b);
    return rc;
}

/* ------------------------------------------------------------------ */
/* soft forces: motion.py:200-245                                      */
/* ------------------------------------------------------------------ */
/* Per particle i: ring o1 in {-1,0,1} (y) outer, o0 inner; within a cell
 * j ascending; skip j == i; minimum image; skip r2 > cut2 or r2 == 0;
 * s = -(exp(-r/eps) / (eps*r)); f += s*dx.  The pair table is indexed
 * t_i * 2 + t_j (t = 0 when type is NULL).  When pairs != NULL the
 * accumulated (i, j) are written in accumulation order (serial only). */
static int64_t force_one(const or_bins *b, const double *pos,
                         const uint8_t *type, int64_t i, double size0,
                         double size1, int per0, int per1,
                         const double *eps_tab, const double *cut2_tab,
                         double *fx_out, double *fy_out, int64_t *pairs,
                         int64_t cap, int64_t npairs) {
    const int64_t n0 = b->n0, n1 = b->n1;
    double fx = 0.0, fy = 0.0;
    const double xi = pos[2 * i], yi = pos[2 * i + 1];
    const int ti = type ? type[i] : 0;
    for (int o1 = -1; o1 <= 1; o1++) {
        int64_t g1 = b->cy[i] + o1;
        if (per1) {
            if (n1 == 1 && o1 != 0) continue;
            if (n1 == 2 && o1 == 1) continue;
            g1 = pymod(g1, n1);
        } else if (g1 < 0 || g1 >= n1) {
            continue;
        }
        for (int o0 = -1; o0 <= 1; o0++) {
            int64_t g0 = b->cx[i] + o0;
            if (per0) {
                if (n0 == 1 && o0 != 0) continue;
                if (n0 == 2 && o0 == 1) continue;
                g0 = pymod(g0, n0);
            } else if (g0 < 0 || g0 >= n0) {
                continue;
            }
            const int64_t f = g1 * n0 + g0;
            for (int64_t k = b->starts[f]; k < b->starts[f + 1]; k++) {
                const int64_t j = b->order[k];
                if (j == i) continue;
                double dx0 = pos[2 * j] - xi;
                double dx1 = pos[2 * j + 1] - yi;
                if (per0) dx0 -= size0 * np_round(dx0 / size0);
                if (per1) dx1 -= size1 * np_round(dx1 / size1);
                const double r2 = dx0 * dx0 + dx1 * dx1;
                const int t = ti * 2 + (type ? type[j] : 0);
                if (r2 > cut2_tab[t] || r2 == 0.0) continue;
                const double eps = eps_tab[t];
                const double r = sqrt(r2);
                const double s = -(exp(-r / eps) / (eps * r));
                fx += s * dx0;
                fy += s * dx1;
                if (pairs) {
                    if (npairs < cap) {
                        pairs[2 * npairs] = i;
                        pairs[2 * npairs + 1] = j;
                    }
                    npairs++;
                }
            }
        }
    }
    *fx_out = fx;
    *fy_out = fy;
    return npairs;
}

int or_soft_forces(const double *pos, const uint8_t *type, int64_t n,
                   double lo0, double lo1, double size0, double size1,
                   int per0, int per1, const double *eps_tab,
                   const double *cut_tab, double cell_cutoff, double *out,
                   int64_t *pairs, int64_t cap, int64_t *npairs_out,
                   int nthreads) {
    or_bins b;
    if (bins_build(&b, pos, n, lo0, lo1, size0, size1, cell_cutoff)) return -1;
    double cut2[4];
    for (int t = 0; t < 4; t++) cut2[t] = cut_tab[t] * cut_tab[t];
    if (pairs || nthreads <= 1) {
        int64_t np = 0;
        for (int64_t i = 0; i < n; i++)
            np = force_one(&b, pos, type, i, size0, size1, per0, per1, eps_tab,
                           cut2, &out[2 * i], &out[2 * i + 1], pairs, cap, np);
        if (npairs_out) *npairs_out = np;
    } else {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
        for (int64_t i = 0; i < n; i++)
            force_one(&b, pos, type, i, size0, size1, per0, per1, eps_tab, cut2,
                      &out[2 * i], &out[2 * i + 1], NULL, 0, 0);
        if (npairs_out) *npairs_out = -1;
    }
    bins_free(&b);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Euler--Maruyama: motion.py:268-282                                  */
/* ((pos + amp*xi) + drift*dt) + force*dt, amp = sqrt((2.0*D)*dt)      */
/* ------------------------------------------------------------------ */
void or_em_step(const double *pos, const double *diffusion, const double *drift,
                const double *force, const double *xi, double dt, int64_t n,
                double *out, int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; i++) {
        const double amp = sqrt((2.0 * diffusion[i]) * dt);
        for (int a = 0; a < 2; a++) {
            const int64_t k = 2 * i + a;
            out[k] = ((pos[k] + amp * xi[k]) + drift[k] * dt) + force[k] * dt;
        }
    }
}

/* ------------------------------------------------------------------ */
/* boundaries: motion.py:355-402 (serial, partial-update semantics)    */
/* ------------------------------------------------------------------ */
int or_boundaries(double *x, double *anchor, int64_t n, double lo0, double lo1,
                  double hi0, double hi1, int per0, int per1, int64_t *bad_i,
                  int32_t *bad_ax) {
    *bad_i = -1;
    *bad_ax = -1;
    for (int64_t i = 0; i < n; i++) {
        if (!(isfinite(x[2 * i]) && isfinite(x[2 * i + 1]))) {
            *bad_i = i;
            *bad_ax = 0;
            return 1;
        }
    }
    for (int ax = 0; ax < 2; ax++) {
        const double lo = ax == 0 ? lo0 : lo1;
        const double hi = ax == 0 ? hi0 : hi1;
        const int per = ax == 0 ? per0 : per1;
        const double size = hi - lo;
        for (int64_t i = 0; i < n; i++) {
            double v = x[2 * i + ax];
            if (per) {
                const double k = floor((v - lo) / size);
                if (k != 0.0) {
                    const double shift = k * size;
                    v -= shift;
                    anchor[2 * i + ax] -= shift;
                }
                for (int it = 0; it < 2; it++) {
                    if (v >= hi) {
                        v -= size;
                        anchor[2 * i + ax] -= size;
                    } else if (v < lo) {
                        v += size;
                        anchor[2 * i + ax] += size;
                    } else {
                        break;
                    }
                }
                x[2 * i + ax] = v;
            } else {
                if (v > hi + size || v < lo - size) {
                    *bad_i = i;
                    *bad_ax = ax;
                    return 2;
                }
                int settled = 0;
                for (int it = 0; it < 4; it++) {
                    if (v > hi) v = 2.0 * hi - v;
                    else if (v < lo) v = 2.0 * lo - v;
                    else {
                        settled = 1;
                        break;
                    }
                }
                if (!settled) {
                    *bad_i = i;
                    *bad_ax = ax;
                    return 3;
                }
                x[2 * i + ax] = v;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* CIC deposit: coupling.py:113-138                                    */
/* mask selects the particles of the deposited species (the reference  */
/* passes positions[species == s], coupling.py:150).                   */
/* ------------------------------------------------------------------ */
int or_cic_scatter(const double *pos, const uint8_t *mask, int64_t n, int nc,
                   double lo0, double lo1, double d0, double d1, int per,
                   double *out) {
    const int64_t m = (int64_t)nc * nc;
    double *pass = (double *)malloc(sizeof(double) * (size_t)m);
    if (!pass) return -1;
    for (int64_t l = 0; l < m; l++) out[l] = 0.0;
    const double unit = 1.0 / (d0 * d1);
    for (int corner = 0; corner < 4; corner++) {
        for (int64_t l = 0; l < m; l++) pass[l] = 0.0;
        for (int64_t p = 0; p < n; p++) {
            if (mask && !mask[p]) continue;
            const double u0 = (pos[2 * p] - lo0) / d0;
            const double u1 = (pos[2 * p + 1] - lo1) / d1;
            int64_t b0, b1, c0, c1;
            double f0, f1;
            if (per) {
                const double base0 = floor(u0), base1 = floor(u1);
                f0 = u0 - base0;
                f1 = u1 - base1;
                b0 = pymod((int64_t)base0, nc);
                b1 = pymod((int64_t)base1, nc);
                c0 = (b0 + 1) % nc;
                c1 = (b1 + 1) % nc;
            } else {
                b0 = (int64_t)floor(u0);
                b1 = (int64_t)floor(u1);
                if (b0 < 0) b0 = 0;
                if (b0 > nc - 2) b0 = nc - 2;
                if (b1 < 0) b1 = 0;
                if (b1 > nc - 2) b1 = nc - 2;
                f0 = u0 - (double)b0;
                f1 = u1 - (double)b1;
                c0 = b0 + 1;
                c1 = b1 + 1;
            }
            int64_t ix, iy;
            double w;
            switch (corner) {
            case 0: ix = b0; iy = b1; w = (1.0 - f0) * (1.0 - f1); break;
            case 1: ix = c0; iy = b1; w = f0 * (1.0 - f1); break;
            case 2: ix = b0; iy = c1; w = (1.0 - f0) * f1; break;
            default: ix = c0; iy = c1; w = f0 * f1; break;
            }
            pass[iy * nc + ix] += w * unit;
        }
        for (int64_t l = 0; l < m; l++) out[l] += pass[l];
    }
    free(pass);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Gaussian deposit: coupling.py:77-110 (_gauss_scatter_pair)          */
/* route[p]: 0 -> out_a, 1 -> out_b, anything else -> skipped.         */
/* ------------------------------------------------------------------ */
void or_gauss_scatter(const double *pos, const uint8_t *route, int64_t n,
                      int nc, double lo0, double lo1, double d0, double d1,
                      int per, double h, double cutoff, double *out_a,
                      double *out_b) {
    const double inv_norm = 1.0 / (2.0 * M_PI * h * h);
    const double two_h2 = 2.0 * h * h;
    const double cut2 = cutoff * cutoff;
    const int64_t w0 = (int64_t)floor(cutoff / d0 + 0.5);
    const int64_t w1 = (int64_t)floor(cutoff / d1 + 0.5);
    for (int64_t p = 0; p < n; p++) {
        double *out = route[p] == 0 ? out_a : (route[p] == 1 ? out_b : NULL);
        if (!out) continue;
        const double u0 = (pos[2 * p] - lo0) / d0;
        const double u1 = (pos[2 * p + 1] - lo1) / d1;
        const int64_t b0 = (int64_t)floor(u0 + 0.5);
        const int64_t b1 = (int64_t)floor(u1 + 0.5);
        for (int64_t o1 = -w1; o1 <= w1; o1++) {
            int64_t j = b1 + o1;
            if (per) j = pymod(j, nc);
            else if (j < 0 || j >= nc) continue;
            const double dy = (u1 - (double)(b1 + o1)) * d1;
            const double dy2 = dy * dy;
            for (int64_t o0 = -w0; o0 <= w0; o0++) {
                int64_t i = b0 + o0;
                if (per) i = pymod(i, nc);
                else if (i < 0 || i >= nc) continue;
                const double dxp = (u0 - (double)(b0 + o0)) * d0;
                const double r2 = dxp * dxp + dy2;
                if (r2 <= cut2) out[j * nc + i] += inv_norm * exp(-r2 / two_h2);
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* bilinear sampling: coupling.py:216-262                              */
/* ------------------------------------------------------------------ */
int64_t or_bilinear(const double *points, int64_t np, const double *values,
                    int m, double lo0, double lo1, double d0, double d1,
                    int nc, int per, double *out) {
    int64_t clamped = 0;
    const int nm1 = nc - 1;
    for (int64_t p = 0; p < np; p++) {
        double u0 = (points[2 * p] - lo0) / d0;
        double u1 = (points[2 * p + 1] - lo1) / d1;
        int64_t b0, b1, c0, c1;
        double f0, f1;
        if (per) {
            const double f0f = floor(u0), f1f = floor(u1);
            b0 = pymod((int64_t)f0f, nc);
            b1 = pymod((int64_t)f1f, nc);
            f0 = u0 - f0f;
            f1 = u1 - f1f;
            c0 = (b0 + 1) % nc;
            c1 = (b1 + 1) % nc;
        } else {
            if (u0 < 0.0) { u0 = 0.0; clamped++; }
            else if (u0 > nm1) { u0 = (double)nm1; clamped++; }
            if (u1 < 0.0) { u1 = 0.0; clamped++; }
            else if (u1 > nm1) { u1 = (double)nm1; clamped++; }
            b0 = (int64_t)floor(u0);
            if (b0 > nc - 2) b0 = nc - 2;
            b1 = (int64_t)floor(u1);
            if (b1 > nc - 2) b1 = nc - 2;
            f0 = u0 - (double)b0;
            f1 = u1 - (double)b1;
            c0 = b0 + 1;
            c1 = b1 + 1;
        }
        const double w00 = (1.0 - f0) * (1.0 - f1);
        const double w10 = f0 * (1.0 - f1);
        const double w01 = (1.0 - f0) * f1;
        const double w11 = f0 * f1;
        const int64_t r00 = b1 * nc + b0, r10 = b1 * nc + c0;
        const int64_t r01 = c1 * nc + b0, r11 = c1 * nc + c0;
        for (int k = 0; k < m; k++)
            out[p * m + k] = w00 * values[r00 * m + k] + w10 * values[r10 * m + k] +
                             w01 * values[r01 * m + k] + w11 * values[r11 * m + k];
    }
    return clamped;
}

/* ------------------------------------------------------------------ */
/* gradient: field.py:128-137 (_d1_1d), 182-185 (kron), 242-245        */
/* CSR rows hold their entries in ascending column order; scipy's      */
/* csr_matvec accumulates sum = 0 + a0*x0 + a1*x1 (+ a2*x2).           */
/* ------------------------------------------------------------------ */
static inline double d1_row(const double *c, int64_t base, int64_t stride,
                            int64_t i, int nc, int per, double h) {
    const double two_h = 2.0 * h;
    if (per) {
        const int64_t im = (i - 1 + nc) % nc, ip = (i + 1) % nc;
        const double vm = -1.0 / two_h, vp = 1.0 / two_h;
        const double am = vm * c[base + im * stride];
        const double ap = vp * c[base + ip * stride];
        /* ascending column order */
        if (im < ip) return (0.0 + am) + ap;
        return (0.0 + ap) + am;
    }
    if (i == 0) {
        return ((0.0 + (-3.0 / two_h) * c[base]) + (4.0 / two_h) * c[base + stride]) +
               (-1.0 / two_h) * c[base + 2 * stride];
    }
    if (i == nc - 1) {
        return ((0.0 + (1.0 / two_h) * c[base + (nc - 3) * stride]) +
                (-4.0 / two_h) * c[base + (nc - 2) * stride]) +
               (3.0 / two_h) * c[base + (nc - 1) * stride];
    }
    return (0.0 + (-1.0 / two_h) * c[base + (i - 1) * stride]) +
           (1.0 / two_h) * c[base + (i + 1) * stride];
}

void or_gradient(const double *c, int nc, double hx, double hy, int per,
                 double *grad) {
    for (int64_t j = 0; j < nc; j++)
        for (int64_t i = 0; i < nc; i++) {
            const int64_t l = j * nc + i;
            grad[2 * l] = d1_row(c, j * nc, 1, i, nc, per, hx);
            grad[2 * l + 1] = d1_row(c, i, nc, j, nc, per, hy);
        }
}

/* ------------------------------------------------------------------ */
/* explicit part of step_field: field.py:220-227                       */
/* ------------------------------------------------------------------ */
void or_field_rhs(const double *c, const double *rho_a, const double *rho_b,
                  int64_t m, double dt, double k_alpha, double k_beta,
                  double gamma, double *rhs) {
    for (int64_t l = 0; l < m; l++) {
        double r = gamma != 0.0 ? c[l] * (1.0 - dt * gamma) : c[l];
        if (k_alpha != 0.0) r += (dt * k_alpha) * rho_a[l];
        if (k_beta != 0.0) {
            double consumed = rho_b[l] * c[l];
            consumed *= dt * k_beta;
            r -= consumed;
        }
        rhs[l] = r;
    }
}

/* the exp the oracle uses, exported so tests can compare device exp */
double or_exp(double x) { return exp(x); }
