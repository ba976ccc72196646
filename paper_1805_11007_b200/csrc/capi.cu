// capi.cu -- the extern "C" boundary (include/chemo_b200.h).
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace cs {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int Buf::ensure(size_t need) {
    if (need <= bytes && p) return CS_OK;
    if (p) {
        cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    if (need == 0) need = 16;
    cudaError_t e = cudaMalloc(&p, need);
    if (e != cudaSuccess) {
        set_error("cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
        p = nullptr;
        return CS_ERR_NOMEM;
    }
    bytes = need;
    return CS_OK;
}

void Buf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

BinGeom make_geom(const cs_domain &d, double cell_cutoff) {
    BinGeom g;
    g.lo0 = d.lo[0];
    g.lo1 = d.lo[1];
    g.size0 = d.hi[0] - d.lo[0];
    g.size1 = d.hi[1] - d.lo[1];
    // motion.py:171-174: n = max(1, int(size / cutoff)); eff = size / n
    long long n0 = (long long)(g.size0 / cell_cutoff);
    long long n1 = (long long)(g.size1 / cell_cutoff);
    g.n0 = (int)(n0 < 1 ? 1 : n0);
    g.n1 = (int)(n1 < 1 ? 1 : n1);
    g.eff0 = g.size0 / g.n0;
    g.eff1 = g.size1 / g.n1;
    g.per0 = d.periodic[0] != 0;
    g.per1 = d.periodic[1] != 0;
    return g;
}

ExactDiv make_exact_div(double b) {
    ExactDiv d;
    d.b = b;
    d.inv = 1.0 / b;
    int e = 0;
    d.pow2 = (b > 0.0 && frexp(b, &e) == 0.5) ? 1 : 0;
    return d;
}

PairTab make_pairtab(const cs_pair_params &pp) {
    PairTab t;
    for (int k = 0; k < 4; k++) {
        t.eps[k] = pp.eps[k];
        t.cut2[k] = pp.cutoff[k] * pp.cutoff[k];
    }
    return t;
}

GridGeom make_grid_geom(const cs_grid &g) {
    GridGeom gg;
    gg.n = g.n_c;
    gg.per = g.periodic != 0;
    gg.lo0 = g.lo[0];
    gg.lo1 = g.lo[1];
    gg.d0 = g.spacing[0];
    gg.d1 = g.spacing[1];
    return gg;
}

int launch_em_step(cs_ctx *ctx, int prec, const void *pos, const double *D, const double *drift,
                   const double *force, const void *xi, double dt, long long n, void *out,
                   int tamed);
int launch_boundaries(cs_ctx *ctx, int prec, void *x, void *anchor, long long n,
                      const cs_domain &d, DevStatus *st);
int launch_deposit(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type, long long n,
                   const GridGeom &gg, int kind, double h, double cutoff,
                   const unsigned char bits[3], void *ra, void *rb, const DevStatus *st);
bool gauss_too_wide(const GridGeom &gg, double cutoff);
int launch_bilinear(cs_ctx *ctx, int prec, const void *pts, long long np, const void *vals, int m,
                    const GridGeom &gg, void *out, unsigned long long *clamped);
int launch_gradient(cs_ctx *ctx, int prec, const void *c, const GridGeom &gg, void *grad,
                    DevStatus *st, int step, int *zero_q = nullptr);
int field_ops_create(cs_ctx *ctx, int prec, const cs_grid *g, double d_c, double dt,
                     cs_field_ops **out);
void field_ops_destroy(cs_field_ops *ops);
int field_solve_rhs(cs_field_ops *ops, void *out);
int field_rhs(cs_field_ops *ops, const void *c, const void *ra, const void *rb, double ka,
              double kb, double gamma, const DevStatus *st);
int field_load_rhs(cs_field_ops *ops, const void *rhs);
int sim_create(cs_ctx *ctx, const cs_sim_params *p, cs_sim **out);
void sim_destroy(cs_sim *sim);
int sim_step(cs_sim *sim, const cs_sim_state *s, const void *xi, int64_t stride, int k,
             const double *u, int64_t u_stride);
int launch_react(cs_ctx *ctx, uint8_t *type, const double *local_c, double *drift,
                 const double *u, long long n, double p_ab, double r_beta, double dt,
                 DevStatus *st);
int sim_status(cs_sim *sim, cs_status *out);
int sim_reset_status(cs_sim *sim);

__global__ void k_exp(const double *x, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = cs_exp(x[i]);
}

static int check_prec(int prec) {
    if (prec != CS_F64 && prec != CS_F32) {
        set_error("unknown precision %d", prec);
        return CS_ERR_PARAM;
    }
    return CS_OK;
}

static int check_pairs(const cs_pair_params *pp) {
    for (int k = 0; k < 4; k++) {
        if (!(pp->eps[k] > 0) || !(pp->cutoff[k] > 0)) {
            set_error("pair table entries must be positive");
            return CS_ERR_PARAM;
        }
        if (pp->cutoff[k] > pp->cell_cutoff) {
            set_error("cell_cutoff must cover every pair cutoff");
            return CS_ERR_PARAM;
        }
    }
    return CS_OK;
}

// status word for the standalone seams
static int local_status(cs_ctx *ctx, DevStatus **out) {
    CS_TRY(ctx->status.ensure(sizeof(DevStatus)));
    DevStatus init{};
    init.key = ~0ULL;
    init.step = -1;
    CS_CUDA(cudaMemcpyAsync(ctx->status.p, &init, sizeof(init), cudaMemcpyHostToDevice,
                            ctx->stream));
    *out = ctx->dstat();
    return CS_OK;
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_abi_version(void) { return CS_ABI_VERSION; }
const char *cs_last_error(void) { return g_err; }

int cs_ctx_create(int device, void *stream, cs_ctx **out) {
    CS_CUDA(cudaSetDevice(device));
    auto *ctx = new cs_ctx();
    ctx->device = device;
    ctx->stream = (cudaStream_t)stream;
    *out = ctx;
    return CS_OK;
}

int cs_ctx_set_stream(cs_ctx *ctx, void *stream) {
    ctx->stream = (cudaStream_t)stream;
    return CS_OK;
}

int cs_ctx_sync(cs_ctx *ctx) {
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    return CS_OK;
}

int cs_ctx_destroy(cs_ctx *ctx) {
    if (!ctx) return CS_OK;
    cudaStreamSynchronize(ctx->stream);
    for (Buf *b : {&ctx->keys, &ctx->skeys, &ctx->counts, &ctx->starts, &ctx->order,
                   &ctx->force, &ctx->tile_flags, &ctx->tmp, &ctx->coop_sums, &ctx->status, &ctx->pair_counts,
                   &ctx->pair_offsets, &ctx->host_scratch, &ctx->zpar, &ctx->obs, &ctx->spos,
                   &ctx->stype, &ctx->dep_keys, &ctx->dep_counts, &ctx->dep_starts,
                   &ctx->dep_slots, &ctx->dep_pos, &ctx->dep_meta})
        b->release();
    delete ctx;
    return CS_OK;
}

int cs_soft_forces(cs_ctx *ctx, int32_t prec, const void *pos, const uint8_t *type, int64_t n,
                   const cs_domain *dom, const cs_pair_params *pp, double *out) {
    CS_TRY(check_prec(prec));
    CS_TRY(check_pairs(pp));
    const BinGeom g = make_geom(*dom, pp->cell_cutoff);
    CS_TRY(bin_particles(ctx, prec, pos, n, g, type));
    CS_TRY(launch_soft_forces(ctx, prec, pos, type, n, g, make_pairtab(*pp), out, nullptr));
    return CS_OK;
}

int cs_soft_force_pairs(cs_ctx *ctx, int32_t prec, const void *pos, const uint8_t *type,
                        int64_t n, const cs_domain *dom, const cs_pair_params *pp,
                        int64_t *pairs, int64_t cap, int64_t *count) {
    CS_TRY(check_prec(prec));
    CS_TRY(check_pairs(pp));
    const BinGeom g = make_geom(*dom, pp->cell_cutoff);
    CS_TRY(bin_particles(ctx, prec, pos, n, g));
    CS_TRY(run_soft_force_pairs(ctx, prec, pos, type, n, g, make_pairtab(*pp), pairs, cap, count));
    return CS_OK;
}

int cs_em_step(cs_ctx *ctx, int32_t prec, const void *pos, const double *diffusion,
               const double *drift, const double *force, const void *xi, double dt, int64_t n,
               void *out) {
    CS_TRY(check_prec(prec));
    return launch_em_step(ctx, prec, pos, diffusion, drift, force, xi, dt, n, out, 0);
}

int cs_tamed_step(cs_ctx *ctx, int32_t prec, const void *pos, const double *diffusion,
                  const double *drift, const double *force, const void *xi, double dt,
                  int64_t n, void *out) {
    CS_TRY(check_prec(prec));
    return launch_em_step(ctx, prec, pos, diffusion, drift, force, xi, dt, n, out, 1);
}

int cs_apply_boundaries(cs_ctx *ctx, int32_t prec, void *x, void *anchor, void *positions,
                        int64_t n, const cs_domain *dom, int64_t *bad_i, int32_t *bad_ax) {
    CS_TRY(check_prec(prec));
    DevStatus *st;
    CS_TRY(local_status(ctx, &st));
    CS_TRY(launch_boundaries(ctx, prec, x, anchor, n, *dom, st));
    DevStatus d;
    CS_CUDA(cudaMemcpyAsync(&d, st, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *bad_i = -1;
    *bad_ax = -1;
    if (d.key != ~0ULL) {
        const int rank = (int)(d.key >> 60);
        *bad_i = (int64_t)((d.key >> 3) & ((1ULL << 57) - 1));
        *bad_ax = rank >= 1 ? rank - 1 : 0;
        return (int)(d.key & 7ULL);
    }
    if (positions && positions != x && n > 0) {
        const size_t es = prec == CS_F64 ? 8 : 4;
        CS_CUDA(cudaMemcpyAsync(positions, x, (size_t)n * 2 * es, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    }
    return CS_OK;
}

int cs_cell_index(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n, const cs_domain *dom,
                  double cell_side, int32_t *cell_xy, int32_t *order, int32_t *starts,
                  int32_t *n_cells) {
    CS_TRY(check_prec(prec));
    if (!(cell_side > 0.0)) {
        set_error("cell_side must be positive");
        return CS_ERR_PARAM;
    }
    const BinGeom g = make_geom(*dom, cell_side);
    CS_TRY(bin_particles(ctx, prec, pos, n, g));
    const long long nflat = (long long)g.n0 * g.n1;
    if (n > 0)
        CS_CUDA(cudaMemcpyAsync(order, ctx->order.p, sizeof(int) * (size_t)n,
                                cudaMemcpyDeviceToDevice, ctx->stream));
    CS_CUDA(cudaMemcpyAsync(starts, ctx->starts.p, sizeof(int) * (size_t)(nflat + 1),
                            cudaMemcpyDeviceToDevice, ctx->stream));
    CS_TRY(launch_cell_xy(ctx, prec, pos, n, g, cell_xy));
    n_cells[0] = g.n0;
    n_cells[1] = g.n1;
    return CS_OK;
}

int cs_index_forces(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n, const int32_t *cell_xy,
                    const int32_t *order, const int32_t *starts, const cs_domain *dom,
                    const int32_t *n_cells, double epsilon, double cutoff, double *out) {
    CS_TRY(check_prec(prec));
    if (!(epsilon > 0.0) || !(cutoff > 0.0) || n_cells[0] < 1 || n_cells[1] < 1) {
        set_error("epsilon, cutoff and the cell counts must be positive");
        return CS_ERR_PARAM;
    }
    const double lx = dom->hi[0] - dom->lo[0], ly = dom->hi[1] - dom->lo[1];
    return launch_index_forces(ctx, prec, pos, n, cell_xy, order, starts, n_cells[0], n_cells[1],
                               lx / n_cells[0], ly / n_cells[1], dom->periodic[0] != 0,
                               dom->periodic[1] != 0, lx, ly, epsilon, cutoff, out);
}

int cs_deposit_gather(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n, const cs_grid *grid,
                      double span0, double span1, double h, double cutoff, double *out) {
    CS_TRY(check_prec(prec));
    if (!(h > 0) || !(cutoff > 0)) {
        set_error("kernel bandwidth and cutoff must be positive");
        return CS_ERR_PARAM;
    }
    const GridGeom gg = make_grid_geom(*grid);
    const double inv_norm = 1.0 / ((2.0 * M_PI) * (h * h));  // coupling.py:204
    return launch_deposit_gather(ctx, prec, pos, n, gg, span0, span1, h, cutoff, inv_norm, out);
}

int cs_deposit(cs_ctx *ctx, int32_t prec, const void *pos, const uint8_t *route, int64_t n,
               const cs_grid *grid, int32_t kind, double h, double cutoff, void *rho_a,
               void *rho_b) {
    CS_TRY(check_prec(prec));
    const GridGeom gg = make_grid_geom(*grid);
    if (kind == CS_GAUSSIAN) {
        if (!(h > 0) || !(cutoff > 0)) {
            set_error("kernel bandwidth and cutoff must be positive");
            return CS_ERR_PARAM;
        }
        if (gauss_too_wide(gg, cutoff)) {
            set_error("gaussian cutoff spans more than the periodic grid");
            return CS_ERR_PARAM;
        }
    }
    const unsigned char bits[3] = {1, 2, 0};
    void *rb = rho_b;
    Buf *tmp = nullptr;
    if (!rb) {  // single-output call: route everything to rho_a
        tmp = &ctx->tmp;
        CS_TRY(tmp->ensure((size_t)grid->n_c * grid->n_c * (prec == CS_F64 ? 8 : 4)));
        rb = tmp->p;
    }
    return launch_deposit(ctx, prec, pos, route, n, gg, kind, h, cutoff, bits, rho_a, rb, nullptr);
}

int cs_bilinear(cs_ctx *ctx, int32_t prec, const void *points, int64_t np, const void *values,
                int32_t m, const cs_grid *grid, void *out, int64_t *clamped) {
    CS_TRY(check_prec(prec));
    CS_TRY(ctx->tmp.ensure(sizeof(unsigned long long)));
    unsigned long long *cl = ctx->tmp.as<unsigned long long>();
    CS_CUDA(cudaMemsetAsync(cl, 0, sizeof(unsigned long long), ctx->stream));
    CS_TRY(launch_bilinear(ctx, prec, points, np, values, m, make_grid_geom(*grid), out, cl));
    unsigned long long h = 0;
    CS_CUDA(cudaMemcpyAsync(&h, cl, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *clamped = (int64_t)h;
    return CS_OK;
}

int cs_gradient(cs_ctx *ctx, int32_t prec, const void *c, const cs_grid *grid, void *grad) {
    CS_TRY(check_prec(prec));
    return launch_gradient(ctx, prec, c, make_grid_geom(*grid), grad, nullptr, -1);
}

int cs_field_ops_create(cs_ctx *ctx, int32_t prec, const cs_grid *grid, double d_c, double dt,
                        cs_field_ops **out) {
    CS_TRY(check_prec(prec));
    *out = nullptr;
    cs_field_ops *ops = nullptr;
    const int rc = field_ops_create(ctx, prec, grid, d_c, dt, &ops);
    if (rc != CS_OK) {
        field_ops_destroy(ops);
        return rc;
    }
    *out = ops;
    return CS_OK;
}

int cs_field_ops_destroy(cs_field_ops *ops) {
    field_ops_destroy(ops);
    return CS_OK;
}

int cs_field_solve(cs_field_ops *ops, const void *rhs, void *out) {
    CS_TRY(field_load_rhs(ops, rhs));
    return field_solve_rhs(ops, out);
}

int cs_field_step(cs_field_ops *ops, void *c, const void *rho_a, const void *rho_b,
                  double k_alpha, double k_beta, double gamma, int32_t *nonfinite,
                  double *neg_mass) {
    cs_ctx *ctx = ops->ctx;
    const size_t m = (size_t)ops->gg.n * ops->gg.n;
    const size_t es = ops->prec == CS_F64 ? 8 : 4;
    CS_TRY(field_rhs(ops, c, rho_a, rho_b, k_alpha, k_beta, gamma, nullptr));
    // solve into scratch so a non-finite result leaves c untouched
    const size_t off = (m * es + 255) & ~(size_t)255;  // 256-B aligned sub-buffers
    CS_TRY(ctx->tmp.ensure(off + 2 * m * es + 256));
    void *cn = ctx->tmp.p;
    void *grad = (char *)ctx->tmp.p + off;
    CS_TRY(field_solve_rhs(ops, cn));
    DevStatus *st;
    CS_TRY(local_status(ctx, &st));
    CS_TRY(launch_gradient(ctx, ops->prec, cn, ops->gg, grad, st, -1));
    DevStatus d;
    CS_CUDA(cudaMemcpyAsync(&d, st, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *nonfinite = d.field_bad;
    *neg_mass = d.neg_flag ? d.neg_mass : 0.0;
    if (!d.field_bad)
        CS_CUDA(cudaMemcpyAsync(c, cn, m * es, cudaMemcpyDeviceToDevice, ctx->stream));
    return CS_OK;
}

int cs_exp_batch(cs_ctx *ctx, const double *x, double *y, int64_t n) {
    if (n == 0) return CS_OK;
    k_exp<<<grid_for(n, 256), 256, 0, ctx->stream>>>(x, y, n);
    CS_LAUNCH_CHECK();
    return CS_OK;
}

int cs_sim_create(cs_ctx *ctx, const cs_sim_params *p, cs_sim **out) {
    CS_TRY(check_prec(p->prec));
    if (p->interaction == 1) CS_TRY(check_pairs(&p->pairs));
    if (p->field_active && p->deposit_kind == CS_GAUSSIAN &&
        gauss_too_wide(make_grid_geom(p->grid), p->kernel_cutoff)) {
        set_error("gaussian cutoff spans more than the periodic grid");
        return CS_ERR_PARAM;
    }
    *out = nullptr;
    cs_sim *sim = nullptr;
    const int rc = sim_create(ctx, p, &sim);
    if (rc != CS_OK) {
        sim_destroy(sim);
        return rc;
    }
    *out = sim;
    return CS_OK;
}

int cs_sim_destroy(cs_sim *sim) {
    sim_destroy(sim);
    return CS_OK;
}

int cs_sim_step(cs_sim *sim, const cs_sim_state *st, const void *xi, int64_t xi_stride,
                int32_t k_steps) {
    return sim_step(sim, st, xi, xi_stride, k_steps, nullptr, 0);
}

int cs_sim_step_react(cs_sim *sim, const cs_sim_state *st, const void *xi, int64_t xi_stride,
                      const double *u, int64_t u_stride, int32_t k_steps) {
    return sim_step(sim, st, xi, xi_stride, k_steps, u, u_stride);
}

int cs_react(cs_ctx *ctx, uint8_t *type, const double *local_c, double *drift, const double *u,
             int64_t n, double p_ab, double r_beta, double dt, int64_t *flips, double *high) {
    if (n < 0 || !(p_ab >= 0.0) || !(r_beta >= 0.0)) {
        set_error("cs_react: n, p_ab and r_beta must be non-negative");
        return CS_ERR_PARAM;
    }
    DevStatus *st;
    CS_TRY(local_status(ctx, &st));
    CS_TRY(launch_react(ctx, type, local_c, drift, u, n, p_ab, r_beta, dt, st));
    DevStatus d;
    CS_CUDA(cudaMemcpyAsync(&d, st, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (flips) {
        flips[0] = (int64_t)d.react_flips[0];
        flips[1] = (int64_t)d.react_flips[1];
    }
    if (high) {
        *high = 0.0;
        if (d.react_high_n) memcpy(high, &d.react_high_bits, sizeof(double));
    }
    return CS_OK;
}

int cs_sim_status(cs_sim *sim, cs_status *out) { return sim_status(sim, out); }
int cs_sim_reset_status(cs_sim *sim) { return sim_reset_status(sim); }

}  // extern "C"
