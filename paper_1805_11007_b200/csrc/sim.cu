#include <stdlib.h>
#include <string.h>
// sim.cu -- the fused per-step pipeline (Realisation._step_inner,
// engine.py:369-387) run for K steps on the device without host syncs.
//
// Per step, in the reference stage order:
//   field (if active):  zero rho -> deposit -> rhs -> implicit solve -> gradient
//                       (+ non-finite / negative-mass checks, field.py:229-238)
//   forces (if soft):   bin (count, scan, scatter, in-cell sort) -> pair sum
//   update:             bilinear refresh of drift/local_c at the start-of-step
//                       positions (coupling.py:302-325), EM proposal with
//                       xi[k] (motion.py:268-282), boundaries with anchor
//                       bookkeeping and status (motion.py:355-402), commit.
// The refresh is fused into the update kernel: both read only the particle's
// own start-of-step position and the freshly updated field, exactly the
// values the reference's separate refresh stage reads.
#include <utility>
#include <vector>

#include "common.cuh"

namespace cs {

int launch_deposit(cs_ctx *ctx, int prec, const void *pos, const uint8_t *type, long long n,
                   const GridGeom &gg, int kind, double h, double cutoff,
                   const unsigned char bits[3], void *ra, void *rb, const DevStatus *st);
int launch_gradient(cs_ctx *ctx, int prec, const void *c, const GridGeom &gg, void *grad,
                    DevStatus *st, int step, int *zero_q = nullptr);
int field_ops_create(cs_ctx *ctx, int prec, const cs_grid *g, double d_c, double dt,
                     cs_field_ops **out);
void field_ops_destroy(cs_field_ops *ops);
int field_solve_rhs(cs_field_ops *ops, void *out);
int field_rhs(cs_field_ops *ops, const void *c, const void *ra, const void *rb, double ka,
              double kb, double gamma, const DevStatus *st);
int launch_hard_sphere(cs_ctx *ctx, int prec, void *prop, const uint8_t *type, long long n,
                       const cs_domain &dom, double eps, const double D[2], int *n_hits_dev);
int launch_react(cs_ctx *ctx, uint8_t *type, const double *local_c, double *drift,
                 const double *u, long long n, double p_ab, double r_beta, double dt,
                 DevStatus *st);

int ens_create(cs_ctx *ctx, const cs_sim_params *p, int n_real, cs_ens **out);
void ens_destroy(cs_ens *e);
int ens_step(cs_ens *e, const cs_ens_state *s, const double *xi, const double *u, int k);
int ens_status(cs_ens *e, cs_status *out);
int ens_reset_status(cs_ens *e);

struct FastStepCfg {
    const cs_sim_params *p;
    BinGeom g;
    PairTab pt;
    GridGeom gg;
    cs_field_ops *ops;
    unsigned char bits[3];
    int overlap = 0;  // the field solve runs concurrently on a side stream
};
int fast_create(cs_fast **out, long long n, const BinGeom &g, const GridGeom *gg);
void fast_destroy(cs_fast *f);
int fast_import(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                const BinGeom &g, const GridGeom &gg, const unsigned char bits[3], DevStatus *st,
                int step);
int fast_export(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                const GridGeom &gg);
int fast_field(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
               DevStatus *st, int step);
int fast_particles(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
                   const void *xi, DevStatus *st, int step, int part);
bool fast_fused(const cs_fast *f, const cs_sim_params &p);
int fast_resort(cs_ctx *ctx, cs_fast *f, long long n, const cs_sim_params &p, const GridGeom &gg,
                const unsigned char bits[3], int part, DevStatus *st, int step,
                const void *xi_next = nullptr);
void fast_begin_call(cs_fast *f);
bool fast_imported(const cs_fast *f);
int *fast_rho_q(cs_fast *f);
int fast_slab_config(cs_fast *f, const int *bounds, int world, int rank, long long n,
                     cudaStream_t stream);
int fast_slab_import(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                     const GridGeom &gg, const unsigned char bits[3], DevStatus *st, int step);
int fast_slab_claim(cs_ctx *ctx, cs_fast *f, const void *recs, long long n, DevStatus *st,
                    int step);
int fast_slab_outbox(cs_ctx *ctx, cs_fast *f, void **recs, int **dest, long long *count);
int fast_slab_reset_outbox(cs_ctx *ctx, cs_fast *f);
int fast_slab_exchange_cap(cs_fast *f, long long seg);
int fast_slab_outbox_packed(cs_fast *f, void **recs, int **counts, long long *seg);
int fast_slab_claim_packed(cs_ctx *ctx, cs_fast *f, const void *inbox, const int *counts,
                           long long seg, DevStatus *st, int step);
int fast_slab_sort(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const GridGeom &gg,
                   const unsigned char bits[3], DevStatus *st, int step);
int fast_slab_range_host(cs_ctx *ctx, cs_fast *f, long long *lo, long long *hi);
bool fast_slab_gather(const cs_fast *f);
int fast_slab_hist(cs_ctx *ctx, cs_fast *f, int *hist);
int fast_slab_world(const cs_fast *f);
int fast_slab_rank(const cs_fast *f);
int fast_slab_dep_window(cs_fast *f, int j0, int rows);
void *fast_rho_all(cs_fast *f);
int spectral_slab_rows(cs_field_ops *ops, float *c, const int *q, double gamma, double ka,
                       double kb, double scale, int row0, int rows, void *spec, int inverse,
                       const DevStatus *st);
int spectral_slab_cols(cs_field_ops *ops, void *blocks, int kx0, int ncols, int rp,
                       const DevStatus *st);
int launch_gradient_rows(cs_ctx *ctx, const float *c, const GridGeom &gg, float *grad,
                         DevStatus *st, int step, int jbase, int jrows, int own0, int own1);

struct UpdateArgs {
    const void *xi;
    void *pos, *anchor, *next;
    const uint8_t *type;
    const double *force;  // (n, 2) or NULL
    double *drift;        // read when !refresh; written when refresh && store
    double *local_c;
    const void *c, *grad;
    long long n;
    double amp[2], dt, chi[2];
    int chi_pinned[2];
    int refresh, store_samples, store_next, tamed, propose_only;
    cs_domain dom;
    GridGeom gg;
};

template <class P>
__global__ void __launch_bounds__(256) k_update(UpdateArgs a, DevStatus *st, int step) {
    if (st->abort) return;
    const P *xi = (const P *)a.xi;
    P *pos = (P *)a.pos;
    P *anchor = (P *)a.anchor;
    int clamped = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int t = a.type ? (a.type[i] ? 1 : 0) : 0;
        double x, y;
        load2(pos, i, x, y);
        double dr0 = 0.0, dr1 = 0.0;
        if (a.refresh) {
            Bilin b;
            clamped += 2 * bilinear_stencil(x, y, a.gg, b);
            const P *g = (const P *)a.grad;
            dr0 = bilinear_apply(b, g, 2, 0);
            dr1 = bilinear_apply(b, g, 2, 1);
            if (a.chi_pinned[t]) {
                dr0 = 0.0;
                dr1 = 0.0;
            } else if (a.chi[t] != 1.0) {
                dr0 = dmul(dr0, a.chi[t]);
                dr1 = dmul(dr1, a.chi[t]);
            }
            if (a.store_samples) {
                a.local_c[i] = bilinear_apply(b, (const P *)a.c, 1, 0);
                reinterpret_cast<double2 *>(a.drift)[i] = make_double2(dr0, dr1);
            }
        } else if (a.drift) {
            const double2 d = reinterpret_cast<const double2 *>(a.drift)[i];
            dr0 = d.x;
            dr1 = d.y;
        }
        double f0 = 0.0, f1 = 0.0;
        if (a.force) {
            const double2 f = reinterpret_cast<const double2 *>(a.force)[i];
            f0 = f.x;
            f1 = f.y;
        }
        double x0, x1;
        load2(xi, i, x0, x1);
        const double amp = a.amp[t];
        double v[2];
        double i0, i1;
        force_increment(f0, f1, a.dt, a.tamed, i0, i1);
        v[0] = dadd(dadd(dadd(x, dmul(amp, x0)), dmul(dr0, a.dt)), i0);
        v[1] = dadd(dadd(dadd(y, dmul(amp, x1)), dmul(dr1, a.dt)), i1);
        if (a.propose_only) {  // hard spheres: the sweep comes before the boundaries
            store2((P *)a.next, i, v[0], v[1]);
            continue;
        }
        if (!(isfinite(v[0]) && isfinite(v[1]))) {
            atomicMin(&st->key, err_key(0, i, CS_NONFINITE));
            st->abort = 1;
            st->step = step;
            if (a.next) store2((P *)a.next, i, v[0], v[1]);
            continue;
        }
        double an[2];
        load2(anchor, i, an[0], an[1]);
        bool ok = true;
        for (int ax = 0; ax < 2; ax++) {
            const double raw = v[ax];
            const int code = boundary_axis(v[ax], an[ax], a.dom.lo[ax], a.dom.hi[ax],
                                           a.dom.periodic[ax]);
            if (code) {
                atomicMin(&st->key, err_key(1 + ax, i, code));
                st->abort = 1;
                st->step = step;
                v[ax] = raw;
                ok = false;
                break;
            }
        }
        if (a.store_next) store2((P *)a.next, i, v[0], v[1]);
        if (!ok) continue;
        store2(pos, i, v[0], v[1]);
        store2(anchor, i, an[0], an[1]);
    }
    if (clamped) atomicAdd((unsigned long long *)&st->clamped, (unsigned long long)clamped);
}

// apply_boundaries (motion.py:355-430) of the swept proposals and commit
template <class P>
__global__ void __launch_bounds__(256)
k_commit(P *__restrict__ pos, P *__restrict__ anchor, const P *__restrict__ next, long long n,
         cs_domain dom, DevStatus *st, int step) {
    if (st->abort) return;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double v[2], an[2];
        load2(next, i, v[0], v[1]);
        if (!(isfinite(v[0]) && isfinite(v[1]))) {
            atomicMin(&st->key, err_key(0, i, CS_NONFINITE));
            st->abort = 1;
            st->step = step;
            continue;
        }
        load2(anchor, i, an[0], an[1]);
        bool ok = true;
        for (int ax = 0; ax < 2; ax++) {
            const int code = boundary_axis(v[ax], an[ax], dom.lo[ax], dom.hi[ax],
                                           dom.periodic[ax]);
            if (code) {
                atomicMin(&st->key, err_key(1 + ax, i, code));
                st->abort = 1;
                st->step = step;
                ok = false;
                break;
            }
        }
        if (!ok) continue;
        store2(pos, i, v[0], v[1]);
        store2(anchor, i, an[0], an[1]);
    }
}

}  // namespace cs

struct cs_sim {
    cs_ctx *ctx = nullptr;
    cs_sim_params p{};
    cs::BinGeom geom{};
    cs::PairTab pt{};
    cs::GridGeom gg{};
    cs_field_ops *ops = nullptr;
    int steps_done = 0;
    int64_t last_launches = 0;
    unsigned char bits[3] = {0, 0, 0};
    int engine = CS_ENGINE_DIRECT;
    cs_fast *fast = nullptr;
    int slab_g0 = 0, slab_g1 = 0, slab_grad_j0 = 0, slab_grad_rows = 0;  // slab field rows
    cs_ens *ens = nullptr;              // CTA engine: one realisation of the ensemble engine
    cs::Buf cta_drift, cta_lc, cta_type;  // its state rows the caller did not provide
    cs::Buf status;  // this simulation's DevStatus
    cs::DevStatus *dstat() { return status.as<cs::DevStatus>(); }
    // optional per-stage device timing (CUDA events on the step stream)
    int profiling = 0;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    size_t ev_next = 0;
    double stage_ms[CS_N_STAGES] = {};
    // sorted engine: the field solve runs on a high-priority side stream,
    // concurrently with the pair forces (which do not read the field)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int overlap = 0;
    int ensure_side() {
        if (side) return CS_OK;
        int least = 0, greatest = 0;
        CS_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        CS_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, greatest));
        CS_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        CS_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        return CS_OK;
    }
    cudaEvent_t next_event() {
        if (ev_next == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_next++];
    }
};

namespace cs {

int sim_create(cs_ctx *ctx, const cs_sim_params *p, cs_sim **out) {
    if (p->n < 0 || p->n >= (1LL << 31) - 1) {
        set_error("particle count out of range");
        return CS_ERR_PARAM;
    }
    auto *sim = new cs_sim();
    sim->ctx = ctx;
    sim->p = *p;
    // field solve (spectral passes + gradient) concurrent with the pair forces
    // on a high-priority side stream (measured at cfg3, round 2: 1.317 ->
    // 1.278 ms/step; CS_NO_OVERLAP=1 serialises them)
    sim->overlap = getenv("CS_NO_OVERLAP") ? 0 : 1;
    *out = sim;
    if (p->interaction == 1) {
        sim->geom = make_geom(p->domain, p->pairs.cell_cutoff);
        sim->pt = make_pairtab(p->pairs);
        CS_TRY(ctx->force.ensure(sizeof(double) * 2 * (size_t)(p->n > 0 ? p->n : 1)));
    }
    if (p->field_active || p->refresh_active) sim->gg = make_grid_geom(p->grid);
    for (int t = 0; t < 2; t++)
        sim->bits[t] = (unsigned char)((p->secretes[t] ? 1 : 0) | (p->consumes[t] ? 2 : 0));
    sim->bits[2] = 0;
    if (p->field_active) CS_TRY(field_ops_create(ctx, p->prec, &p->grid, p->d_c, p->dt, &sim->ops));
    // engine selection
    {
        const BinGeom g = make_geom(p->domain, p->interaction == 1 ? p->pairs.cell_cutoff : 1e300);
        const double per_cell = (double)p->n / ((double)g.n0 * (double)g.n1);
        bool want_sorted = p->engine == CS_ENGINE_SORTED ||
                           (p->engine == CS_ENGINE_AUTO && p->prec == CS_F32 &&
                            !p->store_samples && !p->store_next && !p->react &&
                            p->integrator == 0 && p->interaction != 2 &&
                            per_cell <= 4.0);
        if (want_sorted && (p->react || p->integrator != 0 || p->interaction == 2)) {
            set_error("reactions, the tamed integrator and hard spheres run on the direct engine only");
            return CS_ERR_PARAM;
        }
        if (want_sorted && p->prec != CS_F32) {
            set_error("the sorted engine stores binary32 records (prec must be CS_F32)");
            return CS_ERR_PARAM;
        }
        const bool grid = p->field_active || p->refresh_active;
        const bool want_cta =
            p->engine == CS_ENGINE_CTA ||
            (p->engine == CS_ENGINE_AUTO && p->prec == CS_F64 && p->n >= 1 && p->n <= 4096 &&
             (p->interaction == 0 || p->interaction == 1) && !p->store_next &&
             (!grid || (!p->grid.periodic && p->grid.n_c <= 64)) && !getenv("CS_NO_CTA"));
        if (want_cta) {
            const int rc = ens_create(ctx, p, 1, &sim->ens);
            if (rc == CS_OK) {
                sim->engine = CS_ENGINE_CTA;
            } else {
                ens_destroy(sim->ens);
                sim->ens = nullptr;
                if (p->engine == CS_ENGINE_CTA) return rc;  // asked for explicitly
            }
        }
        if (want_sorted) {
            sim->engine = CS_ENGINE_SORTED;
            sim->geom = g;
            sim->pt = make_pairtab(p->pairs);
            const GridGeom gg = make_grid_geom(p->grid);
            CS_TRY(fast_create(&sim->fast, p->n, g, p->field_active ? &gg : nullptr));
        }
    }
    CS_TRY(sim->status.ensure(sizeof(DevStatus)));
    DevStatus init{};
    init.key = ~0ULL;
    init.step = -1;
    CS_CUDA(cudaMemcpy(sim->status.p, &init, sizeof(init), cudaMemcpyHostToDevice));
    return CS_OK;
}

void sim_destroy(cs_sim *sim) {
    if (!sim) return;
    field_ops_destroy(sim->ops);
    fast_destroy(sim->fast);
    ens_destroy(sim->ens);
    sim->cta_drift.release();
    sim->cta_lc.release();
    sim->cta_type.release();
    sim->status.release();
    if (sim->side) {
        cudaStreamSynchronize(sim->side);
        cudaStreamDestroy(sim->side);
        cudaEventDestroy(sim->ev_fork);
        cudaEventDestroy(sim->ev_join);
    }
    for (cudaEvent_t e : sim->ev_pool) cudaEventDestroy(e);
    delete sim;
}

int sim_reset_status(cs_sim *sim) {
    if (sim->ens) CS_TRY(ens_reset_status(sim->ens));
    DevStatus init{};
    init.key = ~0ULL;
    init.step = -1;
    CS_CUDA(cudaMemcpyAsync(sim->status.p, &init, sizeof(init), cudaMemcpyHostToDevice,
                            sim->ctx->stream));
    CS_CUDA(cudaStreamSynchronize(sim->ctx->stream));
    sim->steps_done = 0;
    return CS_OK;
}

// Stage timing: a begin event before the stage's first launch and an end
// event after its last; durations are summed when the caller asks.
struct StageMark {
    cs_sim *sim;
    int stage;
    cudaEvent_t b = nullptr;
    StageMark(cs_sim *s, int st) : sim(s), stage(st) {
        if (sim->profiling) {
            b = sim->next_event();
            cudaEventRecord(b, sim->ctx->stream);
        }
    }
    ~StageMark() {
        if (sim->profiling) {
            cudaEvent_t e = sim->next_event();
            cudaEventRecord(e, sim->ctx->stream);
            sim->marks.push_back({stage, {b, e}});
        }
    }
};

int sim_collect_stage_times(cs_sim *sim) {
    if (sim->marks.empty()) return CS_OK;
    CS_CUDA(cudaStreamSynchronize(sim->ctx->stream));
    for (auto &m : sim->marks) {
        float ms = 0.f;
        CS_CUDA(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
        sim->stage_ms[m.first] += ms;
    }
    sim->marks.clear();
    sim->ev_next = 0;
    return CS_OK;
}

int sim_step(cs_sim *sim, const cs_sim_state *s, const void *xi, int64_t stride, int k,
             const double *u, int64_t u_stride) {
    if (sim->p.react && !u) {
        set_error("params.react is set: the step needs the reaction uniforms (cs_sim_step_react)");
        return CS_ERR_PARAM;
    }
    if (sim->p.interaction == 2 && (!s->next_pos || sim->p.n > 65536)) {
        set_error("hard spheres need the next_pos buffer and n <= 65536");
        return CS_ERR_PARAM;
    }
    if (sim->p.react && !s->type) {
        set_error("reactions need the species array");
        return CS_ERR_PARAM;
    }
    cs_ctx *ctx = sim->ctx;
    const cs_sim_params &p = sim->p;
    DevStatus *st = sim->dstat();
    const size_t es = p.prec == CS_F64 ? 8 : 4;
    const long long n = p.n;
    const int64_t l0 = ctx->launches;
    if (sim->engine == CS_ENGINE_CTA) {
        // one launch runs all k steps in shared memory (ensemble.cu, S = 1);
        // its xi / u layouts are (k, 1, n, 2) / (k, 1, n): caller strides of
        // 2n / n run as one call, others one call per step
        cs_ens_state es{};
        const size_t nn = (size_t)n;
        es.pos = (double *)s->pos;
        es.anchor = (double *)s->anchor;
        es.c = (double *)s->c;
        if (s->drift) {
            es.drift = s->drift;
        } else {
            if (!sim->cta_drift.p) {
                CS_TRY(sim->cta_drift.ensure(16 * nn));
                CS_CUDA(cudaMemsetAsync(sim->cta_drift.p, 0, 16 * nn, ctx->stream));
            }
            es.drift = sim->cta_drift.as<double>();
        }
        if (s->local_c) {
            es.local_c = s->local_c;
        } else {
            CS_TRY(sim->cta_lc.ensure(8 * nn));
            es.local_c = sim->cta_lc.as<double>();
        }
        if (s->type) {
            es.type = s->type;
        } else {
            if (!sim->cta_type.p) {
                CS_TRY(sim->cta_type.ensure(nn));
                CS_CUDA(cudaMemsetAsync(sim->cta_type.p, 0, nn, ctx->stream));
            }
            es.type = sim->cta_type.as<uint8_t>();
        }
        StageMark m(sim, CS_STAGE_FORCE);  // the whole fused step
        if (stride == 2 * n && (!u || u_stride == n)) {
            CS_TRY(ens_step(sim->ens, &es, (const double *)xi, u, k));
        } else {
            for (int kk = 0; kk < k; kk++)
                CS_TRY(ens_step(sim->ens, &es, (const double *)xi + (size_t)kk * stride,
                                u ? u + (size_t)kk * u_stride : nullptr, 1));
        }
        sim->steps_done += k;
        sim->last_launches = ctx->launches - l0;
        return CS_OK;
    }
    if (sim->engine == CS_ENGINE_SORTED) {
        FastStepCfg c;
        c.p = &p;
        c.g = sim->geom;
        c.pt = sim->pt;
        c.gg = sim->gg;
        c.ops = sim->ops;
        c.bits[0] = sim->bits[0];
        c.bits[1] = sim->bits[1];
        c.bits[2] = 0;
        if (!fast_imported(sim->fast)) {
            StageMark m(sim, CS_STAGE_BIN);
            CS_TRY(fast_import(ctx, sim->fast, p, s, sim->geom, sim->gg, sim->bits, st,
                               sim->steps_done));
        }
        // fork/join of the field solve (skipped while profiling, so that the
        // stage times stay additive)
        fast_begin_call(sim->fast);  // no increments gathered ahead by an earlier call
        const bool ov = p.field_active && sim->overlap && !sim->profiling &&
                        !fast_fused(sim->fast, p);  // the fused update needs the gradient
        if (ov) CS_TRY(sim->ensure_side());
        c.overlap = ov ? 1 : 0;
        for (int kk = 0; kk < k; kk++) {
            const int step = sim->steps_done + kk;
            const void *xik = (const char *)xi + (size_t)kk * (size_t)stride * es;
            if (p.field_active) {
                cudaStream_t main = ctx->stream;
                if (ov) {
                    CS_CUDA(cudaEventRecord(sim->ev_fork, main));
                    CS_CUDA(cudaStreamWaitEvent(sim->side, sim->ev_fork, 0));
                    ctx->stream = sim->side;
                }
                struct Restore {
                    cs_ctx *c;
                    cudaStream_t s;
                    ~Restore() { c->stream = s; }
                } restore{ctx, main};
                {
                    StageMark m(sim, CS_STAGE_SOLVE);
                    CS_TRY(fast_field(ctx, sim->fast, c, s, st, step));
                }
                {
                    StageMark m(sim, CS_STAGE_GRADIENT);
                    CS_TRY(launch_gradient(ctx, p.prec, s->c, sim->gg, s->grad, st, step,
                                           fast_rho_q(sim->fast)));
                }
                if (ov) CS_CUDA(cudaEventRecord(sim->ev_join, sim->side));
            }
            {
                StageMark m(sim, CS_STAGE_FORCE);
                CS_TRY(fast_particles(ctx, sim->fast, c, s, xik, st, step, 1));
            }
            if (ov) CS_CUDA(cudaStreamWaitEvent(ctx->stream, sim->ev_join, 0));
            {
                StageMark m(sim, CS_STAGE_UPDATE);
                CS_TRY(fast_particles(ctx, sim->fast, c, s, xik, st, step, 2));
            }
            {
                StageMark m(sim, CS_STAGE_BIN);
                // (large systems: the bucket sort also gathers the coming
                // step's increments into slot order when this call holds them)
                const void *xi_next =
                    kk + 1 < k ? (const char *)xik + (size_t)stride * es : nullptr;
                CS_TRY(fast_resort(ctx, sim->fast, n, p, sim->gg, sim->bits, 1, st, step,
                                   xi_next));
            }
            // in-cell id order + deposit for the next step's field
            StageMark m(sim, CS_STAGE_DEPOSIT);
            CS_TRY(fast_resort(ctx, sim->fast, n, p, sim->gg, sim->bits, 2, st, step));
        }
        sim->steps_done += k;
        sim->last_launches = ctx->launches - l0;
        return CS_OK;
    }
    // one step of the direct engine
    if (p.field_active && p.interaction == 1 && sim->overlap && !sim->profiling)
        CS_TRY(sim->ensure_side());
    auto one = [&](int kk) -> int {
        const int step = sim->steps_done + kk;
        const void *xik = (const char *)xi + (size_t)kk * (size_t)stride * es;
        // the cell list and the deposit bins come from the same start-of-step
        // positions: one binning pass builds both (the deposit is a gather
        // over its bins, deposit.cu)
        bool binned = false, dep_binned = false;
        if (p.field_active && p.interaction == 1) {
            StageMark m(sim, CS_STAGE_BIN);
            DepBin db;
            db.gg = sim->gg;
            db.kind = p.deposit_kind;
            for (int t = 0; t < 3; t++) db.route.bits[t] = sim->bits[t];
            CS_TRY(bin_particles(ctx, p.prec, s->pos, n, sim->geom, s->type, &db, &dep_binned));
            binned = true;
        }
        // the field chain (deposit, solve, gradient) only meets the pair
        // forces at the update: it runs on the side stream concurrently
        // (small systems leave most SMs idle in either)
        const bool ovd = binned && sim->overlap && !sim->profiling && sim->side;
        if (p.field_active) {
            cudaStream_t main = ctx->stream;
            if (ovd) {
                CS_CUDA(cudaEventRecord(sim->ev_fork, main));
                CS_CUDA(cudaStreamWaitEvent(sim->side, sim->ev_fork, 0));
                ctx->stream = sim->side;
            }
            struct Restore {
                cs_ctx *c;
                cudaStream_t s;
                ~Restore() { c->stream = s; }
            } restore{ctx, main};
            // a DCT-solved grid takes the solve's rhs from the CIC gather itself
            const bool rhs_fused = dep_binned && p.deposit_kind == CS_CIC &&
                                   sim->ops->kind == 1;
            {
                StageMark m(sim, CS_STAGE_DEPOSIT);
                RhsFuse rf;
                if (rhs_fused) {
                    rf.c = s->c;
                    rf.k = make_rhs_coef(sim->ops->dt, p.k_alpha, p.k_beta, p.gamma);
                    rf.rhs = (double *)sim->ops->rhs;
                }
                if (dep_binned)
                    CS_TRY(launch_deposit_binned(
                        ctx, p.prec, sim->gg, p.deposit_kind, p.kernel_h, p.kernel_cutoff,
                        ctx->starts.as<int>() + (size_t)sim->geom.n0 * sim->geom.n1, (int)n,
                        s->rho_a, s->rho_b, st, rhs_fused ? &rf : nullptr));
                else
                    CS_TRY(launch_deposit(ctx, p.prec, s->pos, s->type, n, sim->gg,
                                          p.deposit_kind, p.kernel_h, p.kernel_cutoff, sim->bits,
                                          s->rho_a, s->rho_b, st));
            }
            {
                StageMark m(sim, CS_STAGE_SOLVE);
                if (spectral_on(sim->ops)) {  // rhs fused into the spectral passes
                    CS_TRY(spectral_step_g(sim->ops, s->c, s->rho_a, s->rho_b, p.gamma,
                                           p.k_alpha, p.k_beta, st));
                } else {
                    if (!rhs_fused)
                        CS_TRY(field_rhs(sim->ops, s->c, s->rho_a, s->rho_b, p.k_alpha,
                                         p.k_beta, p.gamma, st));
                    CS_TRY(field_solve_rhs(sim->ops, s->c));
                }
            }
            {
                StageMark m(sim, CS_STAGE_GRADIENT);
                CS_TRY(launch_gradient(ctx, p.prec, s->c, sim->gg, s->grad, st, step));
            }
            if (ovd) CS_CUDA(cudaEventRecord(sim->ev_join, sim->side));
        }
        const double *force = nullptr;
        if (p.interaction == 1) {
            if (!binned) {
                StageMark m(sim, CS_STAGE_BIN);
                CS_TRY(bin_particles(ctx, p.prec, s->pos, n, sim->geom, s->type));
            }
            StageMark m(sim, CS_STAGE_FORCE);
            CS_TRY(launch_soft_forces(ctx, p.prec, s->pos, s->type, n, sim->geom, sim->pt,
                                      ctx->force.as<double>(), st));
            force = ctx->force.as<double>();
        }
        UpdateArgs a;
        a.xi = xik;
        a.pos = s->pos;
        a.anchor = s->anchor;
        a.next = s->next_pos;
        a.type = s->type;
        a.force = force;
        a.drift = s->drift;
        a.local_c = s->local_c;
        a.c = s->c;
        a.grad = s->grad;
        a.n = n;
        a.amp[0] = p.amp[0];
        a.amp[1] = p.amp[1];
        a.dt = p.dt;
        a.chi[0] = p.chi[0];
        a.chi[1] = p.chi[1];
        a.chi_pinned[0] = p.chi_pinned[0];
        a.chi_pinned[1] = p.chi_pinned[1];
        a.refresh = p.refresh_active;
        // Beta -> Alpha flips read this step's local concentration
        a.store_samples = (p.store_samples || (p.react && p.react_r_beta != 0.0)) && s->drift &&
                          s->local_c;
        a.store_next = p.store_next && s->next_pos;
        a.tamed = p.integrator == 1;
        a.propose_only = p.interaction == 2;
        a.dom = p.domain;
        a.gg = sim->gg;
        if (ovd && p.field_active) CS_CUDA(cudaStreamWaitEvent(ctx->stream, sim->ev_join, 0));
        if (n > 0) {
            StageMark m(sim, CS_STAGE_UPDATE);
            const int B = 256;
            if (p.prec == CS_F64)
                k_update<double><<<grid_for(n, B), B, 0, ctx->stream>>>(a, st, step);
            else
                k_update<float><<<grid_for(n, B), B, 0, ctx->stream>>>(a, st, step);
            CS_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        if (p.interaction == 2 && n > 0) {  // hard spheres (engine.py:384-386)
            StageMark m(sim, CS_STAGE_UPDATE);
            const double D[2] = {p.diffusion[0], p.diffusion[1]};
            CS_TRY(launch_hard_sphere(ctx, p.prec, s->next_pos, s->type, n, p.domain, p.hard_eps, D,
                                      nullptr));
            const int B = 256;
            if (p.prec == CS_F64)
                k_commit<double><<<grid_for(n, B), B, 0, ctx->stream>>>(
                    (double *)s->pos, (double *)s->anchor, (const double *)s->next_pos, n,
                    p.domain, st, step);
            else
                k_commit<float><<<grid_for(n, B), B, 0, ctx->stream>>>(
                    (float *)s->pos, (float *)s->anchor, (const float *)s->next_pos, n, p.domain,
                    st, step);
            CS_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        if (p.react) {  // fixed-step reactions after the boundaries (engine.py:387-393)
            StageMark m(sim, CS_STAGE_UPDATE);
            CS_TRY(launch_react(ctx, s->type, s->local_c, s->drift,
                                u + (size_t)kk * (size_t)u_stride, n, p.react_p_ab,
                                p.react_r_beta, p.dt, st));
        }
            return CS_OK;
    };
    for (int kk = 0; kk < k; kk++) CS_TRY(one(kk));
    sim->steps_done += k;
    sim->last_launches = ctx->launches - l0;
    return CS_OK;
}

int sim_status(cs_sim *sim, cs_status *out) {
    cs_ctx *ctx = sim->ctx;
    if (sim->ens) {
        CS_TRY(ens_status(sim->ens, out));
        out->steps_done = sim->steps_done;
        return CS_OK;
    }
    DevStatus d;
    CS_CUDA(cudaMemcpyAsync(&d, sim->status.p, sizeof(d), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    out->code = CS_OK;
    out->step = -1;
    out->particle = -1;
    out->axis = -1;
    if (d.key != ~0ULL) {
        const int rank = (int)(d.key >> 60);
        out->code = (int)(d.key & 7ULL);
        out->particle = (long long)((d.key >> 3) & ((1ULL << 57) - 1));
        out->axis = rank >= 1 ? rank - 1 : 0;
        out->step = d.step;
        if (out->code == CS_FIELD_NONFINITE || out->code == CS_DEPOSIT_OVERFLOW ||
            out->code == CS_SORT_OVERFLOW) {
            out->particle = -1;
            out->axis = -1;
        }
    }
    out->clamped = d.clamped;
    out->neg_mass_steps = d.neg_steps;
    out->first_neg_mass = d.first_neg;
    out->steps_done = sim->steps_done;
    out->react_high_count = (int64_t)d.react_high_n;
    out->react_high_max = 0.0;
    if (d.react_high_n) memcpy(&out->react_high_max, &d.react_high_bits, sizeof(double));
    return CS_OK;
}

}  // namespace cs

extern "C" int64_t cs_sim_launches(cs_sim *sim) { return sim ? sim->last_launches : 0; }

extern "C" int cs_sim_engine(cs_sim *sim) { return sim->engine; }

extern "C" int cs_sim_import(cs_sim *sim, const cs_sim_state *st) {
    if (sim->engine != CS_ENGINE_SORTED) return CS_OK;
    return cs::fast_import(sim->ctx, sim->fast, sim->p, st, sim->geom, sim->gg, sim->bits,
                           sim->dstat(), sim->steps_done);
}

extern "C" int cs_sim_export(cs_sim *sim, const cs_sim_state *st) {
    if (sim->engine != CS_ENGINE_SORTED) return CS_OK;
    return cs::fast_export(sim->ctx, sim->fast, sim->p, st, sim->gg);
}

extern "C" void *cs_sim_status_device(cs_sim *sim) { return sim ? sim->status.p : nullptr; }
extern "C" int64_t cs_sim_status_bytes(void) { return (int64_t)sizeof(cs::DevStatus); }

extern "C" int cs_sim_set_profiling(cs_sim *sim, int32_t on) {
    CS_TRY(cs::sim_collect_stage_times(sim));
    sim->profiling = on ? 1 : 0;
    for (double &v : sim->stage_ms) v = 0.0;
    return CS_OK;
}

extern "C" int cs_sim_stage_times(cs_sim *sim, double *ms, int32_t n) {
    CS_TRY(cs::sim_collect_stage_times(sim));
    for (int i = 0; i < n && i < CS_N_STAGES; i++) ms[i] = sim->stage_ms[i];
    return CS_OK;
}

// ---------------------------------------------------------------------------
// y-slab mode of the sorted engine: one rank's share of one
// system.  The step is split where records cross ranks: cs_slab_step_local
// (forces + update over the owned slots; leavers and ghost copies go to the
// outbox), the caller's exchange (slabs.py: NCCL all-to-all, or in-process
// copies), cs_slab_claim (received records), cs_slab_finish (bucket sort,
// owned range).
namespace {
cs::FastStepCfg slab_cfg(cs_sim *sim) {
    cs::FastStepCfg c;
    c.p = &sim->p;
    c.g = sim->geom;
    c.pt = sim->pt;
    c.gg = sim->gg;
    c.ops = sim->ops;
    c.bits[0] = sim->bits[0];
    c.bits[1] = sim->bits[1];
    c.bits[2] = 0;
    return c;
}
int slab_check(cs_sim *sim) {
    if (sim->engine != CS_ENGINE_SORTED) {
        cs::set_error("slab mode runs on the sorted engine (prec CS_F32, engine SORTED)");
        return CS_ERR_PARAM;
    }
    return CS_OK;
}
}  // namespace

extern "C" int cs_slab_config(cs_sim *sim, const int32_t *bounds, int32_t world, int32_t rank) {
    CS_TRY(slab_check(sim));
    if (sim->p.refresh_active && !sim->p.field_active) {
        cs::set_error("slab mode: a static field (refresh without field steps) is not supported");
        return CS_ERR_PARAM;
    }
    if (sim->p.field_active &&
        !(sim->ops && cs::spectral_on(sim->ops) && sim->p.grid.periodic && sim->p.prec == CS_F32 &&
          sim->p.deposit_kind == CS_CIC && cs::fast_slab_gather(sim->fast))) {
        cs::set_error("slab mode with the field: periodic binary32 grid of n = 2^k, CIC deposit, "
                      "periodic domain");
        return CS_ERR_PARAM;
    }
    return cs::fast_slab_config(sim->fast, bounds, world, rank, sim->p.n, sim->ctx->stream);
}

// The field of a slab rank: own grid rows [g0, g1) (a multiple of the
// spectral row blocking), the grid rows its particles deposit into (a
// window that includes the own rows) and the rows whose gradient its
// particles sample.
extern "C" int cs_slab_field_config(cs_sim *sim, int32_t g0, int32_t g1, int32_t dep_j0,
                                    int32_t dep_rows, int32_t grad_j0, int32_t grad_rows) {
    CS_TRY(slab_check(sim));
    sim->slab_g0 = g0;
    sim->slab_g1 = g1;
    sim->slab_grad_j0 = grad_j0;
    sim->slab_grad_rows = grad_rows;
    return cs::fast_slab_dep_window(sim->fast, dep_j0, dep_rows);
}

extern "C" void *cs_slab_rho(cs_sim *sim) { return cs::fast_rho_all(sim->fast); }

extern "C" int cs_slab_field_rows(cs_sim *sim, const cs_sim_state *st, void *spec,
                                  int32_t inverse) {
    CS_TRY(slab_check(sim));
    const cs_sim_params &p = sim->p;
    const double scale = (1.0 / 4194304.0) * (1.0 / (sim->gg.d0 * sim->gg.d1));
    return cs::spectral_slab_rows(sim->ops, (float *)st->c, (const int *)cs::fast_rho_all(sim->fast),
                                  p.gamma, p.k_alpha, p.k_beta, scale, sim->slab_g0,
                                  sim->slab_g1 - sim->slab_g0, spec, inverse, sim->dstat());
}

extern "C" int cs_slab_field_cols(cs_sim *sim, void *blocks, int32_t kx0, int32_t ncols,
                                  int32_t rp) {
    CS_TRY(slab_check(sim));
    return cs::spectral_slab_cols(sim->ops, blocks, kx0, ncols, rp, sim->dstat());
}

extern "C" int cs_slab_field_grad(cs_sim *sim, const cs_sim_state *st) {
    CS_TRY(slab_check(sim));
    return cs::launch_gradient_rows(sim->ctx, (const float *)st->c, sim->gg, (float *)st->grad,
                                    sim->dstat(), sim->steps_done, sim->slab_grad_j0,
                                    sim->slab_grad_rows, sim->slab_g0, sim->slab_g1);
}

extern "C" int cs_slab_import(cs_sim *sim, const cs_sim_state *st) {
    CS_TRY(slab_check(sim));
    return cs::fast_slab_import(sim->ctx, sim->fast, sim->p, st, sim->gg, sim->bits, sim->dstat(),
                                sim->steps_done);
}

extern "C" int cs_slab_step_local(cs_sim *sim, const cs_sim_state *st, const void *xi) {
    CS_TRY(slab_check(sim));
    const int64_t l0 = sim->ctx->launches;
    const cs::FastStepCfg c = slab_cfg(sim);
    CS_TRY(cs::fast_slab_reset_outbox(sim->ctx, sim->fast));
    CS_TRY(cs::fast_particles(sim->ctx, sim->fast, c, st, xi, sim->dstat(), sim->steps_done, 1));
    CS_TRY(cs::fast_particles(sim->ctx, sim->fast, c, st, xi, sim->dstat(), sim->steps_done, 2));
    sim->last_launches = sim->ctx->launches - l0;
    return CS_OK;
}

// the two halves of cs_slab_step_local as separate calls (part 1: outbox
// reset + pair forces, part 2: update), so that the caller can run the
// distributed field step -- which the forces do not read -- on another
// stream beside part 1 and join before part 2
extern "C" int cs_slab_step_part(cs_sim *sim, const cs_sim_state *st, const void *xi,
                                 int32_t part) {
    CS_TRY(slab_check(sim));
    if (part != 1 && part != 2) {
        cs::set_error("cs_slab_step_part: part is 1 (forces) or 2 (update)");
        return CS_ERR_PARAM;
    }
    const int64_t l0 = sim->ctx->launches;
    const cs::FastStepCfg c = slab_cfg(sim);
    if (part == 1) CS_TRY(cs::fast_slab_reset_outbox(sim->ctx, sim->fast));
    CS_TRY(cs::fast_particles(sim->ctx, sim->fast, c, st, xi, sim->dstat(), sim->steps_done,
                              part));
    sim->last_launches = (part == 1 ? 0 : sim->last_launches) + sim->ctx->launches - l0;
    return CS_OK;
}

extern "C" int cs_slab_outbox(cs_sim *sim, void **recs, int32_t **dest, int64_t *count) {
    CS_TRY(slab_check(sim));
    long long c = 0;
    CS_TRY(cs::fast_slab_outbox(sim->ctx, sim->fast, recs, dest, &c));
    *count = c;
    return CS_OK;
}

extern "C" int cs_slab_claim(cs_sim *sim, const void *recs, int64_t n) {
    CS_TRY(slab_check(sim));
    return cs::fast_slab_claim(sim->ctx, sim->fast, recs, n, sim->dstat(), sim->steps_done);
}

// Packed exchange (no host round trip in the step): cs_slab_exchange_cap
// gives every destination rank `seg` slots of the outbox and its own device
// counter; cs_slab_outbox_packed returns the device pointers (records
// [world][seg], counts [world]) -- the layout an equal-split all-to-all
// sends as it is; cs_slab_claim_packed claims what was received in the same
// layout.  A destination that gets more than seg records in a step stops the
// run with CS_SORT_OVERFLOW.  seg = 0 returns to the tagged outbox.
extern "C" int cs_slab_exchange_cap(cs_sim *sim, int64_t seg) {
    CS_TRY(slab_check(sim));
    return cs::fast_slab_exchange_cap(sim->fast, seg);
}

extern "C" int cs_slab_outbox_packed(cs_sim *sim, void **recs, int32_t **counts, int64_t *seg) {
    CS_TRY(slab_check(sim));
    long long s = 0;
    CS_TRY(cs::fast_slab_outbox_packed(sim->fast, recs, counts, &s));
    *seg = s;
    return CS_OK;
}

extern "C" int cs_slab_claim_packed(cs_sim *sim, const void *inbox, const int32_t *counts,
                                    int64_t seg) {
    CS_TRY(slab_check(sim));
    return cs::fast_slab_claim_packed(sim->ctx, sim->fast, inbox, counts, seg, sim->dstat(),
                                      sim->steps_done);
}

// Re-balancing: the per-row counts of the owned records (device int[n1]),
// then cs_slab_rebalance with the new bounds (every owned record routed
// under them into the outbox or claimed; the caller exchanges, claims and
// calls cs_slab_finish with advance = 0).
extern "C" int cs_slab_row_counts(cs_sim *sim, int32_t *hist) {
    CS_TRY(slab_check(sim));
    return cs::fast_slab_hist(sim->ctx, sim->fast, hist);
}

extern "C" int cs_slab_rebalance(cs_sim *sim, const int32_t *bounds) {
    CS_TRY(slab_check(sim));
    cs_fast *f = sim->fast;
    CS_TRY(cs::fast_slab_config(f, bounds, cs::fast_slab_world(f), cs::fast_slab_rank(f), sim->p.n,
                                sim->ctx->stream));
    CS_TRY(cs::fast_slab_reset_outbox(sim->ctx, f));
    const cs::FastStepCfg c = slab_cfg(sim);
    return cs::fast_particles(sim->ctx, f, c, nullptr, nullptr, sim->dstat(), sim->steps_done, 4);
}

static int slab_finish(cs_sim *sim, bool advance) {
    CS_TRY(slab_check(sim));
    const int64_t l0 = sim->ctx->launches;
    CS_TRY(cs::fast_slab_sort(sim->ctx, sim->fast, sim->p, sim->gg, sim->bits, sim->dstat(),
                              sim->steps_done));
    // the deposit of the new positions for the next step's field (own
    // particles, into this rank's deposit window)
    CS_TRY(cs::fast_resort(sim->ctx, sim->fast, sim->p.n, sim->p, sim->gg, sim->bits, 2,
                           sim->dstat(), sim->steps_done));
    if (advance) sim->steps_done += 1;
    sim->last_launches += sim->ctx->launches - l0;
    return CS_OK;
}

extern "C" int cs_slab_finish(cs_sim *sim) { return slab_finish(sim, true); }

extern "C" int cs_slab_finish_rebalance(cs_sim *sim) { return slab_finish(sim, false); }

extern "C" int cs_slab_range(cs_sim *sim, int64_t *lo, int64_t *hi) {
    CS_TRY(slab_check(sim));
    long long a = 0, b = 0;
    CS_TRY(cs::fast_slab_range_host(sim->ctx, sim->fast, &a, &b));
    *lo = a;
    *hi = b;
    return CS_OK;
}
