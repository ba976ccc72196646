/*
 * chemo_b200.h -- C ABI of the B200-native chemotaxis hot path.
 *
 * Every entry point takes plain device pointers, sizes and POD parameter
 * structs (no torch or CUDA types in the signatures; streams are passed as
 * void*).  The caller owns every state and output buffer; the library owns
 * only scratch (cell tables, sort buffers, FFT plans, status words) inside a
 * context.  A context is bound to one device and one stream and is not
 * thread-safe.
 *
 * Each function replaces one seam of the reference package (paths relative
 * to /root/reference/pkg/src/chemosim), see INTEGRATION.md for the binding:
 *
 *   cs_soft_forces       motion.py:248-265  soft_forces -> _soft_forces_fused (:165-245)
 *   cs_soft_force_pairs  (pair-set export of the same loop)
 *   cs_em_step           motion.py:268-282  em_step
 *   cs_apply_boundaries  motion.py:405-430  apply_boundaries -> _boundaries_kernel (:355-402)
 *   cs_deposit           coupling.py:141-187 deposit / deposit_both (_cic_scatter :113-138,
 *                                            _gauss_scatter_pair :77-110)
 *   cs_bilinear          coupling.py:216-262 _bilinear (interpolate / field_at / refresh)
 *   cs_gradient          field.py:242-245   gradient (d1x/d1y CSR matvecs, :128-137)
 *   cs_field_ops_*       field.py:173-201   build_operators + Operators.solve (:162-170)
 *   cs_field_step        field.py:209-239   step_field
 *   cs_sim_*             engine.py:369-387  Realisation._step_inner (fused, K steps)
 *
 * Status codes mirror the reference kernel's (motion.py:357-358); the
 * Python layer raises the reference's exception types and messages.
 */
#ifndef CHEMO_B200_H
#define CHEMO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 3

enum cs_code {
    CS_OK = 0,
    CS_NONFINITE = 1,        /* non-finite coordinate (motion.py:361-362) */
    CS_OVERSHOOT = 2,        /* overshoot beyond one width (motion.py:388-389) */
    CS_UNSETTLED = 3,        /* reflection failed to settle (motion.py:399-400) */
    CS_FIELD_NONFINITE = 4,  /* step_field non-finite (field.py:229-231) */
    CS_DEPOSIT_OVERFLOW = 5, /* sorted engine only: a cell holds more particles than its
                                int32 fixed-point deposit can sum exactly (no reference
                                counterpart; the direct engine has no such limit) */
    CS_SORT_OVERFLOW = 6,    /* sorted engine only: a bucket of 256 consecutive cells received
                                more records than its region holds (a local density far
                                above the run's initial one; no reference counterpart) */
    CS_ERR_CUDA = -1,
    CS_ERR_PARAM = -2,
    CS_ERR_NOMEM = -3,
    CS_ERR_CUFFT = -4
};

enum cs_prec { CS_F64 = 0, CS_F32 = 1 };
enum cs_deposit_kind { CS_GAUSSIAN = 0, CS_CIC = 1 };

typedef struct cs_ctx cs_ctx;
typedef struct cs_field_ops cs_field_ops;
typedef struct cs_sim cs_sim;

/* Box [lo, hi] per axis (spatial_index.py:20-62). */
typedef struct {
    double lo[2];
    double hi[2];
    int32_t periodic[2];
} cs_domain;

/* Pair table indexed t_i * 2 + t_j (t = 0 when the type array is NULL).
 * Homogeneous reference: all eps = epsilon, all cutoff = cutoff.
 * cell_cutoff sets the binning: n_ax = max(1, (int)(size_ax / cell_cutoff))
 * (motion.py:171-172); it must be >= every cutoff entry. */
typedef struct {
    double eps[4];
    double cutoff[4];
    double cell_cutoff;
} cs_pair_params;

/* Node-centred grid (field.py:33-80): flat l = j * n_c + i, x fastest. */
typedef struct {
    int32_t n_c;
    int32_t periodic;   /* 0 neumann, 1 periodic */
    double lo[2];
    double spacing[2];
} cs_grid;

int cs_abi_version(void);
const char *cs_last_error(void);

int cs_ctx_create(int device, void *stream, cs_ctx **out);
int cs_ctx_set_stream(cs_ctx *ctx, void *stream);
int cs_ctx_sync(cs_ctx *ctx);
int cs_ctx_destroy(cs_ctx *ctx);

/* out (n, 2) f64 = soft pair forces.  pos is (n, 2) f64 or f32 per prec. */
int cs_soft_forces(cs_ctx *ctx, int32_t prec, const void *pos,
                   const uint8_t *type, int64_t n, const cs_domain *dom,
                   const cs_pair_params *pp, double *out);

/* pairs (cap, 2) int64 (i, j) in the reference accumulation order (i
 * ascending, then ring cell, then j ascending); *count = total pairs (may
 * exceed cap, in which case nothing is written).  out may be NULL. */
int cs_soft_force_pairs(cs_ctx *ctx, int32_t prec, const void *pos,
                        const uint8_t *type, int64_t n, const cs_domain *dom,
                        const cs_pair_params *pp, int64_t *pairs, int64_t cap,
                        int64_t *count);

/* The reference's CellIndex (spatial_index.py:71-122): bucket (n, 2)
 * positions into cells of side >= cell_side (n_cells = max(1,
 * floor(size / cell_side)) per axis, closed upper edge).  Outputs: cell_xy
 * (n, 2) int32, order (n) int32 (ascending id inside a cell), starts
 * (n_cells_x * n_cells_y + 1) int32; n_cells (2) int32. */
int cs_cell_index(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n,
                  const cs_domain *dom, double cell_side, int32_t *cell_xy,
                  int32_t *order, int32_t *starts, int32_t *n_cells);

/* The reference's accumulate_forces (motion.py:107-161): soft pair forces
 * over an index built with any cell side (ring reach ceil(cutoff / eff)
 * per axis, the whole axis once 2 reach + 1 >= n on a periodic axis), single
 * epsilon / cutoff; same summation order and arithmetic.  out (n, 2) f64. */
int cs_index_forces(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n,
                    const int32_t *cell_xy, const int32_t *order,
                    const int32_t *starts, const cs_domain *dom,
                    const int32_t *n_cells, double epsilon, double cutoff,
                    double *out);

/* The reference's deposit_gather (coupling.py:190-213): node-centric
 * gaussian deposit, every node against every particle in index order (the
 * cross-check of the scatter path).  pos (n, 2) of the selected species in
 * prec; span = grid hi - lo (the periodic image span); out (n_c^2) f64. */
int cs_deposit_gather(cs_ctx *ctx, int32_t prec, const void *pos, int64_t n,
                      const cs_grid *grid, double span0, double span1, double h,
                      double cutoff, double *out);

/* out = ((pos + sqrt((2 D) dt) xi) + drift dt) + force dt; pos/xi/out in
 * prec, diffusion (n) f64, drift/force (n, 2) f64 (NULL = zero). */
int cs_em_step(cs_ctx *ctx, int32_t prec, const void *pos,
               const double *diffusion, const double *drift,
               const double *force, const void *xi, double dt, int64_t n,
               void *out);
/* tamed_step (motion.py:283-298): as cs_em_step with the interaction
 * increment (force dt) / (1 + ||force|| dt). */
int cs_tamed_step(cs_ctx *ctx, int32_t prec, const void *pos,
                  const double *diffusion, const double *drift,
                  const double *force, const void *xi, double dt, int64_t n,
                  void *out);

/* Resolves x (the proposal buffer) against the box in place, shifts anchor
 * on periodic wraps and, on success, copies x into positions (may be NULL).
 * Returns CS_OK or the reference status with the first offending particle
 * (non-finite: lowest index; otherwise lowest (axis, index)). */
int cs_apply_boundaries(cs_ctx *ctx, int32_t prec, void *x, void *anchor,
                        void *positions, int64_t n, const cs_domain *dom,
                        int64_t *bad_i, int32_t *bad_ax);

/* rho_a / rho_b (n_c^2, prec) are overwritten.  route[p]: 0 -> rho_a,
 * 1 -> rho_b, other -> skipped (NULL: every particle -> rho_a).  For CS_CIC
 * h and cutoff are ignored.  Returns CS_ERR_PARAM for a periodic gaussian
 * stamp wider than the grid (coupling.py:156-157). */
int cs_deposit(cs_ctx *ctx, int32_t prec, const void *pos,
               const uint8_t *route, int64_t n, const cs_grid *grid,
               int32_t kind, double h, double cutoff, void *rho_a,
               void *rho_b);

/* out (np, m) = bilinear samples of values (n_c^2, m); *clamped = number of
 * clamped coordinates (neumann only). */
int cs_bilinear(cs_ctx *ctx, int32_t prec, const void *points, int64_t np,
                const void *values, int32_t m, const cs_grid *grid, void *out,
                int64_t *clamped);

/* grad (n_c^2, 2) = (d1x c, d1y c). */
int cs_gradient(cs_ctx *ctx, int32_t prec, const void *c, const cs_grid *grid,
                void *grad);

/* Prepared implicit solver for (I - dt d_c L) x = rhs. */
int cs_field_ops_create(cs_ctx *ctx, int32_t prec, const cs_grid *grid,
                        double d_c, double dt, cs_field_ops **out);
int cs_field_ops_destroy(cs_field_ops *ops);
int cs_field_solve(cs_field_ops *ops, const void *rhs, void *out);

/* One semi-implicit step of c in place.  *nonfinite = 1 when the new field
 * has a non-finite value (c is then left unchanged); *neg_mass = weighted
 * mass of the negative entries (0 if none). */
int cs_field_step(cs_field_ops *ops, void *c, const void *rho_a,
                  const void *rho_b, double k_alpha, double k_beta,
                  double gamma, int32_t *nonfinite, double *neg_mass);

/* resolve_hard_sphere (motion.py:301-352) on proposals prop (n, 2) in
 * place: the pairs closer than eps at the start, in ascending (i, j) order,
 * each re-measured and pushed apart by 2 (eps - d) split by the
 * diffusivities (type (n,) u8 or NULL = all Alpha). */
int cs_resolve_hard_sphere(cs_ctx *ctx, int32_t prec, void *prop, const uint8_t *type,
                           int64_t n, const cs_domain *dom, double eps, double d_alpha,
                           double d_beta);

/* y = exp(x) on the device with the glibc-exact restatement (test seam). */
int cs_exp_batch(cs_ctx *ctx, const double *x, double *y, int64_t n);

/* Species switching, one Bernoulli trial per particle against the species
 * snapshot (reactions.py:43-81 fixed_step_reactions; with p_ab = 0 it is
 * beta_step_reactions, reactions.py:141-160): an Alpha (type 0) becomes Beta
 * when u < p_ab; a Beta becomes Alpha when r_beta != 0 and
 * u < (r_beta * max(local_c, 0)) * dt, and its drift row (if drift != NULL)
 * is zeroed.  type (n,) u8 in/out, local_c (n,) f64 (NULL: 0), u (n,) f64
 * uniforms on [0, 1).  flips[0] = Alpha -> Beta, flips[1] = Beta -> Alpha;
 * *high = the largest flip probability above 1 (0 if none), which the
 * reference clamps with a warning (the decisions are the same: u < 1). */
int cs_react(cs_ctx *ctx, uint8_t *type, const double *local_c, double *drift,
             const double *u, int64_t n, double p_ab, double r_beta, double dt,
             int64_t *flips, double *high);

/* ---------------------------------------------------------------------- */
/* Fused K-step pipeline (Realisation._step_inner, engine.py:369-387).      */
/* ---------------------------------------------------------------------- */
typedef struct {
    int64_t n;
    int32_t prec;            /* storage of pos/next/anchor/xi and grid arrays */
    int32_t n_types;         /* 1 (type may be NULL) or 2 */
    cs_domain domain;
    int32_t interaction;     /* 0 none, 1 soft */
    cs_pair_params pairs;
    double amp[2];           /* per-type sqrt((2 D) dt) */
    double dt;
    int32_t field_active;    /* deposit + step_field + gradient each step */
    int32_t refresh_active;  /* bilinear refresh of drift each step */
    cs_grid grid;
    double d_c, k_alpha, k_beta, gamma;
    int32_t deposit_kind;
    double kernel_h, kernel_cutoff;
    int32_t secretes[2];     /* type t deposits into rho_a */
    int32_t consumes[2];     /* type t deposits into rho_b */
    double chi[2];
    int32_t chi_pinned[2];   /* drift of type t is pinned to zero */
    int32_t store_samples;   /* write drift / local_c every step */
    int32_t store_next;      /* write next_pos every step */
    int32_t engine;          /* CS_ENGINE_AUTO / _DIRECT / _SORTED */
    /* fixed-step reactions after the boundaries of every step
     * (engine.py:389-393, reactions.py:43-81), DIRECT engine only: one
     * uniform per particle per step from cs_sim_step_react's u. */
    int32_t react;           /* 0 off, 1 fixed-step Bernoulli flips */
    double react_p_ab;       /* r_alpha * dt */
    double react_r_beta;     /* Beta -> Alpha rate per unit concentration */
    int32_t integrator;      /* 0 Euler-Maruyama, 1 tamed (motion.py:283-298) */
    /* interaction 2 = hard spheres (motion.py:301-352): no soft forces; the
     * proposals get one overlap-correction sweep before the boundaries.
     * DIRECT engine, n <= 65536 (O(n^2) scan), next_pos required. */
    double hard_eps;         /* the sphere diameter epsilon */
    double diffusion[2];     /* D per type (the sweep's split) */
    /* Performance mode (hard part 6), SORTED engine only: the step's
     * increments are consumed in the engine's storage-slot order (cell-sorted
     * records) instead of by particle id -- coalesced reads instead of a
     * random gather.  The increments are i.i.d. N(0,1), so the dynamics are
     * the same in distribution (parity tier T4), not trajectory for
     * trajectory.  0 = by id (the reference's layout). */
    int32_t xi_by_slot;
} cs_sim_params;

/* Engines.  DIRECT keeps the reference layout (rows in id order) and
 * supports every option.  SORTED (fp32 storage only) keeps cell-sorted
 * particle records inside the library: the caller's pos/anchor/rho arrays
 * are read on the first step (or cs_sim_import) and written back only by
 * cs_sim_export; drift/local_c/next_pos are not stored per step.  AUTO picks
 * SORTED for fp32 runs that need none of the per-step stores and whose cell
 * occupancy is low (<= 4 per cell), DIRECT otherwise. */
enum cs_engine { CS_ENGINE_AUTO = 0, CS_ENGINE_DIRECT = 1, CS_ENGINE_SORTED = 2,
                 CS_ENGINE_CTA = 3 };
/* CTA: a small binary64 system (n <= 4096, no grid or a neumann grid of
 * n_c <= 64, soft or no interaction, no next_pos store) held in ONE CTA's
 * shared memory for all k steps of a call -- the ensemble engine (cs_ens_*)
 * with one realisation: one launch per call instead of ~15 per step.  AUTO
 * picks it when the system fits (cs_ens_create succeeds), the DIRECT
 * engine otherwise; the results are the DIRECT engine's bit for bit. */

typedef struct {
    void *pos;               /* (n, 2) prec, in/out */
    void *next_pos;          /* (n, 2) prec, optional */
    void *anchor;            /* (n, 2) prec, in/out */
    uint8_t *type;           /* (n,) or NULL; switched in place by reactions */
    double *drift;           /* (n, 2) f64; read when refresh is off */
    double *local_c;         /* (n,) f64, optional */
    void *c;                 /* (n_c^2) prec */
    void *grad;              /* (n_c^2, 2) prec */
    void *rho_a, *rho_b;     /* (n_c^2) prec */
} cs_sim_state;

typedef struct {
    int32_t code;            /* enum cs_code */
    int32_t step;            /* failing step (relative to the first call since
                                the last reset), -1 if none */
    int64_t particle;
    int32_t axis;
    int64_t clamped;         /* clamped interpolation coordinates */
    int64_t neg_mass_steps;  /* steps with negative weighted mass < -1e-12 */
    double first_neg_mass;
    int64_t steps_done;
    int64_t react_high_count; /* particle-steps whose flip probability exceeded 1 */
    double react_high_max;    /* the largest such probability */
} cs_status;

int cs_sim_create(cs_ctx *ctx, const cs_sim_params *p, cs_sim **out);
int cs_sim_destroy(cs_sim *sim);
/* Enqueue k steps on the context stream (asynchronous).  xi points at the
 * Brownian increments of the first step, (n, 2) prec per step, successive
 * steps xi_stride elements apart. */
int cs_sim_step(cs_sim *sim, const cs_sim_state *st, const void *xi,
                int64_t xi_stride, int32_t k_steps);
/* cs_sim_step with the reaction uniforms of params.react: u points at the
 * (n,) f64 uniforms of the first step, successive steps u_stride apart. */
int cs_sim_step_react(cs_sim *sim, const cs_sim_state *st, const void *xi,
                      int64_t xi_stride, const double *u, int64_t u_stride,
                      int32_t k_steps);
/* Synchronise and read the status accumulated since the last reset. */
int cs_sim_status(cs_sim *sim, cs_status *out);
int cs_sim_reset_status(cs_sim *sim);
/* Engine in use (CS_ENGINE_DIRECT or CS_ENGINE_SORTED). */
int cs_sim_engine(cs_sim *sim);
/* SORTED engine: (re)load the internal state from the caller's arrays /
 * write it back (positions, anchors, deposited densities).  No-ops for
 * DIRECT.  Both are enqueued on the context stream. */
int cs_sim_import(cs_sim *sim, const cs_sim_state *st);
int cs_sim_export(cs_sim *sim, const cs_sim_state *st);
/* Launch count of the most recent cs_sim_step call (kernels of this
 * library; cuFFT's internal kernels are not counted). */
int64_t cs_sim_launches(cs_sim *sim);

/* Per-stage device time (CUDA events around each stage on the context
 * stream).  Enabling resets the accumulators. */
enum cs_stage {
    CS_STAGE_DEPOSIT = 0,   /* zero rho + deposit */
    CS_STAGE_SOLVE = 1,     /* rhs + implicit solve */
    CS_STAGE_GRADIENT = 2,  /* gradient + field checks */
    CS_STAGE_BIN = 3,       /* cell list */
    CS_STAGE_FORCE = 4,     /* pair forces */
    CS_STAGE_UPDATE = 5,    /* refresh + EM + boundaries */
    CS_N_STAGES = 6
};
int cs_sim_set_profiling(cs_sim *sim, int32_t on);
/* Device address and size of the simulation's status word, so a caller can
 * read it back asynchronously (e.g. into pinned memory) after every step. */
void *cs_sim_status_device(cs_sim *sim);
int64_t cs_sim_status_bytes(void);
int cs_sim_stage_times(cs_sim *sim, double *ms, int32_t n);

/* ---------------------------------------------------------------------- */
/* y-slab decomposition of one system over ranks (slabs.py).     */
/* The SORTED engine of rank r owns the global cell rows [bounds[r],        */
/* bounds[r+1]) (bounds: world + 1 ints from 0 to the cell-row count) and   */
/* keeps copies (ghosts) of the neighbours' boundary rows, so that every    */
/* owned particle sees its whole reference ring (motion.py:200-245): the    */
/* forces and the update are the single-domain engine's, bit for bit.  Per  */
/* step: cs_slab_step_local (forces + update over the owned slots; records  */
/* whose new row another rank owns, and ghost copies of records landing in  */
/* a boundary row, go to the outbox), the caller's exchange of the outbox   */
/* records (dest = rank | kind << 30, kind 0 migrant / 1 ghost; 16-byte     */
/* records), cs_slab_claim of the records received, cs_slab_finish (sort).  */
/* ---------------------------------------------------------------------- */
int cs_slab_config(cs_sim *sim, const int32_t *bounds, int32_t world, int32_t rank);
/* the owned rows and the ghost rows of the caller's global (id-ordered)
 * pos / anchor / type arrays -> the engine's records */
int cs_slab_import(cs_sim *sim, const cs_sim_state *st);
/* xi: the step's (n_global, 2) increments by particle id */
int cs_slab_step_local(cs_sim *sim, const cs_sim_state *st, const void *xi);
/* its two halves as separate calls: part 1 = outbox reset + pair forces, part
 * 2 = update (the caller may run the field step on another stream beside
 * part 1 and join before part 2) */
int cs_slab_step_part(cs_sim *sim, const cs_sim_state *st, const void *xi, int32_t part);
/* the outbox after cs_slab_step_local (device pointers; the count is read
 * back to the host: the exchange sizes its transfers with it) */
int cs_slab_outbox(cs_sim *sim, void **recs, int32_t **dest, int64_t *count);
int cs_slab_claim(cs_sim *sim, const void *recs, int64_t n);
int cs_slab_finish(cs_sim *sim);
/* packed exchange, no host round trip in the step: `seg` outbox slots and a
 * device counter per destination rank (0: back to the tagged outbox);
 * records [world][seg] and counts [world] as device pointers -- what an
 * equal-split all-to-all sends as it is -- and the claim of what was received
 * in the same layout.  More than seg records for one rank in a step stop the
 * run with CS_SORT_OVERFLOW. */
int cs_slab_exchange_cap(cs_sim *sim, int64_t seg);
int cs_slab_outbox_packed(cs_sim *sim, void **recs, int32_t **counts, int64_t *seg);
int cs_slab_claim_packed(cs_sim *sim, const void *inbox, const int32_t *counts, int64_t seg);
/* the owned slot range of the sorted records (tests) */
int cs_slab_range(cs_sim *sim, int64_t *lo, int64_t *hi);
/* The field of a slab rank (periodic binary32 grid, n_c = 2^k, CIC): it owns
 * the grid rows [g0, g1) (an even split, rows a multiple of the spectral
 * blocking); its particles deposit (int32 fixed point, exact) into the rows
 * dep_j0 .. dep_j0 + dep_rows - 1 (mod n_c; they include the own rows) --
 * the caller adds the window rows other ranks own into their owners' rows
 * (cs_slab_rho: the 2 n_c^2 int32 deposit grids) -- and sample the gradient
 * of the rows grad_j0 .. grad_j0 + grad_rows - 1 (computed from c rows one
 * wider, which the caller fetches from their owners).  The implicit solve:
 * cs_slab_field_rows (forward: own rows -> half spectrum [kx][g1 - g0]),
 * the caller's all-to-all transpose, cs_slab_field_cols (columns kx0 ..
 * kx0 + ncols of the blocks [rank][ncols][rp]), the transpose back,
 * cs_slab_field_rows (inverse: -> c own rows).  Every pass is the
 * single-domain solve's on the same rows / columns: the decomposed field is
 * the single-domain field bit for bit. */
int cs_slab_field_config(cs_sim *sim, int32_t g0, int32_t g1, int32_t dep_j0, int32_t dep_rows,
                         int32_t grad_j0, int32_t grad_rows);
void *cs_slab_rho(cs_sim *sim);
int cs_slab_field_rows(cs_sim *sim, const cs_sim_state *st, void *spec, int32_t inverse);
int cs_slab_field_cols(cs_sim *sim, void *blocks, int32_t kx0, int32_t ncols, int32_t rp);
int cs_slab_field_grad(cs_sim *sim, const cs_sim_state *st);
/* Re-balancing every M steps: the per-row counts of the owned records
 * (hist: device int32[cell rows], summed over ranks by the caller), then
 * cs_slab_rebalance with the new bounds (every owned record routed under
 * them: claimed, or into the outbox with the ghost copies of the new
 * boundary rows), the caller's exchange and cs_slab_claim, the new deposit /
 * gradient windows (cs_slab_field_config), cs_slab_finish_rebalance. */
int cs_slab_row_counts(cs_sim *sim, int32_t *hist);
int cs_slab_rebalance(cs_sim *sim, const int32_t *bounds);
int cs_slab_finish_rebalance(cs_sim *sim);

/* ---------------------------------------------------------------------- */
/* Ensembles of small realisations (run_ensemble, engine.py:455-484;       */
/* SURVEY 8f rank 1): one CTA per realisation, state in shared memory,      */
/* K steps per launch.  The realisations share one cs_sim_params (n =       */
/* particles per realisation; prec must be CS_F64; a grid, if any, must be  */
/* neumann with n_c <= 64; direct-engine semantics incl. react).            */
/* ---------------------------------------------------------------------- */
typedef struct cs_ens cs_ens;

typedef struct {
    double *pos;             /* (S, n, 2) in/out */
    double *anchor;          /* (S, n, 2) in/out */
    double *drift;           /* (S, n, 2) in/out */
    double *local_c;         /* (S, n) in/out */
    uint8_t *type;           /* (S, n) in/out */
    double *c;               /* (S, n_c^2) in/out; NULL without a grid */
} cs_ens_state;

int cs_ens_create(cs_ctx *ctx, const cs_sim_params *p, int32_t n_real, cs_ens **out);
int cs_ens_destroy(cs_ens *e);
/* xi: (k, S, n, 2) f64 Brownian increments; u: (k, S, n) f64 reaction
 * uniforms (required when p->react).  Asynchronous on the context stream. */
int cs_ens_step(cs_ens *e, const cs_ens_state *st, const double *xi, const double *u,
                int32_t k_steps);
/* Synchronise and read the per-realisation status: out[S]. */
int cs_ens_status(cs_ens *e, cs_status *out);
/* Recorded observables of every realisation (engine.py:343-349), device
 * arrays: n_alpha[S] (int64) and msd[S] (f64, numpy's pairwise mean of the
 * squared displacements from the start anchors, bit-identical). */
int cs_ens_observe(cs_ens *e, const cs_ens_state *st, int64_t *n_alpha, double *msd);

/* numpy's Generator(PCG64) on the device (csrc/rng.cu): n_streams streams
 * with state (n_streams, 4) u64 = {state_hi, state_lo, inc_hi, inc_lo}
 * (numpy's bit_generator.state), advanced in place.  out (k, n_streams, m)
 * f64: out[k][s] = stream s's next m draws of step k -- kind 0:
 * standard_normal (the ziggurat of numpy's distributions.c), kind 1:
 * random ([0, 1) doubles); bit-identical to numpy on the same host libm. */
int cs_rng_fill(cs_ctx *ctx, uint64_t *state, int32_t n_streams, int32_t kind, int32_t k,
                int64_t m, double *out);
/* y = log1p(x) with the glibc-exact restatement (test seam). */
/* Observables of a realisation in numpy's arithmetic (engine.py:230-235,
 * :317-352).  cs_msd: *out (device f64) = mean over particles of
 * (0 + dx^2) + dy^2, dx = pos - anchor in f64, numpy's pairwise reduction
 * order.  cs_hist2d: counts (device, bins x bins u64, [y bin][x bin]) of
 * numpy.histogram2d over the species (-1: all) with the given bin edges
 * (device f64, bins + 1 each, numpy's linspace); per_sample > 0: particles
 * i / per_sample belong to consecutive samples, counts (samples, bins, bins). */
int cs_msd(cs_ctx *ctx, int32_t prec, const void *pos, const void *anchor, int64_t n,
           double *out);
int cs_hist2d(cs_ctx *ctx, int32_t prec, const void *pos, const uint8_t *type, int64_t n,
              int32_t species, const double *edges_x, const double *edges_y, int32_t bins,
              int64_t per_sample, uint64_t *counts);

/* One numpy Generator(PCG64) stream drawn by the whole device, bit for bit:
 * state (host, 4 words) = {state_hi, state_lo, inc_hi, inc_lo} as numpy's
 * bit_generator.state; kind 0 = standard_normal (the ziggurat of
 * distributions.c), 1 = random; m values written to out (f64, or f32 when
 * f32 != 0).  On return state[0..1] is advanced by the raws consumed, so
 * the next draw (here or in numpy) continues the same stream.  Replaces
 * engine.py:272-275's sequential host draws (motion.py:277, reactions.py:57)
 * for large N. */
int cs_rng_fill_stream(cs_ctx *ctx, uint64_t *state, int32_t kind, int64_t m, int32_t f32,
                       void *out);

int cs_log1p_batch(cs_ctx *ctx, const double *x, double *y, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
