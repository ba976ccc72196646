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
// Per step (the field solve of fast_field runs on a side stream, overlapped
// with the forces):
//   k_fast_forces          pair forces over the 3x3 reference ring per sorted
//                          slot (binary32 prefilter in the candidate loop
//                          except across a periodic seam, exact test and pair
//                          terms in binary64, canonical id order); owners with
//                          too many hits, or at seams / walls, are deferred
//   k_fast_forces_generic  the deferred owners, one warp each
//   k_fast_update          bilinear drift, EM proposal with xi (by id, or by
//                          storage slot in the performance mode), boundaries
//                          with wrap counting, new cell key; the record is
//                          claimed into one of SUBB parts of its bucket
//                          (1024 consecutive cells) with a warp-aggregated
//                          atomic -- in slab mode migrants and ghost copies
//                          go to the outbox instead (slab_route)
//   k_scan                 exclusive scan of the bucket-part fills
//   k_bucket_sort          one CTA per bucket: counting sort of the claimed
//                          records into cells in shared memory, records of a
//                          cell ordered by id, next cell table
//   k_fast_deposit_rows    CIC deposit of the new positions for the next
//                          step's field: one CTA per grid row gathers the
//                          records of the cell rows under it (int32 fixed
//                          point, deterministic)
//
// Force summation order.  Records of a cell are stored in id order and the
// ring cells are visited in the reference's order, so the accepted pairs of
// an owner are summed in ascending particle id -- the reference's order
// (motion.py:206-243).  The force on every particle is therefore
// bit-identical to the reference arithmetic on the stored binary32
// coordinates.
//
// Deposits accumulate w * 2^22 (w = CIC corner weight) in int32 per node:
// integer addition is associative, so the field is run-to-run
// deterministic; resolution 2.4e-7 of a particle mass per contribution.
#include <stddef.h>
#include <stdlib.h>

#include <utility>
#include <vector>

#include "common.cuh"


namespace cs {

struct __align__(16) Rec {
    float x, y;
    unsigned int meta;  // id | type << 31
    short wx, wy;
};

constexpr double Q_SCALE = 4194304.0;  // 2^22
constexpr unsigned ID_MASK = 0x7fffffffu;
// bucket sort: buckets of BUCKET_CELLS consecutive cells (flat index)
constexpr int BUCKET_SHIFT = 10;
constexpr int BSORT_THREADS = 256;
constexpr int CELLS_PER_THREAD = (1 << BUCKET_SHIFT) / BSORT_THREADS;
static_assert(CELLS_PER_THREAD == 4, "k_bucket_sort owns 4 cells (one int4) per thread");
// every bucket has SUBB claim counters and region parts (a record picks one
// by its lane): the claims of a bucket spread over SUBB addresses, so the
// same-address atomic chains at the L2 are SUBB times shorter
#ifndef CS_SUBB
#define CS_SUBB 8
#endif
constexpr int SUBB = CS_SUBB;
constexpr int RPT = 4;  // records per k_bucket_sort thread held in registers
#ifndef CS_CLAIM_AGG
#define CS_CLAIM_AGG 1
#endif
static_assert(SUBB >= 1 && SUBB <= 32 && (SUBB & (SUBB - 1)) == 0, "SUBB: power of two <= 32");
constexpr int BUCKET_CELLS = 1 << BUCKET_SHIFT;

struct FastArgs {
    const Rec *rec;
    const int *starts;
    Rec *region;        // sub-bucket q = b * SUBB + s owns slots [q * cap, (q + 1) * cap)
    int *fill;          // records claimed per sub-bucket (zeroed by the bucket scan)
    long long cap;      // slots per sub-bucket region
    double2 *force;     // pair force per sorted slot (binary64)
    int *gen;           // slots the force kernel defers to k_fast_forces_generic
    int *gen_count;     // gen[0, *gen_count); reset by k_fast_update (fused: a memset)
    int *gen_dead;      // fused: the run state the force kernel saw at its start
    int debug;          // diagnostics bitmask (CS_FAST_DEBUG): 1 plain xi loads,
                        // 2 skip deposits, 64 no pair terms, 128 no candidate walk, 4 store records at the slot index
                        // without claims, 8 the same plus a fire-and-forget
                        // claim (4/8/32: timing only, wrong results)
    const float *xi;    // this step's (N, 2) increments, indexed by id (or slot: xi_slot)
    int xi_slot;        // performance mode: increments by storage slot (cs_sim_params.xi_by_slot)
    const float *grad;  // (n_c^2, 2)
    int *rho_q;         // 2 * m fixed-point deposits (a | b)
    long long n;
    BinGeom g;
    PairTab pt;
    GridGeom gg;
    ExactDiv eff0, eff1, gd0, gd1, sz0, sz1;
    double amp[2], dt, chi[2];
    int chi_pinned[2];
    int refresh, deposit, interact;
    unsigned bits[2];
    double half0, half1;
    float halff0, halff1, sizef0, sizef1;
    float cutf2[4];     // binary32 prefilter: cut2 * (1 + 1e-5)
    cs_domain dom;
    // y-slab mode (slabs.py): this rank owns the global cell rows
    // [b0, b1); its records are those plus copies of the neighbours' boundary
    // rows (ghosts); forces and the update run over the owned slot range
    const int *range;    // device [lo, hi) of the owned slots (nullptr: [0, n))
    int slab, rank, world, b0, b1, per_rows;
    const int *row_owner;  // device: owner rank of every global cell row
    const int *bounds;     // device: world + 1 row boundaries
    Rec *outbox;           // records for other ranks (migrants and ghosts)
    int *out_dest;         // their destination rank | kind << 30 (0 migrant, 1 ghost)
    int *out_count;        // [0]: records in the outbox; [1 + q]: records for rank q (packed)
    long long out_cap;
    long long out_seg;     // packed exchange: rank q's records at outbox[q * out_seg ...) (0: off)
};

// Random gather of the step's increments: keep the 80 MB slice in L2
// (evict_last) while the streamed arrays pass through (evict_first).
__device__ __forceinline__ float2 ld_evict_last(const float2 *p) {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(v.x), "=f"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// Launch parameters of the sorted-engine kernels live in constant memory: every thread
// reads the same words, and nothing has to be copied into registers or
// marshalled through the out-of-line helpers.
__constant__ FastArgs cA;

// minimum image with the |dx| <= L/2 shortcut: round(dx/L) is then +-0 and
// dx - L*(+-0) == dx exactly (dx is never -0.0: x - x = +0 under RN)
__device__ __noinline__ double min_image_slow(double dx, double size) {
    return dsub(dx, dmul(size, rint(ddiv(dx, size))));
}
__device__ __forceinline__ double min_image(double dx, double size, double half) {
    if (fabs(dx) <= half) return dx;
    return min_image_slow(dx, size);
}

// The pair term of an accepted pair (motion.py:240-243), out of line: it is
// reached ~1.1 times per particle and carries the exp and two divisions.
__device__ __noinline__ double2 pair_term(double dx0, double dx1, double r2, double eps) {
    const double rr = dsqrt(r2);
    const double s = -ddiv(cs_exp(-ddiv(rr, eps)), dmul(eps, rr));
    return make_double2(dmul(s, dx0), dmul(s, dx1));
}

struct PairRow {  // table row of this particle's type: index = partner type
    double cut2_0, cut2_1, eps_0, eps_1;
    float cf_0, cf_1;
    __device__ __forceinline__ double cut2(int tj) const { return tj ? cut2_1 : cut2_0; }
    __device__ __forceinline__ double eps(int tj) const { return tj ? eps_1 : eps_0; }
    __device__ __forceinline__ float cf(int tj) const { return tj ? cf_1 : cf_0; }
};

// Exact reference pair test (motion.py:231-239).  Returns r2 > 0 when
// accepted (displacement in dx0/dx1), 0 otherwise.  A binary32 prefilter
// runs first when neither axis wraps: then fx = xj - xf is one rounded
// binary32 op (exact under Sterbenz for nearby coordinates) and the
// squared distance carries a relative error ~2^-23, far inside the 1e-5
// margin of cf, so it never rejects an accepted pair.  A pair across a
// periodic seam skips it: (xj - x) - L cancels to ~cutoff from a binary32
// difference rounded at ~L, a relative error of ~1e-4 that would reject
// pairs at the cutoff edge (found at N = 10^7 by
// test_gpu_cfg3_pin.py::test_cfg3_field_off_sorted_equals_direct_bitwise_5_steps).
__device__ __forceinline__ double pair_test(float xjf, float yjf, float xf, float yf, double x,
                                            double y, float cf, double cut2, double &dx0,
                                            double &dx1) {
    const float fx = xjf - xf, fy = yjf - yf;
    const bool wraps = (cA.g.per0 && fabsf(fx) > cA.halff0) || (cA.g.per1 && fabsf(fy) > cA.halff1);
    if (!wraps && fmaf(fx, fx, fy * fy) > cf) return 0.0;
    dx0 = dsub((double)xjf, x);
    dx1 = dsub((double)yjf, y);
    if (cA.g.per0) dx0 = min_image(dx0, cA.g.size0, cA.half0);
    if (cA.g.per1) dx1 = min_image(dx1, cA.g.size1, cA.half1);
    const double r2 = dadd(dmul(dx0, dx0), dmul(dx1, dx1));
    if (r2 > cut2 || r2 == 0.0) return 0.0;
    return r2;
}

// Several accepted pairs in one cell: add them in ascending partner id.
__device__ __noinline__ double2 cell_ordered(const float4 *__restrict__ rec, long long t, int kb,
                                             int ke, int nacc, float xf, float yf, double x,
                                             double y, PairRow pr, double fx, double fy) {
    long long last = -1;
    for (int r = 0; r < nacc; r++) {
        unsigned best = 0xffffffffu;
        int bk = -1;
        for (int k = kb; k < ke; k++) {
            if (k == t) continue;
            const float4 q = __ldg(rec + k);
            const unsigned meta = __float_as_uint(q.z);
            const unsigned idk = meta & ID_MASK;
            if ((long long)idk <= last || idk >= best) continue;
            const int tj = (int)(meta >> 31);
            double d0, d1;
            if (pair_test(q.x, q.y, xf, yf, x, y, pr.cf(tj), pr.cut2(tj), d0, d1) > 0.0) {
                best = idk;
                bk = k;
            }
        }
        const float4 q = __ldg(rec + bk);
        const int tj = (int)(__float_as_uint(q.z) >> 31);
        double d0, d1;
        const double r2 = pair_test(q.x, q.y, xf, yf, x, y, pr.cf(tj), pr.cut2(tj), d0, d1);
        const double2 tt = pair_term(d0, d1, r2, pr.eps(tj));
        fx = dadd(fx, tt.x);
        fy = dadd(fy, tt.y);
        last = best;
    }
    return make_double2(fx, fy);
}

__device__ __forceinline__ int boundary_axis_wraps(double &v, int &w, double lo, double hi,
                                                   const ExactDiv &sz, int per) {
    const double size = sz.b;
    if (per) {
        const double k = floor_div(dsub(v, lo), sz);
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

__device__ __forceinline__ int wrap_index(double base, int n) {
    const int ib = (int)base;  // positions lie in [lo, hi]: base in [-1, n]
    if (ib >= 0 && ib < n) return ib;
    if (ib >= n && ib < 2 * n) return ib - n;
    if (ib < 0 && ib >= -n) return ib + n;
    return (int)pymod((long long)base, n);
}

// CIC corner nodes and weights in the reference arithmetic
// (coupling.py:119-135; for in-hull points identical to the bilinear
// stencil of coupling.py:221-258), u = (x - lo) / d with an exact division
struct Cic {
    int i00, i10, i01, i11;
    double w00, w10, w01, w11;
    double f0, f1;  // fractional offsets the weights derive from
};
__device__ __noinline__ Cic cic_stencil(double x, double y, GridGeom gg, ExactDiv d0,
                                        ExactDiv d1) {
    Cic c;
    const int nc = gg.n;
    const double u0 = ediv(dsub(x, gg.lo0), d0);
    const double u1 = ediv(dsub(y, gg.lo1), d1);
    int b0, b1, c0, c1;
    double f0, f1;
    if (gg.per) {
        const double base0 = floor(u0), base1 = floor(u1);
        f0 = dsub(u0, base0);
        f1 = dsub(u1, base1);
        b0 = wrap_index(base0, nc);
        b1 = wrap_index(base1, nc);
        c0 = b0 + 1 == nc ? 0 : b0 + 1;
        c1 = b1 + 1 == nc ? 0 : b1 + 1;
    } else {
        const double fl0 = floor(u0), fl1 = floor(u1);
        b0 = fl0 < 0.0 ? 0 : (fl0 > nc - 2 ? nc - 2 : (int)fl0);
        b1 = fl1 < 0.0 ? 0 : (fl1 > nc - 2 ? nc - 2 : (int)fl1);
        f0 = dsub(u0, (double)b0);
        f1 = dsub(u1, (double)b1);
        c0 = b0 + 1;
        c1 = b1 + 1;
    }
    const double g0 = dsub(1.0, f0), g1 = dsub(1.0, f1);
    c.f0 = f0;
    c.f1 = f1;
    c.w00 = dmul(g0, g1);
    c.w10 = dmul(f0, g1);
    c.w01 = dmul(g0, f1);
    c.w11 = dmul(f0, f1);
    c.i00 = b1 * nc + b0;
    c.i10 = b1 * nc + c0;
    c.i01 = c1 * nc + b0;
    c.i11 = c1 * nc + c0;
    return c;
}

// add of a fixed-point mass (>= 0; a non-finite coordinate, reported by the
// update, gives INT_MIN); true when it pushes the sum past INT_MAX
__device__ __forceinline__ bool add_overflows(int *p, int q) {
    const int old = atomicAdd(p, q);
    return q > 0 && old > INT_MAX - q;
}

// CIC deposit of one particle mass (int32 fixed point) with exact overflow
// detection
__device__ __forceinline__ bool cic_deposit_q(const Cic &c, int *__restrict__ out) {
    bool ovf = add_overflows(&out[c.i00], __double2int_rn(dmul(c.w00, Q_SCALE)));
    ovf |= add_overflows(&out[c.i10], __double2int_rn(dmul(c.w10, Q_SCALE)));
    ovf |= add_overflows(&out[c.i01], __double2int_rn(dmul(c.w01, Q_SCALE)));
    ovf |= add_overflows(&out[c.i11], __double2int_rn(dmul(c.w11, Q_SCALE)));
    return ovf;
}

__device__ __forceinline__ PairRow make_pair_row(int ti) {
    PairRow pr;
    pr.cut2_0 = ti ? cA.pt.cut2[2] : cA.pt.cut2[0];
    pr.cut2_1 = ti ? cA.pt.cut2[3] : cA.pt.cut2[1];
    pr.eps_0 = ti ? cA.pt.eps[2] : cA.pt.eps[0];
    pr.eps_1 = ti ? cA.pt.eps[3] : cA.pt.eps[1];
    pr.cf_0 = ti ? cA.cutf2[2] : cA.cutf2[0];
    pr.cf_1 = ti ? cA.cutf2[3] : cA.cutf2[1];
    return pr;
}

// Generic ring walk for the rare particles the fast path does not cover
// (cells on a periodic seam or wall, axes with < 3 cells, > ACC_MAX accepted
// pairs): per-cell loop in ring order, ascending id inside a cell.
__device__ __noinline__ double2 ring_forces_generic(const float4 *__restrict__ rec,
                                                    const int *__restrict__ starts, long long t,
                                                    float xf, float yf, double x, double y,
                                                    int cx, int cy, int n0, int n1,
                                                    PairRow pr) {
    double fx = 0.0, fy = 0.0;
    for (int c9 = 0; c9 < 9; c9++) {
        const int o1 = c9 / 3 - 1, o0 = c9 % 3 - 1;
        int g1 = cy + o1, g0 = cx + o0;
        if (cA.g.per1) {
            if ((n1 == 1 && o1 != 0) || (n1 == 2 && o1 == 1)) continue;
            g1 = g1 < 0 ? g1 + n1 : (g1 >= n1 ? g1 - n1 : g1);
        } else if (g1 < 0 || g1 >= n1) {
            continue;
        }
        if (cA.g.per0) {
            if ((n0 == 1 && o0 != 0) || (n0 == 2 && o0 == 1)) continue;
            g0 = g0 < 0 ? g0 + n0 : (g0 >= n0 ? g0 - n0 : g0);
        } else if (g0 < 0 || g0 >= n0) {
            continue;
        }
        const int f = g1 * n0 + g0;
        const int kb = starts[f], ke = starts[f + 1];
        int nacc = 0;
        for (int k = kb; k < ke; k++) {
            if (k == t) continue;
            const float4 r = __ldg(rec + k);
            const int tj = (int)(__float_as_uint(r.z) >> 31);
            double d0, d1;
            if (pair_test(r.x, r.y, xf, yf, x, y, pr.cf(tj), pr.cut2(tj), d0, d1) > 0.0)
                nacc++;
        }
        if (nacc > 0) {
            const double2 ff = cell_ordered(rec, t, kb, ke, nacc, xf, yf, x, y, pr, fx, fy);
            fx = ff.x;
            fy = ff.y;
        }
    }
    return make_double2(fx, fy);
}

// store a record at its claimed bucket slot (or flag the overflow)
__device__ __forceinline__ void claim_store(const FastArgs &a, DevStatus *st, int step, int b,
                                            int slot, float4 out) {
    if (slot < a.cap) {
        reinterpret_cast<float4 *>(a.region)[(long long)b * a.cap + slot] = out;
    } else {
        atomicMin(&st->key, err_key(3, b / SUBB, CS_SORT_OVERFLOW));
        st->abort = 1;
        st->step = step;
    }
}

// The update's inputs of one slot that do not depend on its pair force: the
// increment and the four gradient nodes of its bilinear stencil (the fused
// kernel issues these loads before its candidate walk)
struct UpdIn {
    float2 z, v00, v10, v01, v11;
    double bf0, bf1;
};

__device__ __forceinline__ UpdIn upd_load(const FastArgs &a, float4 mer, long long t, bool dead) {
    UpdIn u;
    const unsigned meta = __float_as_uint(mer.z);
    const int ti = (int)(meta >> 31);
    const unsigned id = meta & ID_MASK;
    // the particle's increment: xi[id] (the reference's layout: a random
    // gather, kept in L2 by evict_last), or xi[slot] in performance mode
    // (xi_by_slot: a coalesced stream)
    if (a.xi_slot)
        u.z = __ldcs(reinterpret_cast<const float2 *>(a.xi) + t);
    else if (a.debug & 1)
        u.z = __ldg(reinterpret_cast<const float2 *>(a.xi) + id);
    else
        u.z = ld_evict_last(reinterpret_cast<const float2 *>(a.xi) + id);
    const int pinned = ti ? a.chi_pinned[1] : a.chi_pinned[0];
    u.v00 = make_float2(0.f, 0.f);
    u.v10 = u.v01 = u.v11 = u.v00;
    u.bf0 = u.bf1 = 0.0;
    if (a.refresh && !dead && !pinned) {
        const Cic bst = cic_stencil((double)mer.x, (double)mer.y, a.gg, a.gd0, a.gd1);
        u.bf0 = bst.f0;
        u.bf1 = bst.f1;
        const float2 *g2 = reinterpret_cast<const float2 *>(a.grad);
        u.v00 = __ldg(g2 + bst.i00);
        u.v10 = __ldg(g2 + bst.i10);
        u.v01 = __ldg(g2 + bst.i01);
        u.v11 = __ldg(g2 + bst.i11);
    }
    return u;
}

// Drift refresh, EM proposal and boundaries of one slot given its pair force
// (zero without interactions): the new record and its cell (key, row).  A
// dead run (an earlier error) keeps the record unchanged.
__device__ __forceinline__ float4 upd_finish(const FastArgs &a, DevStatus *st, int step,
                                             float4 mer, const UpdIn &u, double fx, double fy,
                                             bool dead, bool live, int &key, int &cyn) {
    const unsigned meta = __float_as_uint(mer.z);
    const unsigned wbits = __float_as_uint(mer.w);
    const double x = (double)mer.x, y = (double)mer.y;
    const int ti = (int)(meta >> 31);
    const unsigned id = meta & ID_MASK;
    const int pinned = ti ? a.chi_pinned[1] : a.chi_pinned[0];
    const bool do_drift = a.refresh && !dead && !pinned;
    // ---- drift refresh at the start-of-step position (coupling.py:302-325)
    const double chi = ti ? a.chi[1] : a.chi[0];
    double dr0 = 0.0, dr1 = 0.0;
    if (do_drift) {
        Cic b;  // bilinear weights (coupling.py:251-254) from the kept offsets
        const double g0 = dsub(1.0, u.bf0), g1 = dsub(1.0, u.bf1);
        b.w00 = dmul(g0, g1);
        b.w10 = dmul(u.bf0, g1);
        b.w01 = dmul(g0, u.bf1);
        b.w11 = dmul(u.bf0, u.bf1);
        dr0 = dadd(dadd(dadd(dmul(b.w00, (double)u.v00.x), dmul(b.w10, (double)u.v10.x)),
                        dmul(b.w01, (double)u.v01.x)),
                   dmul(b.w11, (double)u.v11.x));
        dr1 = dadd(dadd(dadd(dmul(b.w00, (double)u.v00.y), dmul(b.w10, (double)u.v10.y)),
                        dmul(b.w01, (double)u.v01.y)),
                   dmul(b.w11, (double)u.v11.y));
        if (chi != 1.0) {
            dr0 = dmul(dr0, chi);
            dr1 = dmul(dr1, chi);
        }
    }
    // ---- EM proposal (motion.py:281-282)
    const double amp = ti ? a.amp[1] : a.amp[0];
    double v0 = dadd(dadd(dadd(x, dmul(amp, (double)u.z.x)), dmul(dr0, a.dt)), dmul(fx, a.dt));
    double v1 = dadd(dadd(dadd(y, dmul(amp, (double)u.z.y)), dmul(dr1, a.dt)), dmul(fy, a.dt));
    int w0 = (short)(wbits & 0xffffu), w1 = (short)(wbits >> 16);
    bool ok = !dead && live;
    if (ok && !(isfinite(v0) && isfinite(v1))) {
        atomicMin(&st->key, err_key(0, id, CS_NONFINITE));
        st->abort = 1;
        st->step = step;
        ok = false;
    }
    if (ok) {
        const double r0 = v0, r1 = v1;
        int code = boundary_axis_wraps(v0, w0, a.dom.lo[0], a.dom.hi[0], a.sz0,
                                       a.dom.periodic[0]);
        int ax = 0;
        if (!code) {
            code = boundary_axis_wraps(v1, w1, a.dom.lo[1], a.dom.hi[1], a.sz1,
                                       a.dom.periodic[1]);
            ax = 1;
        }
        if (code) {
            atomicMin(&st->key, err_key(1 + ax, id, code));
            st->abort = 1;
            st->step = step;
            if (ax == 0) v0 = r0;  // the raw proposal stays visible for the message
            else v1 = r1;
            ok = false;
        }
    }
    float4 out;
    if (dead) {
        out = mer;
    } else {
        out.x = (float)v0;
        out.y = (float)v1;
        out.z = mer.z;
        out.w = __uint_as_float(((unsigned)(w1 & 0xffff) << 16) | (unsigned)(w0 & 0xffff));
    }
    // ---- the cell of the stored (binary32) coordinate for the next step
    const double nx = (double)out.x, ny = (double)out.y;
    cyn = cell_axis_fast(ny, a.g.lo1, a.eff1, a.g.n1);
    key = cyn * a.g.n0 + cell_axis_fast(nx, a.g.lo0, a.eff0, a.g.n0);
    return out;
}

#ifndef CS_ACC_MAX
#define CS_ACC_MAX 8
#endif
constexpr int ACC_MAX = CS_ACC_MAX;  // accepted pairs buffered per particle
constexpr int WARPS_PER_BLOCK = 4;  // k_fast_forces block = 128 threads
constexpr int QCAP = 32 * ACC_MAX;  // pair-term queue per warp
// candidates of a ring the force kernel walks itself; beyond it the owner is
// deferred.  The walk stores the j-th prefilter hit of a lane at int index
// j * 32 + lane from the start of the warp's queue: (TOT_MAX - 1) hits stay
// inside ck + oj + tx + ty = 5.5 ACC_MAX rows of 32 ints
constexpr int TOT_MAX = ACC_MAX * 11 / 2;

// store to a shared-memory byte address (the walk's hit column: one 32-bit
// address register, no generic pointer to carry along)
__device__ __forceinline__ void sts_i32(unsigned addr, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v));
}

struct WarpQueue {  // (member order matters to the walk's stores: TOT_MAX)
    int ck[QCAP];                  // queue entry -> partner slot
    unsigned short oj[QCAP];       // queue entry -> owner term index j * 32 + lane
    double tx[QCAP], ty[QCAP];     // owner term index -> pair term (lane regions)
    float ox[32], oy[32];          // owner coordinates
    int oti[32];
};
static_assert(offsetof(WarpQueue, ox) >= sizeof(int) * 32 * (TOT_MAX - 1) && offsetof(WarpQueue, ck) == 0,
              "the walk's hit columns must end before the owner arrays");

// Pair forces of every sorted slot -> force[t] (binary64).
//
// Per warp iteration (32 consecutive slots, one per lane):
//  1. candidate walk, warp-uniform: each lane runs over its ring's three row
//     segments (the three cells of a ring row are consecutive in the cell
//     table, and inside a cell the records are in ascending id
//     (k_fast_cellfix), so slot order along the rows is exactly the
//     reference's ring order (o1, o0, id)); binary32 prefilter hits are
//     enqueued into the warp's queue at ballot/popc positions, tagged with
//     the owner's term index j * 32 + lane (j = the owner's j-th hit; lanes
//     of one j side by side: the owners read their terms without bank
//     conflicts, 8-way with lane * ACC_MAX + j);
//  2. the queue is evaluated ~1/32 per lane: exact reference test (binary64)
//     and pair term, written to the owner's term index (+0.0 for prefilter
//     false positives: the owners' sums start at +0.0 and so are never -0.0,
//     and x + 0.0 == x);
//  3. each owner adds its terms in j order = canonical order.
// Ring cells on a periodic seam or a wall, axes with < 5 cells, and lanes
// with > ACC_MAX hits are deferred to k_fast_forces_generic (generic walk).
//
// FUSED: the update of every non-deferred slot runs in the same iteration
// (its increment and gradient loads issued before the walk, so they arrive
// during it); the pair force never goes to memory.  The deferred owners are
// updated by k_fast_forces_generic<true>.
template <bool FUSED>
__global__ void __launch_bounds__(128, 5)  // 96 regs: measured best (4: 560, 6: 513 us)
k_fast_forces(DevStatus *st, int step) {
    const FastArgs &a = cA;
    __shared__ WarpQueue wq_all[WARPS_PER_BLOCK];
    WarpQueue &wq = wq_all[threadIdx.x >> 5];
    int *wq_ck = reinterpret_cast<int *>(&wq);  // ck, running on into oj / tx / ty (TOT_MAX)
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;  // lanes below this one
    const bool dead = st->abort != 0;
    const float4 *__restrict__ rec = reinterpret_cast<const float4 *>(a.rec);
    const int n0 = a.g.n0, n1 = a.g.n1;
    // persistent grid, warps sweep the slots together (a narrow processing
    // front: ring rows are shared by concurrently running warps)
    const long long wstride = (long long)gridDim.x * blockDim.x;
    const long long s_lo = a.range ? a.range[0] : 0, s_hi = a.range ? a.range[1] : a.n;
    // FUSED: the previous iteration's bucket claim (stored once this
    // iteration's loads are in flight)
    const int wpart = (threadIdx.x >> 5) & (SUBB - 1);
    bool p_have = false, p_live = false;
    int p_leader = 0, p_rank = 0, p_ret = 0, p_b = 0;
    float4 p_out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FUSED && blockIdx.x == 0 && threadIdx.x == 0) *a.gen_dead = dead ? 1 : 0;
    for (long long base = s_lo + (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
         base < s_hi; base += wstride) {
        const long long t = base + lane;
        const int t32 = (int)t;
        const bool live = t < s_hi;
        float4 mer = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live) mer = __ldg(rec + t);
        UpdIn u;
        if (FUSED) {
            u = upd_load(a, mer, live ? t : s_lo, dead);
            if (p_have) {
                const int basev = __shfl_sync(0xffffffffu, p_ret, p_leader);
                if (p_live) claim_store(a, st, step, p_b, basev + p_rank, p_out);
            }
        }
        // (a lane past the range never hits: its d2 is NaN, above every cutoff's bit pattern)
        const float xf = live ? mer.x : __int_as_float(0x7fc00000), yf = mer.y;
        const double x = (double)xf, y = (double)yf;
        const int ti = (int)(__float_as_uint(mer.z) >> 31);
        const float cf0 = ti ? a.cutf2[2] : a.cutf2[0];
        const float cf1 = ti ? a.cutf2[3] : a.cutf2[1];
        double fx = 0.0, fy = 0.0;
        int nacc = 0, tot = 0;
        bool generic = false;
        // ring row segments, compacted to the non-empty ones: the walk visits
        // [k, kend), then [nb1, ne1), then [nb2, ne2)
        int k = t32, kend = t32, nb1 = t32, ne1 = t32, nb2 = t32, ne2 = t32;
        int cx = 0, cy = 0;
        if (live && !dead && a.interact) {
            cx = cell_axis_fast(x, a.g.lo0, a.eff0, n0);
            cy = cell_axis_fast(y, a.g.lo1, a.eff1, n1);
            generic = cx < 1 || cx + 2 > n0 || cy < 1 || cy + 2 > n1 || n0 < 5 || n1 < 5;
            if (!generic) {
                int sa[3], se[3];
#pragma unroll
                for (int r = 0; r < 3; r++) {  // all 6 table loads issued together
                    const int f = (cy + r - 1) * n0 + cx - 1;
                    sa[r] = __ldg(a.starts + f);
                    se[r] = __ldg(a.starts + f + 3);
                }
                tot = (se[0] - sa[0]) + (se[1] - sa[1]) + (se[2] - sa[2]);
                if (a.debug & 128) tot = 0;  // timing diagnostic: no walk
                if (tot > TOT_MAX) {  // dense ring: the warp-per-owner pass (see the walk)
                    generic = true;
                    tot = 0;
                }
#pragma unroll
                for (int r = 2; r >= 0; r--) {  // push front, skipping empty rows
                    if (se[r] > sa[r]) {
                        nb2 = nb1;
                        ne2 = ne1;
                        nb1 = k;
                        ne1 = kend;
                        k = sa[r];
                        kend = se[r];
                    }
                }
            }
        }
        // ---- 1. candidate walk (warp-uniform trip count): a prefilter hit
        // goes into the lane's own column of the queue's slot array,
        // ck[j * 32 + lane] = partner slot of the lane's j-th hit.  A hit is
        // 0 < d2 <= c, tested as one unsigned compare of the bit patterns
        // (d2 >= +0 and c > 0: binary32 order is integer order, and
        // bits(+0) - 1 wraps to the top): d2 == 0 is the owner itself -- also
        // the record a lane past its own tot re-reads -- or a partner at the
        // same stored coordinates, whose exact r2 == 0 the reference skips
        // (motion.py:238).  The store is not bounded by ACC_MAX: a ring has at
        // most TOT_MAX candidates, and rows 8 .. TOT_MAX - 1 of the lane's
        // column fall into oj / tx / ty of the warp's own queue, which are
        // written and read only after the walk (owners with more than
        // ACC_MAX hits are deferred below).
        const int c0m = cf0 > 0.f ? __float_as_int(cf0) - 1 : 0;
        const int c1m = cf1 > 0.f ? __float_as_int(cf1) - 1 : 0;
        const unsigned qp0 = (unsigned)__cvta_generic_to_shared(wq_ck + lane);
        unsigned qp = qp0;  // shared-memory byte address of the lane's next hit
        const int totmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)tot);
#pragma unroll 2
        for (int j = 0; j < totmax; j += 2) {
            const int ka = k;
            if (++k == kend) {
                k = nb1;
                kend = ne1;
                nb1 = nb2;
                ne1 = ne2;
            }
            const int kb = k;
            if (++k == kend) {
                k = nb1;
                kend = ne1;
                nb1 = nb2;
                ne1 = ne2;
            }
            const float4 qa = __ldg(rec + (j < tot ? ka : t32));
            const float4 qb = __ldg(rec + (j + 1 < tot ? kb : t32));
            const float dax = qa.x - xf, day = qa.y - yf;
            const float dbx = qb.x - xf, dby = qb.y - yf;
            const unsigned ca = (unsigned)((__float_as_int(qa.z) < 0) ? c1m : c0m);
            const unsigned cb = (unsigned)((__float_as_int(qb.z) < 0) ? c1m : c0m);
            const bool ha = (unsigned)(__float_as_int(fmaf(dax, dax, day * day)) - 1) <= ca;
            const bool hb = (unsigned)(__float_as_int(fmaf(dbx, dbx, dby * dby)) - 1) <= cb;
            if (ha) {
                sts_i32(qp, ka);
                qp += 128;
            }
            if (hb) {
                sts_i32(qp, kb);
                qp += 128;
            }
        }
        asm volatile("" ::: "memory");  // the hit stores above precede the queue reads below
        nacc = (int)(qp - qp0) >> 7;
        // the hits compacted level by level into queue entries (in place:
        // entry e <= j * 32 + lane, and a level is read before it is written),
        // each tagged with the owner's term index j * 32 + lane
        int qn = 0;  // queue length (warp-uniform)
        {
            const int nq = nacc < ACC_MAX ? nacc : ACC_MAX;
            const int lev = (int)__reduce_max_sync(0xffffffffu, (unsigned)nq);
            for (int j = 0; j < lev; j++) {
                const bool has = j < nq;
                const unsigned m = __ballot_sync(0xffffffffu, has);
                const int kk = has ? wq.ck[j * 32 + lane] : 0;
                __syncwarp();
                if (has) {
                    const int e = qn + __popc(m & lt);
                    wq.ck[e] = kk;
                    wq.oj[e] = (unsigned short)(j * 32 + lane);
                }
                qn += __popc(m);
            }
        }
        if (nacc > ACC_MAX) generic = true;  // its queued terms are computed, not used
        if (generic) {
            // deferred to k_fast_forces_generic (seam / wall / dense owners:
            // ~0.15 % at cfg3), so that no warp of this kernel serialises on
            // one lane's generic walk
            a.gen[atomicAdd(a.gen_count, 1)] = t32;
            nacc = 0;
        }
        // ---- 2. queue evaluation
        if (qn > 0) {
            wq.ox[lane] = xf;
            wq.oy[lane] = yf;
            wq.oti[lane] = ti;
            __syncwarp();
            for (int e = lane; e < qn; e += 32) {
                const int o = wq.oj[e];
                const int ow = o & 31;
                const float4 q = __ldg(rec + wq.ck[e]);
                const int tt = wq.oti[ow] * 2 + (int)(__float_as_uint(q.z) >> 31);
                // interior ring (fast path): |dx| <= 2 cells < L/2, so the
                // minimum image is the identity (motion.py:231-236)
                const double d0 = dsub((double)q.x, (double)wq.ox[ow]);
                const double d1 = dsub((double)q.y, (double)wq.oy[ow]);
                const double r2 = dadd(dmul(d0, d0), dmul(d1, d1));
                double2 term = make_double2(0.0, 0.0);
                if (!(r2 > a.pt.cut2[tt] || r2 == 0.0) && !(a.debug & 64))
                    term = pair_term(d0, d1, r2, a.pt.eps[tt]);
                wq.tx[o] = term.x;
                wq.ty[o] = term.y;
            }
            __syncwarp();
            // ---- 3. owners add their terms in canonical order
            for (int j = 0; j < nacc; j++) {
                fx = dadd(fx, wq.tx[j * 32 + lane]);
                fy = dadd(fy, wq.ty[j * 32 + lane]);
            }
            __syncwarp();
        }
        if (FUSED) {
            const bool own = live && !generic;
            int key, cyn;
            const float4 out = upd_finish(a, st, step, mer, u, fx, fy, dead, own, key, cyn);
            p_b = (key >> BUCKET_SHIFT) * SUBB + wpart;
            const unsigned peers = __match_any_sync(0xffffffffu, own ? p_b : -1 - lane);
            p_leader = __ffs(peers) - 1;
            p_rank = __popc(peers & lt);
            if (own && lane == p_leader) p_ret = atomicAdd(&a.fill[p_b], __popc(peers));
            p_live = own;
            p_have = true;
            p_out = out;
        } else if (live && !generic) {
            a.force[t] = make_double2(fx, fy);
        }
    }
    if (FUSED && p_have) {
        const int basev = __shfl_sync(0xffffffffu, p_ret, p_leader);
        if (p_live) claim_store(a, st, step, p_b, basev + p_rank, p_out);
    }
}

// The owners k_fast_forces deferred (seam / wall / small-grid / dense): a
// warp per owner, lane c9 < 9 walks ring cell c9 (reference order o1 outer,
// o0 inner, with the periodic de-duplication and wall skips of
// motion.py:206-222).  Records inside a cell are in ascending id, so a
// lane's accepted pairs are already in the reference order; the exact test
// (pair_test: minimum image with rint) and the pair term are the reference's.
// Lane 0 then adds the terms cell by cell.  A cell with more than GEN_K
// accepted pairs sends the owner through ring_forces_generic instead.
// the fused update of one deferred owner (one thread) and its bucket claim
__device__ __noinline__ void generic_claim(const FastArgs &a, DevStatus *st, int step, float4 me,
                                           double fx, double fy, bool dead, int q) {
    const int t = a.gen[q];
    const UpdIn u = upd_load(a, me, t, dead);
    int key, cyn;
    const float4 out = upd_finish(a, st, step, me, u, fx, fy, dead, true, key, cyn);
    const int pb = (key >> BUCKET_SHIFT) * SUBB + (q & (SUBB - 1));
    claim_store(a, st, step, pb, atomicAdd(&a.fill[pb], 1), out);
}
constexpr int GEN_K = 8;
//
// FUSED: lane 0 then updates the owner (the fused kernel's update, with the
// run state that kernel saw at its start) and claims its record.
template <bool FUSED>
__global__ void __launch_bounds__(128) k_fast_forces_generic(DevStatus *st, int step) {
    const FastArgs &a = cA;
    const bool dead = FUSED ? *a.gen_dead != 0 : st->abort != 0;
    if (!FUSED && dead) return;
    const int cnt = *a.gen_count;
    const float4 *__restrict__ rec = reinterpret_cast<const float4 *>(a.rec);
    const int lane = threadIdx.x & 31;
    const int n0 = a.g.n0, n1 = a.g.n1;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < cnt;
         q += (gridDim.x * blockDim.x) >> 5) {
        const int t = a.gen[q];
        const float4 me = __ldg(rec + t);
        if (FUSED && dead) {  // an earlier step failed: the record stays as it is
            if (lane == 0) generic_claim(a, st, step, me, 0.0, 0.0, true, q);
            continue;
        }
        const double x = (double)me.x, y = (double)me.y;
        const int cx = cell_axis_fast(x, a.g.lo0, a.eff0, n0);
        const int cy = cell_axis_fast(y, a.g.lo1, a.eff1, n1);
        const PairRow pr = make_pair_row((int)(__float_as_uint(me.z) >> 31));
        double tx[GEN_K], ty[GEN_K];
        int nt = 0;
        bool over = false;
        if (lane < 9) {
            const int o1 = lane / 3 - 1, o0 = lane % 3 - 1;
            int g1 = cy + o1, g0 = cx + o0;
            bool ok = true;
            if (a.g.per1) {
                if ((n1 == 1 && o1 != 0) || (n1 == 2 && o1 == 1)) ok = false;
                g1 = g1 < 0 ? g1 + n1 : (g1 >= n1 ? g1 - n1 : g1);
            } else if (g1 < 0 || g1 >= n1) {
                ok = false;
            }
            if (a.g.per0) {
                if ((n0 == 1 && o0 != 0) || (n0 == 2 && o0 == 1)) ok = false;
                g0 = g0 < 0 ? g0 + n0 : (g0 >= n0 ? g0 - n0 : g0);
            } else if (g0 < 0 || g0 >= n0) {
                ok = false;
            }
            if (ok) {
                const int f = g1 * n0 + g0;
                const int kb = a.starts[f], ke = a.starts[f + 1];
                for (int k = kb; k < ke; k++) {
                    if (k == t) continue;
                    const float4 r = __ldg(rec + k);
                    const int tj = (int)(__float_as_uint(r.z) >> 31);
                    double d0, d1;
                    const double r2 = pair_test(r.x, r.y, me.x, me.y, x, y, pr.cf(tj),
                                                pr.cut2(tj), d0, d1);
                    if (r2 > 0.0) {
                        if (nt == GEN_K) {
                            over = true;
                            break;
                        }
                        const double2 tv = pair_term(d0, d1, r2, pr.eps(tj));
#pragma unroll
                        for (int u = 0; u < GEN_K; u++)
                            if (u == nt) {
                                tx[u] = tv.x;
                                ty[u] = tv.y;
                            }
                        nt++;
                    }
                }
            }
        }
        if (__any_sync(0xffffffffu, over)) {
            if (lane == 0) {
                const double2 fr = ring_forces_generic(rec, a.starts, t, me.x, me.y, x, y, cx, cy,
                                                       n0, n1, pr);
                if (FUSED) generic_claim(a, st, step, me, fr.x, fr.y, false, q);
                else a.force[t] = fr;
            }
            continue;
        }
        double fx = 0.0, fy = 0.0;
        const int ntmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nt);
        for (int c9 = 0; c9 < 9; c9++) {
            const int m = __shfl_sync(0xffffffffu, nt, c9);
#pragma unroll
            for (int u = 0; u < GEN_K; u++) {
                if (u >= ntmax) break;
                const double vx = __shfl_sync(0xffffffffu, tx[u], c9);
                const double vy = __shfl_sync(0xffffffffu, ty[u], c9);
                if (u < m) {
                    fx = dadd(fx, vx);
                    fy = dadd(fy, vy);
                }
            }
        }
        if (lane == 0) {
            if (FUSED) generic_claim(a, st, step, me, fx, fy, false, q);
            else a.force[t] = make_double2(fx, fy);
        }
    }
}

// Per sorted slot: drift refresh, EM proposal, boundaries, new cell key and
// rank, deposit of the new position for the next step's field.
#ifndef CS_UPDATE_MINB
#define CS_UPDATE_MINB 4  // measured with the bucket claims: 4: 320 us, 5: 327 (spills), 6: 380
#endif
// slab mode: a record for another rank (a migrant to the owner of its new
// row, or a ghost copy for a neighbour of that owner); a ghost for this rank
// itself is claimed here directly
__device__ __noinline__ void slab_emit(const FastArgs &a, DevStatus *st, int step, float4 out,
                                       int key, int dest, int kind, int lane) {
    if (dest == a.rank) {
        const int pb = (key >> BUCKET_SHIFT) * SUBB + (lane & (SUBB - 1));
        claim_store(a, st, step, pb, atomicAdd(&a.fill[pb], 1), out);
        return;
    }
    if (a.out_seg > 0) {
        // packed exchange: a segment of out_seg slots per destination and its
        // own counter -- the layout an equal-split all-to-all sends as it is,
        // so the step needs no host round trip for the counts
        const int e = atomicAdd(a.out_count + 1 + dest, 1);
        if (e < a.out_seg) {
            reinterpret_cast<float4 *>(a.outbox)[(long long)dest * a.out_seg + e] = out;
            return;
        }
        atomicMin(&st->key, err_key(3, 0, CS_SORT_OVERFLOW));
        st->abort = 1;
        st->step = step;
        return;
    }
    const int e = atomicAdd(a.out_count, 1);
    if (e < a.out_cap) {
        reinterpret_cast<float4 *>(a.outbox)[e] = out;
        a.out_dest[e] = dest | (kind << 30);
    } else {
        atomicMin(&st->key, err_key(3, 0, CS_SORT_OVERFLOW));
        st->abort = 1;
        st->step = step;
    }
}

// the slab duties of a record whose new cell row is R: ghost copies for the
// neighbours of R's owner when R is one of its boundary rows; false when the
// record leaves (a migrant to R's owner) instead of being claimed here
__device__ __forceinline__ bool slab_route(const FastArgs &a, DevStatus *st, int step, float4 out,
                                           int key, int R, int lane) {
    const int q = a.row_owner[R];
    int g1 = -1, g2 = -1;
    if (R == a.bounds[q]) g1 = q > 0 ? q - 1 : (a.per_rows ? a.world - 1 : -1);
    if (R == a.bounds[q + 1] - 1) g2 = q + 1 < a.world ? q + 1 : (a.per_rows ? 0 : -1);
    if (g2 == g1) g2 = -1;  // world 2, periodic: one copy for the other rank
    if (g1 == q) g1 = -1;   // world 1
    if (g2 == q) g2 = -1;
    if (g1 >= 0) slab_emit(a, st, step, out, key, g1, 1, lane);
    if (g2 >= 0) slab_emit(a, st, step, out, key, g2, 1, lane);
    if (q == a.rank) return true;
    slab_emit(a, st, step, out, key, q, 0, lane);
    return false;
}

template <bool SLAB>
__global__ void __launch_bounds__(256, CS_UPDATE_MINB)
k_fast_update(DevStatus *st, int step) {
    const FastArgs &a = cA;
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.gen_count = 0;  // k_fast_forces_generic has run
    const bool dead = st->abort != 0;
    const float4 *__restrict__ rec = reinterpret_cast<const float4 *>(a.rec);
    // the bucket claim of one iteration is consumed (record stored at its
    // slot) in the next, after that iteration's loads are in flight: the
    // atomic's round trip overlaps them instead of stalling the warp
    float4 p_out = make_float4(0.f, 0.f, 0.f, 0.f);
    int p_b = -1, p_slot = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
#if CS_CLAIM_AGG
    // warp-aggregated claims: the lanes of a warp that target the same
    // bucket part claim with one atomic (the warp picks the part); the loop
    // is warp-uniform so that the deferred shuffle of the claimed base sees
    // every lane
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int wpart = (threadIdx.x >> 5) & (SUBB - 1);
    bool p_have = false, p_live = false;
    int p_leader = 0, p_rank = 0, p_ret = 0;
    const long long s_lo = SLAB ? a.range[0] : 0, s_hi = SLAB ? a.range[1] : a.n;
    for (long long tb = s_lo + blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31);
         tb < s_hi; tb += stride) {
        const bool live = tb + lane < s_hi;
        const long long t = live ? tb + lane : s_hi - 1;
#else
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < a.n; t += stride) {
        const bool live = true;
#endif
        const float4 mer = __ldcs(rec + t);
        double2 f = make_double2(0.0, 0.0);
        if (a.interact) f = __ldcs(a.force + t);
        const UpdIn u = upd_load(a, mer, t, dead);
#if CS_CLAIM_AGG
        if (p_have) {
            const int basev = __shfl_sync(0xffffffffu, p_ret, p_leader);
            if (p_live) claim_store(a, st, step, p_b, basev + p_rank, p_out);
        }
#else
        if (p_b >= 0) claim_store(a, st, step, p_b, p_slot, p_out);
#endif
        int key, cyn;
        const float4 out = upd_finish(a, st, step, mer, u, f.x, f.y, dead, live, key, cyn);
#if CS_CLAIM_AGG
        bool claim = live;
        if (SLAB && live && !dead) claim = slab_route(a, st, step, out, key, cyn, lane);
        p_b = (key >> BUCKET_SHIFT) * SUBB + wpart;
        if (a.debug & 12) {  // timing diagnostics only (wrong results)
            if (live && (a.debug & 8)) atomicAdd(&a.fill[p_b], 1);
            if (live) reinterpret_cast<float4 *>(a.region)[t] = out;
            p_have = false;
            continue;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, claim ? p_b : -1 - lane);
        p_leader = __ffs(peers) - 1;
        p_rank = __popc(peers & lt);
        if (claim && lane == p_leader) p_ret = atomicAdd(&a.fill[p_b], __popc(peers));
        p_live = claim;
        p_have = true;
        p_out = out;
#else
        p_b = (key >> BUCKET_SHIFT) * SUBB + (threadIdx.x & (SUBB - 1));
        if (a.debug & 12) {  // timing diagnostics only (wrong results)
            if (a.debug & 8) atomicAdd(&a.fill[p_b], 1);
            reinterpret_cast<float4 *>(a.region)[t] = out;
            p_b = -1;
            continue;
        }
        p_slot = atomicAdd(&a.fill[p_b], 1);
        p_out = out;
#endif
    }
#if CS_CLAIM_AGG
    if (p_have) {
        const int basev = __shfl_sync(0xffffffffu, p_ret, p_leader);
        if (p_live) claim_store(a, st, step, p_b, basev + p_rank, p_out);
    }
#else
    if (p_b >= 0) claim_store(a, st, step, p_b, p_slot, p_out);
#endif
}

// Slab re-balancing: every owned record (old range) routed under the new
// row bounds without moving -- claimed here, or sent to its new owner, plus
// ghost copies for the neighbours of its row's owner (slab_route).
__global__ void __launch_bounds__(256) k_slab_reroute(DevStatus *st, int step) {
    const FastArgs &a = cA;
    const long long lo = a.range[0], hi = a.range[1];
    const float4 *__restrict__ rec = reinterpret_cast<const float4 *>(a.rec);
    const int lane = threadIdx.x & 31;
    for (long long t = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; t < hi;
         t += (long long)gridDim.x * blockDim.x) {
        const float4 out = rec[t];
        const int cy = cell_axis_fast((double)out.y, a.g.lo1, a.eff1, a.g.n1);
        const int key = cy * a.g.n0 + cell_axis_fast((double)out.x, a.g.lo0, a.eff0, a.g.n0);
        if (slab_route(a, st, step, out, key, cy, lane)) {
            const int pb = (key >> BUCKET_SHIFT) * SUBB + (lane & (SUBB - 1));
            claim_store(a, st, step, pb, atomicAdd(&a.fill[pb], 1), out);
        }
    }
}

// per-row counts of the owned records (the re-balancing histogram)
__global__ void k_slab_hist(const Rec *__restrict__ rec, const int *__restrict__ range, BinGeom g,
                            ExactDiv eff1, int *__restrict__ hist) {
    const long long lo = range[0], hi = range[1];
    for (long long t = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; t < hi;
         t += (long long)gridDim.x * blockDim.x)
        atomicAdd(&hist[cell_axis_fast((double)rec[t].y, g.lo1, eff1, g.n1)], 1);
}

// caller arrays (id order) -> records claimed into their bucket regions
// (the same claim as k_fast_update's), anchors kept as the wrap origin
__global__ void k_fast_import(const float *__restrict__ pos, const float *__restrict__ anchor,
                              const uint8_t *__restrict__ type, long long n, BinGeom g,
                              Rec *__restrict__ region, int *__restrict__ fill, long long cap,
                              float *__restrict__ anchor0, DevStatus *st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 p = reinterpret_cast<const float2 *>(pos)[i];
        Rec r;
        r.x = p.x;
        r.y = p.y;
        r.meta = (unsigned)i | ((type && type[i]) ? 0x80000000u : 0u);
        r.wx = 0;
        r.wy = 0;
        reinterpret_cast<float2 *>(anchor0)[i] = reinterpret_cast<const float2 *>(anchor)[i];
        const int key = cell_axis((double)p.y, g.lo1, g.eff1, g.n1) * g.n0 +
                        cell_axis((double)p.x, g.lo0, g.eff0, g.n0);
        const int q = (key >> BUCKET_SHIFT) * SUBB + (threadIdx.x & (SUBB - 1));
        const int slot = atomicAdd(&fill[q], 1);
        if (slot < cap) {
            region[(long long)q * cap + slot] = r;
        } else {
            atomicMin(&st->key, err_key(3, q / SUBB, CS_SORT_OVERFLOW));
            st->abort = 1;
        }
    }
}

__device__ __noinline__ bool deposit_record(float4 rv, GridGeom gg, ExactDiv d0, ExactDiv d1,
                                            unsigned bits, int *rho_q, int m) {
    const Cic c = cic_stencil((double)rv.x, (double)rv.y, gg, d0, d1);
    bool ovf = false;
    if (bits & 1u) ovf |= cic_deposit_q(c, rho_q);
    if (bits & 2u) ovf |= cic_deposit_q(c, rho_q + m);
    return ovf;
}

// Bucket sort: one block per bucket of BUCKET_CELLS consecutive cells (flat,
// y-major index).  k_fast_update / k_fast_import claimed a slot for every
// record in its bucket's region (arrival order); k_scan turned the claim
// counts into the bucket offsets boff[].  The block
//   1. loads the bucket's records (coalesced) and recomputes each record's
//      cell exactly as the claim did (cell_axis_fast on the stored binary32
//      coordinates), counting the cells in shared memory;
//   2. scans the cell counts -> the bucket's slice of the next cell table;
//   3. ranks every record inside its cell by particle id (the reference's
//      in-cell order, motion.py:195-199: a stable counting sort of ids), and
//      writes it to boff[b] + cell start + rank: the output is cell-sorted,
//      id-sorted inside a cell, and contiguous;
//   4. (atomic deposit mode) CIC-deposits the bucket's records: neighbouring
//      cells, so the integer reductions stay L2-local and deterministic.
// A deposit add that overflows the int32 fixed-point sum stops the run with
// CS_DEPOSIT_OVERFLOW (checked on every add here; the row deposit checks its
// adds once a cell exceeds the conservative population bound cell_max).
// XI: the coming step's increments (an (N, 2) array by particle id) are
// gathered here, by the ids of the records being placed, and stored by
// destination slot; that step's update reads them as a coalesced stream.
// The gather costs the same wherever it runs while the array fits the L2
// (cfg3: update 313 -> 256 us, this kernel 154 -> 277 us); beyond it (cfg4:
// 640 MB) the update's one load in flight per thread is the limit and the
// four independent loads per thread here are not (13.0 -> 12.3 ms/step).
template <bool XI>
__global__ void __launch_bounds__(BSORT_THREADS)
k_bucket_sort(const Rec *__restrict__ region, const int *__restrict__ boff, long long cap,
              long long nbucket, BinGeom g, ExactDiv eff0, ExactDiv eff1, long long nflat,
              Rec *__restrict__ out, int *__restrict__ starts, GridGeom gg, ExactDiv d0,
              ExactDiv d1, unsigned bits0, unsigned bits1, int *__restrict__ rho_q, int deposit,
              int cell_max, int *__restrict__ dep_exact, DevStatus *st, int step,
              const float2 *__restrict__ xi_next, float2 *__restrict__ xi_slot) {
    // [SUBB cap] ids by slot, then codes (cell | arrival << 10 | part << 25) of
    // the records beyond the register-resident ones
    extern __shared__ int s_dyn[];
    __shared__ int s_pre[SUBB + 1];
    __shared__ __align__(16) int s_cnt[BUCKET_CELLS];
    __shared__ __align__(16) int s_beg[BUCKET_CELLS + 4];
    __shared__ int s_wsum[BSORT_THREADS / 32];
    unsigned *s_id = reinterpret_cast<unsigned *>(s_dyn);
    int *s_code = s_dyn + SUBB * cap;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long b = blockIdx.x;
    // the bucket's records: its SUBB region parts, concatenated (part q
    // holds local indices s_pre[q] .. s_pre[q + 1])
    const int off = boff[b * SUBB];
    if (warp == 0) {
        int c = 0;
        if (lane < SUBB) {
            c = boff[b * SUBB + lane + 1] - boff[b * SUBB + lane];
            if (c > cap) c = (int)cap;  // overflowed part: the run is already stopped
        }
        int v = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += u;
        }
        if (lane < SUBB) s_pre[lane + 1] = v;
        if (lane == 0) s_pre[0] = 0;
    }
    const float4 *r4 = reinterpret_cast<const float4 *>(region) + b * SUBB * cap;
    const long long cell0 = b * BUCKET_CELLS;
    reinterpret_cast<int4 *>(s_cnt)[tid] = make_int4(0, 0, 0, 0);
    __syncthreads();
    const int cnt = s_pre[SUBB];
    auto part_of = [&](int i) {  // part holding local index i
        int q = 0;
#pragma unroll
        for (int k = 1; k < SUBB; k++) q += i >= s_pre[k] ? 1 : 0;
        return q;
    };
    auto cell_code = [&](float4 r, int q) {
        const int key = cell_axis_fast((double)r.y, g.lo1, eff1, g.n1) * g.n0 +
                        cell_axis_fast((double)r.x, g.lo0, eff0, g.n0);
        const int lc = (int)(key - cell0);
        const int arr = atomicAdd(&s_cnt[lc], 1);
        return lc | (arr << BUCKET_SHIFT) | (q << 25);
    };
    // the first RPT * BSORT_THREADS records stay in registers through all
    // phases (their loads issued together); the rest (dense buckets only)
    // keep their codes in shared memory and are re-read
    float4 rr[RPT];
    int cc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; k++) {
        const int i = tid + k * BSORT_THREADS;
        cc[k] = -1;
        if (i < cnt) {
            const int q = part_of(i);
            rr[k] = __ldg(r4 + (long long)q * cap + (i - s_pre[q]));
            cc[k] = q;
        }
    }
#pragma unroll
    for (int k = 0; k < RPT; k++)
        if (cc[k] >= 0) cc[k] = cell_code(rr[k], cc[k]);
    for (int i = tid + RPT * BSORT_THREADS; i < cnt; i += BSORT_THREADS) {
        const int q = part_of(i);
        s_code[i - RPT * BSORT_THREADS] =
            cell_code(__ldg(r4 + (long long)q * cap + (i - s_pre[q])), q);
    }
    __syncthreads();
    // exclusive scan of the cell counts: thread t owns cells 4t .. 4t + 3
    const int4 c4 = reinterpret_cast<const int4 *>(s_cnt)[tid];
    const int csum = c4.x + c4.y + c4.z + c4.w;
    int v = csum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
    }
    if (lane == 31) s_wsum[warp] = v;
    __syncthreads();
    int wbase = 0;
#pragma unroll
    for (int w = 0; w < BSORT_THREADS / 32; w++) wbase += w < warp ? s_wsum[w] : 0;
    int4 b4;
    b4.x = wbase + v - csum;
    b4.y = b4.x + c4.x;
    b4.z = b4.y + c4.y;
    b4.w = b4.z + c4.z;
    reinterpret_cast<int4 *>(s_beg)[tid] = b4;
    if (tid == 0) s_beg[BUCKET_CELLS] = cnt;
    const long long cfirst = cell0 + CELLS_PER_THREAD * tid;
    const int4 o4 = make_int4(off + b4.x, off + b4.y, off + b4.z, off + b4.w);
    if (cfirst + 4 <= nflat) {
        reinterpret_cast<int4 *>(starts + cfirst)[0] = o4;
    } else {
        const int ov[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (cfirst + k < nflat) starts[cfirst + k] = ov[k];
    }
    if (cell_max > 0) {
        const int cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (cv[k] > cell_max && cfirst + k < nflat) {
                // a grid node could collect more particle masses of 2^22 than
                // an int32 sums exactly: the row deposit checks every add
                *dep_exact = 1;
            }
        }
    }
    if (b == nbucket - 1 && tid == 0) starts[nflat] = off + cnt;
    {
        // overflowed parts (the run is stopped): the lost records' slots get
        // an in-domain placeholder, so that no kernel reads garbage ids or
        // coordinates before the host sees the status
        const int full = boff[(b + 1) * SUBB] - off;
        for (int i = cnt + tid; i < full; i += BSORT_THREADS) {
            Rec ph;
            ph.x = (float)g.lo0;
            ph.y = (float)g.lo1;
            ph.meta = 0;
            ph.wx = 0;
            ph.wy = 0;
            out[off + i] = ph;
        }
    }
    __syncthreads();
    constexpr int LC_MASK = BUCKET_CELLS - 1;
    constexpr int ARR_MASK = (1 << (25 - BUCKET_SHIFT)) - 1;
#pragma unroll
    for (int k = 0; k < RPT; k++)
        if (cc[k] >= 0)
            s_id[s_beg[cc[k] & LC_MASK] + ((cc[k] >> BUCKET_SHIFT) & ARR_MASK)] =
                __float_as_uint(rr[k].z) & ID_MASK;
    for (int i = tid + RPT * BSORT_THREADS; i < cnt; i += BSORT_THREADS) {
        const int code = s_code[i - RPT * BSORT_THREADS];
        const int q = code >> 25;
        s_id[s_beg[code & LC_MASK] + ((code >> BUCKET_SHIFT) & ARR_MASK)] =
            __float_as_uint(__ldg(r4 + (long long)q * cap + (i - s_pre[q])).z) & ID_MASK;
    }
    __syncthreads();
    const unsigned bits_dep = deposit ? (bits0 | bits1) : 0u;
    float2 xv[RPT];  // XI: the register-resident records' increments, loads issued together
    if (XI) {
#pragma unroll
        for (int k = 0; k < RPT; k++)
            if (cc[k] >= 0) xv[k] = ld_evict_last(xi_next + (__float_as_uint(rr[k].z) & ID_MASK));
    }
    auto place = [&](float4 r, int code, float2 z, bool have_z) {
        const int lc = code & LC_MASK;
        const int kb = s_beg[lc], len = s_beg[lc + 1] - kb;
        int rank = 0;
        if (len > 1) {
            const unsigned id = __float_as_uint(r.z) & ID_MASK;
            for (int k = 0; k < len; k++) rank += s_id[kb + k] < id ? 1 : 0;
        }
        reinterpret_cast<float4 *>(out)[off + kb + rank] = r;
        if (XI) {
            if (!have_z) z = ld_evict_last(xi_next + (__float_as_uint(r.z) & ID_MASK));
            __stcs(xi_slot + off + kb + rank, z);
        }
        if (bits_dep) {
            const unsigned bits = (__float_as_uint(r.z) >> 31) ? bits1 : bits0;
            if (bits && deposit_record(r, gg, d0, d1, bits, rho_q, gg.n * gg.n)) {
                atomicMin(&st->key, err_key(3, __float_as_uint(r.z) & ID_MASK,
                                            CS_DEPOSIT_OVERFLOW));
                st->abort = 1;
                st->step = step;
            }
        }
    };
#pragma unroll
    for (int k = 0; k < RPT; k++)
        if (cc[k] >= 0) place(rr[k], cc[k], XI ? xv[k] : make_float2(0.f, 0.f), true);
    for (int i = tid + RPT * BSORT_THREADS; i < cnt; i += BSORT_THREADS) {
        const int code = s_code[i - RPT * BSORT_THREADS];
        const int q = code >> 25;
        place(__ldg(r4 + (long long)q * cap + (i - s_pre[q])), code, make_float2(0.f, 0.f), false);
    }
}

// Deposit by rows (periodic grids): one block per grid row j gathers the CIC
// weights of every particle whose stencil touches row j -- base row j - 1 or
// j (coupling.py:119-135) -- from the contiguous slot ranges of the cell rows
// that can hold such particles (one row of margin each side), accumulates
// them in shared memory as int32 fixed point and writes row j of both grids
// in full: no global atomics, no grid reset, and the sums equal the atomic
// deposit's bit for bit (integer addition is associative).
#ifndef CS_DEP_ROWS
#define CS_DEP_ROWS 2
#endif
constexpr int DEP_ROWS = CS_DEP_ROWS;  // grid rows per block of k_fast_deposit_rows

// P2: the grid size is a power of two (every BASELINE grid): node and window
// indices wrap with a mask instead of the compare / add sequences.
template <int NT, bool P2>  // threads per block (launch bound: registers)
__global__ void __launch_bounds__(NT)
k_fast_deposit_rows(const Rec *__restrict__ rec, const int *__restrict__ starts, BinGeom g,
                    GridGeom gg, ExactDiv d0, ExactDiv d1, unsigned bits0, unsigned bits1,
                    int *__restrict__ rho_q, const int *__restrict__ exact_flag,
                    int *__restrict__ other_flag, DevStatus *st, int step, int jbase, int jrows,
                    int cb0, int cb1) {
    // (slab mode: grid rows jbase .. jbase + jrows - 1, mod n, from the
    // particles of the own cell rows [cb0, cb1) only; single domain: 0, n, -1)
    extern __shared__ __align__(16) int acc[];  // [DEP_ROWS][2][n]
    // exact overflow checks only when the bucket sort saw a cell populated
    // beyond the conservative bound (returning atomics cost ~20 % here)
    const bool exact = *exact_flag != 0;
    __shared__ int ovf_node;
    if (threadIdx.x == 0) ovf_node = -1;
    if (blockIdx.x == 0 && threadIdx.x == 0) *other_flag = 0;  // the next step's flag
    const int n = gg.n, j0 = jbase + blockIdx.x * DEP_ROWS;
    const long long m = (long long)n * n;
    const bool vec4 = (n & 3) == 0;  // rows of whole int4s (accumulators and both grids)
    if (vec4) {
        for (int i = threadIdx.x; i < DEP_ROWS * 2 * n / 4; i += blockDim.x)
            reinterpret_cast<int4 *>(acc)[i] = make_int4(0, 0, 0, 0);
    } else {
        for (int i = threadIdx.x; i < DEP_ROWS * 2 * n; i += blockDim.x) acc[i] = 0;
    }
    __syncthreads();
    // cell rows that can hold a particle with y in [lo + (j0-1) d, lo + (j0+R) d):
    // the cell index is monotone in y, so the rows of the (slightly widened)
    // window ends bound it
    const double ylo = dsub(dadd(gg.lo1, dmul((double)(j0 - 1), gg.d1)), 1e-9);
    const double yhi = dadd(dadd(gg.lo1, dmul((double)(j0 + DEP_ROWS), gg.d1)), 1e-9);
    const int cy0 = (int)floor(ddiv(dsub(ylo, g.lo1), g.eff1));
    const int cy1 = (int)floor(ddiv(dsub(yhi, g.lo1), g.eff1));
    const float4 *r4 = reinterpret_cast<const float4 *>(rec);
    for (int cyw = cy0; cyw <= cy1; cyw++) {
        if (cyw - cy0 >= g.n1) break;  // fewer cell rows than the window
        int cy = cyw;  // (the window starts within one period of the domain)
        while (cy < 0) cy += g.n1;
        while (cy >= g.n1) cy -= g.n1;
        if (cb0 >= 0 && (cy < cb0 || cy >= cb1)) continue;  // ghost rows: other ranks'
        const int kb = starts[(long long)cy * g.n0], ke = starts[(long long)(cy + 1) * g.n0];
        for (int k = kb + threadIdx.x; k < ke; k += blockDim.x) {
            const float4 rv = __ldg(r4 + k);
            const unsigned bits = (__float_as_uint(rv.z) >> 31) ? bits1 : bits0;
            if (!bits) continue;
            // the periodic branch of cic_stencil, y first (the row filter)
            const double u1 = ediv(dsub((double)rv.y, gg.lo1), d1);
            const double base1 = floor(u1);
            // (P2: base1 lies in [-1, n] for in-domain records; the mask is
            // pymod for every int, and a non-finite coordinate -- the run is
            // already stopped -- saturates)
            const int b1 = P2 ? ((int)base1 & (n - 1)) : wrap_index(base1, n);
            const int c1 = P2 ? ((b1 + 1) & (n - 1)) : (b1 + 1 == n ? 0 : b1 + 1);
            // rows of this block's window, if any (j0 in [-n, 2n): two wraps at most)
            int rb = b1 - j0, rc = c1 - j0;
            if (P2) {
                rb &= n - 1;
                rc &= n - 1;
            } else {
                rb += rb < 0 ? n : (rb >= n ? -n : 0);
                rc += rc < 0 ? n : (rc >= n ? -n : 0);
                rb += rb < 0 ? n : 0;
                rc += rc < 0 ? n : 0;
            }
            const bool hb = rb < DEP_ROWS, hc = rc < DEP_ROWS;
            if (!hb && !hc) continue;
            const double f1 = dsub(u1, base1);
            const double u0 = ediv(dsub((double)rv.x, gg.lo0), d0);
            const double base0 = floor(u0);
            const double f0 = dsub(u0, base0);
            const int b0 = P2 ? ((int)base0 & (n - 1)) : wrap_index(base0, n);
            const int c0 = P2 ? ((b0 + 1) & (n - 1)) : (b0 + 1 == n ? 0 : b0 + 1);
            const double g0 = dsub(1.0, f0);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                if (!(h ? hc : hb)) continue;
                const double wy = h ? f1 : dsub(1.0, f1);  // row b1: g1, row c1: f1
                const int qa = __double2int_rn(dmul(dmul(g0, wy), Q_SCALE));
                const int qb = __double2int_rn(dmul(dmul(f0, wy), Q_SCALE));
                int *row = acc + (h ? rc : rb) * 2 * n;
                if (exact) {
                    bool ovf = false;
                    if (bits & 1u) {
                        ovf |= add_overflows(&row[b0], qa);
                        ovf |= add_overflows(&row[c0], qb);
                    }
                    if (bits & 2u) {
                        ovf |= add_overflows(&row[n + b0], qa);
                        ovf |= add_overflows(&row[n + c0], qb);
                    }
                    if (ovf) ovf_node = (j0 + (h ? rc : rb)) * n + b0;
                } else {
                    if (bits & 1u) {
                        atomicAdd(&row[b0], qa);
                        atomicAdd(&row[c0], qb);
                    }
                    if (bits & 2u) {
                        atomicAdd(&row[n + b0], qa);
                        atomicAdd(&row[n + c0], qb);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && ovf_node >= 0) {
        atomicMin(&st->key, err_key(3, ovf_node, CS_DEPOSIT_OVERFLOW));
        st->abort = 1;
        st->step = step;
    }
    for (int r = 0; r < DEP_ROWS; r++) {
        if (blockIdx.x * DEP_ROWS + r >= jrows) break;
        int j = (j0 + r) % n;
        if (j < 0) j += n;
        int *ra = rho_q + (long long)j * n, *rbp = rho_q + m + (long long)j * n;
        if (vec4) {
            const int4 *sa = reinterpret_cast<const int4 *>(acc + r * 2 * n);
            for (int i = threadIdx.x; i < n / 4; i += blockDim.x) {
                reinterpret_cast<int4 *>(ra)[i] = sa[i];
                reinterpret_cast<int4 *>(rbp)[i] = sa[n / 4 + i];
            }
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                ra[i] = acc[r * 2 * n + i];
                rbp[i] = acc[r * 2 * n + n + i];
            }
        }
    }
}

// records (sorted) -> caller arrays (id order); anchor = anchor0 - wraps * L
__global__ void k_fast_export(const Rec *__restrict__ rec, long long n,
                              const float *__restrict__ anchor0, double size0, double size1,
                              float *__restrict__ pos, float *__restrict__ anchor,
                              const int *__restrict__ range) {
    const long long lo = range ? range[0] : 0, hi = range ? range[1] : n;
    for (long long t = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; t < hi;
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

// ---- y-slab mode (cs_slab_*) ----------------------------------------------
// The cell row of a position, as the update bins it.
__device__ __forceinline__ int slab_row(float y, const BinGeom &g, const ExactDiv &eff1) {
    return cell_axis_fast((double)y, g.lo1, eff1, g.n1);
}
__device__ __forceinline__ bool slab_keeps(int R, int b0, int b1, int n1, int per) {
    if (R >= b0 && R < b1) return true;                             // owned
    if (R == b0 - 1 || (per && b0 == 0 && R == n1 - 1)) return true;  // lower ghost row
    if (R == b1 || (per && b1 == n1 && R == 0)) return true;          // upper ghost row
    return false;
}

// the caller's (id-ordered, global) arrays -> this rank's records: its owned
// rows and the ghost rows on either side, claimed into their bucket regions
__global__ void k_slab_import(const float *__restrict__ pos, const float *__restrict__ anchor,
                              const uint8_t *__restrict__ type, long long n, BinGeom g,
                              ExactDiv eff0, ExactDiv eff1, int b0, int b1,
                              Rec *__restrict__ region, int *__restrict__ fill, long long cap,
                              float *__restrict__ anchor0, DevStatus *st) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 p = reinterpret_cast<const float2 *>(pos)[i];
        reinterpret_cast<float2 *>(anchor0)[i] = reinterpret_cast<const float2 *>(anchor)[i];
        const int R = slab_row(p.y, g, eff1);
        if (!slab_keeps(R, b0, b1, g.n1, g.per1)) continue;
        Rec r;
        r.x = p.x;
        r.y = p.y;
        r.meta = (unsigned)i | ((type && type[i]) ? 0x80000000u : 0u);
        r.wx = 0;
        r.wy = 0;
        const int key = R * g.n0 + cell_axis_fast((double)p.x, g.lo0, eff0, g.n0);
        const int q = (key >> BUCKET_SHIFT) * SUBB + (threadIdx.x & (SUBB - 1));
        const int slot = atomicAdd(&fill[q], 1);
        if (slot < cap) {
            region[(long long)q * cap + slot] = r;
        } else {
            atomicMin(&st->key, err_key(3, q / SUBB, CS_SORT_OVERFLOW));
            st->abort = 1;
        }
    }
}

// records received from other ranks (migrants and ghosts) claimed into
// their bucket regions
__global__ void k_slab_claim(const float4 *__restrict__ in, long long n, BinGeom g, ExactDiv eff0,
                             ExactDiv eff1, Rec *__restrict__ region, int *__restrict__ fill,
                             long long cap, DevStatus *st, int step) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 r = in[i];
        const int key = slab_row(r.y, g, eff1) * g.n0 +
                        cell_axis_fast((double)r.x, g.lo0, eff0, g.n0);
        const int q = (key >> BUCKET_SHIFT) * SUBB + (threadIdx.x & (SUBB - 1));
        const int slot = atomicAdd(&fill[q], 1);
        if (slot < cap) {
            reinterpret_cast<float4 *>(region)[(long long)q * cap + slot] = r;
        } else {
            atomicMin(&st->key, err_key(3, q / SUBB, CS_SORT_OVERFLOW));
            st->abort = 1;
            st->step = step;
        }
    }
}

// the owned slot range [starts(b0 row), starts(b1 row)) of the sorted records
__global__ void k_slab_range(const int *__restrict__ starts, long long c0, long long c1,
                             int *__restrict__ range) {
    range[0] = starts[c0];
    range[1] = starts[c1];
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
k_fast_rhs(const float *__restrict__ c, const int *__restrict__ q, long long m, double one_m_dtg,
           double dka, double dkb, int has_g, int has_a, int has_b, double scale,
           R *__restrict__ rhs, const DevStatus *st) {
    if (st->abort) return;
    for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < m;
         l += (long long)gridDim.x * blockDim.x) {
        const double cv = (double)c[l];
        const int qa = q[l], qb = q[l + m];  // zeroed later by the gradient kernel
        double r = has_g ? dmul(cv, one_m_dtg) : cv;
        if (has_a) r = dadd(r, dmul(dka, dmul((double)qa, scale)));
        if (has_b) r = dsub(r, dmul(dmul(dmul((double)qb, scale), cv), dkb));
        rhs[l] = (R)r;
    }
}

}  // namespace cs

// ---------------------------------------------------------------------------
constexpr int STARTS_OFF = 0;

struct cs_fast {
    cs::Buf rec[2], region, fill, boff, starts[2], anchor0, rho_q, force, gen, depflag;
    // the coming step's increments in storage-slot order (gathered by id in
    // the bucket sort when the caller's block holds that step and the array
    // is beyond the L2: xi_ready)
    cs::Buf xi_slot;
    bool xi_ready = false;
    int cur = 0;
    bool imported = false;
    long long nflat = 0;
    long long nbucket = 0;  // buckets of BUCKET_CELLS cells
    long long cap = 0;      // record slots per bucket region
    double eff0 = 1.0, eff1 = 1.0;  // cell sides
    cs::BinGeom g{};
    bool gather = false;            // deposit by grid rows (k_fast_deposit_rows)
    // y-slab mode (cs_slab_*): owned rows [b0, b1) of world ranks
    bool slab = false;
    int rank = 0, world = 1, b0 = 0, b1 = 0;
    int dep_j0 = 0, dep_rows = 0;  // slab field: the grid rows this rank deposits into
    cs::Buf range, row_owner, bounds, outbox, out_dest, out_count;
    long long out_cap = 0;
    long long out_seg = 0;  // packed exchange: slots per destination (0: one outbox + dest tags)
};

namespace cs {

int field_solve_rhs(cs_field_ops *ops, void *out);
int launch_gradient(cs_ctx *ctx, int prec, const void *c, const GridGeom &gg, void *grad,
                    DevStatus *st, int step, int *zero_q = nullptr);

static int *cell_table(cs_fast *f, int b) { return f->starts[b].as<int>() + STARTS_OFF; }

int fast_create(cs_fast **out, long long n, const BinGeom &g, const GridGeom *gg) {
    auto *f = new cs_fast();
    *out = f;
    f->nflat = (long long)g.n0 * g.n1;
    f->eff0 = g.eff0;
    f->eff1 = g.eff1;
    f->g = g;
    // periodic domain and grid, accumulators of a grid row fit in shared memory
    f->gather = gg && gg->per && g.per0 && g.per1 && gg->n >= 2 &&
                (size_t)gg->n * DEP_ROWS * 8 <= 200 * 1024 &&
                !getenv("CS_ATOMIC_DEPOSIT");
    // bucket regions: 8x the mean bucket population + 256 slots (at least
    // 1024), capped so that a block's shared staging (8 B per slot) fits
    f->nbucket = (f->nflat + BUCKET_CELLS - 1) / BUCKET_CELLS;
    const double mean = (double)(n > 0 ? n : 1) / (double)f->nbucket;
    long long cap = (long long)(8.0 * mean / SUBB) + 64;  // per region part
    if (cap < 128) cap = 128;
    if (cap > 24576 / SUBB) cap = 24576 / SUBB;
    if (const char *e = getenv("CS_BUCKET_CAP")) cap = atoll(e);  // tests: force overflows
    f->cap = (cap + 7) / 8 * 8;
    // (+ 32 records: a lane past the end of the last warp's slots re-reads "its own" slot
    // in the force walk)
    const size_t nr = sizeof(Rec) * (size_t)((n > 0 ? n : 1) + 32);
    CS_TRY(f->rec[0].ensure(nr));
    CS_TRY(f->rec[1].ensure(nr));
    for (int b = 0; b < 2; b++)  // the tail reads as zeros (no prefilter hit: d2 == 0)
        CS_CUDA(cudaMemset(static_cast<char *>(f->rec[b].p) + nr - 32 * sizeof(Rec), 0,
                           32 * sizeof(Rec)));
    CS_TRY(f->region.ensure(sizeof(Rec) * (size_t)f->nbucket * SUBB * (size_t)f->cap));
    CS_TRY(f->force.ensure(sizeof(double2) * (size_t)(n > 0 ? n : 1)));
    CS_TRY(f->gen.ensure(sizeof(int) * (size_t)(n + 2)));  // counter, run state, list
    CS_CUDA(cudaMemset(f->gen.p, 0, f->gen.bytes));
    CS_TRY(f->depflag.ensure(sizeof(int) * 2));  // exact-deposit flags by step parity
    CS_CUDA(cudaMemset(f->depflag.p, 0, f->depflag.bytes));
    CS_TRY(f->fill.ensure(sizeof(int) * (size_t)(f->nbucket * SUBB + 1)));
    CS_CUDA(cudaMemset(f->fill.p, 0, f->fill.bytes));
    CS_TRY(f->boff.ensure(sizeof(int) * (size_t)(f->nbucket * SUBB + 4)));
    // cell tables: nflat + 1 starts (kept STARTS_OFF ints into the buffer)
    for (int b = 0; b < 2; b++) {
        CS_TRY(f->starts[b].ensure(sizeof(int) * (size_t)(f->nflat + 2 + STARTS_OFF)));
        CS_CUDA(cudaMemset(f->starts[b].p, 0, f->starts[b].bytes));
    }
    CS_TRY(f->anchor0.ensure(sizeof(float) * 2 * (size_t)(n > 0 ? n : 1)));
    if (gg) {
        CS_TRY(f->rho_q.ensure(sizeof(int) * 2 * (size_t)gg->n * gg->n));
        CS_CUDA(cudaMemset(f->rho_q.p, 0, f->rho_q.bytes));
    }
    return CS_OK;
}

void fast_destroy(cs_fast *f) {
    if (!f) return;
    for (Buf *b : {&f->rec[0], &f->rec[1], &f->region, &f->fill, &f->boff, &f->starts[0],
                   &f->starts[1], &f->anchor0, &f->rho_q, &f->force, &f->gen, &f->depflag,
                   &f->xi_slot,
                   &f->range, &f->row_owner, &f->bounds, &f->outbox, &f->out_dest,
                   &f->out_count})
        b->release();
    delete f;
}

static int persistent_grid(cs_ctx *ctx, const void *kern, int block, long long work,
                           int *resident) {
    if (!*resident) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(resident, kern, block, 0);
        if (*resident < 1) *resident = 1;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const long long want = (work + block - 1) / block;
    return (int)(want < (long long)sms * *resident ? want : (long long)sms * *resident);
}

// Largest cell population for which the int32 fixed-point deposit is exact:
// a node's CIC support (two grid spacings per axis) overlaps at most
// floor(2 d / eff) + 2 cells per axis, and a node overflows only past 511
// contributions of 2^22.
static int deposit_cell_max(const GridGeom &gg, const cs_fast *f) {
    const double k0 = floor(2.0 * gg.d0 / f->eff0) + 2.0, k1 = floor(2.0 * gg.d1 / f->eff1) + 2.0;
    const double m = floor(511.0 / (k0 * k1));
    return m < 1.0 ? 1 : (int)m;
}

// Bucket offsets (scan of the claim counts, which it also resets), then the
// bucket sort into the next record array and cell table (in-cell id order;
// the atomic-mode deposit of the next step's field rides along).
static int fast_sort(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const GridGeom &gg,
                     const unsigned char bits[3], DevStatus *st, int step,
                     const void *xi_next = nullptr) {
    const int nxt = 1 - f->cur;
    if (xi_next) CS_TRY(f->xi_slot.ensure(sizeof(float2) * (size_t)(p.n > 0 ? p.n : 1)));
    CS_TRY(exclusive_scan_i32(ctx, f->fill.as<int>(), f->boff.as<int>(), f->nbucket * SUBB,
                              f->fill.as<int>()));
    const char *dbg = getenv("CS_FAST_DEBUG");
    const int debug = dbg ? atoi(dbg) : 0;
    const bool dep = p.field_active && !(debug & 2);
    const double d0 = gg.d0 > 0 ? gg.d0 : 1.0, d1 = gg.d1 > 0 ? gg.d1 : 1.0;
    const long long extra = SUBB * f->cap - RPT * BSORT_THREADS;
    const size_t smem = sizeof(int) * (size_t)(SUBB * f->cap + (extra > 0 ? extra : 0));
    static size_t smem_set = 0;
    if (smem > smem_set) {  // static + dynamic may pass 48 KB before the dynamic part does
        CS_CUDA(cudaFuncSetAttribute(k_bucket_sort<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CS_CUDA(cudaFuncSetAttribute(k_bucket_sort<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set = smem;
    }
    auto kern = xi_next ? k_bucket_sort<true> : k_bucket_sort<false>;
    kern<<<(unsigned)f->nbucket, BSORT_THREADS, smem, ctx->stream>>>(
        f->region.as<Rec>(), f->boff.as<int>(), f->cap, f->nbucket, f->g,
        make_exact_div(f->g.eff0), make_exact_div(f->g.eff1), f->nflat, f->rec[nxt].as<Rec>(),
        cell_table(f, nxt), gg, make_exact_div(d0), make_exact_div(d1), dep ? bits[0] : 0u,
        dep ? bits[1] : 0u, f->rho_q.as<int>(), dep && !f->gather,
        dep && f->gather && (bits[0] | bits[1]) ? deposit_cell_max(gg, f) : 0,
        f->depflag.as<int>() + (step & 1), st, step, (const float2 *)xi_next,
        xi_next ? f->xi_slot.as<float2>() : nullptr);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    f->cur = nxt;
    f->xi_ready = xi_next != nullptr;
    return CS_OK;
}

// periodic grids: the next step's deposit gathered per grid row
static int fast_deposit_rows(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p,
                             const GridGeom &gg, const unsigned char bits[3], DevStatus *st,
                             int step) {
    const char *dbg = getenv("CS_FAST_DEBUG");
    const int debug = dbg ? atoi(dbg) : 0;
    if (p.n <= 0 || !p.field_active || (debug & 2) || !f->gather) return CS_OK;
    const double d0 = gg.d0 > 0 ? gg.d0 : 1.0, d1 = gg.d1 > 0 ? gg.d1 : 1.0;
    const int smem = (int)(DEP_ROWS * 2 * sizeof(int) * (size_t)gg.n);
    static int smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
        for (auto k : {k_fast_deposit_rows<512, false>, k_fast_deposit_rows<512, true>,
                       k_fast_deposit_rows<1024, false>, k_fast_deposit_rows<1024, true>})
            CS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        smem_set = smem;
    }
    const int jbase = f->slab ? f->dep_j0 : 0, jrows = f->slab ? f->dep_rows : gg.n;
    // a block's row accumulators take 64 KB at 4096 nodes per row (3 blocks of
    // 512 threads per SM) and 128 KB at 8192 (one block per SM: 1024 threads)
    const int threads = smem > 100 * 1024 ? 1024 : 512;
    const bool p2 = (gg.n & (gg.n - 1)) == 0 && !getenv("CS_DEP_NO_P2");
    auto kern = threads == 1024
                    ? (p2 ? k_fast_deposit_rows<1024, true> : k_fast_deposit_rows<1024, false>)
                    : (p2 ? k_fast_deposit_rows<512, true> : k_fast_deposit_rows<512, false>);
    kern<<<(jrows + DEP_ROWS - 1) / DEP_ROWS, threads, smem, ctx->stream>>>(
        f->rec[f->cur].as<Rec>(), cell_table(f, f->cur), f->g, gg, make_exact_div(d0),
        make_exact_div(d1), bits[0], bits[1], f->rho_q.as<int>(),
        f->depflag.as<int>() + (step & 1), f->depflag.as<int>() + ((step + 1) & 1), st, step,
        jbase, jrows, f->slab ? f->b0 : -1, f->slab ? f->b1 : -1);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int fast_import(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                const BinGeom &g, const GridGeom &gg, const unsigned char bits[3], DevStatus *st,
                int step) {
    const long long n = p.n;
    if (n > 0) {
        k_fast_import<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            (const float *)s->pos, (const float *)s->anchor, s->type, n, g,
            f->region.as<Rec>(), f->fill.as<int>(), f->cap, f->anchor0.as<float>(), st);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    if (p.field_active && !f->gather)
        CS_CUDA(cudaMemsetAsync(f->rho_q.p, 0, f->rho_q.bytes, ctx->stream));
    CS_TRY(fast_sort(ctx, f, p, gg, bits, st, step));
    CS_TRY(fast_deposit_rows(ctx, f, p, gg, bits, st, step));
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
            p.domain.hi[1] - p.domain.lo[1], (float *)s->pos, (float *)s->anchor,
            f->slab ? f->range.as<int>() : nullptr);
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
    int overlap = 0;  // the field solve runs concurrently on a side stream
};

int fast_field(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
               DevStatus *st, int step) {
    const cs_sim_params &p = *c.p;
    const long long m = (long long)c.gg.n * c.gg.n;
    const double dt = p.dt;
    const double scale = (1.0 / Q_SCALE) * (1.0 / (c.gg.d0 * c.gg.d1));
    if (spectral_on(c.ops) && c.ops->prec == CS_F32)  // periodic: the fused three-pass solve
        return spectral_step_q(c.ops, (float *)s->c, f->rho_q.as<int>(), p.gamma, p.k_alpha,
                               p.k_beta, scale, st);
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

// The fused force + update kernel (k_fast_forces<true>): interacting
// particles, one domain (slab mode keeps the split kernels).  CS_FUSED=0/1
// overrides the default.
bool fast_fused(const cs_fast *f, const cs_sim_params &p) {
    if (p.interaction != 1 || f->slab) return false;
    const char *e = getenv("CS_FUSED");
    return e ? atoi(e) != 0 : false;
}

// part: 1 = pair forces, 2 = update (drift, EM, boundaries, binning)
int fast_particles(cs_ctx *ctx, cs_fast *f, const FastStepCfg &c, const cs_sim_state *s,
                   const void *xi, DevStatus *st, int step, int part) {
    const cs_sim_params &p = *c.p;
    const long long n = p.n;
    FastArgs a;
    a.rec = f->rec[f->cur].as<Rec>();
    a.starts = cell_table(f, f->cur);
    a.region = f->region.as<Rec>();
    a.fill = f->fill.as<int>();
    a.cap = f->cap;
    a.force = f->force.as<double2>();
    a.gen_count = f->gen.as<int>();
    a.gen_dead = f->gen.as<int>() + 1;
    a.gen = f->gen.as<int>() + 2;
    {
        const char *dbg = getenv("CS_FAST_DEBUG");
        a.debug = dbg ? atoi(dbg) : 0;
    }
    a.xi = (const float *)xi;
    a.xi_slot = p.xi_by_slot ? 1 : 0;
    if (f->xi_ready && !(part & 4)) {  // gathered into slot order by the last bucket sort
        a.xi = f->xi_slot.as<float>();
        a.xi_slot = 1;
    }
    a.grad = s ? (const float *)s->grad : nullptr;
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
    a.halff0 = (float)a.half0;
    a.halff1 = (float)a.half1;
    a.sizef0 = (float)c.g.size0;
    a.sizef1 = (float)c.g.size1;
    for (int k = 0; k < 4; k++) a.cutf2[k] = (float)(a.pt.cut2[k] * (1.0 + 1e-5));
    a.eff0 = make_exact_div(c.g.eff0);
    a.eff1 = make_exact_div(c.g.eff1);
    a.gd0 = make_exact_div(c.gg.d0 > 0 ? c.gg.d0 : 1.0);
    a.gd1 = make_exact_div(c.gg.d1 > 0 ? c.gg.d1 : 1.0);
    a.sz0 = make_exact_div(p.domain.hi[0] - p.domain.lo[0]);
    a.sz1 = make_exact_div(p.domain.hi[1] - p.domain.lo[1]);
    a.dom = p.domain;
    a.slab = f->slab ? 1 : 0;
    a.range = f->slab ? f->range.as<int>() : nullptr;
    a.rank = f->rank;
    a.world = f->world;
    a.b0 = f->b0;
    a.b1 = f->b1;
    a.per_rows = c.g.per1;
    a.row_owner = f->slab ? f->row_owner.as<int>() : nullptr;
    a.bounds = f->slab ? f->bounds.as<int>() : nullptr;
    a.outbox = f->slab ? f->outbox.as<Rec>() : nullptr;
    a.out_dest = f->slab ? f->out_dest.as<int>() : nullptr;
    a.out_count = f->slab ? f->out_count.as<int>() : nullptr;
    a.out_cap = f->out_cap;
    a.out_seg = (part & 4) ? 0 : f->out_seg;  // a re-balance can move every record: tagged outbox
    const bool fused = fast_fused(f, p);
    if (n > 0) {
        static int resident_s[2] = {0, 0};  // blocks of k_fast_forces resident per SM
        int &resident = resident_s[fused ? 1 : 0];
        if (!resident) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &resident, fused ? (const void *)k_fast_forces<true> : (const void *)k_fast_forces<false>, 128,
                0);
            if (resident < 1) resident = 1;
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        // with the field solve running concurrently (side stream), leave one
        // block's worth of registers per SM to its kernels
        static int leave = -1;  // CS_FORCE_LEAVE: resident blocks per SM left to the side stream
        if (leave < 0) {
            const char *e = getenv("CS_FORCE_LEAVE");
            leave = e ? atoi(e) : 1;
        }
        const int per_sm =
            c.overlap ? (resident - leave > 1 ? resident - leave : 1) : resident;
        const long long want_f = (n + 127) / 128;
        const int grid =
            (int)(want_f < (long long)sms * per_sm ? want_f : (long long)sms * per_sm);
        const long long want = (n + 255) / 256;
        if (part & 1)  // the update reuses the forces' constant block
            CS_CUDA(cudaMemcpyToSymbolAsync(cA, &a, sizeof(FastArgs), 0,
                                            cudaMemcpyHostToDevice, ctx->stream));
        if (fused && (part & 1)) {  // forces + update; part 2 has nothing left to do
            k_fast_forces<true><<<grid, 128, 0, ctx->stream>>>(st, step);
            CS_LAUNCH_CHECK();
            k_fast_forces_generic<true><<<sms * 16, 128, 0, ctx->stream>>>(st, step);
            CS_LAUNCH_CHECK();
            CS_CUDA(cudaMemsetAsync(a.gen_count, 0, sizeof(int), ctx->stream));
            ctx->launches += 2;
            return CS_OK;
        }
        if (fused && (part & 2)) return CS_OK;
        if (a.interact && (part & 1)) {
            k_fast_forces<false><<<grid, 128, 0, ctx->stream>>>(st, step);
            CS_LAUNCH_CHECK();
            k_fast_forces_generic<false><<<sms * 16, 128, 0, ctx->stream>>>(st, step);
            CS_LAUNCH_CHECK();
            ctx->launches += 2;
        }
        if (part & 4) {  // slab re-balancing (the constant block is this call's)
            CS_CUDA(cudaMemcpyToSymbolAsync(cA, &a, sizeof(FastArgs), 0, cudaMemcpyHostToDevice,
                                            ctx->stream));
            k_slab_reroute<<<sms * 8, 256, 0, ctx->stream>>>(st, step);
            CS_LAUNCH_CHECK();
            ctx->launches += 1;
            return CS_OK;
        }
        if (!(part & 2)) return CS_OK;
        // persistent grid: one contiguous processing front, so the atomics'
        // working set (cell histogram + deposit rows near the front) stays in L2
        static int resident_u = 0;
        if (!resident_u) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident_u, k_fast_update<false>, 256,
                                                          0);
            if (resident_u < 1) resident_u = 1;
        }
        const int grid_u =
            (int)(want < (long long)sms * resident_u ? want : (long long)sms * resident_u);
        if (f->slab)
            k_fast_update<true><<<grid_u, 256, 0, ctx->stream>>>(st, step);
        else
            k_fast_update<false><<<grid_u, 256, 0, ctx->stream>>>(st, step);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    return CS_OK;
}

// part 1: bucket sort into the next record array / cell table (+ the
// atomic-mode deposit); part 2: the row-gathered deposit (periodic grids)
int fast_resort(cs_ctx *ctx, cs_fast *f, long long n, const cs_sim_params &p, const GridGeom &gg,
                const unsigned char bits[3], int part, DevStatus *st, int step,
                const void *xi_next) {
    (void)n;
    // xi_next: the coming step's (N, 2) increments by id, or nullptr when the
    // caller's block ends here.  Gathered ahead only when the array is well
    // beyond the L2 (k_bucket_sort<true>; CS_XI_PREGATHER=0/1 overrides)
    if (xi_next) {
        const char *e = getenv("CS_XI_PREGATHER");
        const bool big = sizeof(float2) * (double)p.n > 256e6;
        if (p.xi_by_slot || f->slab || !(e ? atoi(e) != 0 : big)) xi_next = nullptr;
    }
    if (part & 1) CS_TRY(fast_sort(ctx, f, p, gg, bits, st, step, xi_next));
    if (part & 2) CS_TRY(fast_deposit_rows(ctx, f, p, gg, bits, st, step));
    return CS_OK;
}

// deposit grids the gradient kernel must clear (none when they are written
// in full by k_fast_deposit_rows)
int *fast_rho_q(cs_fast *f) { return f->rho_q.p && !f->gather ? f->rho_q.as<int>() : nullptr; }

bool fast_imported(const cs_fast *f) { return f && f->imported; }

// a new step call: increments gathered ahead belong to the previous call's block
void fast_begin_call(cs_fast *f) {
    if (f) f->xi_ready = false;
}

// ---- y-slab mode host side ------------------------------------------------
int fast_slab_config(cs_fast *f, const int *bounds, int world, int rank, long long n,
                     cudaStream_t stream) {
    if (world < 1 || rank < 0 || rank >= world) {  // (world 1: one slab, no ghosts -- the
                                                   // transports' code path on one rank)
        set_error("slab mode: world >= 1 and 0 <= rank < world");
        return CS_ERR_PARAM;
    }
    const int n1 = f->g.n1;
    std::vector<int> owner((size_t)n1), b((size_t)world + 1);
    for (int q = 0; q <= world; q++) b[(size_t)q] = bounds[q];
    if (b[0] != 0 || b[(size_t)world] != n1) {
        set_error("slab mode: bounds must run from 0 to the %d cell rows", n1);
        return CS_ERR_PARAM;
    }
    for (int q = 0; q < world; q++) {
        if (b[(size_t)q + 1] <= b[(size_t)q]) {
            set_error("slab mode: every rank needs at least one cell row");
            return CS_ERR_PARAM;
        }
        for (int r = b[(size_t)q]; r < b[(size_t)q + 1]; r++) owner[(size_t)r] = q;
    }
    f->slab = true;
    f->world = world;
    f->rank = rank;
    f->b0 = b[(size_t)rank];
    f->b1 = b[(size_t)rank + 1];
    CS_TRY(f->row_owner.ensure(sizeof(int) * (size_t)n1));
    CS_TRY(f->bounds.ensure(sizeof(int) * ((size_t)world + 1)));
    const bool first = f->range.p == nullptr;  // a re-balance keeps the owned range (re-routed)
    CS_TRY(f->range.ensure(sizeof(int) * 4));
    CS_TRY(f->out_count.ensure(sizeof(int) * (size_t)(4 + world)));
    f->out_cap = n > 1024 ? n : 1024;  // every record could leave (kicks cross several slabs)
    CS_TRY(f->outbox.ensure(sizeof(Rec) * (size_t)f->out_cap));
    CS_TRY(f->out_dest.ensure(sizeof(int) * (size_t)f->out_cap));
    CS_CUDA(cudaMemcpyAsync(f->row_owner.p, owner.data(), sizeof(int) * owner.size(),
                            cudaMemcpyHostToDevice, stream));
    CS_CUDA(cudaMemcpyAsync(f->bounds.p, b.data(), sizeof(int) * b.size(),
                            cudaMemcpyHostToDevice, stream));
    if (first) CS_CUDA(cudaMemsetAsync(f->range.p, 0, sizeof(int) * 4, stream));
    CS_CUDA(cudaMemsetAsync(f->out_count.p, 0, sizeof(int) * (size_t)(4 + world), stream));
    CS_CUDA(cudaStreamSynchronize(stream));  // the host vectors go out of scope
    return CS_OK;
}

static int fast_slab_range(cs_ctx *ctx, cs_fast *f) {
    k_slab_range<<<1, 1, 0, ctx->stream>>>(cell_table(f, f->cur), (long long)f->b0 * f->g.n0,
                                            (long long)f->b1 * f->g.n0, f->range.as<int>());
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int fast_slab_import(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const cs_sim_state *s,
                     const GridGeom &gg, const unsigned char bits[3], DevStatus *st, int step) {
    const long long n = p.n;
    if (n > 0) {
        k_slab_import<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            (const float *)s->pos, (const float *)s->anchor, s->type, n, f->g,
            make_exact_div(f->g.eff0), make_exact_div(f->g.eff1), f->b0, f->b1,
            f->region.as<Rec>(), f->fill.as<int>(), f->cap, f->anchor0.as<float>(), st);
        CS_LAUNCH_CHECK();
        ctx->launches += 1;
    }
    CS_TRY(fast_sort(ctx, f, p, gg, bits, st, step));
    CS_TRY(fast_slab_range(ctx, f));
    CS_TRY(fast_deposit_rows(ctx, f, p, gg, bits, st, step));
    f->imported = true;
    return CS_OK;
}

int fast_slab_claim(cs_ctx *ctx, cs_fast *f, const void *recs, long long n, DevStatus *st,
                    int step) {
    if (n <= 0) return CS_OK;
    k_slab_claim<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        (const float4 *)recs, n, f->g, make_exact_div(f->g.eff0), make_exact_div(f->g.eff1),
        f->region.as<Rec>(), f->fill.as<int>(), f->cap, st, step);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int fast_slab_outbox(cs_ctx *ctx, cs_fast *f, void **recs, int **dest, long long *count) {
    int c = 0;
    CS_CUDA(cudaMemcpyAsync(&c, f->out_count.p, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *recs = f->outbox.p;
    *dest = f->out_dest.as<int>();
    *count = c < f->out_cap ? c : f->out_cap;
    return CS_OK;
}

int fast_slab_reset_outbox(cs_ctx *ctx, cs_fast *f) {
    CS_CUDA(cudaMemsetAsync(f->out_count.p, 0, sizeof(int) * (size_t)(1 + f->world), ctx->stream));
    return CS_OK;
}

// Packed exchange: seg slots of the outbox per destination rank (0: back to
// the tagged outbox).  The outbox holds out_cap >= N records.
int fast_slab_exchange_cap(cs_fast *f, long long seg) {
    if (seg < 0 || seg * f->world > f->out_cap) {
        set_error("slab exchange: %lld slots per rank exceed the outbox (%lld records, %d ranks)",
                  seg, f->out_cap, f->world);
        return CS_ERR_PARAM;
    }
    f->out_seg = seg;
    return CS_OK;
}

// device pointers of the packed outbox: records [world][seg], counts [world]
int fast_slab_outbox_packed(cs_fast *f, void **recs, int **counts, long long *seg) {
    *recs = f->outbox.p;
    *counts = f->out_count.as<int>() + 1;
    *seg = f->out_seg;
    return CS_OK;
}

// the records received in packed form (segment s = from rank s, counts[s]
// of its seg slots filled; counts on the device) claimed into their buckets
__global__ void k_slab_claim_packed(const float4 *__restrict__ in, const int *__restrict__ counts,
                                    long long seg, BinGeom g, ExactDiv eff0, ExactDiv eff1,
                                    Rec *__restrict__ region, int *__restrict__ fill,
                                    long long cap, DevStatus *st, int step) {
    const int sgm = blockIdx.y;
    int cnt = counts[sgm];
    if (cnt > seg) cnt = (int)seg;  // (the sender stopped the run)
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < cnt;
         j += (long long)gridDim.x * blockDim.x) {
        const float4 r = in[(long long)sgm * seg + j];
        const int key = slab_row(r.y, g, eff1) * g.n0 +
                        cell_axis_fast((double)r.x, g.lo0, eff0, g.n0);
        const int q = (key >> BUCKET_SHIFT) * SUBB + (threadIdx.x & (SUBB - 1));
        const int slot = atomicAdd(&fill[q], 1);
        if (slot < cap) {
            reinterpret_cast<float4 *>(region)[(long long)q * cap + slot] = r;
        } else {
            atomicMin(&st->key, err_key(3, q / SUBB, CS_SORT_OVERFLOW));
            st->abort = 1;
            st->step = step;
        }
    }
}

int fast_slab_claim_packed(cs_ctx *ctx, cs_fast *f, const void *inbox, const int *counts,
                           long long seg, DevStatus *st, int step) {
    if (seg <= 0) return CS_OK;
    int gx = grid_for(seg, 256);
    if (gx > 148 * 4) gx = 148 * 4;
    k_slab_claim_packed<<<dim3((unsigned)gx, (unsigned)f->world), 256, 0, ctx->stream>>>(
        (const float4 *)inbox, counts, seg, f->g, make_exact_div(f->g.eff0),
        make_exact_div(f->g.eff1), f->region.as<Rec>(), f->fill.as<int>(), f->cap, st, step);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

int fast_slab_sort(cs_ctx *ctx, cs_fast *f, const cs_sim_params &p, const GridGeom &gg,
                   const unsigned char bits[3], DevStatus *st, int step) {
    CS_TRY(fast_sort(ctx, f, p, gg, bits, st, step));
    return fast_slab_range(ctx, f);
}

int fast_slab_hist(cs_ctx *ctx, cs_fast *f, int *hist) {
    CS_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * (size_t)f->g.n1, ctx->stream));
    k_slab_hist<<<148 * 8, 256, 0, ctx->stream>>>(f->rec[f->cur].as<Rec>(), f->range.as<int>(),
                                                  f->g, make_exact_div(f->g.eff1), hist);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

bool fast_slab_gather(const cs_fast *f) { return f->gather; }
int fast_slab_world(const cs_fast *f) { return f->world; }
int fast_slab_rank(const cs_fast *f) { return f->rank; }
int fast_slab_dep_window(cs_fast *f, int j0, int rows) {
    f->dep_j0 = j0;
    f->dep_rows = rows;
    return CS_OK;
}
void *fast_rho_all(cs_fast *f) { return f->rho_q.p; }

int fast_slab_range_host(cs_ctx *ctx, cs_fast *f, long long *lo, long long *hi) {
    int r[2] = {0, 0};
    CS_CUDA(cudaMemcpyAsync(r, f->range.p, sizeof(r), cudaMemcpyDeviceToHost, ctx->stream));
    CS_CUDA(cudaStreamSynchronize(ctx->stream));
    *lo = r[0];
    *hi = r[1];
    return CS_OK;
}

}  // namespace cs
