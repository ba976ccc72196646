// react.cu -- stochastic species switching (chemosim/reactions.py).
//
// fixed_step_reactions (reactions.py:43-81): one uniform u per particle per
// step, decisions against the species snapshot (each particle reads only its
// own label, so a particle flips at most once), Alpha -> Beta when
// u < r_alpha dt, Beta -> Alpha when u < (r_beta * max(c_local, 0)) * dt with
// the drift row of a new Alpha zeroed (_flip_to_alpha, :37-39).  A
// probability above 1 is clamped by the reference with a warning; u < 1
// always, so the clamped and unclamped decisions agree and the kernel only
// records the largest such probability for the host's warning.
// beta_step_reactions (:141-160) is the same kernel with p_ab = 0.
#include "common.cuh"

namespace cs {

__global__ void __launch_bounds__(256)
k_react(uint8_t *__restrict__ type, const double *__restrict__ local_c,
        double *__restrict__ drift, const double *__restrict__ u, long long n, double p_ab,
        double r_beta, double dt, DevStatus *st) {
    if (st->abort) return;  // the step failed before the reactions (engine.py:384-387)
    unsigned long long f_ab = 0, f_ba = 0, hn = 0;
    double high = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double ui = u[i];
        if (type[i] == 0) {
            if (p_ab > 1.0) {
                hn++;
                high = fmax(high, p_ab);
            }
            if (ui < p_ab) {
                type[i] = 1;
                f_ab++;
            }
        } else if (r_beta != 0.0) {
            const double c = local_c ? local_c[i] : 0.0;
            const double conc = c > 0.0 || c != c ? c : 0.0;  // np.maximum(c, 0.0)
            const double p = dmul(dmul(r_beta, conc), dt);
            if (p > 1.0) {
                hn++;
                high = fmax(high, p);
            }
            if (ui < p) {
                type[i] = 0;
                if (drift) reinterpret_cast<double2 *>(drift)[i] = make_double2(0.0, 0.0);
                f_ba++;
            }
        }
    }
    // warp-reduce the counters before the atomics
    for (int o = 16; o > 0; o >>= 1) {
        f_ab += __shfl_down_sync(0xffffffffu, f_ab, o);
        f_ba += __shfl_down_sync(0xffffffffu, f_ba, o);
        hn += __shfl_down_sync(0xffffffffu, hn, o);
        high = fmax(high, __shfl_down_sync(0xffffffffu, high, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (f_ab) atomicAdd(&st->react_flips[0], f_ab);
        if (f_ba) atomicAdd(&st->react_flips[1], f_ba);
        if (hn) {
            atomicAdd(&st->react_high_n, hn);
            atomicMax(&st->react_high_bits, (unsigned long long)__double_as_longlong(high));
        }
    }
}

int launch_react(cs_ctx *ctx, uint8_t *type, const double *local_c, double *drift,
                 const double *u, long long n, double p_ab, double r_beta, double dt,
                 DevStatus *st) {
    if (n <= 0) return CS_OK;
    k_react<<<grid_for(n, 256), 256, 0, ctx->stream>>>(type, local_c, drift, u, n, p_ab, r_beta,
                                                      dt, st);
    CS_LAUNCH_CHECK();
    ctx->launches += 1;
    return CS_OK;
}

}  // namespace cs
