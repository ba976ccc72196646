"""Species switching restated on numpy -- TEST INFRASTRUCTURE ONLY.

Follows chemosim/reactions.py:43-81 (fixed_step_reactions: one uniform per
particle, decisions against the species snapshot, Alpha -> Beta when
u < r_alpha dt, Beta -> Alpha when u < (r_beta * max(c, 0)) * dt, the new
Alphas' drift rows zeroed, :37-39) and :141-160 (beta_step_reactions = the
same with the Alpha channel off).  Pinned against the reference by
tests/test_oracle_golden.py (tests/golden/reactions.npz).
"""

from __future__ import annotations

import numpy as np


def fixed_step(types, local_c, drift, u, p_ab, r_beta, dt):
    """-> (new types, new drift, (n_ab, n_ba), high) where high is the largest
    flip probability above 1 (0.0 if none), the value the reference warns
    about."""
    types = np.asarray(types, dtype=np.uint8)
    u = np.asarray(u, dtype=np.float64)
    is_alpha = types == 0
    is_beta = ~is_alpha
    high = 0.0
    if is_alpha.any() and p_ab > 1.0:
        high = float(p_ab)
    to_beta = is_alpha & (u < p_ab)
    to_alpha = np.zeros_like(is_alpha)
    if r_beta != 0.0:
        conc = np.maximum(np.asarray(local_c, dtype=np.float64), 0.0)
        p_ba = r_beta * conc * dt
        if is_beta.any():
            m = float(p_ba[is_beta].max())
            if m > 1.0:
                high = max(high, m)
        to_alpha = is_beta & (u < p_ba)
    out = types.copy()
    out[to_beta] = 1
    out[to_alpha] = 0
    d = np.array(drift, dtype=np.float64, copy=True)
    d[to_alpha] = 0.0
    return out, d, (int(to_beta.sum()), int(to_alpha.sum())), high


def tamed_step(pos, dcoef, drift, force, xi, dt):
    """chemosim/motion.py:283-298 restated (numpy, the reference's own
    operation order): ((x + sqrt((2 D) dt) xi) + drift dt) + (f dt) /
    (1 + ||f|| dt)."""
    pos = np.asarray(pos, dtype=np.float64)
    amp = np.sqrt(2.0 * np.asarray(dcoef, dtype=np.float64) * dt)[:, None]
    f = np.asarray(force, dtype=np.float64)
    fnorm = np.sqrt((f * f).sum(axis=-1, keepdims=True))
    tamed = f * dt / (1.0 + fnorm * dt)
    return pos + amp * np.asarray(xi) + np.asarray(drift) * dt + tamed
