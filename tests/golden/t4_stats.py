"""Per-realisation statistics of the parity tier T4: per-type
MSD, in-cutoff pair count, g(r) histogram inside the cutoff, field weighted
mass and L2 norm.  Pure numpy: used by make_t4.py on the reference's
Realisation and by tests/test_gpu_t4.py on ours."""

from __future__ import annotations

import numpy as np

# the T4 configuration: two species, periodic box and grid, secretion by
# Alpha, consumption by Beta, chemotaxis (Beta repelled), soft pair forces;
# fp32 on our side selects the sorted engine
T4_CONFIG = dict(n_alpha_0=2000, n_beta_0=2000, d_alpha=1.0, d_beta=0.5, chi=-0.5,
                 epsilon=0.002, soft_cutoff_factor=2.0, dt=1e-5, t_final=2e-3, r_alpha=0.0,
                 r_beta=0.0, periodic=True, n_c=64, deposit="cic", d_c=1.0, k_alpha=0.1,
                 k_beta=0.03, gamma=0.1, output_every=50)
GR_BINS = 4
NAMES = ["msd_alpha", "msd_beta", "pairs"] + [f"gr{k}" for k in range(GR_BINS)] + \
    ["mass", "l2"]


def pair_distances(pos: np.ndarray, size: float, cutoff: float) -> np.ndarray:
    """Distances of all unordered pairs within the cutoff (periodic minimum
    image, scipy's periodic k-d tree)."""
    from scipy.spatial import cKDTree
    p = np.mod(pos + 0.5 * size, size)
    p[p >= size] = 0.0
    tree = cKDTree(p, boxsize=size)
    pairs = tree.query_pairs(cutoff, output_type="ndarray")
    if len(pairs) == 0:
        return np.zeros(0)
    d = pos[pairs[:, 1]] - pos[pairs[:, 0]]
    d -= size * np.round(d / size)
    r = np.sqrt((d * d).sum(axis=1))
    return r[r <= cutoff]


def sample_stats(positions, start_anchor, species, c, weights, size, cutoff) -> np.ndarray:
    d = positions - start_anchor
    sq = (d * d).sum(axis=1)
    r = pair_distances(positions, size, cutoff)
    gr, _ = np.histogram(r, bins=GR_BINS, range=(0.0, cutoff))
    mass = float(weights @ c)
    l2 = float(np.sqrt(weights @ (c * c)))
    return np.array([sq[species == 0].mean(), sq[species == 1].mean(), r.size, *gr, mass, l2],
                    dtype=np.float64)


def compare(ref: np.ndarray, ours: np.ndarray, k: float = 3.0):
    """Per statistic: |mean difference| <= k combined standard errors."""
    mr, mo = ref.mean(axis=0), ours.mean(axis=0)
    se = np.sqrt(ref.var(axis=0, ddof=1) / len(ref) + ours.var(axis=0, ddof=1) / len(ours))
    z = np.abs(mo - mr) / np.where(se > 0, se, np.inf)
    return z, mr, mo, se
