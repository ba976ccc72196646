"""Reference ensemble for the parity tier T4, run through the
reference's own Realisation (numba, fp64) in this container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_t4.py

writes tests/golden/t4_reference.npz: per-sample statistics (t4_stats.py) of
samples 0..S-1 of T4_CONFIG (seed_base 0) after t_final."""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import chemosim as cs  # noqa: E402
from t4_stats import NAMES, T4_CONFIG, sample_stats  # noqa: E402

S = int(os.environ.get("T4_SAMPLES", "48"))


def main():
    cfg = cs.SimConfig(**T4_CONFIG, seed_base=0)
    rows = []
    t0 = time.time()
    for s in range(S):
        real = cs.Realisation(cfg, s)
        real.run()
        pop = real.pop
        grid = real.grid
        rows.append(sample_stats(pop.positions, pop.start_anchor, pop.species, real.field.c,
                                 grid.quadrature_weights(), cfg.domain_size,
                                 cfg.soft_cutoff_factor * cfg.epsilon))
    stats = np.array(rows)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "t4_reference.npz")
    np.savez(out, stats=stats, names=np.array(NAMES))
    print(f"{S} samples in {time.time() - t0:.1f} s -> {out}")
    for k, nm in enumerate(NAMES):
        print(f"  {nm:10s} {stats[:, k].mean():.6g} +- {stats[:, k].std(ddof=1) / np.sqrt(S):.3g}")


if __name__ == "__main__":
    main()
