"""Golden vectors of the reference's CellIndex / Neighbor query API,
accumulate_forces and deposit_gather (chemosim/spatial_index.py:65-178,
motion.py:107-161, coupling.py:190-213), produced by the reference itself:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_index.py      -> tests/golden/index.npz
"""

from __future__ import annotations

import os

import numpy as np

import chemosim as cs

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "index.npz")


def main():
    g = {}
    rng = np.random.default_rng(20)
    # index builds: (n, cell_side, periodic); the last rows sit on the closed
    # upper edge and on lo
    builds = [(400, 0.1, False), (400, 0.3, True), (300, 0.45, True), (50, 2.0, False)]
    for k, (n, side, per) in enumerate(builds):
        pos = rng.uniform(-0.5, 0.5, (n, 2))
        pos[-1] = [0.5, 0.5]
        pos[-2] = [-0.5, 0.5]
        pos[-3] = [0.5, -0.5]
        dom = cs.Domain.square(1.0, periodic=per)
        idx = cs.CellIndex.build(pos, dom, side)
        g[f"b{k}_pos"], g[f"b{k}_meta"] = pos, np.array([side, per])
        g[f"b{k}_order"], g[f"b{k}_starts"] = idx.order, idx.starts
        g[f"b{k}_cell_xy"], g[f"b{k}_n_cells"] = idx.cell_xy, idx.n_cells
        # queries: inside radius, wider than a cell, across the periodic seam
        qs = [((0.0, 0.0), 0.05), ((0.49, -0.49), 0.12), ((0.1, 0.2), 0.31), ((-0.5, 0.5), 0.2)]
        for q, (pt, rad) in enumerate(qs):
            nb = idx.query(np.array(pt), rad)
            g[f"b{k}_q{q}_ids"] = np.array([x.id for x in nb], dtype=np.int64)
            g[f"b{k}_q{q}_dx"] = np.array([x.dx for x in nb]).reshape(-1, 2)
            g[f"b{k}_q{q}_dist"] = np.array([x.distance for x in nb])
            g[f"b{k}_q{q}_pt"], g[f"b{k}_q{q}_rad"] = np.array(pt), rad
    g["n_builds"], g["n_queries"] = len(builds), 4
    # accumulate_forces: reach 1 / 2 / 3 cells, periodic axes with 2 and 3
    # cells (whole-axis rings), walls
    forces = [(2000, 0.02, 0.05, 0.05, False), (2000, 0.02, 0.05, 0.025, True),
              (2000, 0.02, 0.05, 0.017, False), (300, 0.1, 0.3, 0.4, True),
              (300, 0.1, 0.3, 0.3, True), (600, 0.05, 0.12, 0.04, True)]
    for k, (n, eps, cut, side, per) in enumerate(forces):
        pos = rng.uniform(-0.5, 0.5, (n, 2))
        dom = cs.Domain.square(1.0, periodic=per)
        pop = cs.Population(ids=np.arange(n), positions=pos.copy(), next_positions=pos.copy(),
                            species=np.ones(n, np.uint8), drift=np.zeros((n, 2)),
                            local_concentration=np.zeros(n), start_anchor=pos.copy())
        params = cs.MotionParams(epsilon=eps, cutoff=cut, dt=1e-9)
        idx = cs.CellIndex.build(pos, dom, side)
        g[f"f{k}_pos"], g[f"f{k}_meta"] = pos, np.array([eps, cut, side, per])
        g[f"f{k}_force"] = cs.accumulate_forces(pop, idx, params)
    g["n_forces"] = len(forces)
    # deposit_gather: neumann and periodic grids
    gathers = [(32, "neumann", 0.02), (32, "periodic", 0.03), (17, "neumann", 0.05)]
    for k, (nc, bnd, h) in enumerate(gathers):
        n = 300
        pos = rng.uniform(-0.5, 0.5, (n, 2))
        sp = (rng.random(n) < 0.5).astype(np.uint8)
        pop = cs.Population(ids=np.arange(n), positions=pos.copy(), next_positions=pos.copy(),
                            species=sp, drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                            start_anchor=pos.copy())
        grid = cs.Grid.square(nc, 1.0, bnd)
        ker = cs.Kernel("gaussian", h, 3.0 * h)
        g[f"g{k}_pos"], g[f"g{k}_sp"] = pos, sp
        g[f"g{k}_meta"] = np.array([nc, bnd == "periodic", h])
        g[f"g{k}_rho_a"] = cs.deposit_gather(pop, grid, ker, cs.Species.ALPHA)
        g[f"g{k}_rho_b"] = cs.deposit_gather(pop, grid, ker, cs.Species.BETA)
    g["n_gathers"] = len(gathers)
    np.savez(OUT, **g)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
