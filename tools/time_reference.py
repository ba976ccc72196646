"""Time the reference's own functions on the bench workload.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    NUMBA_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 \
        python tools/time_reference.py --config cfg3 --steps 2 \
        --out profiles/r02/reference_numba_cfg3.json

Runs the reference (`chemosim`, imported from /root/reference -- this
container only; it does not travel to the GPU box) in Realisation._step_inner
order (engine.py:369-387) on the bench's seeded state, one core, timing each
stage with perf_counter after one untimed JIT warm-up step:
deposit_both (CIC), gradient, refresh_particle_fields, soft_forces, em_step,
apply_boundaries.  The periodic implicit field step is SuperLU on a
(n_c^2)^2 system: infeasible at 4096^2, so it is reported as
such and the stage sum excludes it.  The reference has one epsilon for all
pairs; the two-radius pair table of cfg3 (BASELINE) is timed with epsilon =
r_B and cutoff = 2 r_B: the same cells and candidates, and at least as many
accepted pairs.  Replica rate = cores x the 1-core rate (the reference's
only parallelism is one realisation per process, engine.py:463-467).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from chemosim import coupling, field, motion, particles, spatial_index
    cfg = bench.CONFIGS[args.config]
    n, n_c = cfg["n"], cfg["n_c"]
    rng = np.random.default_rng(bench.SEED)
    pos = bench.initial_positions(cfg, rng)
    sp = (np.arange(n) >= n // 2).astype(np.uint8) if cfg["types"] == "half" \
        else np.ones(n, np.uint8)
    pop = particles.Population(ids=np.arange(n), positions=pos.copy(),
                               next_positions=pos.copy(), species=sp,
                               drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                               start_anchor=pos.copy())
    dom = spatial_index.Domain.square(1.0, periodic=cfg["periodic"])
    eps = cfg["radii"][1] if cfg["radii"] else cfg["eps"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = motion.MotionParams(d_alpha=cfg["D"][0], d_beta=cfg["D"][1], chi=1.0, epsilon=eps,
                                 dt=bench.DT, cutoff=2 * eps)
    grid = field.Grid.square(n_c, 1.0, cfg.get("boundary", "periodic")) if cfg["field"] else None
    fp = field.FieldParams(d_c=cfg.get("d_c", 0.0), k_alpha=cfg.get("k_alpha", 0.0),
                           k_beta=cfg.get("k_beta", 0.0), gamma=cfg.get("gamma", 0.0)) \
        if cfg["field"] else None
    xi_rng = np.random.default_rng(bench.SEED + 1)
    D = mp.diffusion_of(sp)
    stages = {}
    ops = None
    pde_ops = None
    if grid is not None and n_c <= 512:  # the reference's own implicit step is feasible
        pde_ops = field.build_operators(grid, fp, bench.DT)
    if grid is not None:
        # the gradient operator only (the solve's SuperLU factorisation at
        # 4096^2 periodic is the infeasible part)
        f = field.Field(c=np.zeros(n_c * n_c), grad=np.zeros((n_c * n_c, 2)),
                        rho_alpha=np.zeros(n_c * n_c), rho_beta=np.zeros(n_c * n_c))
        from scipy import sparse as sp_
        d1 = field._d1_1d(n_c, grid.spacing[0], grid.boundary == "periodic")
        eye = sp_.identity(n_c, format="csr")

        class _Ops:
            dx = sp_.kron(eye, d1, format="csr")
            dy = sp_.kron(d1, eye, format="csr")
        ops = _Ops()
    kern = coupling.Kernel(kind="cic", h=0.0, cutoff=0.0) if grid is not None else None

    def tick(name, t0, timed):
        t1 = time.perf_counter()
        if timed:
            stages[name] = stages.get(name, 0.0) + (t1 - t0)
        return t1

    for s in range(args.steps + 1):
        timed = s > 0
        t0 = time.perf_counter()
        if grid is not None:
            f.rho_alpha, f.rho_beta = coupling.deposit_both(pop, grid, kern)
            t0 = tick("deposit", t0, timed)
            if pde_ops is not None:
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    field.step_field(f, pde_ops, fp, bench.DT)
                t0 = tick("pde", t0, timed)
            f.grad[:, 0] = ops.dx @ f.c
            f.grad[:, 1] = ops.dy @ f.c
            t0 = tick("gradient", t0, timed)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                coupling.refresh_particle_fields(pop, f, grid, 1.0)
            t0 = tick("refresh", t0, timed)
        force = motion.soft_forces(pop, dom, mp)
        t0 = tick("force", t0, timed)
        xi = xi_rng.standard_normal((n, 2))

        class _Fixed:
            def standard_normal(self, shape):
                return xi
        pop.next_positions[:] = motion.em_step(pop.positions, D, pop.drift, force, bench.DT,
                                               _Fixed())
        t0 = tick("em", t0, timed)
        motion.apply_boundaries(pop, dom)
        tick("boundaries", t0, timed)
        print(f"step {s}: {time.perf_counter():.1f}", file=sys.stderr)
    per_step = {k: v / args.steps for k, v in stages.items()}
    total = sum(per_step.values())
    cores = os.cpu_count() or 1
    model = bench.cpu_model()
    out = {"config": args.config, "n": n, "steps_timed": args.steps,
           "threads": 1, "cpu_model": model, "host": platform.node(), "cores": cores,
           "stage_s_per_step": {k: round(v, 4) for k, v in per_step.items()},
           "pde": ("timed (field.step_field)" if pde_ops is not None else
                   "periodic SuperLU at %d^2: infeasible (SURVEY 6), excluded" % n_c)
           if grid is not None else "no field",
           "value_1core": n / total, "unit": bench.UNIT,
           "value_replicas": cores * n / total,
           "note": "reference chemosim functions on one core in _step_inner order, "
                   "build container (the reference does not travel to the GPU box); "
                   "soft forces with epsilon = r_B, cutoff = 2 r_B (the reference has "
                   "one epsilon); replicas = cores x one core"}
    print(json.dumps(out, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
