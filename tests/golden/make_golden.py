"""Generate the golden fixtures from the reference implementation itself.

Run in the builder container (the reference is NOT present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

Every array below is produced by calling the reference's public functions
(chemosim.*) on seeded inputs; the inputs are stored next to the outputs so
the tests can replay them through the oracle and the CUDA path without the
reference.  Nothing here is copied from the reference's test suite: the
cases are new seeded draws chosen to cover the same edge cases (tiny
periodic boxes, seams, walls, exact overlaps, sharp cutoff, all boundary
statuses).
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

import chemosim as cs
from chemosim.motion import _boundaries_kernel, _soft_forces_fused

OUT = os.path.dirname(os.path.abspath(__file__))


def mkpop(pos, species=None):
    pos = np.atleast_2d(np.asarray(pos, dtype=float))
    n = pos.shape[0]
    sp = np.zeros(n, np.uint8) if species is None else np.asarray(species, np.uint8)
    return cs.Population(ids=np.arange(n, dtype=np.int64), positions=pos.copy(),
                         next_positions=pos.copy(), species=sp.copy(),
                         drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                         start_anchor=pos.copy())


def forces_cases():
    rng = np.random.default_rng(2024)
    cases = []
    # random boxes, both boundary kinds, varied density
    for periodic in (False, True):
        for k in range(12):
            size = float(rng.choice([1.0, 0.5, 2.0]))
            eps = float(rng.uniform(0.01, 0.06)) * size
            factor = float(rng.choice([2.0, 5.0, 3.3]))
            n = int(rng.integers(2, 400))
            pos = rng.uniform(-size / 2, size / 2, (n, 2))
            cases.append((pos, size, periodic, eps, factor))
    # tiny periodic boxes: 1 and 2 cells per axis (ring deduplication)
    for size in (0.08, 0.11, 0.16, 0.25):
        pos = rng.uniform(-size / 2, size / 2, (25, 2))
        cases.append((pos, size, True, 0.01, 5.0))
    # exact overlaps, seam pair, on-face particles, sharp cutoff
    pos = np.array([[0.1, 0.1], [0.1, 0.1], [0.495, 0.0], [-0.495, 0.0],
                    [0.5, 0.5], [-0.5, -0.5], [0.2, 0.2], [0.2 + 0.01, 0.2]])
    cases.append((pos, 1.0, True, 0.005, 2.0))
    cases.append((pos, 1.0, False, 0.005, 2.0))
    # BASELINE config-0 density (N = 1000, eps 0.005, cutoff 2 eps)
    pos = rng.uniform(-0.5, 0.5, (1000, 2))
    cases.append((pos, 1.0, False, 0.005, 2.0))
    cases.append((pos, 1.0, True, 0.005, 2.0))
    # dense (config-2-like candidate counts) small box
    pos = rng.uniform(-0.1, 0.1, (600, 2))
    cases.append((pos, 0.2, True, 0.0075, 8.0 / 3.0))
    out = {}
    for idx, (pos, size, periodic, eps, factor) in enumerate(cases):
        domain = cs.Domain.square(size, periodic=periodic)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            params = cs.MotionParams(epsilon=eps, dt=1e-9, interaction="soft",
                                     cutoff=factor * eps)
        f = cs.soft_forces(mkpop(pos), domain, params)
        out[f"c{idx}_pos"] = pos
        out[f"c{idx}_meta"] = np.array([size, float(periodic), eps, params.cutoff])
        out[f"c{idx}_force"] = f
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "forces.npz"), **out)


def em_cases():
    rng = np.random.default_rng(7)
    n = 500
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    species = rng.integers(0, 2, n).astype(np.uint8)
    mp = cs.MotionParams(d_alpha=0.1, d_beta=1.0, dt=1e-5, interaction="none")
    dcoef = mp.diffusion_of(species)
    drift = rng.standard_normal((n, 2))
    force = rng.standard_normal((n, 2)) * 100
    out = cs.em_step(pos, dcoef, drift, force, mp.dt, np.random.default_rng(99))
    xi = np.random.default_rng(99).standard_normal((n, 2))
    np.savez_compressed(os.path.join(OUT, "em.npz"), pos=pos, species=species,
                        dcoef=dcoef, drift=drift, force=force, xi=xi, dt=mp.dt,
                        out=out)


def boundary_cases():
    rng = np.random.default_rng(8)
    res = {}
    k = 0
    for periodic in (False, True):
        for size in (1.0, 2.0):
            n = 300
            x = rng.uniform(-size / 2 - 0.4 * size, size / 2 + 0.4 * size, (n, 2))
            x[:5] = [[size / 2, -size / 2], [-size / 2, size / 2], [0.0, 0.0],
                     [size / 2 + 1e-17, 0.0], [np.nextafter(size / 2, 9), 0.1]]
            anchor = rng.uniform(-1, 1, (n, 2))
            xx, aa = x.copy(), anchor.copy()
            lo, hi = -size / 2, size / 2
            st, i, ax = _boundaries_kernel(xx, aa, lo, lo, hi, hi, periodic, periodic)
            res[f"b{k}_in"] = x
            res[f"b{k}_anchor_in"] = anchor
            res[f"b{k}_out"] = xx
            res[f"b{k}_anchor_out"] = aa
            res[f"b{k}_meta"] = np.array([size, float(periodic), st, i, ax])
            k += 1
    # error statuses: non-finite (min index), overshoot, unsettled is
    # unreachable after the overshoot guard; periodic never errors
    for x, periodic in (
        (np.array([[0.0, 0.0], [0.1, np.nan], [np.inf, 0.0]]), False),
        (np.array([[0.0, 0.0], [0.2, 1.7], [1.8, 0.0]]), False),
        (np.array([[0.0, 0.0], [0.2, 1.7], [0.3, 0.0]]), False),
        (np.array([[2.9, -3.7], [0.2, 1.7], [-1.3, 0.2]]), True),
    ):
        anchor = np.zeros_like(x)
        xx, aa = x.copy(), anchor.copy()
        st, i, ax = _boundaries_kernel(xx, aa, -0.5, -0.5, 0.5, 0.5, periodic, periodic)
        res[f"b{k}_in"] = x
        res[f"b{k}_anchor_in"] = anchor
        res[f"b{k}_out"] = xx
        res[f"b{k}_anchor_out"] = aa
        res[f"b{k}_meta"] = np.array([1.0, float(periodic), st, i, ax])
        k += 1
    res["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "boundaries.npz"), **res)


def field_cases():
    rng = np.random.default_rng(9)
    res = {}
    k = 0
    for boundary, n_c in (("neumann", 24), ("periodic", 24), ("neumann", 33),
                          ("periodic", 32)):
        g = cs.Grid.square(n_c, 1.0, boundary)
        params = cs.FieldParams(d_c=0.8, k_alpha=0.2, k_beta=0.05, gamma=0.3)
        dt = 2e-3
        ops = cs.build_operators(g, params, dt)
        f = cs.Field.zeros(g)
        f.c = rng.random(n_c * n_c)
        f.rho_alpha = rng.random(n_c * n_c) * 10
        f.rho_beta = rng.random(n_c * n_c) * 10
        res[f"f{k}_c"] = f.c.copy()
        res[f"f{k}_ra"] = f.rho_alpha.copy()
        res[f"f{k}_rb"] = f.rho_beta.copy()
        res[f"f{k}_meta"] = np.array([n_c, float(boundary == "periodic"),
                                      params.d_c, params.k_alpha, params.k_beta,
                                      params.gamma, dt])
        rhs = rng.standard_normal(n_c * n_c)
        res[f"f{k}_rhs"] = rhs
        res[f"f{k}_solve"] = ops.solve(rhs)
        cs.step_field(f, ops, params, dt)
        res[f"f{k}_cnew"] = f.c.copy()
        cs.gradient(f, ops)
        res[f"f{k}_grad"] = f.grad.copy()
        k += 1
    res["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "field.npz"), **res)


def coupling_cases():
    rng = np.random.default_rng(10)
    res = {}
    k = 0
    for boundary, n_c, kind in (("neumann", 27, "cic"), ("periodic", 26, "cic"),
                                ("neumann", 41, "gaussian"),
                                ("periodic", 40, "gaussian"),
                                ("neumann", 128, "cic")):
        g = cs.Grid.square(n_c, 1.0, boundary)
        kernel = cs.Kernel(kind=kind, h=0.02, cutoff=0.06)
        n = 300
        pos = rng.uniform(-0.5, 0.5, (n, 2))
        pos[:4] = [[0.5, 0.5], [-0.5, -0.5], [0.5, -0.5], [0.25, -0.25]]
        species = rng.integers(0, 2, n).astype(np.uint8)
        pop = mkpop(pos, species)
        ra, rb = cs.deposit_both(pop, g, kernel)
        f = cs.Field.zeros(g)
        f.c = rng.random(n_c * n_c)
        f.grad = rng.standard_normal((n_c * n_c, 2))
        cs.refresh_particle_fields(pop, f, g, 1.7)
        res[f"k{k}_pos"] = pos
        res[f"k{k}_species"] = species
        res[f"k{k}_meta"] = np.array([n_c, float(boundary == "periodic"),
                                      float(kind == "cic"), 0.02, 0.06, 1.7])
        res[f"k{k}_ra"] = ra
        res[f"k{k}_rb"] = rb
        res[f"k{k}_c"] = f.c
        res[f"k{k}_grad"] = f.grad
        res[f"k{k}_drift"] = pop.drift.copy()
        res[f"k{k}_conc"] = pop.local_concentration.copy()
        k += 1
    res["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "coupling.npz"), **res)


def cfg0_trajectory():
    """BASELINE config 0 run through the reference's Realisation unmodified
    (SURVEY 8d mapping); positions after 1, 10, 100 steps."""
    cfg = cs.SimConfig(n_alpha_0=0, n_beta_0=1000, d_beta=1.0, chi=0.0,
                       epsilon=0.005, soft_cutoff_factor=2.0, dt=1e-5,
                       t_final=0.01, r_alpha=0.0, r_beta=0.0, d_c=0.0,
                       k_alpha=0.0, k_beta=0.0, gamma=0.0, periodic=False,
                       seed_base=0)
    real = cs.Realisation(cfg, 0)
    res = {"pos0": real.pop.positions.copy()}
    for s in range(1, 101):
        real.step()
        if s in (1, 10, 100):
            res[f"pos{s}"] = real.pop.positions.copy()
    res["seed"] = np.array(cfg.sample_seed(0))
    np.savez_compressed(os.path.join(OUT, "cfg0_traj.npz"), **res)


def composed_cfg1_small():
    """Config-1 semantics at reduced size (N=400, 32^2 grid, 10 steps) through
    the reference's public functions (SURVEY 8d composed driver): a single
    drifting, secreting type (Beta, chi=1, D=1), CIC secretion fed into
    rho_alpha, Neumann grid, D_c=1, gamma=0.1, c0=x, reflective walls."""
    rng = np.random.default_rng(11)
    n, n_c, steps, dt = 400, 32, 10, 1e-5
    domain = cs.Domain.square(1.0)
    grid = cs.Grid.square(n_c, 1.0, "neumann")
    fp = cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.0, gamma=0.1)
    mp = cs.MotionParams(d_alpha=0.1, d_beta=1.0, chi=1.0, epsilon=0.005, dt=dt,
                         interaction="soft", cutoff=0.01)
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    pop = mkpop(pos, np.ones(n, np.uint8))
    f = cs.Field.zeros(grid)
    f.c = grid.node_positions()[:, 0].copy()
    ops = cs.build_operators(grid, fp, dt)
    cs.gradient(f, ops)
    cs.refresh_particle_fields(pop, f, grid, mp.chi)
    xi = rng.standard_normal((steps, n, 2))
    kern = cs.Kernel(kind="cic")
    res = {"pos0": pos.copy(), "xi": xi}
    for s in range(steps):
        f.rho_alpha = cs.deposit(pop, grid, kern, cs.Species.BETA)
        f.rho_beta = np.zeros(n_c * n_c)
        cs.step_field(f, ops, fp, dt)
        cs.gradient(f, ops)
        cs.refresh_particle_fields(pop, f, grid, mp.chi)
        force = cs.soft_forces(pop, domain, mp)
        pop.next_positions[:] = cs.em_step(pop.positions,
                                           mp.diffusion_of(pop.species),
                                           pop.drift, force, dt,
                                           _Replay(xi[s]))
        cs.apply_boundaries(pop, domain)
        res[f"pos{s + 1}"] = pop.positions.copy()
        res[f"c{s + 1}"] = f.c.copy()
    np.savez_compressed(os.path.join(OUT, "cfg1_small.npz"), **res)


def composed_cfg2_small():
    """Config-2 semantics at reduced size with EQUAL radii (the reference's
    homogeneous kernel): Alpha secretes, Beta consumes and drifts, periodic
    box and 32^2 periodic grid, CIC, 8 steps."""
    rng = np.random.default_rng(12)
    n, n_c, steps, dt = 600, 32, 8, 1e-5
    domain = cs.Domain.square(1.0, periodic=True)
    grid = cs.Grid.square(n_c, 1.0, "periodic")
    fp = cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1)
    mp = cs.MotionParams(d_alpha=1.0, d_beta=0.5, chi=-0.5, epsilon=0.01, dt=dt,
                         interaction="soft", cutoff=0.02)
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    species = np.r_[np.zeros(n // 2), np.ones(n - n // 2)].astype(np.uint8)
    pop = mkpop(pos, species)
    f = cs.Field.zeros(grid)
    ops = cs.build_operators(grid, fp, dt)
    kern = cs.Kernel(kind="cic")
    xi = rng.standard_normal((steps, n, 2))
    res = {"pos0": pos.copy(), "species": species, "xi": xi}
    for s in range(steps):
        f.rho_alpha, f.rho_beta = cs.deposit_both(pop, grid, kern)
        cs.step_field(f, ops, fp, dt)
        cs.gradient(f, ops)
        cs.refresh_particle_fields(pop, f, grid, mp.chi)
        force = cs.soft_forces(pop, domain, mp)
        pop.next_positions[:] = cs.em_step(pop.positions,
                                           mp.diffusion_of(pop.species),
                                           pop.drift, force, dt,
                                           _Replay(xi[s]))
        cs.apply_boundaries(pop, domain)
        res[f"pos{s + 1}"] = pop.positions.copy()
        res[f"anchor{s + 1}"] = pop.start_anchor.copy()
        res[f"c{s + 1}"] = f.c.copy()
    np.savez_compressed(os.path.join(OUT, "cfg2_small.npz"), **res)


def reaction_cases():
    """fixed_step_reactions / beta_step_reactions on seeded populations
    (mixed species, negative / zero / large local concentrations, nonzero
    drift rows so the zeroing of new Alphas shows), including clamped
    probabilities; AlphaEventClock event sequences."""
    rng = np.random.default_rng(31)
    res = {}
    cases = [(10.0, 0.0, 1e-3), (10.0, 50.0, 1e-3), (0.0, 80.0, 2e-3),
             (600.0, 0.0, 2e-3), (5.0, 400.0, 3e-3), (0.0, 0.0, 1e-3)]
    for k, (ra, rb, dt) in enumerate(cases):
        n = int(rng.integers(50, 400))
        species = rng.integers(0, 2, n).astype(np.uint8)
        local_c = rng.normal(2.0, 3.0, n)
        local_c[:5] = [0.0, -0.0, -1.0, 1e3, 0.5]
        drift = rng.normal(0.0, 1.0, (n, 2))
        pop = mkpop(rng.uniform(-0.5, 0.5, (n, 2)), species)
        pop.local_concentration[:] = local_c
        pop.drift[:] = drift
        seed = 1000 + k
        u = np.random.default_rng(seed).random(n)
        params = cs.ReactionParams(r_alpha=ra, r_beta=rb)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            cnt = cs.fixed_step_reactions(pop, params, dt, np.random.default_rng(seed))
        res[f"f{k}_in"] = np.array([ra, rb, dt])
        res[f"f{k}_species"] = species
        res[f"f{k}_local_c"] = local_c
        res[f"f{k}_drift"] = drift
        res[f"f{k}_u"] = u
        res[f"f{k}_out_species"] = pop.species.copy()
        res[f"f{k}_out_drift"] = pop.drift.copy()
        res[f"f{k}_counts"] = np.array(cnt)
        res[f"f{k}_warned"] = np.array(len(w))
        # the Beta channel alone (gillespie companion)
        pop2 = mkpop(pop.positions, species)
        pop2.local_concentration[:] = local_c
        pop2.drift[:] = drift
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            nb = cs.beta_step_reactions(pop2, params, dt, np.random.default_rng(seed))
        res[f"b{k}_out_species"] = pop2.species.copy()
        res[f"b{k}_out_drift"] = pop2.drift.copy()
        res[f"b{k}_count"] = np.array(nb)
        res[f"b{k}_warned"] = np.array(len(w))
    res["n_fixed"] = np.array(len(cases))
    # event clock: species after successive advances and the clock times
    species = rng.integers(0, 2, 120).astype(np.uint8)
    pop = mkpop(rng.uniform(-0.5, 0.5, (120, 2)), species)
    crng = np.random.default_rng(77)
    clock = cs.AlphaEventClock(pop.n_alpha, 40.0, 0.0, crng)
    res["clock_species0"] = species
    times = [clock.next_time]
    fired = []
    for until in (0.001, 0.004, 0.01, 0.02, 0.05):
        fired.append(clock.advance(pop, until, crng))
        times.append(clock.next_time)
        res[f"clock_species_{until}"] = pop.species.copy()
    res["clock_times"] = np.array(times)
    res["clock_fired"] = np.array(fired)
    np.savez_compressed(os.path.join(OUT, "reactions.npz"), **res)


def reaction_trajectories():
    """fig1-like runs with reactions through the reference's Realisation
    unmodified: 40 particles, soft forces, gaussian deposit on the Neumann
    52^2 grid, both schedulers; rates raised so that flips (both ways) and,
    in one case, clamped probabilities occur within the recorded steps."""
    res = {}
    runs = {
        "fixed": dict(r_alpha=8000.0, r_beta=3000.0, scheduler="fixed"),
        "gillespie": dict(r_alpha=3000.0, r_beta=3000.0, scheduler="gillespie"),
        "fixed_clamp": dict(r_alpha=3.0e5, r_beta=0.0, scheduler="fixed"),
        "counts": dict(r_alpha=3000.0, r_beta=0.0, scheduler="fixed",
                       interaction="none", d_c=0.0, k_alpha=0.0, k_beta=0.0, dt=1e-4),
    }
    for name, kw in runs.items():
        cfg = cs.SimConfig(n_alpha_0=20, n_beta_0=20, t_final=1.0, seed_base=5, **kw)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            real = cs.Realisation(cfg, 1)
            res[f"{name}_pos0"] = real.pop.positions.copy()
            for s in range(1, 31):
                real.step()
                if s in (1, 5, 10, 20, 30):
                    res[f"{name}_pos{s}"] = real.pop.positions.copy()
                    res[f"{name}_species{s}"] = real.pop.species.copy()
            res[f"{name}_warned"] = np.array(
                sum("flip probability" in str(x.message) for x in w))
    np.savez_compressed(os.path.join(OUT, "reaction_traj.npz"), **res)


def tamed_cases():
    """tamed_step on seeded inputs (force magnitudes from tiny to huge, so
    the taming factor spans 1 .. ~0) and a fig1-like Realisation with the
    tamed integrator."""
    rng = np.random.default_rng(41)
    n = 500
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    dcoef = rng.choice([0.0, 0.1, 1.0], n)
    drift = rng.normal(0.0, 1.0, (n, 2))
    force = rng.normal(0.0, 1.0, (n, 2)) * 10.0 ** rng.uniform(-3, 6, (n, 1))
    force[:3] = 0.0
    dt = 1e-4
    xi = np.random.default_rng(5).standard_normal((n, 2))
    out = cs.tamed_step(pos, dcoef, drift, force, dt, np.random.default_rng(5))
    res = dict(pos=pos, dcoef=dcoef, drift=drift, force=force, dt=np.array(dt), xi=xi, out=out)
    cfg = cs.SimConfig(n_alpha_0=20, n_beta_0=20, t_final=1.0, seed_base=8, r_alpha=0.0,
                       integrator="tamed", epsilon=0.05)
    real = cs.Realisation(cfg, 0)
    res["traj_pos0"] = real.pop.positions.copy()
    for s in range(1, 21):
        real.step()
        if s in (1, 5, 20):
            res[f"traj_pos{s}"] = real.pop.positions.copy()
    np.savez_compressed(os.path.join(OUT, "tamed.npz"), **res)


def hard_sphere_cases():
    """resolve_hard_sphere on seeded dense proposals (chains, immobile
    partners, periodic seams, both species) and a Realisation with hard
    spheres."""
    rng = np.random.default_rng(61)
    res = {}
    cases = [(1.0, False, 0.02, 300), (1.0, True, 0.02, 300), (0.3, True, 0.03, 150),
             (10.0, False, 0.02, 60)]
    for k, (size, per, eps, n) in enumerate(cases):
        domain = cs.Domain.square(size, periodic=per)
        params = cs.MotionParams(epsilon=eps, d_alpha=rng.choice([0.0, 0.1]), d_beta=1.0,
                                 dt=1e-7, interaction="hard")
        pos = rng.uniform(-size / 2, size / 2, (n, 2))
        if k == 3:  # overlapping chains along x
            pos = np.stack([np.arange(n) * 0.9 * eps - 0.3, np.repeat([0.0, 0.011, -0.013], n // 3 + 1)[:n]], 1)
        pos[:4] = pos[4:8] + 0.3 * eps  # guaranteed overlaps
        species = rng.integers(0, 2, n).astype(np.uint8)
        pop = mkpop(pos, species)
        pop.next_positions[:] = pos + rng.normal(0, 0.2 * eps, (n, 2))
        before = pop.next_positions.copy()
        cs.resolve_hard_sphere(pop, domain, params)
        res[f"h{k}_meta"] = np.array([size, per, eps, params.d_alpha, params.d_beta])
        res[f"h{k}_species"] = species
        res[f"h{k}_in"] = before
        res[f"h{k}_out"] = pop.next_positions.copy()
    res["n_cases"] = np.array(len(cases))
    cfg = cs.SimConfig(n_alpha_0=30, n_beta_0=30, t_final=1.0, seed_base=9, r_alpha=0.0,
                       interaction="hard", epsilon=0.05)
    real = cs.Realisation(cfg, 0)
    res["traj_pos0"] = real.pop.positions.copy()
    for s_ in range(1, 21):
        real.step()
        if s_ in (1, 5, 20):
            res[f"traj_pos{s_}"] = real.pop.positions.copy()
    np.savez_compressed(os.path.join(OUT, "hard.npz"), **res)


class _Replay:
    """Generator stand-in handing em_step a pre-drawn block."""

    def __init__(self, block):
        self.block = block

    def standard_normal(self, shape):
        assert tuple(shape) == self.block.shape
        return self.block


if __name__ == "__main__":
    np.random.seed(0)
    forces_cases()
    em_cases()
    boundary_cases()
    field_cases()
    coupling_cases()
    cfg0_trajectory()
    composed_cfg1_small()
    composed_cfg2_small()
    reaction_cases()
    reaction_trajectories()
    tamed_cases()
    hard_sphere_cases()
    for name in sorted(os.listdir(OUT)):
        if name.endswith(".npz"):
            print(name, os.path.getsize(os.path.join(OUT, name)))
    sys.exit(0)
