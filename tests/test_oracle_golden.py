"""Pin the oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  These run on CPU only; the GPU parity tests
then compare the CUDA path with the pinned oracle."""

import numpy as np
import pytest

import oracle
from oracle.field import build_operators
from oracle.sim import OracleSim

from conftest import cfg0_xi, load_golden


def test_force_cases_bitwise():
    g = load_golden("forces.npz")
    for k in range(int(g["n_cases"])):
        pos = g[f"c{k}_pos"]
        size, per, eps, cut = g[f"c{k}_meta"]
        eps_tab, cut_tab, cell = oracle.pair_table(epsilon=eps, cutoff=cut)
        f = oracle.soft_forces(pos, [-size / 2] * 2, [size, size],
                               [bool(per)] * 2, eps_tab, cut_tab, cell)
        assert np.array_equal(f, g[f"c{k}_force"]), k


def test_force_openmp_matches_serial():
    g = load_golden("forces.npz")
    k = int(g["n_cases"]) - 2
    pos = g[f"c{k}_pos"]
    size, per, eps, cut = g[f"c{k}_meta"]
    eps_tab, cut_tab, cell = oracle.pair_table(epsilon=eps, cutoff=cut)
    a = oracle.soft_forces(pos, [-size / 2] * 2, [size] * 2, [bool(per)] * 2,
                           eps_tab, cut_tab, cell, nthreads=1)
    b = oracle.soft_forces(pos, [-size / 2] * 2, [size] * 2, [bool(per)] * 2,
                           eps_tab, cut_tab, cell, nthreads=4)
    assert np.array_equal(a, b)


def test_hetero_table_reduces_to_homogeneous():
    """restated(r_A = r_B = eps) == soft_forces(cutoff = 2 eps)."""
    g = load_golden("forces.npz")
    for k in range(int(g["n_cases"])):
        size, per, eps, cut = g[f"c{k}_meta"]
        if cut != 2.0 * eps:
            continue
        pos = g[f"c{k}_pos"]
        types = np.arange(pos.shape[0]) % 2
        e, c, cell = oracle.pair_table(radii=(eps, eps))
        f = oracle.soft_forces(pos, [-size / 2] * 2, [size] * 2, [bool(per)] * 2,
                               e, c, cell, types=types)
        assert np.array_equal(f, g[f"c{k}_force"]), k


def test_pair_set_is_symmetric_and_matches_brute_force():
    rng = np.random.default_rng(5)
    for per in (False, True):
        pos = rng.uniform(-0.5, 0.5, (700, 2))
        e, c, cell = oracle.pair_table(radii=(0.005, 0.01))
        types = (np.arange(700) >= 350).astype(np.uint8)
        _, pairs = oracle.soft_force_pairs(pos, [-0.5] * 2, [1.0] * 2, [per] * 2,
                                           e, c, cell, types=types)
        s = set(map(tuple, pairs.tolist()))
        assert all((j, i) in s for i, j in s)
        # brute force with the same r2 arithmetic (no FMA)
        d = pos[None, :, :] - pos[:, None, :]
        if per:
            d = d - np.round(d)
        r2 = d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]
        cut2 = (c * c).reshape(2, 2)[types[:, None], types[None, :]]
        m = (r2 <= cut2) & (r2 > 0)
        np.fill_diagonal(m, False)
        brute = set(zip(*np.nonzero(m)))
        assert s == {(int(i), int(j)) for i, j in brute}


def test_em_bitwise():
    g = load_golden("em.npz")
    out = oracle.em_step(g["pos"], g["dcoef"], g["drift"], g["force"], g["xi"],
                         float(g["dt"]))
    assert np.array_equal(out, g["out"])


def test_boundaries_bitwise_and_status():
    g = load_golden("boundaries.npz")
    for k in range(int(g["n_cases"])):
        size, per, st, i, ax = g[f"b{k}_meta"]
        x = g[f"b{k}_in"].copy()
        a = g[f"b{k}_anchor_in"].copy()
        got = oracle.apply_boundaries(x, a, [-size / 2] * 2, [size / 2] * 2,
                                      [bool(per)] * 2)
        assert got == (int(st), int(i), int(ax)), k
        assert np.array_equal(x, g[f"b{k}_out"], equal_nan=True), k
        assert np.array_equal(a, g[f"b{k}_anchor_out"]), k


def test_field_cases():
    g = load_golden("field.npz")
    for k in range(int(g["n_cases"])):
        n_c, per, d_c, ka, kb, gam, dt = g[f"f{k}_meta"]
        n_c = int(n_c)
        spacing = np.array([1.0, 1.0]) / (n_c if per else n_c - 1)
        ops = build_operators(n_c, spacing, bool(per), d_c, dt)
        got = ops.solve(g[f"f{k}_rhs"])
        # same numpy/scipy calls as the reference: bitwise on this host
        assert np.array_equal(got, g[f"f{k}_solve"]), k
        rhs = oracle.field_rhs(g[f"f{k}_c"], g[f"f{k}_ra"], g[f"f{k}_rb"], dt,
                               ka, kb, gam)
        cnew = ops.solve(rhs)
        assert np.array_equal(cnew, g[f"f{k}_cnew"]), k
        grad = oracle.gradient(cnew, n_c, spacing, bool(per))
        assert np.array_equal(grad, g[f"f{k}_grad"]), k


def test_fft_periodic_solve_matches_splu():
    g = load_golden("field.npz")
    for k in range(int(g["n_cases"])):
        n_c, per, d_c, ka, kb, gam, dt = g[f"f{k}_meta"]
        if not per:
            continue
        n_c = int(n_c)
        spacing = np.array([1.0, 1.0]) / n_c
        ops = build_operators(n_c, spacing, True, d_c, dt, splu_max=0)
        assert ops.kind == "fft"
        got = ops.solve(g[f"f{k}_rhs"])
        assert np.allclose(got, g[f"f{k}_solve"], rtol=1e-11, atol=1e-13)


def test_coupling_cases_bitwise():
    g = load_golden("coupling.npz")
    for k in range(int(g["n_cases"])):
        n_c, per, cic, h, kcut, chi = g[f"k{k}_meta"]
        n_c = int(n_c)
        pos, sp = g[f"k{k}_pos"], g[f"k{k}_species"]
        spacing = np.array([1.0, 1.0]) / (n_c if per else n_c - 1)
        lo = [-0.5, -0.5]
        if cic:
            ra = oracle.cic_deposit(pos, sp == 0, n_c, lo, spacing, bool(per))
            rb = oracle.cic_deposit(pos, sp == 1, n_c, lo, spacing, bool(per))
        else:
            ra, rb = oracle.gauss_deposit(pos, sp, n_c, lo, spacing, bool(per),
                                          h, kcut)
        assert np.array_equal(ra, g[f"k{k}_ra"]), k
        assert np.array_equal(rb, g[f"k{k}_rb"]), k
        conc, _ = oracle.bilinear(pos, g[f"k{k}_c"], n_c, lo, spacing, bool(per))
        drift, _ = oracle.bilinear(pos, g[f"k{k}_grad"], n_c, lo, spacing,
                                   bool(per))
        drift *= chi
        drift[sp == 0] = 0.0
        assert np.array_equal(conc, g[f"k{k}_conc"]), k
        assert np.array_equal(drift, g[f"k{k}_drift"]), k


def test_cfg0_trajectory_bitwise():
    """BASELINE config 0 through the oracle's composed driver equals the
    reference Realisation bit for bit after 1, 10 and 100 steps."""
    g = load_golden("cfg0_traj.npz")
    pos0 = g["pos0"]
    n = pos0.shape[0]
    xi = cfg0_xi(int(g["seed"]), 100, n)
    e, c, cell = oracle.pair_table(epsilon=0.005, cutoff=2.0 * 0.005)
    sim = OracleSim(pos0, np.ones(n, np.uint8), lo=[-0.5] * 2, hi=[0.5] * 2,
                    periodic=(False, False), dt=1e-5, diffusion=(0.1, 1.0),
                    eps_tab=e, cut_tab=c, cell_cutoff=cell)
    for s in range(100):
        sim.step(xi[s])
        if s + 1 in (1, 10, 100):
            assert np.array_equal(sim.pos, g[f"pos{s + 1}"]), s + 1


def _cfg1_small_sim(g):
    pos0 = g["pos0"]
    n = pos0.shape[0]
    n_c = 32
    xs = -0.5 + (1.0 / (n_c - 1)) * np.arange(n_c)
    e, c, cell = oracle.pair_table(epsilon=0.005, cutoff=0.01)
    field = dict(n_c=n_c, boundary="neumann", d_c=1.0, k_alpha=0.1, k_beta=0.0,
                 gamma=0.1, kernel="cic", secretes=(False, True),
                 consumes=(False, False), c0=np.tile(xs, n_c))
    return OracleSim(pos0, np.ones(n, np.uint8), lo=[-0.5] * 2, hi=[0.5] * 2,
                     periodic=(False, False), dt=1e-5, diffusion=(0.1, 1.0),
                     eps_tab=e, cut_tab=c, cell_cutoff=cell, chi=(0.0, 1.0),
                     chi_pinned=(True, False), field=field)


def test_cfg1_small_trajectory():
    g = load_golden("cfg1_small.npz")
    sim = _cfg1_small_sim(g)
    for s in range(10):
        sim.step(g["xi"][s])
        assert np.array_equal(sim.c, g[f"c{s + 1}"]), s
        assert np.array_equal(sim.pos, g[f"pos{s + 1}"]), s


def test_cfg2_small_trajectory():
    g = load_golden("cfg2_small.npz")
    pos0, sp = g["pos0"], g["species"]
    n_c = 32
    e, c, cell = oracle.pair_table(epsilon=0.01, cutoff=0.02)
    field = dict(n_c=n_c, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03,
                 gamma=0.1, kernel="cic", secretes=(True, False),
                 consumes=(False, True), c0=np.zeros(n_c * n_c))
    sim = OracleSim(pos0, sp, lo=[-0.5] * 2, hi=[0.5] * 2, periodic=(True, True),
                    dt=1e-5, diffusion=(1.0, 0.5), eps_tab=e, cut_tab=c,
                    cell_cutoff=cell, chi=(0.0, -0.5), chi_pinned=(True, False),
                    field=field)
    for s in range(8):
        sim.step(g["xi"][s])
        assert np.allclose(sim.c, g[f"c{s + 1}"], rtol=1e-12, atol=1e-14), s
        assert np.array_equal(sim.pos, g[f"pos{s + 1}"]), s
        assert np.array_equal(sim.anchor, g[f"anchor{s + 1}"]), s


def test_glibc_exp_restatement_matches_host_libm():
    """The device exp (csrc/glibc_exp.cuh) is a restatement of glibc's
    table-driven exp; its host twin (tools/exp_table.py) must agree with
    the host libm bit for bit."""
    from tools.exp_table import py_exp
    rng = np.random.default_rng(3)
    xs = np.concatenate([-rng.random(20000) * 50, -rng.random(20000) * 4.5,
                         (rng.random(20000) - 0.5) * 1400,
                         [0.0, -0.0, 1e-300, -745.2, 709.8, np.inf, -np.inf]])
    for x in xs:
        a = oracle.host_exp(float(x))
        b = py_exp(float(x))
        assert a == b or (np.isnan(a) and np.isnan(b)), x


def test_reaction_restatement_matches_reference_golden():
    """oracle/react.py against fixed_step_reactions / beta_step_reactions of
    the reference (tests/golden/reactions.npz): switched species, zeroed
    drift rows, flip counts and the clamp warning, bit for bit."""
    from oracle.react import fixed_step
    r = load_golden("reactions.npz")
    for k in range(int(r["n_fixed"])):
        ra, rb, dt = r[f"f{k}_in"]
        args = (r[f"f{k}_species"], r[f"f{k}_local_c"], r[f"f{k}_drift"], r[f"f{k}_u"])
        t, d, c, h = fixed_step(*args, ra * dt, rb, dt)
        assert np.array_equal(t, r[f"f{k}_out_species"]), k
        assert np.array_equal(d, r[f"f{k}_out_drift"]), k
        assert c == tuple(int(v) for v in r[f"f{k}_counts"]), k
        assert (h > 1.0) == bool(r[f"f{k}_warned"]), k
        t, d, c, h = fixed_step(*args, 0.0, rb, dt)
        assert np.array_equal(t, r[f"b{k}_out_species"]), k
        assert np.array_equal(d, r[f"b{k}_out_drift"]), k
        assert c[1] == int(r[f"b{k}_count"]) and (h > 1.0) == bool(r[f"b{k}_warned"]), k


def test_rng_restatement_matches_numpy():
    """oracle/rng.py (PCG64 + numpy's ziggurat with the tables read from
    numpy's own library) against Generator.standard_normal / random."""
    from oracle.rng import PCG64
    for seed in (0, 5, 2**33 + 1):
        g = np.random.default_rng(np.random.SeedSequence(seed).spawn(3)[1])
        p = PCG64.of(g)
        a = g.standard_normal(60000)
        b = np.array([p.standard_normal() for _ in range(60000)])
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), seed
        assert np.array_equal(g.random(500), np.array([p.next_double() for _ in range(500)]))


def test_tamed_restatement_matches_reference_golden():
    from oracle.react import tamed_step
    g = load_golden("tamed.npz")
    out = tamed_step(g["pos"], g["dcoef"], g["drift"], g["force"], g["xi"], float(g["dt"]))
    assert np.array_equal(out, g["out"])


def test_hard_sphere_restatement_matches_reference_golden():
    from oracle.hard import resolve_hard_sphere
    g = load_golden("hard.npz")
    for k in range(int(g["n_cases"])):
        size, per, eps, da, db = g[f"h{k}_meta"]
        out = resolve_hard_sphere(g[f"h{k}_in"], g[f"h{k}_species"], (size, size),
                                  (bool(per), bool(per)), eps, da, db)
        assert np.array_equal(out, g[f"h{k}_out"]), k
