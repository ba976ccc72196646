"""Parity of the CUDA path (through the C ABI) with the pinned oracle and the
reference's own golden outputs.  Tier T1/T2 of SURVEY 8c:

  pair sets, forces, EM, boundaries, gradient, bilinear : bit-exact (fp64)
  deposits (node gathers in the reference's particle order): bit-exact
  implicit solve (GEMM / FFT vs OpenBLAS / SuperLU)      : rtol 1e-11, atol 1e-13
  multi-step trajectories with the field on             : 1e-10 absolute
  fp32 storage                                          : bit-exact vs the fp64
                                                          oracle run on binary32
                                                          values, rounded per step
"""

import math
import os

import numpy as np
import pytest

import oracle
from oracle.sim import OracleSim

from conftest import cfg0_xi, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402
from paper_1805_11007_b200 import _native as N  # noqa: E402


def _pop(pos, species=None, dtype=np.float64):
    pos = np.asarray(pos, dtype=dtype)
    n = pos.shape[0]
    sp = np.zeros(n, np.uint8) if species is None else np.asarray(species, np.uint8)
    return cs.Population(ids=np.arange(n), positions=pos.copy(), next_positions=pos.copy(),
                         species=sp, drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                         start_anchor=pos.copy())


def _params(eps, cutoff, **kw):
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return cs.MotionParams(epsilon=eps, dt=1e-9, interaction="soft", cutoff=cutoff, **kw)


# ------------------------------------------------------------------- exp
def test_device_exp_matches_host_libm_bitwise():
    rng = np.random.default_rng(1)
    x = np.concatenate([-rng.random(400000) * 40.0, -rng.random(400000) * 4.5,
                        (rng.random(200000) - 0.5) * 1480.0,
                        [0.0, -0.0, 1e-300, -745.2, -745.1, 709.8, 709.7, np.inf, -np.inf]])
    xt = torch.as_tensor(x, device="cuda")
    yt = torch.empty_like(xt)
    N.check(N.load_library().cs_exp_batch(N.context(), N.ptr(xt), N.ptr(yt), x.size), "exp")
    y = yt.cpu().numpy()
    host = np.array([oracle.host_exp(v) for v in x[::7]])
    assert np.array_equal(y[::7].view(np.uint64), host.view(np.uint64))
    ref = np.exp(x)  # numpy's vectorised exp differs from libm on ~5%: a 1-ulp bound
    m = np.abs(x) < 700
    assert np.allclose(y[m], ref[m], rtol=4.5e-16, atol=0)


# ------------------------------------------------------------------- forces
def test_forces_bitwise_vs_reference_golden():
    g = load_golden("forces.npz")
    for k in range(int(g["n_cases"])):
        pos = g[f"c{k}_pos"]
        size, per, eps, cut = g[f"c{k}_meta"]
        f = cs.soft_forces(_pop(pos), cs.Domain.square(size, periodic=bool(per)),
                           _params(eps, cut))
        assert np.array_equal(f, g[f"c{k}_force"]), k


@pytest.mark.parametrize("periodic", [False, True])
def test_pair_sets_bit_exact_hetero(periodic):
    rng = np.random.default_rng(11 + periodic)
    n = 3000
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    params = _params(0.005, 0.01, radius_alpha=0.005, radius_beta=0.01)
    dom = cs.Domain.square(1.0, periodic=periodic)
    gpu_pairs = cs.soft_force_pairs(_pop(pos, sp), dom, params)
    e, c, cell = params.pair_table()
    f_or, pairs = oracle.soft_force_pairs(pos, dom.lo, dom.size, dom.periodic, e, c, cell,
                                          types=sp)
    assert np.array_equal(gpu_pairs, pairs)
    f = cs.soft_forces(_pop(pos, sp), dom, params)
    assert np.array_equal(f, f_or)


@pytest.mark.parametrize("kernel", ["auto", "warp", "lane"])
@pytest.mark.parametrize("case", ["cfg2_periodic", "cfg2_walls", "dense_ring", "two_cells"])
def test_dense_cell_forces_bitwise(case, kernel, monkeypatch):
    """Dense cell lists: BASELINE cfg2's density (~40 particles per cell,
    ~360 ring candidates, ~75 accepted pairs per particle, periodic and
    walled), ~1500-candidate rings, and 2-cell periodic axes (ring
    de-duplication), bitwise against the oracle -- with the kernel the
    library picks (cfg2: a warp per owner), with the warp-per-owner kernel
    forced and with the lane-per-owner kernels."""
    if kernel != "auto":
        monkeypatch.setenv("CS_WARP_FORCES", "1" if kernel == "warp" else "0")
    rng = np.random.default_rng({"cfg2_periodic": 21, "cfg2_walls": 22, "dense_ring": 23,
                                 "two_cells": 24}[case])
    periodic = case != "cfg2_walls"
    if case == "dense_ring":
        n, radii = 24000, (0.02, 0.04)
    elif case == "two_cells":  # 2 x 2 cells of side 0.5
        n, radii = 600, (0.1, 0.25)
    else:
        n, radii = 100_000, (0.005, 0.01)
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    params = _params(radii[0], 2 * radii[0], radius_alpha=radii[0], radius_beta=radii[1])
    dom = cs.Domain.square(1.0, periodic=periodic)
    f = cs.soft_forces(_pop(pos, sp), dom, params)
    e, c, cell = params.pair_table()
    ref = oracle.soft_forces(pos, dom.lo, dom.size, dom.periodic, e, c, cell, types=sp,
                             nthreads=os.cpu_count() or 1)
    assert np.array_equal(f, ref)


def test_forces_fp32_storage_bitwise_vs_fp64_oracle_on_binary32_values():
    rng = np.random.default_rng(13)
    n = 20000
    pos32 = rng.uniform(-0.5, 0.5, (n, 2)).astype(np.float32)
    sp = (rng.random(n) < 0.5).astype(np.uint8)
    params = _params(0.002, 0.004, radius_alpha=0.002, radius_beta=0.004)
    dom = cs.Domain.square(1.0, periodic=True)
    f = cs.soft_forces(_pop(pos32, sp, dtype=np.float32), dom, params)
    e, c, cell = params.pair_table()
    ref = oracle.soft_forces(pos32.astype(np.float64), dom.lo, dom.size, dom.periodic, e, c,
                             cell, types=sp)
    assert np.array_equal(f, ref)


def test_forces_device_tensor_in_device_tensor_out():
    rng = np.random.default_rng(14)
    pos = rng.uniform(-0.5, 0.5, (500, 2))
    t = torch.as_tensor(pos, device="cuda")
    pop = _pop(pos)
    pop.positions = t
    f = cs.soft_forces(pop, cs.Domain.square(1.0), _params(0.01, 0.02))
    assert isinstance(f, torch.Tensor) and f.is_cuda
    assert np.array_equal(f.cpu().numpy(), cs.soft_forces(_pop(pos), cs.Domain.square(1.0),
                                                          _params(0.01, 0.02)))


# ------------------------------------------------------------------- motion
def test_em_step_bitwise():
    g = load_golden("em.npz")
    out = cs.em_step(g["pos"], g["dcoef"], g["drift"], g["force"], float(g["dt"]), xi=g["xi"])
    assert np.array_equal(out, g["out"])
    out2 = cs.em_step(g["pos"], g["dcoef"], g["drift"], g["force"], float(g["dt"]),
                      np.random.default_rng(99))
    assert np.array_equal(out2, g["out"])


def test_em_step_single_particle_and_scalar_args():
    out = cs.em_step(np.array([[0.1, 0.2]]), 0.0, np.array([2.0, 0.0]),
                     np.array([0.0, -4.0]), 0.5, np.random.default_rng(0))
    assert np.array_equal(out, [[0.1 + 1.0, 0.2 - 2.0]])


def test_boundaries_vs_reference_golden():
    g = load_golden("boundaries.npz")
    for k in range(int(g["n_cases"])):
        size, per, st, i, ax = g[f"b{k}_meta"]
        pop = _pop(np.zeros_like(g[f"b{k}_in"]))
        pop.next_positions = g[f"b{k}_in"].copy()
        pop.start_anchor = g[f"b{k}_anchor_in"].copy()
        dom = cs.Domain.square(size, periodic=bool(per))
        if st == 0:
            cs.apply_boundaries(pop, dom)
            assert np.array_equal(pop.positions, g[f"b{k}_out"]), k
            assert np.array_equal(pop.start_anchor, g[f"b{k}_anchor_out"]), k
        else:
            match = {1: "non-finite", 2: f"particle {int(i)} overshot axis {int(ax)}",
                     3: "failed to settle"}[int(st)]
            with pytest.raises(cs.SimulationError, match=match):
                cs.apply_boundaries(pop, dom)


# ------------------------------------------------------------------- field
def test_field_golden():
    g = load_golden("field.npz")
    for k in range(int(g["n_cases"])):
        n_c, per, d_c, ka, kb, gam, dt = g[f"f{k}_meta"]
        grid = cs.Grid.square(int(n_c), 1.0, "periodic" if per else "neumann")
        fp = cs.FieldParams(d_c=d_c, k_alpha=ka, k_beta=kb, gamma=gam)
        ops = cs.build_operators(grid, fp, dt)
        assert np.allclose(ops.solve(g[f"f{k}_rhs"]), g[f"f{k}_solve"], rtol=1e-11, atol=1e-13)
        f = cs.Field(c=g[f"f{k}_c"].copy(), grad=np.zeros((int(n_c) ** 2, 2)),
                     rho_alpha=g[f"f{k}_ra"], rho_beta=g[f"f{k}_rb"])
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            cs.step_field(f, ops, fp, dt)
        assert np.allclose(f.c, g[f"f{k}_cnew"], rtol=1e-11, atol=1e-13), k
        # gradient of the reference's own c_new: bit-exact stencil
        f.c = g[f"f{k}_cnew"].copy()
        cs.gradient(f, ops)
        assert np.array_equal(f.grad, g[f"f{k}_grad"]), k


def test_field_nonfinite_raises_and_negative_mass_warns():
    grid = cs.Grid.square(10, 1.0, "neumann")
    fp = cs.FieldParams(d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0)
    ops = cs.build_operators(grid, fp, 1e-3)
    f = cs.Field.zeros(grid)
    f.c[0] = np.inf
    with pytest.raises(FloatingPointError, match="non-finite"):
        cs.step_field(f, ops, fp, 1e-3)
    fp = cs.FieldParams(d_c=0.0, k_alpha=0.0, k_beta=50.0, gamma=0.0)
    ops = cs.build_operators(grid, fp, 0.1)
    f = cs.Field.zeros(grid)
    f.c[:] = 1.0
    f.rho_beta[:] = 1.0
    with pytest.warns(UserWarning, match="negative"):
        cs.step_field(f, ops, fp, 0.1)


def test_periodic_fft_solve_large_matches_oracle():
    n = 512
    grid = cs.Grid.square(n, 1.0, "periodic")
    fp = cs.FieldParams(d_c=1.0)
    ops = cs.build_operators(grid, fp, 1e-5)
    rhs = np.random.default_rng(3).standard_normal(n * n)
    got = ops.solve(rhs)
    ref = oracle.build_operators(n, grid.spacing, True, 1.0, 1e-5, splu_max=0).solve(rhs)
    assert np.allclose(got, ref, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 512, 1024, 2048])
def test_spectral_periodic_solve_vs_oracle_and_cufft(n, monkeypatch):
    """The own three-pass spectral solve (csrc/spectral.cu) for every
    power-of-two periodic grid: binary64 against the oracle's solve (SuperLU
    up to 64^2, FFT diagonalisation above) at the T1 solve tolerance, and
    binary64 / binary32 against the cuFFT path (CS_CUFFT=1)."""
    grid = cs.Grid.square(n, 1.0, "periodic")
    fp = cs.FieldParams(d_c=1.0)
    dt = 1e-5 if n >= 512 else 1e-3
    rhs = np.random.default_rng(n).standard_normal(n * n)
    got = cs.build_operators(grid, fp, dt).solve(rhs)
    ref = oracle.build_operators(n, grid.spacing, True, 1.0, dt,
                                 splu_max=64).solve(rhs)
    assert np.allclose(got, ref, rtol=1e-11, atol=1e-12)
    r32 = torch.as_tensor(rhs, device="cuda").float()
    got32 = cs.build_operators(grid, fp, dt).solve(r32).double().cpu().numpy()
    monkeypatch.setenv("CS_CUFFT", "1")
    lib64 = cs.build_operators(grid, fp, dt).solve(rhs)
    lib32 = cs.build_operators(grid, fp, dt).solve(r32).double().cpu().numpy()
    monkeypatch.delenv("CS_CUFFT")
    assert np.max(np.abs(got - lib64)) <= 1e-13 * np.abs(lib64).max()
    assert np.max(np.abs(got32 - lib32)) <= 2e-6 * np.abs(lib32).max()
    assert np.max(np.abs(got32 - ref)) <= 2e-6 * np.abs(ref).max()


@pytest.mark.parametrize("n", [4096, 8192])
def test_spectral_binary32_as_accurate_as_cufft(n, monkeypatch):
    """At the cfg3 / cfg4 grid sizes: the own binary32 solve's error against
    the binary64 solve (itself within 1e-13 of cuFFT's D2Z/Z2D) is at most
    1.5x cuFFT's binary32 R2C/C2R error, in max and in rms."""
    grid = cs.Grid.square(n, 1.0, "periodic")
    fp = cs.FieldParams(d_c=1.0)
    rhs = torch.as_tensor(0.5 + 0.1 * np.random.default_rng(n).standard_normal(n * n),
                          device="cuda")
    ref = cs.build_operators(grid, fp, 1e-5).solve(rhs)
    own = cs.build_operators(grid, fp, 1e-5).solve(rhs.float()).double()
    monkeypatch.setenv("CS_CUFFT", "1")
    lib = cs.build_operators(grid, fp, 1e-5).solve(rhs.float()).double()
    lib64 = cs.build_operators(grid, fp, 1e-5).solve(rhs)
    monkeypatch.delenv("CS_CUFFT")
    assert float((ref - lib64).abs().max()) <= 1e-13 * float(ref.abs().max())
    e_own, e_lib = (own - ref).abs(), (lib - ref).abs()
    assert float(e_own.max()) <= 1.5 * float(e_lib.max())
    assert float(e_own.square().mean().sqrt()) <= 1.5 * float(e_lib.square().mean().sqrt())


def test_coupling_golden():
    g = load_golden("coupling.npz")
    for k in range(int(g["n_cases"])):
        n_c, per, cic, h, kcut, chi = g[f"k{k}_meta"]
        grid = cs.Grid.square(int(n_c), 1.0, "periodic" if per else "neumann")
        kern = cs.Kernel(kind="cic" if cic else "gaussian", h=h, cutoff=kcut)
        pop = _pop(g[f"k{k}_pos"], g[f"k{k}_species"])
        ra, rb = cs.deposit_both(pop, grid, kern)
        for got, ref in ((ra, g[f"k{k}_ra"]), (rb, g[f"k{k}_rb"])):
            assert np.array_equal(got, ref), k
        f = cs.Field(c=g[f"k{k}_c"], grad=g[f"k{k}_grad"], rho_alpha=ra, rho_beta=rb)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            cs.refresh_particle_fields(pop, f, grid, chi)
        assert np.array_equal(pop.local_concentration, g[f"k{k}_conc"]), k
        assert np.array_equal(pop.drift, g[f"k{k}_drift"]), k


@pytest.mark.parametrize("kind,per,n,n_c,clustered", [
    ("cic", False, 10_000, 128, False),     # cfg1-like
    ("cic", True, 100_000, 512, False),     # cfg2-like
    ("cic", True, 50_000, 64, True),        # dense cells
    ("gaussian", False, 1_000, 52, True),   # fig1-like clusters: > 48 stamps per node
    ("gaussian", True, 20_000, 128, False),
])
def test_deposit_bitwise_vs_oracle_and_rerun(kind, per, n, n_c, clustered):
    """deposit_both at sizes beyond the goldens: bit for bit the oracle's
    particle-order sums (pinned to the reference), and identical on a rerun
    (no atomics in the summation order)."""
    rng = np.random.default_rng(n + n_c)
    if clustered:
        centres = rng.uniform(-0.3, 0.3, (4, 2))
        pos = centres[rng.integers(0, 4, n)] + rng.normal(0, 0.03, (n, 2))
        pos = np.clip(pos, -0.5, 0.4999)
    else:
        pos = rng.uniform(-0.5, 0.5, (n, 2))
    sp = rng.integers(0, 2, n).astype(np.uint8)
    grid = cs.Grid.square(n_c, 1.0, "periodic" if per else "neumann")
    h = 0.02 if kind == "gaussian" else 0.0
    kern = cs.Kernel(kind="cic") if kind == "cic" else cs.Kernel("gaussian", h, 3 * h)
    pop = _pop(pos, sp)
    ra, rb = cs.deposit_both(pop, grid, kern)
    ra2, rb2 = cs.deposit_both(pop, grid, kern)
    assert np.array_equal(ra, ra2) and np.array_equal(rb, rb2)
    lo = list(grid.lo)
    if kind == "cic":
        ea = oracle.cic_deposit(pos, sp == 0, n_c, lo, grid.spacing, per)
        eb = oracle.cic_deposit(pos, sp == 1, n_c, lo, grid.spacing, per)
    else:
        ea, eb = oracle.gauss_deposit(pos, sp, n_c, lo, grid.spacing, per, h, 3 * h)
    assert np.array_equal(ra, ea)
    assert np.array_equal(rb, eb)


def test_gaussian_cutoff_wider_than_periodic_grid_rejected():
    g = cs.Grid.square(5, 1.0, "periodic")
    with pytest.raises(ValueError, match="cutoff"):
        cs.deposit(_pop([[0.0, 0.0]]), g, cs.Kernel(kind="gaussian", h=0.2, cutoff=0.6),
                   cs.Species.ALPHA)


def test_interpolate_clamps_with_warning():
    g = cs.Grid.square(11, 1.0, "neumann")
    values = g.node_positions()[:, 0].copy()
    with pytest.warns(UserWarning, match="clamped"):
        got = cs.interpolate(g, values, np.array([[0.7, 0.0], [0.0, 0.0]]))
    assert got[0] == pytest.approx(0.5, abs=1e-14)


# ------------------------------------------------------------------- pipeline
def _cfg0():
    return cs.SimConfig(n_alpha_0=0, n_beta_0=1000, d_beta=1.0, chi=0.0, epsilon=0.005,
                        soft_cutoff_factor=2.0, dt=1e-5, t_final=0.01, r_alpha=0.0,
                        r_beta=0.0, d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0,
                        periodic=False, seed_base=0)


def test_cfg0_realisation_bitwise_vs_reference():
    """BASELINE config 0 through the drop-in Realisation: positions after
    1, 10 and 100 steps are bit-identical to the reference's Realisation."""
    g = load_golden("cfg0_traj.npz")
    real = cs.Realisation(_cfg0(), 0)
    assert np.array_equal(real.pop.positions, g["pos0"])
    for s in range(1, 101):
        real.step()
        if s in (1, 10, 100):
            assert np.array_equal(real.pop.positions, g[f"pos{s}"]), s


def test_cfg0_full_run_matches_oracle_1000_steps():
    """T3: K = 1000 steps of config 0, run() in device blocks, bitwise vs the
    oracle (itself pinned bitwise to the reference for 100 steps)."""
    cfg = _cfg0()
    real = cs.Realisation(cfg, 0)
    pos0 = real.pop.positions
    obs = real.run()
    xi = cfg0_xi(cfg.sample_seed(0), 1000, 1000)
    e, c, cell = oracle.pair_table(epsilon=0.005, cutoff=0.01)
    sim = OracleSim(pos0, np.ones(1000, np.uint8), lo=[-0.5] * 2, hi=[0.5] * 2,
                    periodic=(False, False), dt=1e-5, diffusion=(0.1, 1.0), eps_tab=e,
                    cut_tab=c, cell_cutoff=cell)
    for s in range(1000):
        sim.step(xi[s])
    assert np.array_equal(real.pop.positions, sim.pos)
    assert obs.msd.shape == (51,)


def _composed_sim(pos, species, *, periodic, n_c, boundary, fp, kernel, chi, chi_pinned,
                  secretes, consumes, c0, radii=None, eps=0.005, cutoff=0.01,
                  diffusion=(0.1, 1.0), dtype=torch.float64, dt=1e-5):
    n = pos.shape[0]
    dom = cs.Domain.square(1.0, periodic=periodic)
    grid = cs.Grid.square(n_c, 1.0, boundary)
    mp = _params(eps, cutoff, d_alpha=diffusion[0], d_beta=diffusion[1],
                 radius_alpha=None if radii is None else radii[0],
                 radius_beta=None if radii is None else radii[1])
    mp.dt = dt
    state = dict(pos=torch.as_tensor(pos, device="cuda").to(dtype).contiguous(),
                 next_pos=torch.as_tensor(pos, device="cuda").to(dtype).contiguous(),
                 anchor=torch.as_tensor(pos, device="cuda").to(dtype).contiguous(),
                 species=torch.as_tensor(species, device="cuda").to(torch.uint8),
                 drift=torch.zeros((n, 2), dtype=torch.float64, device="cuda"),
                 local_c=torch.zeros(n, dtype=torch.float64, device="cuda"),
                 c=torch.as_tensor(c0, device="cuda").to(dtype).contiguous(),
                 grad=torch.zeros((n_c * n_c, 2), dtype=dtype, device="cuda"),
                 rho_a=torch.zeros(n_c * n_c, dtype=dtype, device="cuda"),
                 rho_b=torch.zeros(n_c * n_c, dtype=dtype, device="cuda"))
    params = cs.sim_params_struct(
        n=n, prec=N.prec_code(dtype), domain=dom, motion=mp, dt=dt, field_active=True,
        refresh_active=True, grid=grid, fparams=fp, kernel=kernel, secretes=secretes,
        consumes=consumes, chi=chi, chi_pinned=chi_pinned, store_samples=True,
        store_next=True)
    return cs.DeviceSim(params, state), state


def test_cfg1_small_composed_trajectory_vs_reference():
    g = load_golden("cfg1_small.npz")
    n_c = 32
    xs = -0.5 + (1.0 / (n_c - 1)) * np.arange(n_c)
    sim, st = _composed_sim(
        g["pos0"], np.ones(400, np.uint8), periodic=False, n_c=n_c, boundary="neumann",
        fp=cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.0, gamma=0.1),
        kernel=cs.Kernel(kind="cic"), chi=(0.0, 1.0), chi_pinned=(True, False),
        secretes=(False, True), consumes=(False, False), c0=np.tile(xs, n_c))
    xi = torch.as_tensor(g["xi"], device="cuda")
    for s in range(10):
        sim.step(xi[s], 1)
        status = sim.status()
        assert status.code == 0
        assert np.allclose(st["c"].cpu().numpy(), g[f"c{s + 1}"], rtol=0, atol=1e-12), s
        assert np.allclose(st["pos"].cpu().numpy(), g[f"pos{s + 1}"], rtol=0, atol=1e-10), s
    assert sim.status().neg_mass_steps == 10  # c0 = x is negative on x < 0


def test_cfg2_small_composed_trajectory_vs_reference():
    g = load_golden("cfg2_small.npz")
    n_c = 32
    sim, st = _composed_sim(
        g["pos0"], g["species"], periodic=True, n_c=n_c, boundary="periodic",
        fp=cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1),
        kernel=cs.Kernel(kind="cic"), chi=(0.0, -0.5), chi_pinned=(True, False),
        secretes=(True, False), consumes=(False, True), c0=np.zeros(n_c * n_c),
        eps=0.01, cutoff=0.02, diffusion=(1.0, 0.5))
    xi = torch.as_tensor(g["xi"], device="cuda")
    sim.step(xi, 8)
    assert sim.status().code == 0
    assert np.allclose(st["c"].cpu().numpy(), g["c8"], rtol=0, atol=1e-12)
    assert np.allclose(st["pos"].cpu().numpy(), g["pos8"], rtol=0, atol=1e-10)
    assert np.allclose(st["anchor"].cpu().numpy(), g["anchor8"], rtol=0, atol=1e-10)


def test_cfg2_hetero_fp32_one_step_vs_oracle():
    """BASELINE config 2 semantics (radii 0.005/0.01, D 1/0.5, chi +1/-0.5,
    periodic 512^2, CIC) at N = 20000, fp32 storage: one step vs the fp64
    oracle run on binary32 values and rounded to binary32."""
    rng = np.random.default_rng(21)
    n, n_c = 20000, 512
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32).astype(np.float64)
    sp = np.r_[np.zeros(n // 2), np.ones(n - n // 2)].astype(np.uint8)
    fpar = cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1)
    sim, st = _composed_sim(pos, sp, periodic=True, n_c=n_c, boundary="periodic", fp=fpar,
                            kernel=cs.Kernel(kind="cic"), chi=(1.0, -0.5),
                            chi_pinned=(False, False), secretes=(True, False),
                            consumes=(False, True), c0=np.zeros(n_c * n_c),
                            radii=(0.005, 0.01), diffusion=(1.0, 0.5), dtype=torch.float32)
    xi = rng.standard_normal((n, 2)).astype(np.float32)
    sim.step(torch.as_tensor(xi, device="cuda"), 1)
    assert sim.status().code == 0
    e, c, cell = oracle.pair_table(radii=(0.005, 0.01))
    field = dict(n_c=n_c, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                 kernel="cic", secretes=(True, False), consumes=(False, True),
                 c0=np.zeros(n_c * n_c), splu_max=0)
    osim = OracleSim(pos, sp, lo=[-0.5] * 2, hi=[0.5] * 2, periodic=(True, True), dt=1e-5,
                     diffusion=(1.0, 0.5), eps_tab=e, cut_tab=c, cell_cutoff=cell,
                     chi=(1.0, -0.5), chi_pinned=(False, False), field=field, fp32=True,
                     nthreads=os.cpu_count())
    osim.step(xi.astype(np.float64))
    got = st["pos"].double().cpu().numpy()
    # fp32 tolerance: the drift comes from an fp32 grid/FFT (rel ~1e-6 of a
    # ~1e-5 displacement); positions agree to a few binary32 ulps of 0.5
    assert np.max(np.abs(got - osim.pos)) <= 4 * 2.0 ** -24
    cg = st["c"].double().cpu().numpy()
    assert np.max(np.abs(cg - osim.c)) <= 1e-5 * max(1.0, np.abs(osim.c).max())


def test_realisation_errors_map_to_reference_exceptions():
    cfg = cs.SimConfig(n_alpha_0=0, n_beta_0=3, d_beta=1.0, chi=0.0, epsilon=0.005,
                       soft_cutoff_factor=2.0, dt=1e-5, t_final=1e-4, r_alpha=0.0,
                       r_beta=0.0, d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0, seed_base=0)
    real = cs.Realisation(cfg, 0)
    real.device_state["pos"][1, 1] = float("nan")
    with pytest.raises(cs.SimulationError, match=r"step 0: non-finite coordinate for particle 1"):
        real.step()
    real = cs.Realisation(cfg, 0)
    real.device_state["pos"][2, 0] = 1.7
    with pytest.raises(cs.SimulationError, match=r"step 0: particle 2 overshot axis 0"):
        real.step()


def test_sorted_engine_refuses_what_it_cannot_run():
    """Reactions, the tamed integrator and hard spheres run on the direct
    engine; asking the sorted engine for them is a parameter error."""
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for kw in (dict(interaction="hard"), dict(integrator="tamed"), dict(r_alpha=5.0)):
            cfg = cs.SimConfig(precision="fp32", engine="sorted", **{"r_alpha": 0.0, **kw})
            with pytest.raises(N.NativeError, match="direct engine"):
                cs.Realisation(cfg, 0)


def test_default_fig1_config_runs_on_the_device():
    """The reference's default SimConfig (the fig1 clustering experiment:
    reactions on, gaussian deposit, Neumann 52^2 field) steps through the
    drop-in Realisation."""
    real = cs.Realisation(cs.SimConfig(), 0)
    for _ in range(5):
        real.step()
    assert real.step_index == 5 and len(real.pop) == 200


# ------------------------------------------------------------------- full size
def test_cfg3_full_size_one_step_properties_and_force_parity():
    """BASELINE config 3 size (N = 1e7, 4096^2 periodic grid, fp32 storage):
    one device step; size-independent checks (CIC mass = N, sum of forces
    ~ 0, every particle inside [lo, hi]) and bitwise force parity with the
    oracle on the same binary32 positions."""
    n, n_c = 10_000_000, 4096
    rng = np.random.default_rng(33)
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    params = _params(6.1804e-5, 2 * 6.1804e-5, radius_alpha=6.1804e-5, radius_beta=1.2361e-4)
    dom = cs.Domain.square(1.0, periodic=True)
    pop = _pop(pos, sp, dtype=np.float32)
    pop.positions = torch.as_tensor(pos, device="cuda")
    pop.species = torch.as_tensor(sp, device="cuda")
    f = cs.soft_forces(pop, dom, params).cpu().numpy()
    s = f.sum(axis=0)
    assert np.all(np.abs(s) <= 1e-9 * np.abs(f).sum(axis=0) + 1e-12)
    e, c, cell = params.pair_table()
    ref = oracle.soft_forces(pos.astype(np.float64), dom.lo, dom.size, dom.periodic, e, c, cell,
                             types=sp, nthreads=os.cpu_count())
    assert np.array_equal(f, ref)
    grid = cs.Grid.square(n_c, 1.0, "periodic")
    ra, rb = cs.deposit_both(pop, grid, cs.Kernel(kind="cic"))
    h2 = float(np.prod(grid.spacing))
    assert abs(float(ra.double().sum()) * h2 - n // 2) <= 1e-4 * n
    assert abs(float(rb.double().sum()) * h2 - (n - n // 2)) <= 1e-4 * n
