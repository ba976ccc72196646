"""The sorted (large-N) engine against the direct engine and the oracle.

The sorted engine keeps particles in cell-sorted records and sums forces in
the reference's canonical order regardless of storage order, so with the
field off it must reproduce the direct engine bit for bit; with the field on
it deposits in integer fixed point (deterministic) and must stay within the
fp32 tolerance of the oracle."""

import os

import numpy as np
import pytest

import oracle
from oracle.sim import OracleSim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402


def _sim(pos, sp, *, engine, field, n_c=256, radii=(0.002, 0.004), periodic=True,
         chi=(1.0, -0.5), chi_pinned=(False, False), diffusion=(1.0, 0.5), dt=1e-5,
         boundary="periodic", c0=None):
    import warnings
    n = pos.shape[0]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = cs.MotionParams(d_alpha=diffusion[0], d_beta=diffusion[1], epsilon=radii[0],
                             cutoff=2 * radii[0], dt=dt, radius_alpha=radii[0],
                             radius_beta=radii[1])
    dom = cs.Domain.square(1.0, periodic=periodic)
    grid = cs.Grid.square(n_c, 1.0, boundary)
    fp = cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1)
    f32 = torch.float32
    c0 = np.zeros(n_c * n_c) if c0 is None else c0
    st = dict(pos=torch.as_tensor(pos, device="cuda").to(f32).contiguous(),
              next_pos=None,
              anchor=torch.as_tensor(pos, device="cuda").to(f32).contiguous(),
              species=torch.as_tensor(sp, device="cuda"),
              drift=torch.zeros((n, 2), dtype=torch.float64, device="cuda"), local_c=None,
              c=torch.as_tensor(c0, device="cuda").to(f32).contiguous(),
              grad=torch.zeros((n_c * n_c, 2), dtype=f32, device="cuda"),
              rho_a=torch.zeros(n_c * n_c, dtype=f32, device="cuda"),
              rho_b=torch.zeros(n_c * n_c, dtype=f32, device="cuda"))
    params = cs.sim_params_struct(
        n=n, prec=1, domain=dom, motion=mp, dt=dt, field_active=field, refresh_active=field,
        grid=grid, fparams=fp, kernel=cs.Kernel(kind="cic"), secretes=(True, False),
        consumes=(False, True), chi=chi, chi_pinned=chi_pinned, store_samples=False,
        store_next=False, engine=engine)
    return cs.DeviceSim(params, st), st


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    xi = rng.standard_normal((12, n, 2)).astype(np.float32)
    return pos, sp, xi


@pytest.mark.parametrize("periodic", [True, False])
def test_sorted_equals_direct_bitwise_without_field(periodic):
    pos, sp, xi = _inputs(60000, 1)
    a, sa = _sim(pos, sp, engine="sorted", field=False, periodic=periodic)
    b, sb = _sim(pos, sp, engine="direct", field=False, periodic=periodic)
    assert a.engine == "sorted" and b.engine == "direct"
    x = torch.as_tensor(xi, device="cuda")
    a.step(x, 12)
    b.step(x, 12)
    a.export_state()
    assert a.status().code == 0 and b.status().code == 0
    assert torch.equal(sa["pos"], sb["pos"])


@pytest.mark.parametrize("periodic", [True, False])
def test_sorted_equals_direct_bitwise_clustered(periodic):
    """BASELINE cfg4's initial condition at 1/400 scale: 64 gaussian clusters
    (sigma 0.02) whose cores hold several times the mean 0.8 particles per
    cell, so owners with more than the fast path's 8 hits go through the
    deferred warp-per-owner pass and bucket populations run well above the
    mean: still the direct engine's result bit for bit."""
    rng = np.random.default_rng(8)
    n = 200_000
    centres = -0.5 + rng.random((64, 2))
    pos = centres[rng.integers(0, 64, n)] + 0.02 * rng.standard_normal((n, 2))
    if periodic:
        pos = np.mod(pos + 0.5, 1.0) - 0.5
    else:
        pos = np.clip(pos, -0.5, 0.5)
    pos = pos.astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    xi = rng.standard_normal((6, n, 2)).astype(np.float32)
    radii = (4.9e-4, 9.8e-4)  # area fraction 0.3 over the unit square
    a, sa = _sim(pos, sp, engine="sorted", field=False, periodic=periodic, radii=radii)
    b, sb = _sim(pos, sp, engine="direct", field=False, periodic=periodic, radii=radii)
    x = torch.as_tensor(xi, device="cuda")
    a.step(x, 6)
    b.step(x, 6)
    a.export_state()
    assert a.status().code == 0 and b.status().code == 0
    assert torch.equal(sa["pos"], sb["pos"])


@pytest.mark.parametrize("r_b", [0.0035, 0.005, 0.0075])
def test_sorted_equals_direct_bitwise_dense_rings(r_b):
    """Uniform systems of 2, 4 and 9 particles per cell (rings of ~18, ~36 and
    ~83 candidates): the force walk's hit columns run past the 8 buffered hits
    into the rest of the warp's queue, owners with more than 8 hits and rings
    beyond the walk's candidate bound (44) go to the deferred warp-per-owner
    pass -- the direct engine's positions bit for bit (a small dt keeps the
    overlapping particles' displacements inside the box)."""
    rng = np.random.default_rng(21)
    n = 40_000
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    xi = rng.standard_normal((3, n, 2)).astype(np.float32)
    radii = (r_b / 2, r_b)
    a, sa = _sim(pos, sp, engine="sorted", field=False, radii=radii, dt=1e-10)
    b, sb = _sim(pos, sp, engine="direct", field=False, radii=radii, dt=1e-10)
    x = torch.as_tensor(xi, device="cuda")
    a.step(x, 3)
    b.step(x, 3)
    a.export_state()
    assert a.status().code == 0 and b.status().code == 0
    assert torch.equal(sa["pos"], sb["pos"])
    assert not torch.equal(sa["pos"], torch.as_tensor(pos, device="cuda"))


@pytest.mark.parametrize("pregather", [False, True])
@pytest.mark.parametrize("clustered", [False, True])
def test_block_call_equals_single_step_calls_bitwise(clustered, pregather, monkeypatch):
    """One k-step call (the bench's timed region: the field solve forked to
    the side stream every step) against k one-step calls: the same records,
    anchors and field, bit for bit -- uniform and with cfg4-like clusters.
    pregather: the block call's bucket sort also gathers the coming step's
    increments into storage-slot order (what large systems do, forced here
    by CS_XI_PREGATHER=1), so its updates read them as a stream while the
    one-step calls gather them by id."""
    monkeypatch.setenv("CS_XI_PREGATHER", "1" if pregather else "0")
    rng = np.random.default_rng(21)
    n, k = 150_000, 5
    if clustered:
        centres = -0.5 + rng.random((64, 2))
        pos = centres[rng.integers(0, 64, n)] + 0.02 * rng.standard_normal((n, 2))
        pos = (np.mod(pos + 0.5, 1.0) - 0.5).astype(np.float32)
    else:
        pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    xi = torch.as_tensor(rng.standard_normal((k, n, 2)).astype(np.float32), device="cuda")
    radii = (5e-4, 1e-3)
    a, sa = _sim(pos, sp, engine="sorted", field=True, radii=radii)
    b, sb = _sim(pos, sp, engine="sorted", field=True, radii=radii)
    a.step(xi, k)
    for j in range(k):
        b.step(xi[j], 1)
    a.export_state()
    b.export_state()
    assert a.status().code == 0 and b.status().code == 0
    assert torch.equal(sa["pos"], sb["pos"])
    assert torch.equal(sa["anchor"], sb["anchor"])
    assert torch.equal(sa["c"], sb["c"])


def test_sorted_engine_field_one_step_vs_oracle_and_deterministic():
    n, n_c = 40000, 256
    pos, sp, xi = _inputs(n, 2)
    a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c)
    x = torch.as_tensor(xi, device="cuda")
    a.step(x[0], 1)
    a.export_state()
    assert a.status().code == 0
    e, c, cell = oracle.pair_table(radii=(0.002, 0.004))
    field = dict(n_c=n_c, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                 kernel="cic", secretes=(True, False), consumes=(False, True),
                 c0=np.zeros(n_c * n_c), splu_max=0)
    o = OracleSim(pos.astype(np.float64), sp, lo=[-0.5] * 2, hi=[0.5] * 2,
                  periodic=(True, True), dt=1e-5, diffusion=(1.0, 0.5), eps_tab=e, cut_tab=c,
                  cell_cutoff=cell, chi=(1.0, -0.5), chi_pinned=(False, False), field=field,
                  fp32=True, anchor_mode="wraps", nthreads=os.cpu_count())
    o.step(xi[0].astype(np.float64))
    got = sa["pos"].double().cpu().numpy()
    assert np.max(np.abs(got - o.pos)) <= 4 * 2.0 ** -24
    cg = sa["c"].double().cpu().numpy()
    assert np.max(np.abs(cg - o.c)) <= 1e-5 * max(1.0, np.abs(o.c).max())
    # deposited densities (fixed point) vs the oracle's fp64 CIC
    ra = sa["rho_a"].double().cpu().numpy()
    # rho_a now holds the deposit of the NEW positions; compare its mass
    h2 = (1.0 / n_c) ** 2
    assert abs(ra.sum() * h2 - n // 2) <= 1e-3
    # determinism: a second run gives identical bits
    b, sb = _sim(pos, sp, engine="sorted", field=True, n_c=n_c)
    b.step(x[0], 1)
    b.export_state()
    assert torch.equal(sa["pos"], sb["pos"]) and torch.equal(sa["c"], sb["c"])


def test_sorted_engine_multi_step_field_deterministic_and_anchor_exact():
    n, n_c = 50000, 512
    pos, sp, xi = _inputs(n, 3)
    x = torch.as_tensor(xi, device="cuda")
    outs = []
    for _ in range(2):
        a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c)
        a.step(x, 12)
        a.export_state()
        assert a.status().code == 0
        outs.append({k: v.clone() for k, v in sa.items() if v is not None})
    for k in ("pos", "anchor", "c", "grad", "rho_a", "rho_b"):
        assert torch.equal(outs[0][k], outs[1][k]), k
    # anchor follows wraps exactly: pos - anchor is the unwrapped displacement
    d = (outs[0]["pos"].double() - outs[0]["anchor"].double()).cpu().numpy() \
        - (pos.astype(np.float64) - pos.astype(np.float64))
    assert np.all(np.abs(d) < 0.1)


def test_sorted_engine_reports_nonfinite_with_reference_message():
    cfg = cs.SimConfig(n_alpha_0=2000, n_beta_0=2000, d_alpha=1.0, d_beta=0.5, chi=-0.5,
                       epsilon=0.002, soft_cutoff_factor=2.0, radius_alpha=0.002,
                       radius_beta=0.004, dt=1e-5, t_final=1e-4, r_alpha=0.0, r_beta=0.0,
                       periodic=True, n_c=64, deposit="cic", precision="fp32",
                       alpha_init="uniform", seed_base=3)
    real = cs.Realisation(cfg, 0)
    assert real._sim.engine == "sorted"
    real.step()
    real._sim._st  # noqa: B018
    real.device_state["pos"][17, 0] = float("nan")
    real._sim.import_state()
    with pytest.raises(cs.SimulationError, match=r"step 1: non-finite coordinate for particle 17"):
        real.step()


def test_fused_spectral_solve_4096_vs_oracle_and_cufft(monkeypatch):
    """The fused three-pass periodic solve (csrc/spectral.cu, used for a
    binary32 4096^2 grid): one step against the fp64 oracle (the tolerance of
    the 256^2 test above) and against the same engine's cuFFT path, from a
    non-zero field so that decay, secretion and consumption all enter."""
    n, n_c = 200_000, 4096
    pos, sp, xi = _inputs(n, 5)
    rng = np.random.default_rng(9)
    c0 = (0.5 + 0.1 * rng.standard_normal(n_c * n_c)).astype(np.float32).astype(np.float64)
    x = torch.as_tensor(xi, device="cuda")
    res = {}
    for mode in ("fused", "cufft"):
        if mode == "cufft":
            monkeypatch.setenv("CS_CUFFT", "1")
        else:
            monkeypatch.delenv("CS_CUFFT", raising=False)
        a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c, c0=c0)
        a.step(x[0], 1)
        a.export_state()
        assert a.status().code == 0
        res[mode] = {k: sa[k].double().cpu().numpy() for k in ("pos", "c", "grad")}
    monkeypatch.delenv("CS_CUFFT", raising=False)
    cmax = np.abs(res["cufft"]["c"]).max()
    assert np.max(np.abs(res["fused"]["c"] - res["cufft"]["c"])) <= 1e-6 * cmax
    e, c, cell = oracle.pair_table(radii=(0.002, 0.004))
    field = dict(n_c=n_c, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                 kernel="cic", secretes=(True, False), consumes=(False, True),
                 c0=c0, splu_max=0)
    o = OracleSim(pos.astype(np.float64), sp, lo=[-0.5] * 2, hi=[0.5] * 2,
                  periodic=(True, True), dt=1e-5, diffusion=(1.0, 0.5), eps_tab=e, cut_tab=c,
                  cell_cutoff=cell, chi=(1.0, -0.5), chi_pinned=(False, False), field=field,
                  fp32=True, anchor_mode="wraps", nthreads=os.cpu_count())
    o.step(xi[0].astype(np.float64))
    assert np.max(np.abs(res["fused"]["c"] - o.c)) <= 1e-5 * max(1.0, np.abs(o.c).max())
    assert np.max(np.abs(res["fused"]["pos"] - o.pos)) <= 4 * 2.0 ** -24


def test_vectorized_periodic_gradient_bitwise_equals_generic(monkeypatch):
    """k_gradient_per4 (16-byte accesses, periodic binary32 grids) against the
    generic k_gradient: identical bits over several coupled steps."""
    n, n_c = 60_000, 512
    pos, sp, xi = _inputs(n, 11)
    rng = np.random.default_rng(2)
    c0 = (0.2 + 0.05 * rng.standard_normal(n_c * n_c)).astype(np.float32).astype(np.float64)
    x = torch.as_tensor(xi, device="cuda")
    out = {}
    for mode in ("vec", "generic"):
        if mode == "generic":
            monkeypatch.setenv("CS_GRAD_GENERIC", "1")
        else:
            monkeypatch.delenv("CS_GRAD_GENERIC", raising=False)
        a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c, c0=c0)
        a.step(x, 5)
        a.export_state()
        assert a.status().code == 0
        out[mode] = {k: sa[k].clone() for k in ("pos", "c", "grad")}
    monkeypatch.delenv("CS_GRAD_GENERIC", raising=False)
    for k in ("pos", "c", "grad"):
        assert torch.equal(out["vec"][k], out["generic"][k]), k


@pytest.mark.parametrize("mode", ["rows", "atomic"])
def test_sorted_engine_reports_fixed_point_deposit_overflow(mode, monkeypatch):
    """A grid node collecting more particle masses than the int32 fixed-point
    deposit sums exactly (2^31 / 2^22 = 511 masses) stops the sorted engine
    with CS_DEPOSIT_OVERFLOW instead of wrapping silently: 600 particles
    sitting exactly on one node overflow it, 500 do not (the row-gathered
    deposit of periodic grids switches to checked adds once a cell exceeds
    the conservative bound; the atomic deposit checks every add)."""
    n, n_c = 20_000, 256
    if mode == "atomic":
        monkeypatch.setenv("CS_ATOMIC_DEPOSIT", "1")
    else:
        monkeypatch.delenv("CS_ATOMIC_DEPOSIT", raising=False)
    pos, sp, xi = _inputs(n, 4)
    sp[:] = 0  # every particle secretes into rho_alpha
    node = np.float32(-0.5 + 154.0 / 256.0)  # a grid node, exact in binary32
    pos[:600] = node
    a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c)
    a.step(torch.as_tensor(xi[0], device="cuda"), 1)
    assert a.status().code == cs._native.CS_DEPOSIT_OVERFLOW
    b, sb = _sim(pos[100:], sp[100:], engine="sorted", field=True, n_c=n_c)
    b.step(torch.as_tensor(xi[0, 100:], device="cuda"), 1)
    assert b.status().code == 0
    monkeypatch.delenv("CS_ATOMIC_DEPOSIT", raising=False)


def test_sorted_engine_dense_cells_below_the_node_limit_run():
    """Cells above the conservative population bound whose nodes stay below
    511 masses (coarse grid, fine cells: the bound is 511 / 81 = 6 per cell
    here) run, with the checked row deposit equal to the atomic one."""
    n, n_c = 4000, 64
    pos, sp, xi = _inputs(n, 5)
    pos[:40] = np.float32(0.1)  # 40 particles in one cell
    x = torch.as_tensor(xi, device="cuda")
    a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c, radii=(0.002, 0.002))
    a.step(x, 3)
    a.export_state()
    assert a.status().code == 0


@pytest.mark.parametrize("n_c,generic_wrap", [(512, False), (512, True), (384, False),
                                              (250, False)])
def test_row_gather_deposit_bitwise_equals_atomic_deposit(n_c, generic_wrap, monkeypatch):
    """k_fast_deposit_rows (periodic grids: deposit gathered per grid row, no
    atomics to HBM) against the atomic deposit: identical fixed-point grids,
    hence identical fields and positions, over several steps -- on a
    power-of-two grid with the mask wraps and with the generic ones
    (CS_DEP_NO_P2), and on grids that are not powers of two (384: int4 row
    copies; 250: scalar ones; their solve is cuFFT's)."""
    n = 60_000
    pos, sp, xi = _inputs(n, 13)
    x = torch.as_tensor(xi, device="cuda")
    out = {}
    if generic_wrap:
        monkeypatch.setenv("CS_DEP_NO_P2", "1")
    for mode in ("rows", "atomic"):
        if mode == "atomic":
            monkeypatch.setenv("CS_ATOMIC_DEPOSIT", "1")
        else:
            monkeypatch.delenv("CS_ATOMIC_DEPOSIT", raising=False)
        a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c)
        a.step(x, 6)
        a.export_state()
        assert a.status().code == 0
        out[mode] = {k: sa[k].clone() for k in ("pos", "c", "grad", "rho_a", "rho_b")}
    monkeypatch.delenv("CS_ATOMIC_DEPOSIT", raising=False)
    monkeypatch.delenv("CS_DEP_NO_P2", raising=False)
    for k in out["rows"]:
        assert torch.equal(out["rows"][k], out["atomic"][k]), k


def test_sorted_engine_reports_bucket_overflow(monkeypatch):
    """More records in a bucket of 256 consecutive cells than its region
    holds stops the sorted engine with CS_SORT_OVERFLOW (no record is lost
    silently); the same input with roomy regions runs and matches the direct
    engine bit for bit."""
    n = 20_000
    pos, sp, xi = _inputs(n, 6)
    pos[:3000, 1] = np.float32(0.2)  # 3000 particles in one cell row: a few buckets
    x = torch.as_tensor(xi[:2], device="cuda")
    monkeypatch.setenv("CS_BUCKET_CAP", "16")
    a, sa = _sim(pos, sp, engine="sorted", field=False)
    a.step(x, 1)
    assert a.status().code == cs._native.CS_SORT_OVERFLOW
    monkeypatch.delenv("CS_BUCKET_CAP")
    b, sb = _sim(pos, sp, engine="sorted", field=False)
    c, sc = _sim(pos, sp, engine="direct", field=False)
    b.step(x, 2)
    c.step(x, 2)
    b.export_state()
    assert b.status().code == 0 and c.status().code == 0
    assert torch.equal(sb["pos"], sc["pos"])


@pytest.mark.parametrize("n_c,n", [(512, 100_000), (8192, 400_000)])
def test_spectral_solve_sorted_engine_vs_cufft(n_c, n, monkeypatch):
    """cfg2f32's 512^2 and cfg4's 8192^2 periodic binary32 grids on the own
    spectral solve: one field-on step from a non-zero field against the same
    engine on cuFFT (c within binary32 FFT rounding: 3e-5 of max|c| at the
    largest of 67 M nodes; the accuracy of both transforms against binary64
    is compared in test_gpu_parity.py)."""
    pos, sp, xi = _inputs(n, 11)
    rng = np.random.default_rng(12)
    c0 = (0.5 + 0.1 * rng.standard_normal(n_c * n_c)).astype(np.float32).astype(np.float64)
    x = torch.as_tensor(xi, device="cuda")
    res = {}
    for mode in ("own", "cufft"):
        if mode == "cufft":
            monkeypatch.setenv("CS_CUFFT", "1")
        a, sa = _sim(pos, sp, engine="sorted", field=True, n_c=n_c, c0=c0,
                     radii=(2e-4, 4e-4))
        a.step(x[:2], 2)
        a.export_state()
        assert a.status().code == 0
        res[mode] = {k: sa[k].double().cpu().numpy() for k in ("pos", "c")}
    monkeypatch.delenv("CS_CUFFT", raising=False)
    cmax = np.abs(res["cufft"]["c"]).max()
    assert np.max(np.abs(res["own"]["c"] - res["cufft"]["c"])) <= 3e-5 * cmax
