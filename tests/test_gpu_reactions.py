"""Species reactions on the device against the reference.

The fixtures in tests/golden/reactions.npz and reaction_traj.npz were made by
the reference itself (tests/golden/make_golden.py): fixed_step_reactions /
beta_step_reactions on seeded populations, and fig1-like Realisations with
both schedulers.  Flip decisions compare u with a probability computed in
the reference's arithmetic, so species must match exactly; positions of the
field-coupled runs follow the cfg1/cfg2 composed-trajectory tolerance
(1e-10: the implicit solve's GEMM accumulation order differs from
OpenBLAS), the field-free "counts" run is bitwise."""

import warnings

import numpy as np
import pytest

from conftest import load_golden
from oracle.react import fixed_step

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402


class _Fixed:
    """Generator stand-in handing the reaction functions a pre-drawn block."""

    def __init__(self, u):
        self.u = u

    def random(self, n):
        assert n == self.u.shape[0]
        return self.u


def _pop(species, local_c, drift, device):
    n = species.shape[0]
    if device:
        t = lambda a, dt: torch.as_tensor(np.array(a), device="cuda").to(dt)  # noqa: E731
        return cs.Population(ids=np.arange(n), positions=t(np.zeros((n, 2)), torch.float64),
                             next_positions=t(np.zeros((n, 2)), torch.float64),
                             species=t(species, torch.uint8),
                             drift=t(drift, torch.float64),
                             local_concentration=t(local_c, torch.float64),
                             start_anchor=t(np.zeros((n, 2)), torch.float64))
    return cs.Population(ids=np.arange(n), positions=np.zeros((n, 2)),
                         next_positions=np.zeros((n, 2)), species=species.copy(),
                         drift=drift.copy(), local_concentration=local_c.copy(),
                         start_anchor=np.zeros((n, 2)))


@pytest.mark.parametrize("device", [False, True])
def test_fixed_and_beta_step_reactions_match_reference_golden(device):
    r = load_golden("reactions.npz")
    np_ = lambda a: a.cpu().numpy() if hasattr(a, "cpu") else a  # noqa: E731
    for k in range(int(r["n_fixed"])):
        ra, rb, dt = (float(v) for v in r[f"f{k}_in"])
        params = cs.ReactionParams(r_alpha=ra, r_beta=rb)
        pop = _pop(r[f"f{k}_species"], r[f"f{k}_local_c"], r[f"f{k}_drift"], device)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            cnt = cs.fixed_step_reactions(pop, params, dt, _Fixed(r[f"f{k}_u"]))
        assert np.array_equal(np_(pop.species), r[f"f{k}_out_species"]), k
        assert np.array_equal(np_(pop.drift), r[f"f{k}_out_drift"]), k
        assert cnt == tuple(int(v) for v in r[f"f{k}_counts"]), k
        assert len(w) == int(r[f"f{k}_warned"]), k
        pop = _pop(r[f"f{k}_species"], r[f"f{k}_local_c"], r[f"f{k}_drift"], device)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            nb = cs.beta_step_reactions(pop, params, dt, _Fixed(r[f"f{k}_u"]))
        assert np.array_equal(np_(pop.species), r[f"b{k}_out_species"]), k
        assert np.array_equal(np_(pop.drift), r[f"b{k}_out_drift"]), k
        assert nb == int(r[f"b{k}_count"]) and len(w) == int(r[f"b{k}_warned"]), k


def test_device_reactions_match_oracle_at_large_n():
    rng = np.random.default_rng(8)
    n = 3_000_000
    species = rng.integers(0, 2, n).astype(np.uint8)
    local_c = rng.normal(1.0, 2.0, n)
    drift = rng.normal(0.0, 1.0, (n, 2))
    u = rng.random(n)
    for p_ab, r_beta, dt in ((0.01, 40.0, 1e-3), (1.7, 0.0, 1e-3), (0.0, 600.0, 1e-3)):
        pop = _pop(species, local_c, drift, True)
        cs.fixed_step_reactions(pop, cs.ReactionParams(r_alpha=p_ab / dt, r_beta=r_beta), dt,
                                _Fixed(u)) if p_ab else cs.beta_step_reactions(
            pop, cs.ReactionParams(r_alpha=0.0, r_beta=r_beta), dt, _Fixed(u))
        t, d, _, _ = fixed_step(species, local_c, drift, u, (p_ab / dt) * dt, r_beta, dt)
        assert np.array_equal(pop.species.cpu().numpy(), t)
        assert np.array_equal(pop.drift.cpu().numpy(), d)


@pytest.mark.parametrize("name", ["fixed", "gillespie", "fixed_clamp", "counts"])
def test_realisation_with_reactions_matches_reference(name):
    g = load_golden("reaction_traj.npz")
    kw = {
        "fixed": dict(r_alpha=8000.0, r_beta=3000.0, scheduler="fixed"),
        "gillespie": dict(r_alpha=3000.0, r_beta=3000.0, scheduler="gillespie"),
        "fixed_clamp": dict(r_alpha=3.0e5, r_beta=0.0, scheduler="fixed"),
        "counts": dict(r_alpha=3000.0, r_beta=0.0, scheduler="fixed", interaction="none",
                       d_c=0.0, k_alpha=0.0, k_beta=0.0, dt=1e-4),
    }[name]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # the config's coarse-dt warning is not under test
        cfg = cs.SimConfig(n_alpha_0=20, n_beta_0=20, t_final=1.0, seed_base=5, **kw)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        real = cs.Realisation(cfg, 1)
        assert np.array_equal(real.pop.positions, g[f"{name}_pos0"])
        for s in range(1, 31):
            real.step()
            if s in (1, 5, 10, 20, 30):
                pop = real.pop
                assert np.array_equal(pop.species, g[f"{name}_species{s}"]), s
                if name == "counts":
                    assert np.array_equal(pop.positions, g[f"{name}_pos{s}"]), s
                else:
                    np.testing.assert_allclose(pop.positions, g[f"{name}_pos{s}"], rtol=0,
                                               atol=1e-10, err_msg=f"step {s}")
    warned = sum("exceeded 1 and was clamped" in str(x.message) for x in w)
    assert (warned > 0) == (int(g[f"{name}_warned"]) > 0)


@pytest.mark.parametrize("scheduler", ["fixed", "gillespie"])
def test_run_blocks_equal_single_steps_with_reactions(scheduler):
    """run() draws the increments and the reaction uniforms of several steps
    as one block: bit-identical to step() one at a time."""
    kw = dict(n_alpha_0=30, n_beta_0=30, r_alpha=4000.0, r_beta=2000.0, scheduler=scheduler,
              seed_base=9)
    cfg = cs.SimConfig(**kw)
    cfg = cs.SimConfig(**kw, t_final=40 * cfg.dt)
    a = cs.Realisation(cfg, 0)
    obs = a.run()
    b = cs.Realisation(cfg, 0)
    for _ in range(b.n_steps):
        b.step()
    assert a.step_index == b.step_index == 40
    assert np.array_equal(a.pop.positions, b.pop.positions)
    assert np.array_equal(a.pop.species, b.pop.species)
    assert obs.counts[-1].sum() == 60


def test_tamed_step_bitwise_vs_reference_golden():
    g = load_golden("tamed.npz")
    out = cs.tamed_step(g["pos"], g["dcoef"], g["drift"], g["force"], float(g["dt"]), xi=g["xi"])
    assert np.array_equal(out, g["out"])
    zero = cs.tamed_step(g["pos"], g["dcoef"], g["drift"], np.zeros_like(g["force"]),
                         float(g["dt"]), xi=g["xi"])
    assert np.array_equal(zero, cs.em_step(g["pos"], g["dcoef"], g["drift"],
                                           np.zeros_like(g["force"]), float(g["dt"]),
                                           xi=g["xi"]))


def test_tamed_realisation_matches_reference_trajectory():
    g = load_golden("tamed.npz")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = cs.SimConfig(n_alpha_0=20, n_beta_0=20, t_final=1.0, seed_base=8, r_alpha=0.0,
                           integrator="tamed", epsilon=0.05)
    real = cs.Realisation(cfg, 0)
    assert np.array_equal(real.pop.positions, g["traj_pos0"])
    for s in range(1, 21):
        real.step()
        if s in (1, 5, 20):
            np.testing.assert_allclose(real.pop.positions, g[f"traj_pos{s}"], rtol=0,
                                       atol=1e-10, err_msg=f"step {s}")


def test_hard_sphere_sweep_bitwise_vs_reference_golden():
    g = load_golden("hard.npz")
    for k in range(int(g["n_cases"])):
        size, per, eps, da, db = (float(v) for v in g[f"h{k}_meta"])
        n = g[f"h{k}_in"].shape[0]
        pop = cs.Population(ids=np.arange(n), positions=np.zeros((n, 2)),
                            next_positions=g[f"h{k}_in"].copy(), species=g[f"h{k}_species"],
                            drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                            start_anchor=np.zeros((n, 2)))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            params = cs.MotionParams(epsilon=eps, d_alpha=da, d_beta=db, dt=1e-7,
                                     interaction="hard")
        cs.resolve_hard_sphere(pop, cs.Domain.square(size, periodic=bool(per)), params)
        assert np.array_equal(pop.next_positions, g[f"h{k}_out"]), k


def test_hard_sphere_realisation_matches_reference_trajectory():
    g = load_golden("hard.npz")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = cs.SimConfig(n_alpha_0=30, n_beta_0=30, t_final=1.0, seed_base=9, r_alpha=0.0,
                           interaction="hard", epsilon=0.05)
    real = cs.Realisation(cfg, 0)
    for s in range(1, 21):
        real.step()
        if s in (1, 5, 20):
            np.testing.assert_allclose(real.pop.positions, g[f"traj_pos{s}"], rtol=0,
                                       atol=1e-10, err_msg=f"step {s}")
