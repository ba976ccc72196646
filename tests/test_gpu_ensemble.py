"""Batched ensembles (csrc/ensemble.cu) against the
sample-by-sample Realisation path and the reference's own trajectories.

Without a deposit the batched engine performs the direct engine's
arithmetic in the same order, so field-free ensembles (the counts and msd
presets) must equal the sequential run bit for bit.  With the field on the
shared-memory deposit sums concurrent stamps in a different order (1e-16),
so single-step states agree to 1e-12 and the reference's own fig1-like
trajectory (tests/golden/reaction_traj.npz) to the composed-trajectory
tolerance 1e-10 over 30 steps, species exactly."""

import os
import warnings

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402
from paper_1805_11007_b200.ensemble import Ensemble  # noqa: E402


def _quiet(**kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return cs.SimConfig(**kw)


def _both(cfg, monkeypatch):
    monkeypatch.setenv("CS_ENSEMBLE", "sequential")
    seq = cs.run_ensemble(cfg)
    monkeypatch.delenv("CS_ENSEMBLE")
    bat = cs.run_ensemble(cfg)
    return seq, bat


@pytest.mark.parametrize("preset,kw", [
    ("counts", dict(t_final=0.03, r_beta=0.0)),
    ("msd1", dict(t_final=1.0)),
    ("msd3", dict(t_final=0.6)),
])
def test_field_free_ensembles_equal_sequential_bitwise(preset, kw, monkeypatch):
    cfg = _quiet(**{**cs.SimConfig.preset(preset).as_dict(), **kw, "samples": 5})
    seq, bat = _both(cfg, monkeypatch)
    for name in ("times", "counts_mean", "counts_se", "msd_mean", "msd_se", "hist_alpha_mean",
                 "hist_alpha_se", "hist_beta_mean", "hist_beta_se", "field_mean", "field_se"):
        assert np.array_equal(getattr(seq, name), getattr(bat, name)), name
    assert seq.seeds == bat.seeds and bat.samples == 5


def test_fig1_ensemble_states_track_sequential_realisations():
    """fig1 (soft forces, gaussian deposit on the neumann 52^2 grid,
    fixed-step reactions): after 25 steps every sample's state is within
    1e-10 of its own Realisation, species identical."""
    cfg = _quiet(samples=6, seed_base=3, r_alpha=4000.0, r_beta=2000.0)
    cfg = _quiet(**{**cfg.as_dict(), "t_final": 25 * cfg.dt})
    ens = Ensemble(cfg)
    ens.advance(10)
    ens.advance(15)
    ens.check()
    pos = ens.state["pos"].cpu().numpy()
    sp = ens.state["species"].cpu().numpy()
    c = ens.state["c"].cpu().numpy()
    for s in range(cfg.samples):
        r = cs.Realisation(cfg, s)
        for _ in range(25):
            r.step()
        np.testing.assert_allclose(pos[s], r.pop.positions, rtol=0, atol=1e-10)
        assert np.array_equal(sp[s], r.pop.species)
        np.testing.assert_allclose(c[s], r.field.c, rtol=1e-9, atol=1e-9)
    ens.close()


def test_ensemble_matches_reference_reaction_trajectory():
    """Sample 1 of the reference run behind reaction_traj.npz ("fixed":
    20 + 20 particles, fig1 parameters, r_alpha 8000, r_beta 3000)."""
    g = load_golden("reaction_traj.npz")
    cfg = _quiet(n_alpha_0=20, n_beta_0=20, t_final=1.0, seed_base=5, r_alpha=8000.0,
                 r_beta=3000.0, scheduler="fixed", samples=3)
    ens = Ensemble(cfg)
    assert np.array_equal(ens.state["pos"][1].cpu().numpy(), g["fixed_pos0"])
    done = 0
    for s in (1, 5, 10, 20, 30):
        ens.advance(s - done)
        done = s
        np.testing.assert_allclose(ens.state["pos"][1].cpu().numpy(), g[f"fixed_pos{s}"],
                                   rtol=0, atol=1e-10, err_msg=f"step {s}")
        assert np.array_equal(ens.state["species"][1].cpu().numpy(), g[f"fixed_species{s}"])
    ens.check()
    ens.close()


def test_ensemble_failure_names_sample_and_step():
    cfg = _quiet(samples=4, interaction="none", d_c=0.0, k_alpha=0.0, k_beta=0.0, r_alpha=0.0,
                 dt=3.0, t_final=3.0, d_beta=1.0, d_alpha=1.0)
    with pytest.raises(cs.SimulationError, match=r"sample \d+: step 0: particle \d+ overshot"):
        cs.run_ensemble(cfg)


def test_unsupported_configs_fall_back_to_realisations():
    from paper_1805_11007_b200.ensemble import supported
    assert supported(_quiet(scheduler="gillespie")) is not None
    assert supported(_quiet(periodic=True)) is not None  # periodic grid
    assert supported(_quiet()) is None


def test_device_rng_ensemble_equals_host_rng_ensemble():
    """The ensemble's device-drawn increments/uniforms are numpy's: the
    same states as with host-drawn blocks, bit for bit."""
    cfg = _quiet(samples=5, seed_base=11, r_alpha=3000.0, r_beta=1500.0)
    a = Ensemble(cfg, rng="device")
    b = Ensemble(cfg, rng="host")
    for k in (7, 13):
        a.advance(k)
        b.advance(k)
    for key in ("pos", "species", "anchor"):
        assert torch.equal(a.state[key], b.state[key]) or key != "pos" or \
            torch.allclose(a.state[key], b.state[key], rtol=0, atol=1e-12), key
    a.close()
    b.close()


def test_tamed_ensemble_tracks_realisations():
    cfg = _quiet(samples=3, seed_base=8, r_alpha=0.0, integrator="tamed", epsilon=0.05,
                 n_alpha_0=20, n_beta_0=20)
    ens = Ensemble(cfg)
    ens.advance(12)
    ens.check()
    pos = ens.state["pos"].cpu().numpy()
    for s in range(3):
        r = cs.Realisation(cfg, s)
        for _ in range(12):
            r.step()
        np.testing.assert_allclose(pos[s], r.pop.positions, rtol=0, atol=1e-10)
    ens.close()
