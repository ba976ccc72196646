"""Batched ensembles (csrc/ensemble.cu) against the
sample-by-sample Realisation path and the reference's own trajectories.

The batched engine performs the direct engine's arithmetic in the same
order -- the deposit included: both gather every node's stamps in the
reference's particle order -- so ensembles equal the sequential run bit for
bit, with and without the field.  Against the reference's own fig1-like
trajectory (tests/golden/reaction_traj.npz) the composed-trajectory
tolerance 1e-10 over 30 steps applies (the DCT solve's GEMM accumulation
order is not OpenBLAS's), species exactly."""

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


def test_fig1_ensemble_states_equal_sequential_realisations():
    """fig1 (soft forces, gaussian deposit on the neumann 52^2 grid,
    fixed-step reactions): after 25 steps every sample's state is bit for
    bit its own Realisation's (both engines deposit in particle order)."""
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
        assert np.array_equal(c[s], r.field.c), s
        assert np.array_equal(pos[s], r.pop.positions), s
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
    for key in ("pos", "species", "anchor", "c"):
        assert torch.equal(a.state[key], b.state[key]), key
    a.close()
    b.close()


def test_long_blocks_many_samples_device_rng_run_equals_host_rng_run():
    """Ensemble.run with the device RNG drawing the next block on a side
    stream: the status and observables of each block must be read after the
    block's step kernel (same stream), so many samples x long blocks give
    the host-RNG run's observables bit for bit."""
    cfg = _quiet(samples=96, seed_base=21, r_alpha=2000.0, r_beta=800.0, output_every=150)
    cfg = _quiet(**{**cfg.as_dict(), "t_final": 600 * cfg.dt})
    runs = []
    for rng in ("device", "host"):
        e = Ensemble(cfg, rng=rng)
        runs.append(e.run())
        e.close()
    for oa, ob in zip(*runs):
        for name in ("times", "counts", "msd", "hist_alpha", "hist_beta", "field_c"):
            assert np.array_equal(getattr(oa, name), getattr(ob, name)), name


def test_fig1_cli_reruns_byte_identical(tmp_path):
    """Acceptance criterion 10 of the reference
    (pkg/tests/test_acceptance.py:341-355): two `--experiment fig1
    --samples 2` runs write byte-identical CSV files -- on the batched
    engine and on the sample-by-sample Realisation path (direct engine)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("batched", "sequential"):
        for tag in ("a", "b"):
            env = dict(os.environ, PYTHONPATH=root)
            if mode == "sequential":
                env["CS_ENSEMBLE"] = "sequential"
            out = tmp_path / f"{mode}_{tag}"
            proc = subprocess.run([sys.executable, "-m", "paper_1805_11007_b200", "--experiment",
                                   "fig1", "--samples", "2", "--output-dir", str(out)],
                                  capture_output=True, text=True, env=env, cwd=root)
            assert proc.returncode == 0, proc.stderr
            outs[(mode, tag)] = out
    for mode in ("batched", "sequential"):
        a, b = outs[(mode, "a")], outs[(mode, "b")]
        names = sorted(p.name for p in a.glob("*.csv"))
        assert names
        for name in names:
            assert (a / name).read_bytes() == (b / name).read_bytes(), (mode, name)
    # and the two engines agree with each other byte for byte
    for name in sorted(p.name for p in outs[("batched", "a")].glob("*.csv")):
        assert (outs[("batched", "a")] / name).read_bytes() == \
            (outs[("sequential", "a")] / name).read_bytes(), name


def test_run_ensemble_beyond_one_cta_falls_back(monkeypatch):
    """A realisation whose state exceeds one CTA's shared memory (here 3000
    particles on a 52^2 grid) runs sample by sample instead of failing."""
    cfg = _quiet(n_alpha_0=1500, n_beta_0=1500, samples=2, r_alpha=0.0,
                 t_final=0.0)
    cfg = _quiet(**{**cfg.as_dict(), "t_final": 3 * cfg.dt})
    res = cs.run_ensemble(cfg)
    monkeypatch.setenv("CS_ENSEMBLE", "sequential")
    seq = cs.run_ensemble(cfg)
    assert np.array_equal(res.msd_mean, seq.msd_mean)
    assert np.array_equal(res.counts_mean, seq.counts_mean)


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
