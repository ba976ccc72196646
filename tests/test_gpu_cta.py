"""The CTA engine (cs_sim with one realisation of the ensemble engine: the
whole system in one CTA's shared memory for all k steps of a call) against
the direct engine and the oracle, bit for bit.

It runs the direct engine's arithmetic in the same order (the deposit a
gather in particle order, the DCT solve the same k-ordered GEMMs), so a
K-step run through it equals the direct engine's and, at BASELINE cfg0, the
oracle's (pinned to the reference's own Realisation)."""

import os
import sys

import numpy as np
import pytest

import oracle
from oracle.sim import OracleSim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1805_11007_b200 as cs  # noqa: E402


def _make(cfg, engine):
    orig = cs.sim_params_struct

    def forced(*a, **kw):
        kw["engine"] = engine
        return orig(*a, **kw)
    cs.sim_params_struct = forced
    try:
        return bench.make_state(cfg, 0)
    finally:
        cs.sim_params_struct = orig


def test_cfg0_cta_engine_1000_steps_one_call_equals_oracle():
    cfg = bench.CONFIGS["cfg0"]
    sim, st, pos, sp = bench.make_state(cfg, 0)
    assert sim.engine == "cta"
    xi = np.random.default_rng(5).standard_normal((1000, cfg["n"], 2))
    sim.step(torch.as_tensor(xi, device="cuda"), 1000)
    assert sim.status().code == 0
    e, c, cell = oracle.pair_table(epsilon=cfg["eps"], cutoff=2 * cfg["eps"])
    o = OracleSim(pos, sp, lo=[-0.5] * 2, hi=[0.5] * 2, periodic=(False, False), dt=bench.DT,
                  diffusion=cfg["D"], eps_tab=e, cut_tab=c, cell_cutoff=cell,
                  chi=cfg["chi"], chi_pinned=cfg["chi_pinned"])
    for k in range(1000):
        o.step(xi[k])
    assert np.array_equal(st["pos"].cpu().numpy(), o.pos)


@pytest.mark.parametrize("field", [False, True])
def test_cta_engine_equals_direct_engine(field):
    """cfg1's configuration at 1/10 scale (1000 Beta particles, 48^2
    neumann CIC field with decay and secretion, chemotaxis): 300 steps in
    one call on the CTA engine, 300 per-step calls on the direct engine."""
    cfg = dict(bench.CONFIGS["cfg1"], n=1000, n_c=48 if field else 0, field=field,
               c0="linear_x" if field else "zero")
    if not field:
        cfg.update(chi_pinned=(True, True))
    a, sa, _, _ = _make(cfg, "auto")
    b, sb, _, _ = _make(cfg, "direct")
    assert a.engine == "cta" and b.engine == "direct"
    xi = torch.as_tensor(np.random.default_rng(7).standard_normal((300, cfg["n"], 2)),
                         device="cuda")
    a.step(xi, 300)
    for k in range(300):
        b.step(xi[k], 1)
    assert a.status().code == 0 and b.status().code == 0
    assert torch.equal(sa["pos"], sb["pos"])
    assert torch.equal(sa["anchor"], sb["anchor"])
    if field:
        assert torch.equal(sa["c"], sb["c"])


def test_cta_engine_reports_the_failing_step_and_particle():
    cfg = dict(bench.CONFIGS["cfg0"])
    sim, st, pos, sp = bench.make_state(cfg, 0)
    xi = torch.zeros((4, cfg["n"], 2), dtype=torch.float64, device="cuda")
    xi[2, 17, 1] = 1e9  # overshoots the walls by far more than a domain width
    sim.step(xi, 4)
    s = sim.status()
    assert s.code == 2 and s.step == 2 and s.particle == 17 and s.axis == 1
