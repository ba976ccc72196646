"""Parity tier T4: ensemble statistics of our Realisation
against the reference's own ensemble (tests/golden/t4_reference.npz, made
by tests/golden/make_t4.py from the reference's Realisation, fp64).

Per-type MSD, the in-cutoff pair count, the g(r) histogram inside the cutoff
and the field's weighted mass and L2 norm after t_final, each within 3
combined standard errors of the reference's mean.  Our samples use other
seeds (seed_base 1000), so this is a statistical check, not a trajectory one:
it covers the binary32 sorted engine, whose trajectories are not comparable
with the fp64 reference beyond a few steps (tier T1 pins its one-step error),
and the fp64 direct engine on the same footing."""

import os
import sys
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from t4_stats import NAMES, T4_CONFIG, compare, sample_stats  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "t4_reference.npz")


@pytest.mark.parametrize("precision,engine,xi_order", [("fp32", "sorted", "id"),
                                                      ("fp32", "sorted", "slot"),
                                                      ("fp64", "direct", "id")])
def test_t4_ensemble_statistics_vs_reference(precision, engine, xi_order):
    """xi_order='slot' is the sorted engine's performance mode (increments
    consumed by storage slot): the same distribution, so the same statistics."""
    ref = np.load(GOLDEN)["stats"]
    cfg = cs.SimConfig(**T4_CONFIG, seed_base=1000, precision=precision, xi_order=xi_order)
    rows = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for s in range(64):
            real = cs.Realisation(cfg, s)
            assert real._sim.engine == engine
            real.run()
            real._sim.export_state()
            pop = real.pop
            rows.append(sample_stats(pop.positions, pop.start_anchor, pop.species,
                                     real.field.c, real.grid.quadrature_weights(),
                                     cfg.domain_size, cfg.soft_cutoff_factor * cfg.epsilon))
    ours = np.array(rows)
    z, mr, mo, se = compare(ref, ours)
    report = "\n".join(f"{nm:10s} ref {a:.6g} ours {b:.6g} se {c:.3g} z {d:.2f}"
                       for nm, a, b, c, d in zip(NAMES, mr, mo, se, z))
    assert np.all(z <= 3.0), report
