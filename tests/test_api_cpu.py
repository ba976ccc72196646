"""CPU-only checks of the host side: the C-ABI library loads and exports
every symbol include/chemo_b200.h declares, parameter objects validate like
the reference's, and the pair-table / status plumbing is right.  No compute
call is made (there is no GPU here)."""

import ctypes
import math
import re
import warnings

import numpy as np
import pytest

import paper_1805_11007_b200 as cs
from paper_1805_11007_b200 import _native as N

from conftest import ROOT


def _declared():
    src = open(f"{ROOT}/include/chemo_b200.h").read()
    return set(re.findall(r"^\s*(?:int|int64_t|void \*|const char \*)\s*\**\s*(cs_\w+)\(",
                          src, re.M))


def test_library_exports_every_declared_symbol():
    lib = N.load_library()
    decl = _declared()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
    assert {n for n, _, _ in N.SIGNATURES} == decl
    assert lib.cs_abi_version() == 3


def test_struct_layouts_match_header():
    # offsets that the C side relies on (x86-64 SysV)
    assert ctypes.sizeof(N.Domain_t) == 40
    assert ctypes.sizeof(N.PairParams_t) == 72
    assert ctypes.sizeof(N.Grid_t) == 40
    assert N.SimParams_t.store_next.offset + 4 <= ctypes.sizeof(N.SimParams_t)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.SO_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_compute_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    pop = cs.Population(ids=np.arange(2), positions=np.zeros((2, 2)),
                        next_positions=np.zeros((2, 2)), species=np.zeros(2, np.uint8),
                        drift=np.zeros((2, 2)), local_concentration=np.zeros(2),
                        start_anchor=np.zeros((2, 2)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cs.soft_forces(pop, cs.Domain.square(1.0), cs.MotionParams(dt=1e-7))


def test_pair_table_reduces_to_homogeneous_bitwise():
    eps = 0.005
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        homo = cs.MotionParams(epsilon=eps, cutoff=2.0 * eps, dt=1e-9)
        het = cs.MotionParams(epsilon=eps, cutoff=2.0 * eps, dt=1e-9, radius_alpha=eps,
                              radius_beta=eps)
    assert homo.pair_table() == het.pair_table()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        het = cs.MotionParams(epsilon=eps, dt=1e-9, radius_alpha=0.005, radius_beta=0.01)
    e, c, cell = het.pair_table()
    assert e == [0.005, 0.0075, 0.0075, 0.01]
    assert c == [0.01, 0.015, 0.015, 0.02] and cell == 0.02


def test_simconfig_matches_reference_defaults_and_validation():
    c = cs.SimConfig.preset("fig1")
    assert c.dt == pytest.approx((0.23 * 0.02) ** 2 / 4.0, rel=1e-15)
    assert c.n_steps == 9452
    assert c.motion_params().cutoff == 0.1
    with pytest.raises(ValueError, match="unknown experiment"):
        cs.SimConfig(experiment="warp")
    with pytest.raises(ValueError, match="at least one particle"):
        cs.SimConfig(n_alpha_0=0, n_beta_0=0)
    with pytest.raises(ValueError, match="precision"):
        cs.SimConfig(precision="fp16", r_alpha=0.0)
    with pytest.warns(UserWarning, match="destabilise"):
        cs.SimConfig(n_alpha_0=5, n_beta_0=5, gamma=200.0, dt=0.01, r_alpha=0.0,
                     interaction="none", n_c=11)


def test_sim_params_struct_amplitudes_match_numpy():
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = cs.MotionParams(d_alpha=1.0, d_beta=0.5, epsilon=0.005, cutoff=0.01, dt=1e-5)
    p = cs.sim_params_struct(n=10, prec=N.CS_F64, domain=cs.Domain.square(1.0), motion=mp,
                             dt=1e-5, field_active=False, refresh_active=False, grid=None,
                             fparams=None, kernel=None, secretes=(1, 0), consumes=(0, 1),
                             chi=(0.0, 1.0), chi_pinned=(1, 0), store_samples=0, store_next=0)
    amp = np.sqrt(2.0 * np.array([1.0, 0.5]) * 1e-5)
    assert p.amp[0] == amp[0] and p.amp[1] == amp[1]
    assert p.pairs.cell_cutoff == 0.01


def test_clustered_positions_wrap_into_box():
    dom = cs.Domain.square(1.0, periodic=True)
    pos = cs.clustered_positions(100000, dom, np.random.default_rng(0))
    assert np.all(pos >= -0.5) and np.all(pos < 0.5)


def test_reaction_params_validate_like_reference():
    with pytest.raises(ValueError, match="non-negative"):
        cs.ReactionParams(r_alpha=-1.0)
    with pytest.raises(ValueError, match="unknown reaction scheduler"):
        cs.ReactionParams(scheduler="tau")
    assert cs.SimConfig().reaction_params() == cs.ReactionParams(10.0, 0.0, "fixed")


def test_exponential_waiting_time_and_event_clock_match_reference_golden():
    """The event clock is host logic (reactions.py:84-138): on a host
    population it must reproduce the reference's picks and times exactly."""
    from conftest import load_golden
    r = load_golden("reactions.npz")
    assert cs.exponential_waiting_time(0, 5.0, np.random.default_rng(0)) == np.inf
    assert cs.exponential_waiting_time(3, 0.0, np.random.default_rng(0)) == np.inf
    species = r["clock_species0"].copy()
    n = species.shape[0]
    pop = cs.Population(ids=np.arange(n), positions=np.zeros((n, 2)),
                        next_positions=np.zeros((n, 2)), species=species,
                        drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                        start_anchor=np.zeros((n, 2)))
    rng = np.random.default_rng(77)
    clock = cs.AlphaEventClock(pop.n_alpha, 40.0, 0.0, rng)
    times, fired = [clock.next_time], []
    for until in (0.001, 0.004, 0.01, 0.02, 0.05):
        fired.append(clock.advance(pop, until, rng))
        times.append(clock.next_time)
        assert np.array_equal(pop.species, r[f"clock_species_{until}"]), until
    assert np.array_equal(np.array(times), r["clock_times"])
    assert np.array_equal(np.array(fired), r["clock_fired"])


def test_t4_reference_fixture_and_statistics_helper():
    """The T4 fixture (tests/golden/make_t4.py, the reference's own
    ensemble) holds 64 samples of every statistic, and the statistics helper
    counts pairs / MSD / field moments as defined (small known case)."""
    import os
    import sys
    import numpy as np
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from t4_stats import NAMES, compare, sample_stats
    g = np.load(os.path.join(here, "t4_reference.npz"))
    assert g["stats"].shape == (64, len(NAMES))
    assert list(g["names"]) == NAMES
    pos = np.array([[0.0, 0.0], [0.003, 0.0], [0.4999, 0.1], [-0.4999, 0.1]])
    st = sample_stats(pos, np.zeros_like(pos), np.array([0, 0, 1, 1]), np.ones(4),
                      np.full(4, 0.25), 1.0, 0.004)
    assert st[NAMES.index("pairs")] == 2  # one direct pair, one across the periodic seam
    assert st[NAMES.index("mass")] == 1.0 and abs(st[NAMES.index("l2")] - 1.0) < 1e-15
    assert abs(st[NAMES.index("msd_alpha")] - 0.003 ** 2 / 2) < 1e-18
    z, *_ = compare(g["stats"], g["stats"])
    assert np.all(z == 0)
