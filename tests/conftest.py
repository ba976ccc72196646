"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on a CPU-only host."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def cfg0_xi(seed, steps, n):
    """The reference's motion stream: SeedSequence(seed).spawn(3)[1]
    (engine.py:272-275), one (N, 2) block per step (motion.py:277)."""
    streams = np.random.SeedSequence(seed).spawn(3)
    return np.random.default_rng(streams[1]).standard_normal((steps, n, 2))
