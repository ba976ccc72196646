"""Stochastic switching between the two cell species.

Mirror of chemosim/reactions.py.  Alpha cells convert to Beta at a constant
rate r_alpha; Beta cells convert back at r_beta * c(X).  The per-step
Bernoulli trials (``fixed_step_reactions``, ``beta_step_reactions``) run on
the device (``cs_react``, csrc/react.cu) against the same uniforms the
reference draws -- one ``rng.random(N)`` block per call, drawn on the host
from the caller's generator, so the stream layout is the reference's.  The
event clock of the constant-rate channel (``AlphaEventClock``) is scalar
host logic with the reference's draw order; its flips are single-element
writes into the (device) species array.

Inside a ``Realisation`` the fixed scheduler is fused into the device step
(cs_sim_step_react): the uniforms of K steps are drawn as one (K, N) block,
bit-identical to K successive ``rng.random(N)`` draws.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _arrays as A
from . import _native as N
from .particles import Population, Species


@dataclass(frozen=True)
class ReactionParams:
    """reactions.py:21-31."""
    r_alpha: float = 10.0
    r_beta: float = 0.0
    scheduler: str = "fixed"

    def __post_init__(self):
        if self.r_alpha < 0 or self.r_beta < 0:
            raise ValueError("reaction rates must be non-negative")
        if self.scheduler not in ("fixed", "gillespie"):
            raise ValueError(f"unknown reaction scheduler {self.scheduler!r}")


def _device_species(pop: Population):
    """(species, local_c, drift) as CUDA tensors: the population's own
    tensors when it is device-resident, otherwise uploaded copies."""
    torch = N.require_cuda()
    sp = pop.species
    host = not A.on_device(sp)
    species = A.dev(sp, torch.uint8)
    local_c = A.dev(pop.local_concentration, torch.float64)
    drift = A.dev(pop.drift, torch.float64)
    return species, local_c, drift, host


def _react(pop: Population, u: np.ndarray, p_ab: float, r_beta: float, dt: float):
    torch = N.require_cuda()
    species, local_c, drift, host = _device_species(pop)
    ud = A.dev(u, torch.float64)
    flips = (ctypes.c_int64 * 2)()
    high = ctypes.c_double(0.0)
    N.check(N.load_library().cs_react(N.context(), N.ptr(species), N.ptr(local_c),
                                      N.ptr(drift), N.ptr(ud), len(pop), float(p_ab),
                                      float(r_beta), float(dt), flips, ctypes.byref(high)),
            "cs_react")
    if host:  # write the switched labels / zeroed drift rows back (in place)
        pop.species[...] = species.cpu().numpy()
        pop.drift[...] = drift.cpu().numpy()
    elif drift.data_ptr() != pop.drift.data_ptr():
        pop.drift.copy_(drift)
    return int(flips[0]), int(flips[1]), float(high.value)


def fixed_step_reactions(pop: Population, params: ReactionParams, dt: float,
                         rng: np.random.Generator) -> tuple[int, int]:
    """One Bernoulli trial per particle against its species' flip
    probability (reactions.py:43-81); returns (alpha->beta, beta->alpha)."""
    u = rng.random(len(pop))
    p_ab = params.r_alpha * dt
    n_ab, n_ba, high = _react(pop, u, p_ab, params.r_beta, dt)
    if high > 1.0:
        # the reference's `high` (p_ab when an Alpha exists, else the Beta
        # maximum): the kernel reports the largest probability above 1
        warnings.warn(f"flip probability {high:.3g} exceeded 1 and was "
                      "clamped; reduce dt", stacklevel=2)
    return n_ab, n_ba


def exponential_waiting_time(n_alpha: int, r_alpha: float,
                             rng: np.random.Generator) -> float:
    """reactions.py:84-97: ln(1/zeta) / (n_alpha r_alpha), zeta uniform."""
    total = n_alpha * r_alpha
    if total <= 0.0:
        return np.inf
    zeta = rng.random()
    if zeta == 0.0:
        return np.inf
    return np.log(1.0 / zeta) / total


class AlphaEventClock:
    """Exact event scheduler for the constant-rate Alpha -> Beta channel
    (reactions.py:100-138)."""

    def __init__(self, n_alpha: int, r_alpha: float, now: float,
                 rng: np.random.Generator):
        self.r_alpha = r_alpha
        self.next_time = now + exponential_waiting_time(n_alpha, r_alpha, rng)

    def reschedule(self, n_alpha: int, now: float, rng: np.random.Generator) -> None:
        self.next_time = now + exponential_waiting_time(n_alpha, self.r_alpha, rng)

    def advance(self, pop: Population, until: float, rng: np.random.Generator) -> int:
        """Fire every conversion scheduled up to `until`: each flips one
        uniformly chosen Alpha (ascending index order, as np.flatnonzero)."""
        fired = 0
        species = None
        while self.next_time <= until:
            if species is None:
                species = A.to_numpy(pop.species).copy()
            alphas = np.flatnonzero(species == Species.ALPHA)
            if alphas.size == 0:
                self.next_time = np.inf
                break
            pick = int(alphas[rng.integers(alphas.size)])
            species[pick] = Species.BETA
            pop.species[pick] = int(Species.BETA)
            fired += 1
            self.reschedule(alphas.size - 1, self.next_time, rng)
        return fired


def beta_step_reactions(pop: Population, params: ReactionParams, dt: float,
                        rng: np.random.Generator) -> int:
    """Per-step Bernoulli trials for the Beta -> Alpha channel only
    (reactions.py:141-160)."""
    if params.r_beta == 0.0:
        return 0
    u = rng.random(len(pop))
    _, n_ba, high = _react(pop, u, 0.0, params.r_beta, dt)
    if high > 1.0:
        warnings.warn(f"flip probability {high:.3g} exceeded 1 "
                      "and was clamped; reduce dt", stacklevel=2)
    return n_ba
