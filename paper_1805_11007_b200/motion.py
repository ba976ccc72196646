"""Overdamped Brownian motion with soft repulsion -- device implementation.

Mirror of chemosim/motion.py: same names, signatures, validation, warnings
and error messages.  The per-step work runs in the sm_100a library:

  soft_forces        -> cs_soft_forces       (motion.py:248-265, :165-245)
  em_step            -> cs_em_step           (motion.py:268-282)
  apply_boundaries   -> cs_apply_boundaries  (motion.py:405-430, :355-402)

Extensions (additive keyword fields): per-type radii
(``radius_alpha``/``radius_beta``) give the pair table eps_ij = (r_i+r_j)/2,
cut_ij = cutoff_factor * eps_ij (BASELINE configs 2-4); with equal radii
and cutoff_factor 2 it is bitwise the reference's homogeneous table.
The tamed integrator (motion.py:283-298) and the hard-sphere sweep
(motion.py:301-352) run on the device.
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _arrays as A
from . import _native as N
from .particles import Population, Species
from .spatial_index import Domain


class SimulationError(RuntimeError):
    """A realisation reached a non-recoverable state (NaN position, runaway
    overshoot); the run should be aborted rather than patched over."""


@dataclass
class MotionParams:
    d_alpha: float = 0.1
    d_beta: float = 1.0
    chi: float = 1.0
    epsilon: float = 0.02
    dt: float = 5.29e-6
    interaction: str = "soft"
    cutoff: float = field(default=0.0)  # absolute force cutoff; 0 -> 5 epsilon
    integrator: str = "em"
    # extensions (None = reference semantics)
    radius_alpha: float | None = None
    radius_beta: float | None = None
    cutoff_factor: float = 2.0

    def __post_init__(self):
        if self.d_alpha < 0 or self.d_beta < 0:
            raise ValueError("diffusion coefficients must be non-negative")
        if not self.dt > 0:
            raise ValueError("dt must be positive")
        if self.interaction not in ("soft", "hard", "none"):
            raise ValueError(f"unknown interaction model {self.interaction!r}")
        if self.integrator not in ("em", "tamed"):
            raise ValueError(f"unknown integrator {self.integrator!r}")
        if (self.radius_alpha is None) != (self.radius_beta is None):
            raise ValueError("give both per-type radii or neither")
        if self.radius_alpha is not None and not (self.radius_alpha > 0 and self.radius_beta > 0):
            raise ValueError("per-type radii must be positive")
        if self.interaction != "none":
            if not self.epsilon > 0:
                raise ValueError("epsilon must be positive for interacting runs")
            if self.cutoff == 0.0:
                self.cutoff = 5.0 * self.epsilon
            step_scale = math.sqrt(2.0 * (self.d_alpha + self.d_beta) * self.dt)
            eps_min = self.epsilon if self.radius_alpha is None else min(
                self.radius_alpha, self.radius_beta)
            if step_scale > eps_min:
                warnings.warn(
                    f"dt resolution guard violated: rms pair step {step_scale:.3g} "
                    f"exceeds epsilon {eps_min:.3g}; encounters may be skipped",
                    stacklevel=2)

    def diffusion_of(self, species):
        if A.is_tensor(species):
            import torch
            return torch.where(species == Species.ALPHA, self.d_alpha, self.d_beta).to(
                torch.float64)
        return np.where(np.asarray(species) == Species.ALPHA, self.d_alpha, self.d_beta)

    def pair_table(self):
        """(eps[4], cutoff[4], cell_cutoff) indexed t_i * 2 + t_j."""
        if self.radius_alpha is None:
            eps = [float(self.epsilon)] * 4
            cut = [float(self.cutoff)] * 4
        else:
            r = (float(self.radius_alpha), float(self.radius_beta))
            eps = [(r[a] + r[b]) / 2.0 for a in range(2) for b in range(2)]
            cut = [self.cutoff_factor * e for e in eps]
        return eps, cut, max(cut)

    @property
    def heterogeneous(self) -> bool:
        return self.radius_alpha is not None


def pair_force(dx, r: float, epsilon: float):
    """Force on particle i from u(r) = exp(-r / epsilon) (motion.py:77-88):
    -(1/epsilon) exp(-r/epsilon) dx / r, zero at exact overlap.  Analytic
    scalar helper (not on the per-step path)."""
    dx = np.asarray(dx, dtype=float)
    if r == 0.0:
        return np.zeros_like(dx)
    return -(np.exp(-r / epsilon) / (epsilon * r)) * dx


def _domain_struct(domain: Domain):
    return N.domain_struct(domain.lo, domain.hi, domain.periodic)


def _force_inputs(pop: Population, params: MotionParams):
    pos_t = A.dev(pop.positions, A.float_dtype_of(pop.positions))
    types = None
    if params.heterogeneous:
        import torch
        types = A.dev(pop.species, torch.uint8)
    eps, cut, cell = params.pair_table()
    return pos_t, types, N.pair_struct(eps, cut, cell)


def soft_forces(pop: Population, domain: Domain, params: MotionParams):
    """Soft pair forces (motion.py:248-265), binned internally on the device
    into cells of side >= the cutoff, summed in the reference order."""
    import torch
    host = not A.on_device(pop.positions)
    pos_t, types, pp = _force_inputs(pop, params)
    n = pos_t.shape[0]
    out = A.empty((n, 2), torch.float64)
    ctx = N.context()
    N.check(N.load_library().cs_soft_forces(
        ctx, N.prec_code(pos_t.dtype), N.ptr(pos_t), N.ptr(types), n,
        ctypes.byref(_domain_struct(domain)), ctypes.byref(pp), N.ptr(out)), "cs_soft_forces")
    return A.back(out, host)


def accumulate_forces(pop: Population, index, params: MotionParams):
    """Sum of pair_force over all neighbours within params.cutoff, per
    particle, through a CellIndex (motion.py:146-161, _soft_forces :107-143):
    any cell side (ring reach ceil(cutoff / eff) per axis), single epsilon and
    cutoff, the reference's summation order and arithmetic, on the device."""
    import torch
    host = not A.on_device(pop.positions)
    d = index._dev
    pos_t = d["pos"]
    n = pos_t.shape[0]
    out = A.empty((n, 2), torch.float64)
    nc = (ctypes.c_int32 * 2)(int(index.n_cells[0]), int(index.n_cells[1]))
    dom = index.domain
    N.check(N.load_library().cs_index_forces(
        N.context(), N.prec_code(pos_t.dtype), N.ptr(pos_t), n, N.ptr(d["cell_xy"]),
        N.ptr(d["order"]), N.ptr(d["starts"]),
        ctypes.byref(N.domain_struct(dom.lo, dom.hi, dom.periodic)), nc,
        float(params.epsilon), float(params.cutoff), N.ptr(out)), "cs_index_forces")
    return A.back(out, host)


def soft_force_pairs(pop: Population, domain: Domain, params: MotionParams):
    """(P, 2) int64 pairs (i, j) the force kernel accumulates, in its
    accumulation order (i ascending, ring cell, j ascending): the bit-exact
    pair set of SURVEY 8c."""
    import torch
    pos_t, types, pp = _force_inputs(pop, params)
    n = pos_t.shape[0]
    lib, ctx = N.load_library(), N.context()
    cnt = ctypes.c_int64(0)
    dom = _domain_struct(domain)
    N.check(lib.cs_soft_force_pairs(ctx, N.prec_code(pos_t.dtype), N.ptr(pos_t), N.ptr(types),
                                    n, ctypes.byref(dom), ctypes.byref(pp), N.C_p(0), 0,
                                    ctypes.byref(cnt)), "cs_soft_force_pairs")
    out = A.empty((max(cnt.value, 1), 2), torch.int64)
    N.check(lib.cs_soft_force_pairs(ctx, N.prec_code(pos_t.dtype), N.ptr(pos_t), N.ptr(types),
                                    n, ctypes.byref(dom), ctypes.byref(pp), N.ptr(out),
                                    cnt.value, ctypes.byref(cnt)), "cs_soft_force_pairs")
    return out[:cnt.value].cpu().numpy()


def _proposal(entry, position, diffusion, drift, force, dt, rng, xi):
    import torch
    single = (not A.is_tensor(position)) and np.asarray(position).ndim == 1
    host = not A.on_device(position)
    pdt = A.float_dtype_of(position)
    pos = A.dev(np.atleast_2d(np.asarray(position, dtype=float)) if single else position, pdt)
    n = pos.shape[0]
    if xi is None:
        if rng is None:
            raise ValueError(f"{entry[3:]} needs an rng or a pre-drawn xi")
        xi = rng.standard_normal(tuple(pos.shape))
    xi_t = A.dev(xi, pdt).reshape(n, 2)

    def full(v, shape):
        if A.is_tensor(v):
            t = v.to(device="cuda", dtype=torch.float64)
        else:
            t = torch.as_tensor(np.asarray(v, dtype=float), device="cuda")
        return torch.broadcast_to(t, shape).contiguous()

    d_t = full(diffusion, (n,))
    drift_t = full(drift, (n, 2))
    force_t = full(force, (n, 2))
    out = A.empty((n, 2), pdt)
    N.check(getattr(N.load_library(), entry)(N.context(), N.prec_code(pdt), N.ptr(pos),
                                             N.ptr(d_t), N.ptr(drift_t), N.ptr(force_t),
                                             N.ptr(xi_t), float(dt), n, N.ptr(out)), entry)
    res = A.back(out, host)
    return res[0] if single else res


def em_step(position, diffusion, drift, force, dt: float, rng=None, *, xi=None):
    """Euler--Maruyama proposal X + sqrt(2 D dt) xi + drift dt + force dt
    (motion.py:268-282).  Draws exactly one standard-normal pair per
    particle from `rng` (host numpy Generator, the reference contract), or
    takes a pre-drawn `xi` array/tensor of the position's shape."""
    return _proposal("cs_em_step", position, diffusion, drift, force, dt, rng, xi)


def tamed_step(position, diffusion, drift, force, dt: float, rng=None, *, xi=None):
    """Tamed Euler proposal (motion.py:283-298): the interaction increment
    force dt is scaled by 1 / (1 + ||force|| dt); one standard-normal pair
    per particle as em_step."""
    return _proposal("cs_tamed_step", position, diffusion, drift, force, dt, rng, xi)


def resolve_hard_sphere(pop: Population, domain: Domain, params: MotionParams):
    """Single overlap-correction sweep over the proposed positions
    (motion.py:301-352), on the device: the pairs closer than epsilon at the
    start of the sweep, in ascending (i, j) order, re-measured against the
    current buffer and pushed apart along the centre line, split by the
    diffusivities.  Updates pop.next_positions in place and returns it."""
    prop = pop.next_positions
    n = len(pop)
    if n < 2:
        return prop
    host = not A.on_device(prop)
    pdt = A.float_dtype_of(prop)
    x = A.dev(prop, pdt)
    import torch
    sp = A.dev(pop.species, torch.uint8)
    dom = N.domain_struct(domain.lo, domain.hi, domain.periodic)
    N.check(N.load_library().cs_resolve_hard_sphere(
        N.context(), N.prec_code(pdt), N.ptr(x), N.ptr(sp), n, ctypes.byref(dom),
        float(params.epsilon), float(params.d_alpha), float(params.d_beta)),
        "cs_resolve_hard_sphere")
    if host:
        prop[...] = x.cpu().numpy()
    elif x.data_ptr() != prop.data_ptr():
        prop.copy_(x)
    return prop


def raise_boundary_status(status: int, i: int, ax: int, x) -> None:
    """The reference's exceptions for kernel statuses (motion.py:421-429)."""
    if status == N.CS_NONFINITE:
        row = A.to_numpy(x[i]) if x is not None else "?"
        raise SimulationError(f"non-finite coordinate for particle {i}: {row}")
    if status == N.CS_OVERSHOOT:
        coord = float(x[i, ax]) if x is not None else float("nan")
        raise SimulationError(
            f"particle {i} overshot axis {ax} by more than one "
            f"domain width (coordinate {coord:.6g})")
    if status == N.CS_UNSETTLED:
        raise SimulationError(f"reflection failed to settle on axis {ax}")


def apply_boundaries(pop: Population, domain: Domain) -> None:
    """Resolve the proposal buffer against the box and commit it
    (motion.py:405-430), in place on pop."""
    host = not A.on_device(pop.next_positions)
    pdt = A.float_dtype_of(pop.next_positions)
    x = A.dev(pop.next_positions, pdt)
    anchor = A.dev(pop.start_anchor, pdt)
    n = x.shape[0]
    raw = pop.next_positions
    raw_host = A.to_numpy(raw).copy() if host else None
    bi, ba = ctypes.c_int64(-1), ctypes.c_int32(-1)
    st = N.load_library().cs_apply_boundaries(
        N.context(), N.prec_code(pdt), N.ptr(x), N.ptr(anchor), N.C_p(0), n,
        ctypes.byref(_domain_struct(domain)), ctypes.byref(bi), ctypes.byref(ba))
    N.check(st, "cs_apply_boundaries")
    if st != N.CS_OK:
        raise_boundary_status(st, bi.value, ba.value, raw_host if host else raw)
    if host:
        xs = x.cpu().numpy()
        pop.next_positions[...] = xs
        pop.start_anchor[...] = anchor.cpu().numpy()
        pop.positions[...] = xs
    else:
        if x.data_ptr() != pop.next_positions.data_ptr():
            pop.next_positions.copy_(x)
        if anchor.data_ptr() != pop.start_anchor.data_ptr():
            pop.start_anchor.copy_(anchor)
        pop.positions.copy_(x)
