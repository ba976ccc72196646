"""Particle <-> grid coupling -- device implementation.

Mirror of chemosim/coupling.py: density deposits (gaussian stamp or
cloud-in-cell) and bilinear sampling, in grid units u = (x - lo)/spacing.

  deposit / deposit_both     -> cs_deposit   (coupling.py:141-187)
  interpolate / field_at     -> cs_bilinear  (coupling.py:216-299)
  refresh_particle_fields    -> cs_bilinear  (coupling.py:302-325)
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _arrays as A
from . import _native as N
from .field import Field, Grid
from .particles import Population, Species


@dataclass(frozen=True)
class Kernel:
    kind: str = "gaussian"
    h: float = 0.02
    cutoff: float = 0.06

    def __post_init__(self):
        if self.kind not in ("gaussian", "cic"):
            raise ValueError(f"unknown deposit kernel {self.kind!r}")
        if self.kind == "gaussian":
            if not self.h > 0:
                raise ValueError("kernel bandwidth must be positive")
            if not self.cutoff > 0:
                raise ValueError("kernel cutoff must be positive")


def _deposit(pop: Population, grid: Grid, kernel: Kernel, route, two: bool):
    import torch
    host = not A.on_device(pop.positions)
    pdt = A.float_dtype_of(pop.positions)
    pos = A.dev(pop.positions, pdt)
    r = A.dev(route, torch.uint8)
    m = grid.n_c * grid.n_c
    ra = A.empty((m,), pdt)
    rb = A.empty((m,), pdt) if two else None
    kind = N.CS_CIC if kernel.kind == "cic" else N.CS_GAUSSIAN
    rc = N.load_library().cs_deposit(N.context(), N.prec_code(pdt), N.ptr(pos), N.ptr(r),
                                     pos.shape[0], ctypes.byref(N.grid_struct(grid)), kind,
                                     float(kernel.h), float(kernel.cutoff), N.ptr(ra), N.ptr(rb))
    if rc == -2:
        raise ValueError("gaussian cutoff spans more than the periodic grid")
    N.check(rc, "cs_deposit")
    if two:
        return A.back(ra, host), A.back(rb, host)
    return A.back(ra, host)


def deposit(pop: Population, grid: Grid, kernel: Kernel, species: Species):
    """Nodal number density of one species (coupling.py:141-162)."""
    sp = pop.species
    if A.is_tensor(sp):
        import torch
        route = torch.where(sp == int(species), 0, 2).to(torch.uint8)
    else:
        route = np.where(np.asarray(sp) == int(species), 0, 2).astype(np.uint8)
    return _deposit(pop, grid, kernel, route, two=False)


def deposit_gather(pop: Population, grid: Grid, kernel: Kernel, species: Species):
    """Node-centric reference deposit, gaussian only (coupling.py:190-213):
    every node against every particle of `species` in index order, on the
    device (the cross-check of the scatter path; O(N n_c^2))."""
    import torch
    if kernel.kind != "gaussian":
        raise ValueError("gather reference is defined for the gaussian kernel")
    host = not A.on_device(pop.positions)
    pdt = A.float_dtype_of(pop.positions)
    pos = A.dev(pop.positions, pdt)
    sel = A.dev(pop.species, torch.uint8) == int(species)
    pos = pos[sel].contiguous()
    out = A.zeros(grid.n_c * grid.n_c, torch.float64)
    span = np.asarray(grid.hi, dtype=float) - np.asarray(grid.lo, dtype=float)
    N.check(N.load_library().cs_deposit_gather(
        N.context(), N.prec_code(pdt), N.ptr(pos), pos.shape[0], ctypes.byref(N.grid_struct(grid)),
        float(span[0]), float(span[1]), float(kernel.h), float(kernel.cutoff), N.ptr(out)),
        "cs_deposit_gather")
    return A.back(out, host)


def deposit_both(pop: Population, grid: Grid, kernel: Kernel):
    """(rho_alpha, rho_beta) from one particle sweep (coupling.py:165-187)."""
    return _deposit(pop, grid, kernel, pop.species, two=True)


def _bilinear(grid: Grid, values, points):
    """(out (k, m) tensor, clamped count, host flag)."""
    host = not A.on_device(points)
    pdt = A.float_dtype_of(values)
    pts = A.dev(np.atleast_2d(np.asarray(points, dtype=float)) if not A.is_tensor(points)
                else points, pdt).reshape(-1, 2)
    vals = A.dev(values, pdt)
    m = 1 if vals.dim() == 1 else vals.shape[1]
    vals = vals.reshape(-1, m).contiguous()
    out = A.empty((pts.shape[0], m), pdt)
    clamped = ctypes.c_int64(0)
    N.check(N.load_library().cs_bilinear(N.context(), N.prec_code(pdt), N.ptr(pts),
                                         pts.shape[0], N.ptr(vals), m,
                                         ctypes.byref(N.grid_struct(grid)), N.ptr(out),
                                         ctypes.byref(clamped)), "cs_bilinear")
    return out, clamped.value, host


def interpolate(grid: Grid, values, points):
    """Bilinear sample of one or more nodal arrays (coupling.py:265-292)."""
    squeeze_cols = (A.to_numpy(values).ndim == 1) if not A.is_tensor(values) else values.dim() == 1
    single = (not A.is_tensor(points)) and np.asarray(points).ndim == 1
    out, clamped, host = _bilinear(grid, values, points)
    if clamped:
        warnings.warn(f"{clamped} interpolation point(s) outside the grid hull were clamped",
                      stacklevel=2)
    res = A.back(out, host)
    if squeeze_cols:
        res = res[:, 0]
    if single:
        return res[0]
    return res


def field_at(field: Field, grid: Grid, points):
    """(concentration, gradient) at `points` (coupling.py:295-299)."""
    if A.is_tensor(field.c):
        import torch
        stacked = torch.cat([field.c.reshape(-1, 1), field.grad.reshape(-1, 2)], dim=1)
    else:
        stacked = np.column_stack([field.c, field.grad])
    out = interpolate(grid, stacked, points)
    if np.ndim(out) == 1:
        out = out[None, :]
    return out[:, 0], out[:, 1:3]


def refresh_particle_fields(pop: Population, field: Field, grid: Grid, chi: float) -> None:
    """Cached per-particle samples and chemotactic drift (coupling.py:302-325):
    Beta drift = chi * grad c, Alpha drift pinned to 0, local concentration
    for both."""
    conc, cl1, host = _bilinear(grid, field.c, pop.positions)
    drift, cl2, _ = _bilinear(grid, field.grad, pop.positions)
    if cl1 + cl2:
        warnings.warn(f"{cl1 + cl2} interpolation point(s) outside the grid hull were clamped",
                      stacklevel=2)
    drift = drift.to(dtype=__import__("torch").float64)
    if chi != 1.0:
        drift.mul_(float(chi))
    sp = A.dev(pop.species)
    drift[sp == int(Species.ALPHA)] = 0.0
    if host:
        pop.local_concentration[:] = conc[:, 0].cpu().numpy()
        pop.drift[...] = drift.cpu().numpy()
    else:
        pop.local_concentration.copy_(conc[:, 0])
        pop.drift.copy_(drift)
