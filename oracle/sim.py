"""Composed step driver of the oracle -- TEST INFRASTRUCTURE ONLY.

Runs the reference per-step pipeline, Realisation._step_inner
(engine.py:369-387), stage for stage on the oracle kernels:

  deposit -> step_field -> gradient        (if the field is active)
  refresh_particle_fields                  (if refresh is active)
  soft_forces -> em_step -> apply_boundaries

with the BASELINE extensions spelled out in SURVEY 8d: per-type radii via
the pair table, per-type chi, per-type secretion/consumption masks and an
fp32 storage mode (positions rounded to binary32 after every step, all
arithmetic in binary64 on the binary32 values).  With the extensions at
their reference defaults it is the reference pipeline.
"""

from __future__ import annotations

import time
import warnings

import numpy as np

from . import (apply_boundaries, bilinear, cic_deposit, em_step, field_rhs,
               gauss_deposit, gradient, soft_forces)
from .field import build_operators, quadrature_weights


class OracleStepError(RuntimeError):
    def __init__(self, status, i, ax, msg):
        super().__init__(msg)
        self.status, self.i, self.ax = status, i, ax


class OracleSim:
    def __init__(self, pos, types, *, lo, hi, periodic, dt, diffusion,
                 interaction="soft", eps_tab=None, cut_tab=None,
                 cell_cutoff=None, chi=(0.0, 1.0), chi_pinned=(True, False),
                 field=None, refresh_active=None, fp32=False, nthreads=1,
                 anchor_mode="round"):
        self.fp32 = bool(fp32)
        # fp32 anchors: "round" = rounded to binary32 after every step (the
        # direct engine's storage); "wraps" = start - k L kept exactly and
        # rounded only when read (the sorted engine's wrap counters)
        self.anchor_mode = anchor_mode
        self.pos = np.array(pos, dtype=np.float64).reshape(-1, 2)
        if self.fp32:
            self.pos = self.pos.astype(np.float32).astype(np.float64)
        self.n = self.pos.shape[0]
        self.types = np.asarray(types, dtype=np.uint8).copy()
        self.anchor = self.pos.copy()
        self.lo = np.asarray(lo, dtype=float)
        self.hi = np.asarray(hi, dtype=float)
        self.size = self.hi - self.lo
        self.periodic = tuple(bool(p) for p in periodic)
        self.dt = float(dt)
        self.dcoef = np.asarray(diffusion, dtype=float)[self.types]
        self.interaction = interaction
        self.eps_tab, self.cut_tab, self.cell_cutoff = eps_tab, cut_tab, cell_cutoff
        self.chi = tuple(float(c) for c in chi)
        self.chi_pinned = tuple(bool(p) for p in chi_pinned)
        self.nthreads = nthreads
        self.drift = np.zeros((self.n, 2))
        self.local_c = np.zeros(self.n)
        self.field = field
        self.step_index = 0
        self.timings = {}
        self.field_active = False
        if field is not None:
            nc = field["n_c"]
            per = field["boundary"] == "periodic"
            div = nc if per else nc - 1
            self.spacing = self.size / div
            self.grid_lo = self.lo.copy()
            self.nc = nc
            self.grid_periodic = per
            fp = field
            self.field_active = (fp["d_c"] > 0 or fp["k_alpha"] > 0
                                 or fp["k_beta"] > 0 or fp["gamma"] > 0)
            self.ops = build_operators(nc, self.spacing, per, fp["d_c"], self.dt,
                                       splu_max=fp.get("splu_max", 256))
            self.weights = quadrature_weights(nc, self.spacing, per)
            self.c = np.array(fp["c0"], dtype=float).reshape(nc * nc).copy()
            self.grad = gradient(self.c, nc, self.spacing, per)
            self.sec_mask = np.asarray(fp["secretes"], dtype=bool)[self.types]
            self.con_mask = np.asarray(fp["consumes"], dtype=bool)[self.types]
            if refresh_active is None:
                refresh_active = self.field_active or bool(np.any(self.c != 0.0))
        self.refresh_active = bool(refresh_active) if field is not None else False
        self.clamped = 0
        self.neg_mass_warnings = 0
        if self.refresh_active:
            self._refresh()

    # ---- stages -------------------------------------------------------
    def _deposit(self):
        f = self.field
        nc, per = self.nc, self.grid_periodic
        if f["kernel"] == "cic":
            ra = cic_deposit(self.pos, self.sec_mask, nc, self.grid_lo,
                             self.spacing, per)
            rb = cic_deposit(self.pos, self.con_mask, nc, self.grid_lo,
                             self.spacing, per)
        else:
            route_a = np.where(self.sec_mask, 0, 2).astype(np.uint8)
            route_b = np.where(self.con_mask, 1, 2).astype(np.uint8)
            ra, _ = gauss_deposit(self.pos, route_a, nc, self.grid_lo,
                                  self.spacing, per, f["h"], f["kernel_cutoff"])
            _, rb = gauss_deposit(self.pos, route_b, nc, self.grid_lo,
                                  self.spacing, per, f["h"], f["kernel_cutoff"])
        self.rho_a, self.rho_b = ra, rb

    def _step_field(self):
        f = self.field
        rhs = field_rhs(self.c, self.rho_a, self.rho_b, self.dt, f["k_alpha"],
                        f["k_beta"], f["gamma"])
        c_new = self.ops.solve(rhs)
        if not np.isfinite(c_new.sum()) and not np.all(np.isfinite(c_new)):
            raise FloatingPointError("field update produced non-finite values")
        if c_new.min() < 0.0:
            neg = c_new < 0.0
            if float(self.weights[neg] @ c_new[neg]) < -1e-12:
                self.neg_mass_warnings += 1
        self.c = c_new

    def _refresh(self):
        conc, cl1 = bilinear(self.pos, self.c, self.nc, self.grid_lo,
                             self.spacing, self.grid_periodic)
        drift, cl2 = bilinear(self.pos, self.grad, self.nc, self.grid_lo,
                              self.spacing, self.grid_periodic)
        self.clamped += cl1 + cl2
        self.local_c = conc
        for t in range(2):
            sel = self.types == t
            if self.chi_pinned[t]:
                drift[sel] = 0.0
            elif self.chi[t] != 1.0:
                drift[sel] *= self.chi[t]
        self.drift = drift

    def _tick(self, name, t0):
        t1 = time.perf_counter()
        self.timings[name] = self.timings.get(name, 0.0) + (t1 - t0)
        return t1

    def step(self, xi):
        t0 = time.perf_counter()
        if self.field_active:
            self._deposit()
            t0 = self._tick("deposit", t0)
            self._step_field()
            t0 = self._tick("pde", t0)
            self.grad = gradient(self.c, self.nc, self.spacing, self.grid_periodic)
            t0 = self._tick("gradient", t0)
        if self.refresh_active:
            self._refresh()
            t0 = self._tick("refresh", t0)
        if self.interaction == "soft":
            force = soft_forces(self.pos, self.lo, self.size, self.periodic,
                                self.eps_tab, self.cut_tab, self.cell_cutoff,
                                types=self.types, nthreads=self.nthreads)
        else:
            force = np.zeros((self.n, 2))
        t0 = self._tick("force", t0)
        nxt = em_step(self.pos, self.dcoef, self.drift, force,
                      np.asarray(xi, dtype=np.float64), self.dt,
                      nthreads=self.nthreads)
        t0 = self._tick("em", t0)
        st, i, ax = apply_boundaries(nxt, self.anchor, self.lo, self.hi,
                                     self.periodic)
        if st:
            raise OracleStepError(st, i, ax, f"step {self.step_index}: status {st} "
                                  f"particle {i} axis {ax}")
        if self.fp32:
            nxt = nxt.astype(np.float32).astype(np.float64)
            if self.anchor_mode == "round":
                self.anchor = self.anchor.astype(np.float32).astype(np.float64)
        self.pos = nxt
        self._tick("boundaries", t0)
        self.force = force
        self.step_index += 1
