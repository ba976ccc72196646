"""Simulation configuration and the device-resident per-step pipeline.

Mirror of chemosim/engine.py.  ``SimConfig`` keeps every reference field,
default, derived quantity, preset, validation message and warning
(engine.py:56-227); the extension fields below are additive and default to
the reference semantics.  ``Realisation`` keeps the reference seeding
(SeedSequence(seed_base + N * sample).spawn(3) -> init, motion, reactions;
engine.py:272-275) and step order (engine.py:369-387), but holds the state
on the GPU and advances it with the fused library pipeline (cs_sim_step):
one (N, 2) block of standard normals is drawn from the motion stream per
step on the host (the reference's RNG contract, motion.py:277) and uploaded;
everything else happens on the device.

Extensions (BASELINE configs 1-4):
  precision            "fp64" (reference) | "fp32" storage of positions,
                       anchors, Brownian increments and grid arrays; all
                       arithmetic stays binary64, force sums binary64
  radius_alpha/_beta   per-type radii -> pair table eps_ij = (r_i+r_j)/2,
                       cutoff cut_ij = soft_cutoff_factor * eps_ij
  chi_alpha            drift factor of Alpha (None: pinned to 0, reference)
  secrete_*/consume_*  which species deposit into rho_alpha (production)
                       and rho_beta (consumption); reference: Alpha
                       secretes, Beta consumes
  alpha_init           "normal" (reference) | "uniform"
  initial_positions    "default" | "clusters" (n_clusters centres, offset
                       N(0, cluster_sigma^2), wrapped; BASELINE config 4)
Reactions: the fixed scheduler runs on the device after
the boundaries of every step (one rng_react.random(N) block per step, the
reference's stream layout); the gillespie scheduler keeps the reference's
host event clock and runs the Beta -> Alpha trials on the device.  Both run
on the direct engine, as do the tamed integrator (motion.py:283-298) and the
hard-sphere sweep (motion.py:301-352; O(N^2) scan, N <= 65536).
"""

from __future__ import annotations

import ctypes
import math
import multiprocessing
import os
import warnings
from dataclasses import asdict, dataclass

import numpy as np

from . import _arrays as A
from . import _native as N
from .coupling import Kernel
from .field import Field, FieldParams, Grid, Operators
from .motion import MotionParams, SimulationError, raise_boundary_status
from .particles import Population, Species, clustered_positions, init_population
from .reactions import AlphaEventClock, ReactionParams, beta_step_reactions
from .spatial_index import Domain

EXPERIMENTS = ("fig1", "counts", "msd1", "msd2", "msd3", "custom")

_PRESETS: dict[str, dict] = {
    "fig1": {},
    "custom": {},
    "counts": dict(interaction="none", d_c=0.0, k_alpha=0.0, k_beta=0.0, dt=1e-4),
    "msd1": dict(n_alpha_0=100, n_beta_0=0, r_alpha=0.0),
    "msd2": dict(n_alpha_0=0, n_beta_0=100, r_alpha=0.0),
    "msd3": dict(n_alpha_0=50, n_beta_0=50, r_alpha=10.0),
}
for _name in ("msd1", "msd2", "msd3"):
    _PRESETS[_name].update(
        periodic=True, interaction="none", d_alpha=1.0, d_beta=1.0,
        r_beta=0.0, d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0,
        initial_field="linear_x", field_boundary="neumann",
        dt=0.01, t_final=20.0)


@dataclass
class SimConfig:
    experiment: str = "custom"
    n_alpha_0: int = 100
    n_beta_0: int = 100
    sigma: float = 0.1
    domain_size: float = 1.0
    periodic: bool = False
    d_alpha: float = 0.1
    d_beta: float = 1.0
    chi: float = 1.0
    epsilon: float = 0.02
    interaction: str = "soft"
    soft_cutoff_factor: float = 5.0
    integrator: str = "em"
    dt: float | None = None
    t_final: float = 0.05
    r_alpha: float = 10.0
    r_beta: float = 0.0
    scheduler: str = "fixed"
    d_c: float = 1.0
    k_alpha: float = 0.1
    k_beta: float = 0.03
    gamma: float = 0.0
    n_c: int = 52
    deposit: str = "gaussian"
    bandwidth: float | None = None
    kernel_cutoff_factor: float = 3.0
    initial_field: str = "zero"
    field_boundary: str = "auto"
    samples: int = 1
    seed_base: int = 0
    output_every: int = 20
    hist_bins: int = 26
    threads: int = 1
    # ---- extensions (defaults = reference semantics) ----
    precision: str = "fp64"
    radius_alpha: float | None = None
    radius_beta: float | None = None
    chi_alpha: float | None = None
    secrete_alpha: bool = True
    secrete_beta: bool = False
    consume_alpha: bool = False
    consume_beta: bool = True
    alpha_init: str = "normal"
    initial_positions: str = "default"
    n_clusters: int = 64
    cluster_sigma: float = 0.02
    engine: str = "auto"            # auto | direct | sorted (fp32 only)
    rng: str = "auto"               # auto | host | device: where the numpy streams are drawn
    xi_order: str = "id"            # id | slot: performance mode of the sorted engine
                                    # (increments by storage slot; same distribution, T4)

    def __post_init__(self):
        if self.experiment not in EXPERIMENTS:
            raise ValueError(f"unknown experiment {self.experiment!r}")
        if self.n_alpha_0 < 0 or self.n_beta_0 < 0:
            raise ValueError("initial counts must be non-negative")
        if self.n_alpha_0 + self.n_beta_0 < 1:
            raise ValueError("at least one particle is required")
        if not self.domain_size > 0:
            raise ValueError("domain_size must be positive")
        if self.dt is None:
            if not self.d_beta > 0:
                raise ValueError("dt must be given explicitly when d_beta = 0")
            self.dt = (0.23 * self.epsilon) ** 2 / (4.0 * self.d_beta)
        if not self.dt > 0:
            raise ValueError("dt must be positive")
        if self.t_final < 0:
            raise ValueError("t_final must be non-negative")
        if self.bandwidth is None:
            self.bandwidth = self.epsilon
        if self.field_boundary == "auto":
            self.field_boundary = "periodic" if self.periodic else "neumann"
        if self.field_boundary not in ("neumann", "periodic"):
            raise ValueError(f"unknown field_boundary {self.field_boundary!r}")
        if self.initial_field not in ("zero", "linear_x"):
            raise ValueError(f"unknown initial_field {self.initial_field!r}")
        if self.samples < 1:
            raise ValueError("samples must be at least 1")
        if self.seed_base < 0:
            raise ValueError("seed_base must be non-negative")
        if self.output_every < 1:
            raise ValueError("output_every must be at least 1")
        if self.hist_bins < 1:
            raise ValueError("hist_bins must be at least 1")
        if self.threads < 1:
            raise ValueError("threads must be at least 1")
        if not self.kernel_cutoff_factor > 0:
            raise ValueError("kernel_cutoff_factor must be positive")
        if not self.soft_cutoff_factor > 0:
            raise ValueError("soft_cutoff_factor must be positive")
        if self.precision not in ("fp64", "fp32"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.alpha_init not in ("normal", "uniform"):
            raise ValueError(f"unknown alpha_init {self.alpha_init!r}")
        if self.initial_positions not in ("default", "clusters"):
            raise ValueError(f"unknown initial_positions {self.initial_positions!r}")
        if self.engine not in ("auto", "direct", "sorted"):
            raise ValueError(f"unknown engine {self.engine!r}")
        if self.rng not in ("auto", "host", "device"):
            raise ValueError(f"unknown rng {self.rng!r}")
        if self.engine == "sorted" and self.precision != "fp32":
            raise ValueError("the sorted engine needs precision='fp32'")
        if self.xi_order not in ("id", "slot"):
            raise ValueError(f"unknown xi_order {self.xi_order!r}")
        if self.xi_order == "slot" and self.precision != "fp32":
            raise ValueError("xi_order='slot' is the sorted engine's mode (precision='fp32')")
        self.motion_params()
        self.field_params()
        self.kernel()
        self.grid()
        self._warn_explicit_sink()
        if self.scheduler == "fixed" and self.r_alpha * self.dt > 0.1:
            warnings.warn(
                f"per-step flip probability r_alpha dt = "
                f"{self.r_alpha * self.dt:.3g} is coarse; consider a smaller "
                "dt or the event-driven scheduler", stacklevel=2)

    def _warn_explicit_sink(self):
        if self.k_beta == 0.0 and self.gamma == 0.0:
            return
        n_total = self.n_alpha_0 + self.n_beta_0
        if self.deposit == "gaussian":
            rho_max = n_total / (2.0 * math.pi * self.bandwidth ** 2)
        else:
            dx = float(np.prod(self.grid().spacing))
            rho_max = n_total / dx
        if self.dt * (self.gamma + self.k_beta * rho_max) >= 1.0:
            warnings.warn(
                "explicit consumption/decay terms may destabilise the field "
                f"update: dt (gamma + k_beta rho_max) = "
                f"{self.dt * (self.gamma + self.k_beta * rho_max):.3g} >= 1",
                stacklevel=3)

    @classmethod
    def preset(cls, name: str, **overrides) -> "SimConfig":
        if name not in _PRESETS:
            raise ValueError(f"unknown experiment preset {name!r}")
        params = {**_PRESETS[name], **overrides}
        params.setdefault("experiment", name)
        return cls(**params)

    @property
    def n_total(self) -> int:
        return self.n_alpha_0 + self.n_beta_0

    @property
    def n_steps(self) -> int:
        return int(round(self.t_final / self.dt))

    def sample_seed(self, sample: int) -> int:
        return self.seed_base + self.n_total * sample

    def domain(self) -> Domain:
        return Domain.square(self.domain_size, periodic=self.periodic)

    def motion_params(self) -> MotionParams:
        cutoff = (self.soft_cutoff_factor * self.epsilon
                  if self.interaction == "soft" else 0.0)
        return MotionParams(d_alpha=self.d_alpha, d_beta=self.d_beta, chi=self.chi,
                            epsilon=self.epsilon, dt=self.dt, interaction=self.interaction,
                            cutoff=cutoff, integrator=self.integrator,
                            radius_alpha=self.radius_alpha, radius_beta=self.radius_beta,
                            cutoff_factor=self.soft_cutoff_factor)

    def reaction_params(self) -> ReactionParams:
        return ReactionParams(r_alpha=self.r_alpha, r_beta=self.r_beta,
                              scheduler=self.scheduler)

    def field_params(self) -> FieldParams:
        return FieldParams(d_c=self.d_c, k_alpha=self.k_alpha, k_beta=self.k_beta,
                           gamma=self.gamma)

    def kernel(self) -> Kernel:
        return Kernel(kind=self.deposit, h=self.bandwidth,
                      cutoff=self.kernel_cutoff_factor * self.bandwidth)

    def grid(self) -> Grid:
        return Grid.square(self.n_c, self.domain_size, self.field_boundary)

    def as_dict(self) -> dict:
        return asdict(self)

    def reference_dict(self) -> dict:
        """The reference's SimConfig fields (engine.py:56-108), plus the
        extension fields (below '# ---- extensions') whose values differ from
        their defaults: the manifest stays the reference's file contract for
        runs that use no extension."""
        d = asdict(self)
        defaults = SimConfig.__dataclass_fields__
        for name in EXTENSION_FIELDS:
            if d[name] == defaults[name].default:
                del d[name]
        return d


EXTENSION_FIELDS = ("precision", "radius_alpha", "radius_beta", "chi_alpha", "secrete_alpha",
                    "secrete_beta", "consume_alpha", "consume_beta", "alpha_init",
                    "initial_positions", "n_clusters", "cluster_sigma", "engine", "rng",
                    "xi_order")


def msd(pop: Population) -> float:
    """Mean over particles of squared displacement from the start anchor."""
    if len(pop) == 0:
        raise ValueError("msd of an empty population")
    d = A.to_numpy(pop.positions).astype(float) - A.to_numpy(pop.start_anchor).astype(float)
    return float((d * d).sum(axis=1).mean())


@dataclass
class Observables:
    times: np.ndarray
    counts: np.ndarray
    msd: np.ndarray
    snapshot_times: np.ndarray
    hist_alpha: np.ndarray
    hist_beta: np.ndarray
    field_c: np.ndarray


def sim_params_struct(*, n, prec, domain: Domain, motion: MotionParams, dt, field_active,
                      refresh_active, grid: Grid | None, fparams: FieldParams | None,
                      kernel: Kernel | None, secretes, consumes, chi, chi_pinned,
                      store_samples, store_next, engine: str = "auto",
                      reaction: ReactionParams | None = None,
                      xi_by_slot: bool = False) -> N.SimParams_t:
    p = N.SimParams_t()
    p.n = int(n)
    p.prec = prec
    p.n_types = 2
    p.domain = N.domain_struct(domain.lo, domain.hi, domain.periodic)
    p.interaction = {"soft": 1, "hard": 2}.get(motion.interaction, 0)
    p.hard_eps = float(motion.epsilon)
    p.diffusion[0], p.diffusion[1] = float(motion.d_alpha), float(motion.d_beta)
    p.xi_by_slot = 1 if xi_by_slot else 0
    p.integrator = 1 if getattr(motion, "integrator", "em") == "tamed" else 0
    if p.interaction:
        eps, cut, cell = motion.pair_table()
        p.pairs = N.pair_struct(eps, cut, cell)
    for t, d in enumerate((motion.d_alpha, motion.d_beta)):
        # numpy: np.sqrt(2.0 * D * dt) evaluates (2.0 * D) * dt
        p.amp[t] = math.sqrt((2.0 * float(d)) * float(dt))
    p.dt = float(dt)
    p.field_active = int(bool(field_active))
    p.refresh_active = int(bool(refresh_active))
    if grid is not None:
        p.grid = N.grid_struct(grid)
    if fparams is not None:
        p.d_c, p.k_alpha, p.k_beta, p.gamma = (float(fparams.d_c), float(fparams.k_alpha),
                                               float(fparams.k_beta), float(fparams.gamma))
    if kernel is not None:
        p.deposit_kind = N.CS_CIC if kernel.kind == "cic" else N.CS_GAUSSIAN
        p.kernel_h = float(kernel.h)
        p.kernel_cutoff = float(kernel.cutoff)
    for t in range(2):
        p.secretes[t] = int(bool(secretes[t]))
        p.consumes[t] = int(bool(consumes[t]))
        p.chi[t] = float(chi[t])
        p.chi_pinned[t] = int(bool(chi_pinned[t]))
    p.store_samples = int(bool(store_samples))
    p.store_next = int(bool(store_next))
    p.engine = {"auto": N.CS_ENGINE_AUTO, "direct": N.CS_ENGINE_DIRECT,
                "sorted": N.CS_ENGINE_SORTED, "cta": N.CS_ENGINE_CTA}[engine]
    if reaction is not None and reaction.scheduler == "fixed" and (
            reaction.r_alpha > 0 or reaction.r_beta > 0):
        p.react = 1
        p.react_p_ab = float(reaction.r_alpha * dt)  # reactions.py:61
        p.react_r_beta = float(reaction.r_beta)
    return p


class DeviceSim:
    """Owner of a cs_sim handle and the device state tensors it steps.

    State tensors (all on the current CUDA device):
      pos, next_pos, anchor : (N, 2) fp64 or fp32
      species               : (N,) uint8
      drift (N, 2), local_c (N,) : fp64
      c (n_c^2,), grad (n_c^2, 2), rho_a, rho_b (n_c^2,) : grid dtype
    """

    def __init__(self, params: N.SimParams_t, state: dict):
        self.params = params
        self.state = state
        self.n = int(params.n)
        self.prec = int(params.prec)
        h = N.C_p()
        self._ctx = N.context()
        # the stream this simulation was created on: every call rebinds the
        # (process-wide) library context to it, so a later N.context() under
        # another torch stream cannot move the simulation off it
        import torch
        self._stream = N.C_p(torch.cuda.current_stream().cuda_stream)
        N.check(N.load_library().cs_sim_create(self._ctx, ctypes.byref(params),
                                               ctypes.byref(h)), "cs_sim_create")
        self._h = h
        self._st = N.SimState_t()
        s = self._st
        for name in ("pos", "next_pos", "anchor", "drift", "local_c", "c", "grad", "rho_a",
                     "rho_b"):
            t = state.get(name)
            setattr(s, name, None if t is None else t.data_ptr())
        s.type = None if state.get("species") is None else state["species"].data_ptr()

    def step(self, xi, k: int, stride: int | None = None, u=None):
        """Enqueue k steps; xi is a device tensor holding k (N, 2) blocks
        (u: k (N,) f64 blocks of reaction uniforms when params.react)."""
        if stride is None:
            stride = 2 * self.n
        lib = self._bind()
        if u is None:
            N.check(lib.cs_sim_step(self._h, ctypes.byref(self._st), N.ptr(xi), int(stride),
                                    int(k)), "cs_sim_step")
        else:
            N.check(lib.cs_sim_step_react(self._h, ctypes.byref(self._st), N.ptr(xi),
                                          int(stride), N.ptr(u), self.n, int(k)),
                    "cs_sim_step_react")

    def _bind(self):
        lib = N.load_library()
        lib.cs_ctx_set_stream(self._ctx, self._stream)
        return lib

    def status(self) -> N.Status_t:
        st = N.Status_t()
        N.check(self._bind().cs_sim_status(self._h, ctypes.byref(st)), "cs_sim_status")
        return st

    @property
    def engine(self) -> str:
        e = int(N.load_library().cs_sim_engine(self._h))
        return {N.CS_ENGINE_SORTED: "sorted", N.CS_ENGINE_CTA: "cta"}.get(e, "direct")

    def import_state(self) -> None:
        """Reload the engine's internal state from the state tensors."""
        N.check(self._bind().cs_sim_import(self._h, ctypes.byref(self._st)), "cs_sim_import")

    def export_state(self) -> None:
        """Write the engine's internal state back into the state tensors
        (sorted engine; a no-op for the direct engine)."""
        N.check(self._bind().cs_sim_export(self._h, ctypes.byref(self._st)), "cs_sim_export")

    def launches(self) -> int:
        return int(N.load_library().cs_sim_launches(self._h))

    def set_profiling(self, on: bool) -> None:
        N.check(N.load_library().cs_sim_set_profiling(self._h, int(bool(on))),
                "cs_sim_set_profiling")

    def stage_times(self) -> dict:
        """Accumulated device ms per stage since profiling was enabled."""
        buf = (ctypes.c_double * len(N.STAGES))()
        N.check(N.load_library().cs_sim_stage_times(self._h, buf, len(N.STAGES)),
                "cs_sim_stage_times")
        return {k: float(buf[i]) for i, k in enumerate(N.STAGES)}

    def close(self):
        if getattr(self, "_h", None) is not None:
            N.load_library().cs_sim_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class Realisation:
    """One seeded run of the configured experiment, state on the GPU."""

    def __init__(self, config: SimConfig, sample: int):
        if sample < 0:
            raise ValueError("sample must be non-negative")
        torch = N.require_cuda()
        self.config = config
        self.sample = sample
        self.seed = config.sample_seed(sample)
        streams = np.random.SeedSequence(self.seed).spawn(3)
        self.rng_init = np.random.default_rng(streams[0])
        self.rng_motion = np.random.default_rng(streams[1])
        self.rng_react = np.random.default_rng(streams[2])
        self.domain = config.domain()
        self.motion = config.motion_params()
        self.field_params = config.field_params()
        self.kernel = config.kernel()
        self.grid = config.grid()
        self.dt = config.dt
        self.n_steps = config.n_steps
        self.step_index = 0
        self.reaction = config.reaction_params()
        self.reactions_active = self.reaction.r_alpha > 0 or self.reaction.r_beta > 0

        host = init_population(config.n_alpha_0, config.n_beta_0, config.sigma, self.domain,
                               self.rng_init, alpha_init=config.alpha_init)
        if config.initial_positions == "clusters":
            host.positions = clustered_positions(len(host), self.domain, self.rng_init,
                                                 config.n_clusters, config.cluster_sigma)
            host.next_positions = host.positions.copy()
            host.start_anchor = host.positions.copy()
        self.dtype = torch.float64 if config.precision == "fp64" else torch.float32
        dt_ = self.dtype
        dev = "cuda"
        self._state = dict(
            pos=torch.as_tensor(host.positions, device=dev).to(dt_).contiguous(),
            next_pos=torch.as_tensor(host.next_positions, device=dev).to(dt_).contiguous(),
            anchor=torch.as_tensor(host.start_anchor, device=dev).to(dt_).contiguous(),
            species=torch.as_tensor(host.species, device=dev).contiguous(),
            drift=torch.zeros((len(host), 2), dtype=torch.float64, device=dev),
            local_c=torch.zeros(len(host), dtype=torch.float64, device=dev),
        )
        self._ids = host.ids
        fp = self.field_params
        self.field_active = fp.d_c > 0 or fp.k_alpha > 0 or fp.k_beta > 0 or fp.gamma > 0
        m = self.grid.n_c ** 2
        c0 = (self.grid.node_positions()[:, 0].copy() if config.initial_field == "linear_x"
              else np.zeros(m))
        self._state.update(
            c=torch.as_tensor(c0, device=dev).to(dt_).contiguous(),
            grad=torch.zeros((m, 2), dtype=dt_, device=dev),
            rho_a=torch.zeros(m, dtype=dt_, device=dev),
            rho_b=torch.zeros(m, dtype=dt_, device=dev))
        self.ops = Operators(self.grid, fp, self.dt)
        from .field import gradient as _gradient
        from .coupling import refresh_particle_fields as _refresh
        f = Field(c=self._state["c"], grad=self._state["grad"], rho_alpha=self._state["rho_a"],
                  rho_beta=self._state["rho_b"])
        _gradient(f, self.ops)
        self.refresh_active = self.field_active or config.initial_field != "zero"
        chi_alpha = config.chi_alpha
        self._chi = (0.0 if chi_alpha is None else float(chi_alpha), float(self.motion.chi))
        self._chi_pinned = (chi_alpha is None, False)
        if self.refresh_active:
            self._initial_refresh()
        # fp64 keeps the reference's per-step drift / local_c / next_positions
        # stores; fp32 runs drop them so the sorted engine can be used
        self._stores = (config.precision == "fp64" or config.engine == "direct"
                        or self.reactions_active or config.interaction == "hard")
        params = sim_params_struct(
            n=len(host), prec=N.prec_code(dt_), domain=self.domain, motion=self.motion,
            dt=self.dt, field_active=self.field_active, refresh_active=self.refresh_active,
            grid=self.grid, fparams=fp, kernel=self.kernel,
            secretes=(config.secrete_alpha, config.secrete_beta),
            consumes=(config.consume_alpha, config.consume_beta), chi=self._chi,
            chi_pinned=self._chi_pinned, store_samples=self._stores,
            store_next=self._stores, engine=config.engine, reaction=self.reaction,
            xi_by_slot=config.xi_order == "slot")
        self._sim = DeviceSim(params, self._state)
        self._fixed = self.reactions_active and self.reaction.scheduler == "fixed"
        self.clock = None
        if self.reactions_active and self.reaction.scheduler == "gillespie":
            n_a = int(np.count_nonzero(host.species == Species.ALPHA))
            self.clock = AlphaEventClock(n_a, self.reaction.r_alpha, 0.0, self.rng_react)
        self._warned_react = 0
        self._warned_clamp = 0
        self._warned_neg = 0
        self._dead = False
        self._stale = False  # the sorted engine's records are newer than the state tensors
        self._init_recording()

    def _initial_refresh(self):
        from .coupling import _bilinear
        s = self._state
        conc, cl1, _ = _bilinear(self.grid, s["c"], s["pos"])
        drift, cl2, _ = _bilinear(self.grid, s["grad"], s["pos"])
        if cl1 + cl2:
            warnings.warn(f"{cl1 + cl2} interpolation point(s) outside the grid hull were "
                          "clamped", stacklevel=3)
        import torch
        drift = drift.to(torch.float64)
        sp = s["species"]
        for t in range(2):
            sel = sp == t
            if self._chi_pinned[t]:
                drift[sel] = 0.0
            elif self._chi[t] != 1.0:
                drift[sel] = drift[sel] * self._chi[t]
        s["local_c"].copy_(conc[:, 0].to(torch.float64))
        s["drift"].copy_(drift)

    # ---- state views ------------------------------------------------------
    def _sync(self) -> None:
        """Export the sorted engine's records into the (id-ordered) state
        tensors if steps ran since the last export (a no-op for the direct
        engine, whose state tensors are its working arrays)."""
        if self._stale:
            self._sim.export_state()
            self._stale = False

    @property
    def device_state(self) -> dict:
        self._sync()
        return self._state

    @property
    def pop(self) -> Population:
        """Host snapshot of the particle state (numpy, positions float64)."""
        self._sync()
        s = self._state
        return Population(ids=self._ids.copy(),
                          positions=s["pos"].double().cpu().numpy(),
                          next_positions=s["next_pos"].double().cpu().numpy(),
                          species=s["species"].cpu().numpy(),
                          drift=s["drift"].cpu().numpy(),
                          local_concentration=s["local_c"].cpu().numpy(),
                          start_anchor=s["anchor"].double().cpu().numpy())

    @property
    def field(self) -> Field:
        self._sync()
        s = self._state
        return Field(c=s["c"].double().cpu().numpy(), grad=s["grad"].double().cpu().numpy(),
                     rho_alpha=s["rho_a"].double().cpu().numpy(),
                     rho_beta=s["rho_b"].double().cpu().numpy())

    # ---- recording (engine.py:317-352; observables are host-side) ---------
    def _init_recording(self):
        n, every = self.n_steps, self.config.output_every
        flags = np.zeros(n + 1, dtype=bool)
        flags[0] = True
        flags[::every] = True
        flags[n] = True
        self._record_flags = flags
        self._snapshot_steps = [round(k * n / 3) for k in range(4)]
        self._times, self._counts, self._msd = [], [], []
        b = self.config.hist_bins
        self._hist_alpha = np.zeros((4, b, b))
        self._hist_beta = np.zeros((4, b, b))
        self._field_c = np.zeros((4, self.grid.n_c ** 2))
        self._observe(0)

    def _species_hist(self, sp) -> np.ndarray:
        """numpy.histogram2d of one species' positions over the domain
        (engine.py:317-352), normalised by the species count, transposed --
        binned on the device with numpy's edges (cs_hist2d)."""
        import torch
        s = self._state
        b = self.config.hist_bins
        if getattr(self, "_hist_edges", None) is None:
            ex = np.linspace(self.domain.lo[0], self.domain.hi[0], b + 1)
            ey = np.linspace(self.domain.lo[1], self.domain.hi[1], b + 1)
            self._hist_edges = (torch.as_tensor(ex, device="cuda"),
                                torch.as_tensor(ey, device="cuda"),
                                torch.empty((b, b), dtype=torch.int64, device="cuda"))
        ex, ey, cnt = self._hist_edges
        N.check(N.load_library().cs_hist2d(
            N.context(), N.prec_code(s["pos"].dtype), N.ptr(s["pos"]), N.ptr(s["species"]),
            len(self._ids), int(sp), N.ptr(ex), N.ptr(ey), b, 0, N.ptr(cnt)), "cs_hist2d")
        n_sp = int((s["species"] == int(sp)).sum())
        h = cnt.cpu().numpy().astype(np.float64)  # the b x b counts; numpy's division
        return h / n_sp if n_sp else h

    def _device_msd(self) -> float:
        """msd (engine.py:230-235) on the device in numpy's reduction order."""
        import torch
        s = self._state
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        N.check(N.load_library().cs_msd(N.context(), N.prec_code(s["pos"].dtype), N.ptr(s["pos"]),
                                        N.ptr(s["anchor"]), len(self._ids), N.ptr(out)),
                "cs_msd")
        return float(out.item())

    def _observe(self, step: int) -> None:
        snap = [k for k in range(4) if self._snapshot_steps[k] == step]
        if not (self._record_flags[step] or snap):
            return
        self._sync()
        s = self._state
        if self._record_flags[step]:
            n = len(self._ids)
            n_a = int((s["species"] == int(Species.ALPHA)).sum())
            self._times.append(step * self.dt)
            self._counts.append((n_a, n - n_a))
            self._msd.append(self._device_msd())
        for k in snap:
            self._hist_alpha[k] = self._species_hist(Species.ALPHA)
            self._hist_beta[k] = self._species_hist(Species.BETA)
            self._field_c[k] = s["c"].double().cpu().numpy()

    # ---- stepping ----------------------------------------------------------
    @property
    def time(self) -> float:
        return self.step_index * self.dt

    def _advance(self, xi_host: np.ndarray, u_host: np.ndarray | None = None) -> None:
        """Run xi_host.shape[0] steps on the device, then check the status."""
        import torch
        if self._dead:
            raise SimulationError("realisation already failed")
        k = xi_host.shape[0]
        xi = torch.as_tensor(xi_host, device="cuda").to(self.dtype).contiguous()
        u = None if u_host is None else torch.as_tensor(u_host, device="cuda").contiguous()
        self._sim.step(xi, k, u=u)
        self._stale = True  # exported lazily (state views, observables, errors)
        st = self._sim.status()
        self._report_warnings(st)
        if st.code != N.CS_OK:
            self._sync()
            self._dead = True
            self.step_index = int(st.step)
            try:
                if st.code == N.CS_FIELD_NONFINITE:
                    raise FloatingPointError("field update produced non-finite values")
                if st.code == N.CS_DEPOSIT_OVERFLOW:
                    raise SimulationError(
                        "too many particles in one cell for the sorted engine's int32 "
                        "fixed-point deposit; use engine='direct'")
                if st.code == N.CS_SORT_OVERFLOW:
                    raise SimulationError(
                        "local particle density outgrew the sorted engine's bucket regions; "
                        "use engine='direct'")
                src = "next_pos" if self._sim.engine == "direct" else "pos"
                raise_boundary_status(st.code, int(st.particle), int(st.axis),
                                      self._state[src].double().cpu().numpy())
            except (SimulationError, FloatingPointError, ValueError) as exc:
                raise SimulationError(f"step {st.step}: {exc}") from exc
        self.step_index += k

    def _react_host(self, now: float) -> None:
        """Gillespie scheduler after a device step (engine.py:389-400): the
        event clock on the host, the Beta -> Alpha trials on the device."""
        self._sync()
        view = _SpeciesView(self._state)
        self.clock.advance(view, now, self.rng_react)
        flipped = beta_step_reactions(view, self.reaction, self.dt, self.rng_react)
        if flipped:
            n_a = int((self._state["species"] == int(Species.ALPHA)).sum().item())
            self.clock.reschedule(n_a, now, self.rng_react)

    def _report_warnings(self, st) -> None:
        if st.react_high_count > self._warned_react:
            warnings.warn(f"flip probability {st.react_high_max:.3g} exceeded 1 and was "
                          "clamped; reduce dt", stacklevel=3)
            self._warned_react = st.react_high_count
        if st.clamped > self._warned_clamp:
            warnings.warn(f"{st.clamped - self._warned_clamp} interpolation point(s) outside "
                          "the grid hull were clamped", stacklevel=3)
            self._warned_clamp = st.clamped
        if st.neg_mass_steps > self._warned_neg:
            warnings.warn(f"concentration went negative (weighted mass {st.first_neg_mass:.3e})",
                          stacklevel=3)
            self._warned_neg = st.neg_mass_steps

    # draws of at least this many values go to the device (rng="auto")
    DEVICE_DRAW_MIN = 1 << 17

    def _draw(self, k: int):
        """The motion block (k, N, 2) and the fixed scheduler's uniforms
        (k, N) of the next k steps, numpy's values either way: drawn on the
        host, or on the device for large blocks (rng.draw: the same streams,
        bit for bit, the generators advanced identically)."""
        n = len(self._ids)
        dev = self.config.rng == "device" or (self.config.rng == "auto" and
                                              2 * k * n >= self.DEVICE_DRAW_MIN)
        if dev:
            from . import rng as R
            xi = R.draw(self.rng_motion, "normal", (k, n, 2), self.dtype)
            u = R.draw(self.rng_react, "uniform", (k, n)) if self._fixed else None
            return xi, u
        xi = self.rng_motion.standard_normal((k, n, 2))
        u = self.rng_react.random((k, n)) if self._fixed else None
        return xi, u

    def step(self) -> None:
        """Advance the whole system by dt (fixed sub-stage order)."""
        xi, u = self._draw(1)
        self._advance(xi, u)
        if self.clock is not None:
            # step s reacts at now = (s + 1) dt (engine.py:387), s + 1 = step_index
            self._react_host(self.step_index * self.dt)
        self._observe(self.step_index)

    def run(self, max_block_bytes: int = 1 << 28) -> Observables:
        n = len(self._ids)
        per_step = 16 * n
        cap = max(1, max_block_bytes // max(per_step, 1))
        if self.clock is not None:  # host event clock: one step at a time
            while self.step_index < self.n_steps:
                self.step()
            return self._observables()
        while self.step_index < self.n_steps:
            s = self.step_index
            nxt = s + 1
            while (nxt < self.n_steps and not self._record_flags[nxt]
                   and nxt not in self._snapshot_steps and nxt - s < cap):
                nxt += 1
            k = nxt - s
            # one (N, 2) block per step, drawn as one array: bit-identical
            # to k successive draws
            # one (N,) uniform block per step: rng.random((k, n)) is
            # bit-identical to k successive rng.random(n) draws
            xi, u = self._draw(k)
            self._advance(xi, u)
            self._observe(self.step_index)
        return self._observables()

    def _observables(self) -> Observables:
        return Observables(times=np.array(self._times),
                           counts=np.array(self._counts, dtype=np.int64),
                           msd=np.array(self._msd),
                           snapshot_times=np.array(self._snapshot_steps, dtype=float) * self.dt,
                           hist_alpha=self._hist_alpha, hist_beta=self._hist_beta,
                           field_c=self._field_c)


class _SpeciesView:
    """The population slice the reaction functions touch, over the
    Realisation's device tensors."""

    def __init__(self, state: dict):
        self.species = state["species"]
        self.local_concentration = state["local_c"]
        self.drift = state["drift"]

    def __len__(self) -> int:
        return int(self.species.shape[0])


def run_realisation(config: SimConfig, sample: int) -> Observables:
    try:
        return Realisation(config, sample).run()
    except SimulationError as exc:
        raise SimulationError(f"sample {sample}: {exc}") from exc


@dataclass
class EnsembleResult:
    times: np.ndarray
    counts_mean: np.ndarray
    counts_se: np.ndarray
    msd_mean: np.ndarray
    msd_se: np.ndarray
    snapshot_times: np.ndarray
    hist_alpha_mean: np.ndarray
    hist_alpha_se: np.ndarray
    hist_beta_mean: np.ndarray
    hist_beta_se: np.ndarray
    field_mean: np.ndarray
    field_se: np.ndarray
    samples: int
    seeds: list


def _mean_se(stack):
    mean = stack.mean(axis=0)
    s = stack.shape[0]
    if s < 2:
        return mean, np.zeros_like(mean)
    return mean, stack.std(axis=0, ddof=1) / math.sqrt(s)


def run_ensemble(config: SimConfig) -> EnsembleResult:
    """Run samples 0..S-1 and average their observables pointwise
    (engine.py:455-484).  Configurations the batched engine supports
    (ensemble.py: fp64, EM, neumann grid <= 64^2 or none, fixed-step
    reactions, <= 4096 particles) advance all samples together, one CTA per
    sample; the rest run sample by sample through ``Realisation``.  Results
    are reduced in sample order either way; ``threads`` sizes the host pool
    that draws the samples' random blocks."""
    from . import ensemble as E
    ens = None
    if E.supported(config) is None and os.environ.get("CS_ENSEMBLE") != "sequential":
        try:
            ens = E.Ensemble(config, threads=config.threads if config.threads > 1 else None)
        except N.NativeError as exc:
            # a realisation too large for one CTA's shared memory (cs_ens_create
            # reports it): run the samples one by one instead
            if "shared memory" not in str(exc):
                raise
    if ens is not None:
        try:
            all_obs = ens.run()
        finally:
            ens.close()
    else:
        all_obs = [run_realisation(config, s) for s in range(config.samples)]
    cm, cse = _mean_se(np.stack([o.counts for o in all_obs]).astype(float))
    mm, mse = _mean_se(np.stack([o.msd for o in all_obs]))
    ham, hase = _mean_se(np.stack([o.hist_alpha for o in all_obs]))
    hbm, hbse = _mean_se(np.stack([o.hist_beta for o in all_obs]))
    fm, fse = _mean_se(np.stack([o.field_c for o in all_obs]))
    return EnsembleResult(times=all_obs[0].times, counts_mean=cm, counts_se=cse, msd_mean=mm,
                          msd_se=mse, snapshot_times=all_obs[0].snapshot_times,
                          hist_alpha_mean=ham, hist_alpha_se=hase, hist_beta_mean=hbm,
                          hist_beta_se=hbse, field_mean=fm, field_se=fse,
                          samples=config.samples,
                          seeds=[config.sample_seed(s) for s in range(config.samples)])
