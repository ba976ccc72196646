"""Batched ensembles of small realisations.

``run_ensemble`` (engine.py:455-484) runs samples 0..S-1 of one
configuration and averages their observables.  The reference parallelises
only across processes; here every sample is one CTA of ``cs_ens_step``
(csrc/ensemble.cu), all S samples advance together, K steps per launch.

Seeding, initial states and random streams are per sample exactly as in
``Realisation`` (SeedSequence(seed_base + N * s).spawn(3) -> init, motion,
reactions; engine.py:272-275): each sample's increments are one
``standard_normal((K, N, 2))`` block of its own motion stream per launch
(bit-identical to K per-step draws), its reaction uniforms one
``random((K, N))`` block of its reaction stream.  By default the device
draws them (csrc/rng.cu: numpy's PCG64 and ziggurat restated, seeded from
the host generators' states, bit-identical draws); ``rng="host"`` draws
them with numpy on a thread pool while the device runs the previous block.  Observables are
recorded at the reference's steps from the device state and reduced in
sample order with the reference's mean / standard error.
"""

from __future__ import annotations

import ctypes
import os
import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _native as N
from .motion import SimulationError, raise_boundary_status
from .particles import Species, clustered_positions, init_population


def supported(config) -> str | None:
    """None if the batched engine can run `config`, else the reason."""
    if config.precision != "fp64":
        return "precision must be fp64"
    if config.interaction not in ("soft", "none"):
        return "hard-sphere motion"
    if config.engine == "sorted":
        return "engine='sorted' requested"
    r = config.reaction_params()
    if (r.r_alpha > 0 or r.r_beta > 0) and r.scheduler != "fixed":
        return "the gillespie scheduler keeps a host event clock per sample"
    fp = config.field_params()
    field = fp.d_c > 0 or fp.k_alpha > 0 or fp.k_beta > 0 or fp.gamma > 0
    grid_needed = field or config.initial_field != "zero"
    if grid_needed and (config.field_boundary == "periodic" or config.n_c > 64):
        return "the grid must be neumann with n_c <= 64"
    if config.n_total > 4096:
        return "more than 4096 particles per sample"
    return None


class Ensemble:
    """S samples of one SimConfig advanced together on the device."""

    def __init__(self, config, samples: int | None = None, threads: int | None = None,
                 rng: str = "device"):
        from .engine import sim_params_struct  # noqa: circular at import time
        torch = N.require_cuda()
        why = supported(config)
        if why:
            raise ValueError(f"the batched ensemble engine cannot run this config: {why}")
        self.config = config
        self.S = int(config.samples if samples is None else samples)
        if self.S < 1:
            raise ValueError("at least one sample is required")
        self.n = config.n_total
        self.dt = config.dt
        self.n_steps = config.n_steps
        self.domain = config.domain()
        self.grid = config.grid()
        self.motion = config.motion_params()
        self.reaction = config.reaction_params()
        fp = config.field_params()
        self.field_active = fp.d_c > 0 or fp.k_alpha > 0 or fp.k_beta > 0 or fp.gamma > 0
        self.refresh_active = self.field_active or config.initial_field != "zero"
        self.react = self.reaction.r_alpha > 0 or self.reaction.r_beta > 0
        self.threads = max(1, int(threads or min(32, os.cpu_count() or 1)))
        if rng not in ("device", "host"):
            raise ValueError(f"unknown rng {rng!r}")
        self.rng = rng
        n, S = self.n, self.S
        self.seeds = [config.sample_seed(s) for s in range(S)]
        self.rng_motion, self.rng_react = [], []
        pos = np.empty((S, n, 2))
        species = np.empty((S, n), np.uint8)
        for s, seed in enumerate(self.seeds):
            init, motion, react = (np.random.default_rng(q)
                                   for q in np.random.SeedSequence(seed).spawn(3))
            self.rng_motion.append(motion)
            self.rng_react.append(react)
            host = init_population(config.n_alpha_0, config.n_beta_0, config.sigma,
                                   self.domain, init, alpha_init=config.alpha_init)
            if config.initial_positions == "clusters":
                host.positions = clustered_positions(n, self.domain, init,
                                                     config.n_clusters, config.cluster_sigma)
            pos[s] = host.positions
            species[s] = host.species
        dev = "cuda"
        m = self.grid.n_c ** 2
        c0 = (self.grid.node_positions()[:, 0].copy() if config.initial_field == "linear_x"
              else np.zeros(m))
        self.state = dict(
            pos=torch.as_tensor(pos, device=dev).contiguous(),
            anchor=torch.as_tensor(pos, device=dev).contiguous(),
            drift=torch.zeros((S, n, 2), dtype=torch.float64, device=dev),
            local_c=torch.zeros((S, n), dtype=torch.float64, device=dev),
            species=torch.as_tensor(species, device=dev).contiguous(),
            c=torch.as_tensor(np.tile(c0, (S, 1)), device=dev).contiguous())
        chi_alpha = config.chi_alpha
        params = sim_params_struct(
            n=n, prec=N.CS_F64, domain=self.domain, motion=self.motion, dt=self.dt,
            field_active=self.field_active, refresh_active=self.refresh_active,
            grid=self.grid, fparams=fp, kernel=config.kernel(),
            secretes=(config.secrete_alpha, config.secrete_beta),
            consumes=(config.consume_alpha, config.consume_beta),
            chi=(0.0 if chi_alpha is None else float(chi_alpha), float(self.motion.chi)),
            chi_pinned=(chi_alpha is None, False), store_samples=True, store_next=False,
            engine="direct", reaction=self.reaction)
        lib = N.load_library()
        h = N.C_p()
        N.check(lib.cs_ens_create(N.context(), ctypes.byref(params), S, ctypes.byref(h)),
                "cs_ens_create")
        self._h = h
        st = N.EnsState_t()
        st.pos = self.state["pos"].data_ptr()
        st.anchor = self.state["anchor"].data_ptr()
        st.drift = self.state["drift"].data_ptr()
        st.local_c = self.state["local_c"].data_ptr()
        st.type = self.state["species"].data_ptr()
        st.c = self.state["c"].data_ptr()
        self._st = st
        self.step_index = 0
        self._pool = ThreadPoolExecutor(self.threads)
        if rng == "device":
            def words(gens):
                w = np.empty((S, 4), np.uint64)
                for s, g in enumerate(gens):
                    st = g.bit_generator.state["state"]
                    for q, v in enumerate((st["state"] >> 64, st["state"], st["inc"] >> 64,
                                           st["inc"])):
                        w[s, q] = v & 0xFFFFFFFFFFFFFFFF
                return torch.as_tensor(w.view(np.int64), device=dev)
            self._dev_motion = words(self.rng_motion)
            self._dev_react = words(self.rng_react)
        self._warned = dict(clamp=0, neg=0, react=0)

    # ---- random blocks ------------------------------------------------------
    def _draw(self, k: int):
        """(xi (k, S, n, 2), u (k, S, n) or None) from every sample's streams."""
        S, n = self.S, self.n
        xi = np.empty((k, S, n, 2))
        u = np.empty((k, S, n)) if self.react else None

        def fill(lo_hi):
            for s in range(*lo_hi):
                xi[:, s] = self.rng_motion[s].standard_normal((k, n, 2))
                if u is not None:
                    u[:, s] = self.rng_react[s].random((k, n))
        step = (S + self.threads - 1) // self.threads
        list(self._pool.map(fill, [(i, min(S, i + step)) for i in range(0, S, step)]))
        return xi, u

    def _draw_device(self, k: int, into=None):
        """The next k steps' increments (and uniforms) drawn on the device,
        on the current stream (into: preallocated (xi, u) buffers)."""
        import torch
        lib, ctx = N.load_library(), N.context()
        if into is None:
            xd = torch.empty((k, self.S, self.n, 2), dtype=torch.float64, device="cuda")
            ud = (torch.empty((k, self.S, self.n), dtype=torch.float64, device="cuda")
                  if self.react else None)
        else:
            xd = into[0][:k]
            ud = None if into[1] is None else into[1][:k]
        N.check(lib.cs_rng_fill(ctx, N.ptr(self._dev_motion), self.S, 0, int(k), 2 * self.n,
                                N.ptr(xd)), "cs_rng_fill")
        if ud is not None:
            N.check(lib.cs_rng_fill(ctx, N.ptr(self._dev_react), self.S, 1, int(k), self.n,
                                    N.ptr(ud)), "cs_rng_fill")
        return xd, ud

    def advance(self, k: int, drawn=None) -> None:
        """Run k steps of every sample (drawn: a pre-drawn (xi, u) block)."""
        import torch
        if self.rng == "device" and drawn is None:
            xd, ud = self._draw_device(k)
        elif isinstance(drawn, tuple) and torch.is_tensor(drawn[0]):  # device blocks
            xd, ud = drawn
        else:
            xi, u = drawn if drawn is not None else self._draw(k)
            xd = torch.as_tensor(xi, device="cuda")
            ud = None if u is None else torch.as_tensor(u, device="cuda")
        N.context()  # bind the library to the current stream
        N.check(N.load_library().cs_ens_step(self._h, ctypes.byref(self._st), N.ptr(xd),
                                             N.ptr(ud), int(k)), "cs_ens_step")
        self.step_index += k
        self._xd, self._ud = xd, ud  # keep alive until the next sync

    def observe_device(self):
        """(Alpha count (S,) int64, msd (S,) f64) of every sample now."""
        import torch
        if getattr(self, "_obs", None) is None:
            self._obs = (torch.empty(self.S, dtype=torch.int64, device="cuda"),
                         torch.empty(self.S, dtype=torch.float64, device="cuda"))
        na, msd = self._obs
        N.context()  # on the current stream: ordered after the step kernels queued on it
        N.check(N.load_library().cs_ens_observe(self._h, ctypes.byref(self._st), N.ptr(na),
                                                N.ptr(msd)), "cs_ens_observe")
        return na.cpu().numpy(), msd.cpu().numpy()

    def status(self):
        out = (N.Status_t * self.S)()
        N.context()  # the status copy follows the step kernels on the current stream
        N.check(N.load_library().cs_ens_status(self._h, out), "cs_ens_status")
        return out

    def check(self) -> None:
        """Raise the reference's error for the lowest failing sample; warn."""
        st = self.status()
        arr = np.ctypeslib.as_array(st)
        failing = np.flatnonzero(arr["code"] != N.CS_OK)
        for s in failing[:1]:
            x = st[int(s)]
            try:
                try:
                    if x.code == N.CS_FIELD_NONFINITE:
                        raise FloatingPointError("field update produced non-finite values")
                    pos = self.state["pos"][s].cpu().numpy()
                    raise_boundary_status(x.code, int(x.particle), int(x.axis), pos)
                except (SimulationError, FloatingPointError, ValueError) as exc:
                    raise SimulationError(f"step {x.step}: {exc}") from exc
            except SimulationError as exc:
                raise SimulationError(f"sample {s}: {exc}") from exc
        clamp = int(arr["clamped"].sum())
        neg = int(arr["neg_mass_steps"].sum())
        react = int(arr["react_high_count"].sum())
        if clamp > self._warned["clamp"]:
            warnings.warn(f"{clamp - self._warned['clamp']} interpolation point(s) outside the "
                          "grid hull were clamped", stacklevel=3)
        if neg > self._warned["neg"]:
            first = float(arr["first_neg_mass"][np.flatnonzero(arr["neg_mass_steps"])[0]])
            warnings.warn(f"concentration went negative (weighted mass {first:.3e})",
                          stacklevel=3)
        if react > self._warned["react"]:
            high = float(arr["react_high_max"].max())
            warnings.warn(f"flip probability {high:.3g} exceeded 1 and was clamped; reduce dt",
                          stacklevel=3)
        self._warned = dict(clamp=clamp, neg=neg, react=react)

    def close(self):
        if getattr(self, "_h", None) is not None:
            N.load_library().cs_ens_destroy(self._h)
            self._h = None
        if getattr(self, "_pool", None) is not None:
            self._pool.shutdown(wait=False)
            self._pool = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # ---- the reference's recording schedule ------------------------------
    def run(self):
        """All samples to T_f with the reference's observables
        (engine.py:317-352, 402-413) -> list of per-sample Observables."""
        from .engine import Observables
        cfg = self.config
        n_steps, every = self.n_steps, cfg.output_every
        flags = np.zeros(n_steps + 1, dtype=bool)
        flags[0] = True
        flags[::every] = True
        flags[n_steps] = True
        snaps = [round(k * n_steps / 3) for k in range(4)]
        S, b = self.S, cfg.hist_bins
        times, counts, msds = [], [], []
        hist_a = np.zeros((S, 4, b, b))
        hist_b = np.zeros((S, 4, b, b))
        field_c = np.zeros((S, 4, self.grid.n_c ** 2))
        lo, hi = self.domain.lo, self.domain.hi

        import torch
        edges_d = [torch.as_tensor(np.linspace(lo[a], hi[a], b + 1), device="cuda")
                   for a in range(2)]
        hcnt = torch.empty((S, b, b), dtype=torch.int64, device="cuda")

        def observe(step):
            snap = [k for k in range(4) if snaps[k] == step]
            if not (flags[step] or snap):
                return
            if flags[step]:
                # counts and msd on the device (cs_ens_observe: numpy's
                # pairwise mean, bit-identical to engine.py:230-235)
                times.append(step * self.dt)
                n_a, msd = self.observe_device()
                counts.append(np.stack([n_a, self.n - n_a], axis=1))
                msds.append(msd)
            if snap:
                c = self.state["c"].cpu().numpy() if self.field_active or \
                    self.refresh_active else np.zeros((S, self.grid.n_c ** 2))
                species = self.state["species"]
                for sp, out in ((Species.ALPHA, hist_a), (Species.BETA, hist_b)):
                    # numpy.histogram2d of every sample on the device
                    # (cs_hist2d, per_sample = n); numpy's normalisation
                    N.check(N.load_library().cs_hist2d(
                        N.context(), N.CS_F64, N.ptr(self.state["pos"]), N.ptr(species),
                        S * self.n, int(sp), N.ptr(edges_d[0]), N.ptr(edges_d[1]), b, self.n,
                        N.ptr(hcnt)), "cs_hist2d")
                    h = hcnt.cpu().numpy().astype(np.float64)
                    cnt = (species == int(sp)).reshape(S, -1).sum(dim=1).cpu().numpy()
                    nz = cnt > 0
                    h[nz] = h[nz] / cnt[nz][:, None, None]
                    for k in snap:
                        out[:, k] = h
                for k in snap:
                    field_c[:, k] = c

        observe(0)
        # block boundaries at the recording / snapshot steps
        stops = sorted({s for s in range(1, n_steps + 1) if flags[s]} |
                       {s for s in snaps if s > 0})
        prev, pending = 0, None
        blocks = []
        for stop in stops:
            blocks.append(stop - prev)
            prev = stop
        if self.rng == "device":
            # the next block's random numbers are drawn on a side stream while
            # the ensemble kernel runs the current one (two buffer sets)
            import torch
            side = torch.cuda.Stream()
            main = torch.cuda.current_stream()
            kmax = max(blocks) if blocks else 1
            bufs = [(torch.empty((kmax, S, self.n, 2), dtype=torch.float64, device="cuda"),
                     torch.empty((kmax, S, self.n), dtype=torch.float64, device="cuda")
                     if self.react else None) for _ in range(2)]
            ready = [torch.cuda.Event() for _ in range(2)]
            done = [torch.cuda.Event() for _ in range(2)]

            def fill(i, k):
                with torch.cuda.stream(side):
                    if done_used[i]:
                        side.wait_event(done[i])
                    drawn_i = self._draw_device(k, into=bufs[i])
                    ready[i].record(side)
                N.context()  # rebind the library to the main stream
                return drawn_i
            done_used = [False, False]
            side.wait_stream(main)
            pend = fill(0, blocks[0]) if blocks else None
        for bi, k in enumerate(blocks):
            if self.rng == "device":
                i = bi % 2
                main.wait_event(ready[i])
                self.advance(k, pend)
                done[i].record(main)
                done_used[i] = True
                if bi + 1 < len(blocks):
                    pend = fill(1 - i, blocks[bi + 1])
            else:
                drawn = pending.result() if pending is not None else self._draw(k)
                self.advance(k, drawn)
                # draw the next block on the host while the device runs this one
                pending = (self._pool_submit_draw(blocks[bi + 1]) if bi + 1 < len(blocks)
                           else None)
            self.check()
            observe(self.step_index)
        cnt = np.stack(counts, axis=1)        # (S, T, 2)
        msd = np.stack(msds, axis=1)          # (S, T)
        snap_t = np.array(snaps, dtype=float) * self.dt
        return [Observables(times=np.array(times), counts=cnt[s].astype(np.int64),
                            msd=msd[s], snapshot_times=snap_t, hist_alpha=hist_a[s],
                            hist_beta=hist_b[s], field_c=field_c[s]) for s in range(S)]

    def _pool_submit_draw(self, k):
        import concurrent.futures as cf
        ex = cf.ThreadPoolExecutor(1)
        f = ex.submit(self._draw, k)
        ex.shutdown(wait=False)
        return f
