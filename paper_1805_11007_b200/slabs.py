"""y-slab domain decomposition of one system over several GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink).  Rank r owns
the whole cell rows [b_r, b_{r+1}) of the reference's cell grid
(motion.py:171-174: n = int(L / cutoff), eff = L / n), count-balanced at the
start (prefix sum of the per-row particle counts: equal-width slabs cap the
efficiency at 53-83 % for clustered inputs), and an even share of
the field's grid rows.  Each rank runs the SORTED engine in slab mode
(csrc/fast.cu, cs_slab_*) on its particles plus copies of its neighbours'
boundary cell rows (ghosts).  Per step, in the reference stage order
(engine.py:369-387):

  field      deposit window rows (own particles, int32 fixed point) added
             into their owners' rows; the implicit spectral solve as own-row
             passes and own-column passes around two all-to-all transposes
             of the half spectrum; c rows for the gradient window fetched
             from their owners; gradient of the window rows
  particles  pair forces and the update over the owned slots (the update
             kernel routes records whose new row another rank owns --
             migrants -- and copies of records landing in a boundary row --
             ghosts -- into an outbox); one all-to-all of the outbox; the
             received records claimed; bucket sort; the next deposit

Every pass is the single-domain engine's on the same records, rows and
columns, so the decomposed run is the single-domain run bit for bit
(tests/test_gpu_slab_engine.py, ranks emulated in one process).  The grid
exchanges have sizes fixed by the layout.  The particle all-to-all either
sends its per-peer counts first and reads them back (NcclTransport: one host
synchronisation per step) or, once a few such steps have sized it, moves
fixed per-destination segments and their device-side counts
(PackedNcclTransport: no host synchronisation in the step).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


# ----------------------------------------------------------------------------
# layout
# ----------------------------------------------------------------------------
@dataclass
class SlabLayout:
    n_rows: int                 # cell rows of the global cell grid
    bounds: np.ndarray          # (world + 1,) cell-row boundaries

    @property
    def world(self) -> int:
        return len(self.bounds) - 1

    @classmethod
    def even(cls, n_rows: int, world: int) -> "SlabLayout":
        b = np.round(np.linspace(0, n_rows, world + 1)).astype(np.int64)
        return cls(n_rows, b)

    @classmethod
    def balanced(cls, row_counts: np.ndarray, world: int, min_rows: int = 2) -> "SlabLayout":
        """Split so every slab holds ~N/world particles (>= min_rows rows)."""
        n_rows = len(row_counts)
        if world * min_rows > n_rows:
            raise ValueError("too many slabs for the cell grid")
        c = np.concatenate([[0], np.cumsum(row_counts, dtype=np.int64)])
        total = c[-1]
        b = [0]
        for r in range(1, world):
            target = total * r / world
            k = int(np.searchsorted(c, target))
            k = max(k, b[-1] + min_rows)
            k = min(k, n_rows - (world - r) * min_rows)
            b.append(k)
        b.append(n_rows)
        return cls(n_rows, np.asarray(b, dtype=np.int64))

    def owner_of_row(self, rows):
        """Rank owning each cell row (numpy or torch input)."""
        if isinstance(rows, torch.Tensor):
            bt = torch.as_tensor(self.bounds[1:-1], device=rows.device)
            return torch.bucketize(rows, bt, right=True)
        return np.searchsorted(self.bounds[1:-1], rows, side="right")


@dataclass
class CellGeometry:
    """The reference's binning (motion.py:171-190) on one axis (y)."""
    lo: float
    size: float
    n: int
    eff: float

    @classmethod
    def make(cls, lo: float, hi: float, cell_cutoff: float) -> "CellGeometry":
        size = hi - lo
        n = max(1, int(size / cell_cutoff))
        return cls(lo, size, n, size / n)

    def row_of(self, y):
        if isinstance(y, torch.Tensor):
            f = torch.floor((y.double() - self.lo) / self.eff)
            return f.clamp(0, self.n - 1).long()
        f = np.floor((np.asarray(y, dtype=float) - self.lo) / self.eff)
        return np.clip(f, 0, self.n - 1).astype(np.int64)


# ============================================================================
# The device slab engine: each rank's share is the SORTED engine in slab mode
# (csrc/fast.cu, cs_slab_*), records cross ranks as 16-byte device rows
# ============================================================================
class LoopbackHub:
    """All ranks of one process on one device (tests): the exchange hands
    every rank the records the others addressed to it."""

    def __init__(self, world: int):
        self.world = world

    def exchange_all(self, outs):
        """outs[r] = (recs (M, 4) int32, dest (M,) int32) of rank r ->
        received[q] = the records addressed to q, from every rank."""
        got = [[] for _ in range(self.world)]
        for recs, dest in outs:
            if recs.shape[0] == 0:
                continue
            d = (dest & 0x3FFFFFFF).long()
            for q in range(self.world):
                sel = d == q
                if bool(sel.any()):
                    got[q].append(recs[sel])
        return [torch.cat(g) if g else None for g in got]


class NcclTransport:
    """One rank per GPU: the outbox routed by an all-to-all over NCCL
    (NVLink).  The per-destination counts travel first (one P-int
    all-to-all, read back to size the payload -- the only host sync of a
    step), then the 16-byte records."""

    def __init__(self, world: int, group=None):
        self.world, self.group = world, group

    def exchange(self, recs, dest):
        W = self.world
        d = (dest & 0x3FFFFFFF).long()
        order = torch.argsort(d, stable=True)
        sc_t = torch.bincount(d, minlength=W).to(torch.int64)
        rc_t = torch.empty_like(sc_t)
        dist.all_to_all_single(rc_t, sc_t, group=self.group)
        both = torch.stack([sc_t, rc_t]).cpu()
        sc, rc = both[0].tolist(), both[1].tolist()
        out = torch.empty((sum(rc), 4), dtype=torch.int32, device=recs.device)
        send = recs[order].contiguous() if recs.shape[0] else recs
        dist.all_to_all_single(out.view(-1), send.view(-1), [4 * c for c in rc],
                               [4 * c for c in sc], group=self.group)
        return out


class PackedNcclTransport(NcclTransport):
    """The records' exchange without a host round trip: every rank keeps
    `seg` outbox slots and a device counter per destination
    (SlabEngine.set_exchange_cap), so the counts and the records travel as two
    equal-split all-to-alls straight from / into device buffers.  `seg` comes
    from calibrate(): a few steps through the counted exchange of
    NcclTransport, whose per-destination maxima -- reduced over the ranks,
    times a safety factor -- bound a step's traffic; a step that exceeds it
    stops the run (CS_SORT_OVERFLOW), it is never silently dropped."""

    def __init__(self, world: int, group=None, factor: float = 4.0, floor: int = 4096):
        super().__init__(world, group)
        self.factor, self.floor = factor, floor
        self.peak = 0      # largest per-destination count seen by the counted exchange
        self.seg = 0       # slots per destination of the packed exchange (0: not calibrated)
        self.pending = False  # after a re-balance: one counted step, then calibrate() again
        self._inbox = self._in_counts = None

    def exchange(self, recs, dest):
        if recs.shape[0]:
            d = (dest & 0x3FFFFFFF).long()
            self.peak = max(self.peak, int(torch.bincount(d, minlength=self.world).max()))
        return super().exchange(recs, dest)

    def calibrate(self) -> int:
        """Agree on `seg` over the ranks (after some counted exchanges)."""
        t = torch.tensor([self.peak], dtype=torch.int64,
                         device=torch.device("cuda", torch.cuda.current_device()))
        if self.world > 1 or dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        seg = max(self.floor, int(self.factor * int(t.item())))
        self.seg = max(self.seg, (seg + 255) // 256 * 256)
        return self.seg

    def exchange_packed(self, out_recs, out_counts):
        """out_recs (W, seg, 4) int32, out_counts (W,) int32 (device views of
        the engine's outbox) -> (inbox (W, seg, 4), in_counts (W,))."""
        if self._inbox is None or self._inbox.shape != out_recs.shape:
            self._inbox = torch.empty_like(out_recs)
            self._in_counts = torch.empty_like(out_counts)
        dist.all_to_all_single(self._in_counts, out_counts, group=self.group)
        dist.all_to_all_single(self._inbox.view(-1), out_recs.view(-1), group=self.group)
        return self._inbox, self._in_counts


class PackedLoopbackHub(LoopbackHub):
    """The packed exchange between the ranks of one process (tests)."""

    def exchange_all_packed(self, outs):
        """outs[r] = (recs (W, seg, 4), counts (W,)) of rank r ->
        received[q] = (inbox (W, seg, 4), in_counts (W,)): segment s from rank s."""
        W = self.world
        got = []
        for q in range(W):
            inbox = torch.stack([outs[s][0][q] for s in range(W)])
            counts = torch.stack([outs[s][1][q] for s in range(W)])
            got.append((inbox, counts))
        return got


class SlabEngine:
    """One rank's share of a y-slab decomposed system on its GPU: the sorted
    engine (binary32 records, reference summation order) over the owned cell
    rows plus ghost copies of the neighbours' boundary rows.  Bit-identical to
    the single-domain engine: every owned particle sees its whole reference
    ring (ghost rows), rows stay in ascending id inside a cell, and the cell
    geometry is the global one.

    params: cs_sim_params of the WHOLE system (n = N, engine SORTED,
    field off); state: the caller's global id-ordered arrays (pos, anchor,
    species), read at import and written back (own particles) by export."""

    def __init__(self, params, state: dict, bounds, rank: int, world: int,
                 field_plan: "FieldPlan | None" = None):
        from . import _native as N
        from .engine import DeviceSim
        self.N = N
        self.rank, self.world = rank, world
        self.bounds = np.asarray(bounds, dtype=np.int32)
        self.sim = DeviceSim(params, state)
        if self.sim.engine != "sorted":
            raise ValueError("slab mode needs the sorted engine (binary32, engine='sorted')")
        lib = self.sim._bind()
        b = (N.C_i32 * len(self.bounds))(*[int(v) for v in self.bounds])
        N.check(lib.cs_slab_config(self.sim._h, b, world, rank), "cs_slab_config")
        e_, c_, cell = _pair_cell(params)
        self.n1 = max(1, int((params.domain.hi[1] - params.domain.lo[1]) / cell))
        self.field = None
        if field_plan is not None:
            r = rank
            j0, k = field_plan.dep[r]
            gj0, gk = field_plan.grad[r]
            g0 = int(field_plan.g0[r])
            N.check(lib.cs_slab_field_config(self.sim._h, g0, g0 + field_plan.rp, j0, k, gj0,
                                             gk), "cs_slab_field_config")
        N.check(lib.cs_slab_import(self.sim._h, ctypes_byref(self.sim._st)), "cs_slab_import")
        if field_plan is not None:
            self.field = SlabField(self, field_plan)

    # ---- phases ------------------------------------------------------------
    def local(self, xi):
        """Forces + update of the owned particles (xi: the step's global
        (N, 2) increments by id, on this device)."""
        N = self.N
        N.check(self.sim._bind().cs_slab_step_local(self.sim._h, ctypes_byref(self.sim._st),
                                                   N.ptr(xi)), "cs_slab_step_local")

    def forces(self, xi):
        """First half of local(): the outbox reset and the pair forces."""
        N = self.N
        N.check(self.sim._bind().cs_slab_step_part(self.sim._h, ctypes_byref(self.sim._st),
                                                  N.ptr(xi), 1), "cs_slab_step_part")

    def update(self, xi):
        """Second half of local(): the update (needs the field step's gradient)."""
        N = self.N
        N.check(self.sim._bind().cs_slab_step_part(self.sim._h, ctypes_byref(self.sim._st),
                                                  N.ptr(xi), 2), "cs_slab_step_part")

    def outbox(self):
        """(records (M, 4) int32, dest (M,) int32) views of the outbox."""
        import ctypes
        N = self.N
        rp, dp, cnt = N.C_p(), N.C_p(), N.C_i64()
        N.check(self.sim._bind().cs_slab_outbox(self.sim._h, ctypes.byref(rp), ctypes.byref(dp),
                                                ctypes.byref(cnt)), "cs_slab_outbox")
        m = int(cnt.value)
        dev = self.sim.state["pos"].device
        if m == 0:
            z = torch.empty((0, 4), dtype=torch.int32, device=dev)
            return z, torch.empty(0, dtype=torch.int32, device=dev)
        recs = _device_view(rp.value, (m, 4), torch.int32, dev)
        dest = _device_view(dp.value, (m,), torch.int32, dev)
        return recs, dest

    def set_exchange_cap(self, seg: int):
        """Packed exchange with `seg` outbox slots per destination rank
        (0: the tagged outbox of outbox() / claim())."""
        self.N.check(self.sim._bind().cs_slab_exchange_cap(self.sim._h, int(seg)),
                     "cs_slab_exchange_cap")
        self._seg = int(seg)

    def outbox_packed(self):
        """(records (W, seg, 4) int32, counts (W,) int32): device views, no
        host round trip."""
        import ctypes
        N = self.N
        rp, cp, seg = N.C_p(), N.C_p(), N.C_i64()
        N.check(self.sim._bind().cs_slab_outbox_packed(self.sim._h, ctypes.byref(rp),
                                                      ctypes.byref(cp), ctypes.byref(seg)),
                "cs_slab_outbox_packed")
        dev = self.sim.state["pos"].device
        W, sg = self.world, int(seg.value)
        return (_device_view(rp.value, (W, sg, 4), torch.int32, dev),
                _device_view(cp.value, (W,), torch.int32, dev))

    def claim_packed(self, inbox, in_counts):
        N = self.N
        N.check(self.sim._bind().cs_slab_claim_packed(self.sim._h, N.ptr(inbox),
                                                     N.ptr(in_counts), int(inbox.shape[1])),
                "cs_slab_claim_packed")

    def claim(self, recs):
        if recs is None or recs.shape[0] == 0:
            return
        N = self.N
        recs = recs.contiguous()
        N.check(self.sim._bind().cs_slab_claim(self.sim._h, N.ptr(recs), int(recs.shape[0])),
                "cs_slab_claim")
        self._keep = recs  # alive until the claim kernel has run (stream order)

    def finish(self):
        self.N.check(self.sim._bind().cs_slab_finish(self.sim._h), "cs_slab_finish")

    # ---- one step over NCCL (one rank per process) -------------------------
    def step(self, xi, transport: NcclTransport, overlap: bool = True):
        """One step over NCCL.  overlap: the distributed field step (its
        exchanges and transposes included) runs on a side stream beside the
        pair forces, which do not read the field; the update joins them."""
        # (the step after a re-balance goes through the counted exchange and
        # re-sizes the packed one: the boundary rows, hence the ghost traffic,
        # have moved)
        recal = getattr(transport, "pending", False) and getattr(transport, "seg", 0) > 0
        seg = 0 if recal else getattr(transport, "seg", 0)
        if seg != getattr(self, "_seg", 0):
            self.set_exchange_cap(seg)
        if self.field is not None:
            if not hasattr(self, "_nf"):
                self._nf = NcclField(self.field, transport.group)
            if overlap:
                main = torch.cuda.current_stream()
                if not hasattr(self, "_side"):
                    self._side = torch.cuda.Stream(device=main.device)
                self._side.wait_stream(main)  # the deposit of the last finish()
                with torch.cuda.stream(self._side):
                    self._nf.step()
                self.forces(xi)
                main.wait_stream(self._side)
                self.update(xi)
            else:
                self._nf.step()
                self.local(xi)
        else:
            self.local(xi)
        if seg:  # packed: counts and records stay on the device
            self.claim_packed(*transport.exchange_packed(*self.outbox_packed()))
        else:
            recs, dest = self.outbox()
            self.claim(transport.exchange(recs, dest))
        self.finish()
        if recal:
            transport.pending = False
            transport.calibrate()

    def status(self):
        return self.sim.status()

    # ---- re-balancing (every M steps) --------------------------------------
    def row_counts(self):
        """Per-cell-row counts of the owned particles (device int32)."""
        h = torch.empty(int(self.n1), dtype=torch.int32, device=self.sim.state["pos"].device)
        self.N.check(self.sim._bind().cs_slab_row_counts(self.sim._h, self.N.ptr(h)),
                     "cs_slab_row_counts")
        return h

    def rebalance_begin(self, bounds, field_plan: "FieldPlan | None" = None):
        """Adopt new row bounds: the owned records are routed under them
        into the outbox (or claimed); the caller exchanges and claims, then
        calls rebalance_end()."""
        N = self.N
        self.bounds = np.asarray(bounds, dtype=np.int32)
        b = (N.C_i32 * len(self.bounds))(*[int(v) for v in self.bounds])
        lib = self.sim._bind()
        N.check(lib.cs_slab_rebalance(self.sim._h, b), "cs_slab_rebalance")
        if field_plan is not None:
            r = self.rank
            j0, k = field_plan.dep[r]
            gj0, gk = field_plan.grad[r]
            g0 = int(field_plan.g0[r])
            N.check(lib.cs_slab_field_config(self.sim._h, g0, g0 + field_plan.rp, j0, k, gj0,
                                             gk), "cs_slab_field_config")
            self.field = SlabField(self, field_plan)
            if hasattr(self, "_nf"):
                del self._nf

    def rebalance_end(self):
        self.N.check(self.sim._bind().cs_slab_finish_rebalance(self.sim._h),
                     "cs_slab_finish_rebalance")

    def rebalance(self, transport: NcclTransport, n1: int, n_c: int | None = None):
        """One rank's re-balancing over NCCL: the global row histogram
        (all-reduce), count-balanced bounds, the records re-routed."""
        h = self.row_counts().to(torch.int64)
        dist.all_reduce(h, group=transport.group)
        counts = h.cpu().numpy()
        bounds = SlabLayout.balanced(counts, self.world).bounds
        plan = FieldPlan.make(bounds, n1, n_c, self.world) if self.field is not None else None
        self.rebalance_begin(bounds, plan)
        recs, dest = self.outbox()  # (a re-balance always goes through the tagged outbox)
        self.claim(NcclTransport.exchange(transport, recs, dest))
        self.rebalance_end()
        if hasattr(transport, "pending"):
            transport.pending = True

    def export(self):
        """Own particles' positions / anchors into the global state arrays."""
        self.sim.export_state()

    def owned_range(self):
        import ctypes
        lo, hi = self.N.C_i64(), self.N.C_i64()
        self.N.check(self.sim._bind().cs_slab_range(self.sim._h, ctypes.byref(lo),
                                                    ctypes.byref(hi)), "cs_slab_range")
        return int(lo.value), int(hi.value)

    def close(self):
        self.sim.close()


def _pair_cell(params):
    return None, None, float(params.pairs.cell_cutoff)


def rebalance_in_process(engines, hub: LoopbackHub, n_c: int | None = None):
    """Re-balance every in-process rank (tests): the summed row histogram,
    count-balanced bounds, the records re-routed through the hub."""
    counts = sum(e.row_counts().to(torch.int64) for e in engines).cpu().numpy()
    world = len(engines)
    bounds = SlabLayout.balanced(counts, world).bounds
    plan = None
    if engines[0].field is not None:
        plan = FieldPlan.make(bounds, len(counts), n_c, world)
    for e in engines:
        e.rebalance_begin(bounds, plan)
    got = hub.exchange_all([e.outbox() for e in engines])
    for e, g in zip(engines, got):
        e.claim(g)
    for e in engines:
        e.rebalance_end()
    return bounds


def step_in_process(engines, hub: LoopbackHub, xi):
    """One step of every rank of one process (tests): the phases in
    lockstep, the exchange through the hub."""
    if engines[0].field is not None:
        field_in_process([e.field for e in engines], move_in_process)
    for e in engines:
        e.local(xi)
    if getattr(engines[0], "_seg", 0):
        got = hub.exchange_all_packed([e.outbox_packed() for e in engines])
        for e, g in zip(engines, got):
            e.claim_packed(*g)
    else:
        got = hub.exchange_all([e.outbox() for e in engines])
        for e, g in zip(engines, got):
            e.claim(g)
    for e in engines:
        e.finish()


def ctypes_byref(x):
    import ctypes
    return ctypes.byref(x)


def _device_view(ptr: int, shape, dtype, device):
    """A torch tensor aliasing library-owned device memory."""
    typestr = {torch.int32: "<i4", torch.float32: "<f4"}[dtype]

    class _Alias:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3}
    return torch.as_tensor(_Alias(), device=device)


# ---------------------------------------------------------------------------
# the field of the device slab engine
# ---------------------------------------------------------------------------
@dataclass
class FieldPlan:
    """Static row bookkeeping of the distributed field for a layout: every
    rank owns an even share of the grid rows (the spectral passes' unit of
    work), deposits into a window covering its own rows and its particles'
    CIC rows, and samples the gradient of its particles' rows."""
    n: int                      # grid nodes per axis
    world: int
    rp: int                     # grid rows per rank
    g0: np.ndarray              # (world,) own grid rows [g0, g0 + rp)
    dep: list                   # per rank: (j0, rows) deposit window (j0 may be < 0: mod n)
    grad: list                  # per rank: (j0, rows) gradient window
    kx: np.ndarray              # (world + 1,) kx split of the n/2 + 1 half-spectrum columns

    @classmethod
    def make(cls, bounds, n1: int, n: int, world: int, blocking: int = 16) -> "FieldPlan":
        if n % world or (n // world) % 2 or (n // world) % min(blocking, n // world):
            raise ValueError(f"a {n}^2 grid cannot be split into {world} row slabs")
        rp = n // world
        g0 = np.arange(world) * rp
        eff_over_d = n / n1        # cell side over grid spacing (unit box, periodic grid)
        dep, grad = [], []
        for r in range(world):
            b0, b1 = int(bounds[r]), int(bounds[r + 1])
            jlo = int(math.floor(b0 * eff_over_d)) - 1
            jhi = int(math.floor(b1 * eff_over_d)) + 2
            if jhi - jlo > n:
                jlo, jhi = 0, n
            grad.append((jlo, jhi - jlo))
            d0, d1 = min(jlo, int(g0[r])), max(jhi, int(g0[r]) + rp)
            if d1 - d0 > n:
                d0, d1 = 0, n
            dep.append((d0, d1 - d0))
        nh = n // 2 + 1
        kx = np.round(np.linspace(0, nh, world + 1)).astype(np.int64)
        return cls(n, world, rp, g0, dep, grad, kx)

    def owner(self, j):
        return (np.asarray(j) % self.n) // self.rp

    def dep_rows(self, s: int, d: int) -> np.ndarray:
        """Deposit-window rows of rank s that rank d owns (s != d)."""
        j0, k = self.dep[s]
        rows = np.arange(j0, j0 + k) % self.n
        return rows[self.owner(rows) == d]

    def c_rows(self, d: int, s: int) -> np.ndarray:
        """c rows rank d's gradient window needs (one wider) that rank s owns."""
        j0, k = self.grad[d]
        rows = np.unique(np.arange(j0 - 1, j0 + k + 1) % self.n)
        return rows[self.owner(rows) == s]


class SlabField:
    """The field stage of one slab rank (the sorted engine's arrays) with
    the exchanges of its grid rows: deposit window rows into their owners,
    the spectrum transposes of the implicit solve, c rows for the gradient
    window.  ``move(kind, payload_per_dest) -> payload_per_source`` is the
    transport (all-to-all over NCCL, or copies between in-process ranks)."""

    def __init__(self, eng: "SlabEngine", plan: FieldPlan):
        self.eng, self.plan = eng, plan
        r = eng.rank
        lib = eng.sim._bind()
        dev = eng.sim.state["pos"].device
        n = plan.n
        self.rho = _device_view(lib.cs_slab_rho(eng.sim._h), (2, n, n), torch.int32, dev)
        self.c = eng.sim.state["c"].view(n, n)
        nh = n // 2 + 1
        kl = int(plan.kx[r + 1] - plan.kx[r])
        self.spec = torch.empty((nh, plan.rp, 2), dtype=torch.float32, device=dev)
        self.blocks = torch.empty((plan.world, kl, plan.rp, 2), dtype=torch.float32, device=dev)
        W = plan.world
        self.dep_send = [torch.as_tensor(plan.dep_rows(r, d), device=dev) for d in range(W)]
        self.dep_recv = [torch.as_tensor(plan.dep_rows(s, r), device=dev) for s in range(W)]
        self.c_send = [torch.as_tensor(plan.c_rows(d, r), device=dev) for d in range(W)]
        self.c_recv = [torch.as_tensor(plan.c_rows(r, s), device=dev) for s in range(W)]
        for q in (r,):
            self.dep_send[q] = self.dep_send[q][:0]
            self.dep_recv[q] = self.dep_recv[q][:0]
            self.c_send[q] = self.c_send[q][:0]
            self.c_recv[q] = self.c_recv[q][:0]

    # payloads for the transport
    def deposit_out(self):
        return [self.rho[:, rows, :].reshape(-1) for rows in self.dep_send]

    def deposit_in(self, got):
        for rows, g in zip(self.dep_recv, got):
            if rows.numel():
                self.rho[:, rows, :] += g.view(2, rows.numel(), self.plan.n)

    def _lib(self):
        """The library bound to the CURRENT torch stream (SlabEngine.step runs
        the field step on a side stream beside the pair forces)."""
        e = self.eng
        lib = e.N.load_library()
        lib.cs_ctx_set_stream(e.sim._ctx, e.N.C_p(torch.cuda.current_stream().cuda_stream))
        return lib

    def spec_rows(self, inverse: bool):
        e = self.eng
        e.N.check(self._lib().cs_slab_field_rows(e.sim._h, ctypes_byref(e.sim._st),
                                                   e.N.ptr(self.spec), int(inverse)),
                  "cs_slab_field_rows")

    def spec_out(self):
        p = self.plan
        return [self.spec[int(p.kx[q]):int(p.kx[q + 1])].reshape(-1) for q in range(p.world)]

    def spec_in_blocks(self, got):
        for q, g in enumerate(got):
            self.blocks[q].view(-1).copy_(g)

    def cols(self):
        e, p, r = self.eng, self.plan, self.eng.rank
        e.N.check(self._lib().cs_slab_field_cols(
            e.sim._h, e.N.ptr(self.blocks), int(p.kx[r]), int(p.kx[r + 1] - p.kx[r]), p.rp),
            "cs_slab_field_cols")

    def blocks_out(self):
        return [self.blocks[q].reshape(-1) for q in range(self.plan.world)]

    def blocks_in_spec(self, got):
        p = self.plan
        for q, g in enumerate(got):
            self.spec[int(p.kx[q]):int(p.kx[q + 1])].view(-1).copy_(g)

    def c_out(self):
        return [self.c[rows, :].reshape(-1) for rows in self.c_send]

    def c_in(self, got):
        for rows, g in zip(self.c_recv, got):
            if rows.numel():
                self.c[rows, :] = g.view(rows.numel(), self.plan.n)

    def gradient(self):
        e = self.eng
        e.N.check(self._lib().cs_slab_field_grad(e.sim._h, ctypes_byref(e.sim._st)),
                  "cs_slab_field_grad")


def field_in_process(fields, move):
    """The distributed field step of every in-process rank (lockstep)."""
    for f, got in zip(fields, move([f.deposit_out() for f in fields])):
        f.deposit_in(got)
    for f in fields:
        f.spec_rows(inverse=False)
    for f, got in zip(fields, move([f.spec_out() for f in fields])):
        f.spec_in_blocks(got)
    for f in fields:
        f.cols()
    for f, got in zip(fields, move([f.blocks_out() for f in fields])):
        f.blocks_in_spec(got)
    for f in fields:
        f.spec_rows(inverse=True)
    for f, got in zip(fields, move([f.c_out() for f in fields])):
        f.c_in(got)
    for f in fields:
        f.gradient()


def move_in_process(outs):
    """outs[s][d] = the payload rank s sends rank d -> got[d][s]."""
    W = len(outs)
    return [[outs[s][d] for s in range(W)] for d in range(W)]


class NcclField:
    """The transport of one rank's field exchanges over NCCL: every payload
    size is a static function of the layout (row lists, kx split), so the
    all-to-all runs with host-known splits and no synchronisation."""

    def __init__(self, field: SlabField, group=None):
        self.f, self.group = field, group

    def _a2a(self, out, recv_sizes):
        dev = out[0].device
        send = torch.cat([o.reshape(-1) for o in out]) if out else None
        recv = torch.empty(sum(recv_sizes), dtype=out[0].dtype, device=dev)
        dist.all_to_all_single(recv, send, recv_sizes, [o.numel() for o in out],
                               group=self.group)
        return list(recv.split(recv_sizes))

    def step(self):
        f, p = self.f, self.f.plan
        n, W, r = p.n, p.world, self.f.eng.rank
        kl = int(p.kx[r + 1] - p.kx[r])
        f.deposit_in(self._a2a(f.deposit_out(), [2 * n * rows.numel() for rows in f.dep_recv]))
        f.spec_rows(inverse=False)
        # the two spectrum transposes move straight between the engine's
        # buffers: the kx slices of spec (nh, rp, 2) are consecutive and so are
        # the per-rank blocks (W, kl, rp, 2), i.e. the all-to-all's own layout
        by_kx = [int(p.kx[q + 1] - p.kx[q]) * p.rp * 2 for q in range(W)]
        by_rank = [kl * p.rp * 2] * W
        dist.all_to_all_single(f.blocks.view(-1), f.spec.view(-1), by_rank, by_kx,
                               group=self.group)
        f.cols()
        dist.all_to_all_single(f.spec.view(-1), f.blocks.view(-1), by_kx, by_rank,
                               group=self.group)
        f.spec_rows(inverse=True)
        f.c_in(self._a2a(f.c_out(), [n * rows.numel() for rows in f.c_recv]))
        f.gradient()
