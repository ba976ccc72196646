"""y-slab domain decomposition of one system over several GPUs.

One process per GPU (``torch.distributed``, NCCL over NVLink; the same code
runs on gloo/CPU for the tests).  Rank r owns the whole cell rows
[b_r, b_{r+1}) of the reference's cell grid (motion.py:171-174: n = int(L /
cutoff), eff = L / n) and the grid rows whose nodes lie in that y range.
Boundaries are count-balanced (prefix sum of the per-row particle counts),
because equal-width slabs cap the efficiency at 53-83 % for clustered
inputs.

Per step (Realisation._step_inner order, engine.py:369-387):

  field (if active)
    deposit owned particles into local grid rows + one ghost row per side,
    add the ghost rows into their owners            (grid ghost reduce)
    rhs on local rows; distributed spectral solve   (two all-to-all transposes)
    gradient with one ghost row of c per side       (grid ghost fetch)
    one ghost row of grad per side for the bilinear drift
  particles
    halo: every rank sends its first and last owned cell row to its
    neighbours (the cell side is >= the cutoff, so one row covers the ring)
    forces on owned + ghost particles (global cell geometry, rows in id
    order -> the reference summation order), EM, boundaries on owned
    migration: all-to-all by the owner of the new cell row (kicks can cross
    several slabs: 0.46 vs a 0.125-high slab at 8 GPUs)
  status: all-reduce (min error key)

Every collective is ``all_to_all_single`` or ``all_reduce``.  The local
compute comes from a backend object (``DeviceSlabBackend`` below runs the
library's C-ABI ops on the rank's GPU; the tests plug in the oracle).  With
the field off the decomposition is bit-identical to the single-domain run:
ghosts provide every ring neighbour, local rows stay in ascending id, and
the cell geometry is the global one.
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


def grid_row_bounds(layout: SlabLayout, geom: CellGeometry, n_c: int, lo: float,
                    spacing: float) -> np.ndarray:
    """Grid-row boundaries: node row j belongs to the owner of the cell row
    of its y coordinate (nodes are co-partitioned with the particles)."""
    ys = lo + spacing * np.arange(n_c)
    owners = layout.owner_of_row(geom.row_of(ys))
    gb = [0]
    for r in range(1, layout.world):
        gb.append(int(np.searchsorted(owners, r, side="left")))
    gb.append(n_c)
    return np.asarray(gb, dtype=np.int64)


# ----------------------------------------------------------------------------
# collectives
# ----------------------------------------------------------------------------
def exchange(tensors, dest, world: int, group=None):
    """Route rows of every tensor in ``tensors`` (same leading length) to the
    rank in ``dest``; returns the received tensors, rows ordered by source
    rank then by original order.  Two all_to_all_single calls per tensor
    (counts, payload)."""
    dev = dest.device
    order = torch.argsort(dest, stable=True)
    send_counts = torch.bincount(dest, minlength=world).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc = send_counts.cpu().tolist()
    rc = recv_counts.cpu().tolist()
    out = []
    for t in tensors:
        src = t[order]
        tail = tuple(src.shape[1:])
        width = int(np.prod(tail)) if tail else 1
        flat = src.reshape(-1, width) if width > 1 else src.reshape(-1, 1)
        if flat.dtype in (torch.uint8, torch.bool, torch.int16):
            flat = flat.to(torch.int32)
            back = t.dtype
        else:
            back = None
        recv = torch.empty((sum(rc), width), dtype=flat.dtype, device=dev)
        dist.all_to_all_single(recv.view(-1), flat.contiguous().view(-1),
                               [c * width for c in rc], [c * width for c in sc], group=group)
        if back is not None:
            recv = recv.to(back)
        out.append(recv.reshape((sum(rc),) + tail))
    return out


def exchange_flat(blocks, world: int, group=None):
    """All-to-all of arbitrary per-destination blocks (same dtype):
    ``blocks[q]`` goes to rank q; returns the flat 1-D chunks received from
    every rank (the caller knows their shapes)."""
    dev = blocks[0].device
    sc = [int(b.numel()) for b in blocks]
    counts = torch.tensor(sc, dtype=torch.int64, device=dev)
    rcounts = torch.empty_like(counts)
    dist.all_to_all_single(rcounts, counts, group=group)
    rc = rcounts.cpu().tolist()
    send = torch.cat([b.reshape(-1) for b in blocks]).contiguous()
    recv = torch.empty(sum(rc), dtype=send.dtype, device=dev)
    dist.all_to_all_single(recv, send, rc, sc, group=group)
    return list(recv.split(rc))


def exchange_rows(blocks, world: int, group=None):
    """All-to-all of per-destination row blocks with a common width m:
    ``blocks[q]`` (rows, m) goes to rank q; returns the blocks received."""
    m = blocks[0].shape[1]
    return [f.reshape(-1, m) for f in exchange_flat(blocks, world, group)]


# ----------------------------------------------------------------------------
# distributed spectral solve of (I - dt d_c L) c = rhs on a periodic grid
# ----------------------------------------------------------------------------
class DistributedSpectralSolver:
    """Row-slab 2-D real FFT diagonalisation (field.py:162-201's system, the
    periodic closure): rfft along x on local rows, transpose (all-to-all) to
    kx column blocks, FFT along y, multiply by the inverse eigenvalues, and
    back.  Same linear system as the single-GPU cuFFT path."""

    def __init__(self, n: int, spacing, dt: float, d_c: float, grid_bounds, rank: int,
                 world: int, device, group=None):
        self.n, self.rank, self.world, self.group = n, rank, world, group
        self.gb = np.asarray(grid_bounds)
        nh = n // 2 + 1
        self.cb = np.round(np.linspace(0, nh, world + 1)).astype(np.int64)
        hx, hy = float(spacing[0]), float(spacing[1])
        k = np.arange(n)
        lam_x = (2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / hx ** 2
        lam_y = (2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / hy ** 2
        c0, c1 = self.cb[rank], self.cb[rank + 1]
        eig = 1.0 / (1.0 - dt * d_c * (lam_y[:, None] + lam_x[None, c0:c1]))
        self.eig = torch.as_tensor(eig, device=device)

    def solve(self, rhs_rows: torch.Tensor) -> torch.Tensor:
        """rhs_rows: (g1 - g0, n) local rows -> solution rows (same shape)."""
        n, W = self.n, self.world
        spec = torch.fft.rfft(rhs_rows.double(), dim=1)            # (rows, nh)
        blocks = [torch.view_as_real(spec[:, self.cb[q]:self.cb[q + 1]]).contiguous()
                  for q in range(W)]
        got = exchange_flat(blocks, W, self.group)                  # rows from every rank
        ncols = int(self.cb[self.rank + 1] - self.cb[self.rank])
        col = torch.view_as_complex(torch.cat([g.reshape(-1, ncols, 2) for g in got], 0)
                                    .contiguous())
        col = torch.fft.ifft(torch.fft.fft(col, dim=0) * self.eig, dim=0)
        # back: my kx columns, split by the destination's rows
        rows_of = [int(self.gb[q + 1] - self.gb[q]) for q in range(W)]
        back = [torch.view_as_real(b).contiguous() for b in col.split(rows_of, 0)]
        got = exchange_flat(back, W, self.group)
        nh = n // 2 + 1
        mine = rhs_rows.shape[0]
        parts = [torch.view_as_complex(g.reshape(mine, -1, 2).contiguous()) for g in got]
        full = torch.cat(parts, 1)
        assert full.shape[1] == nh
        return torch.fft.irfft(full, n=n, dim=1)


def ghost_rows(local: torch.Tensor, rank: int, world: int, periodic: bool, group=None):
    """(row above the slab's first row, row below its last row) fetched from
    the neighbours (None at a non-periodic wall)."""
    up = (rank - 1) % world
    dn = (rank + 1) % world
    m = local.shape[1]
    empty = local.new_zeros((0, m))
    blocks = [empty] * world
    # my first row goes to the rank above me (it is their "below" ghost),
    # my last row to the rank below
    if world == 1:
        first, last = local[-1:], local[:1]
        return (first if periodic else None), (last if periodic else None)
    blocks = [empty for _ in range(world)]
    if periodic or rank > 0:
        blocks[up] = torch.cat([blocks[up], local[:1]], 0)
    if periodic or rank < world - 1:
        blocks[dn] = torch.cat([blocks[dn], local[-1:]], 0)
    got = exchange_rows(blocks, world, group)
    above = got[up] if (periodic or rank > 0) else None     # last row of the rank above
    below = got[dn] if (periodic or rank < world - 1) else None
    if above is not None and above.shape[0] == 2:           # world == 2, periodic: both
        above = above[1:]
    if below is not None and below.shape[0] == 2:
        below = below[:1]
    return above, below


def reduce_ghost_rows(top: torch.Tensor, bottom: torch.Tensor, rank: int, world: int,
                      periodic: bool, group=None):
    """Send the deposit rows that belong to the neighbours (``top`` = the row
    just above my first row, ``bottom`` = just below my last row) and return
    (what the rank above sent for my first row, what the rank below sent for
    my last row) to be added."""
    m = top.shape[1]
    empty = top.new_zeros((0, m))
    if world == 1:
        return (bottom if periodic else torch.zeros_like(top)), \
               (top if periodic else torch.zeros_like(bottom))
    up = (rank - 1) % world
    dn = (rank + 1) % world
    blocks = [empty for _ in range(world)]
    if periodic or rank > 0:
        blocks[up] = torch.cat([blocks[up], top], 0)
    if periodic or rank < world - 1:
        blocks[dn] = torch.cat([blocks[dn], bottom], 0)
    got = exchange_rows(blocks, world, group)
    z = torch.zeros_like(top)
    # the rank above sent its "bottom" (my first row); the rank below its "top"
    from_up = got[up] if (periodic or rank > 0) else z
    from_dn = got[dn] if (periodic or rank < world - 1) else z
    if world == 2 and periodic:
        # up == dn: that rank sent [top, bottom] in this order
        pair = got[up]
        from_dn, from_up = pair[:1], pair[1:]
    return from_up, from_dn


# ----------------------------------------------------------------------------
# particle state of one rank
# ----------------------------------------------------------------------------
@dataclass
class SlabState:
    ids: torch.Tensor        # (n_r,) int64, ascending
    pos: torch.Tensor        # (n_r, 2)
    anchor: torch.Tensor     # (n_r, 2)
    types: torch.Tensor      # (n_r,) uint8

    def sort_by_id(self) -> "SlabState":
        o = torch.argsort(self.ids)
        return SlabState(self.ids[o], self.pos[o], self.anchor[o], self.types[o])


def scatter_initial(ids, pos, types, layout: SlabLayout, geom: CellGeometry, rank: int,
                    device, dtype) -> SlabState:
    """Every rank keeps the particles of its slab (inputs replicated)."""
    rows = geom.row_of(pos[:, 1])
    mine = layout.owner_of_row(rows) == rank
    p = torch.as_tensor(pos[mine], device=device).to(dtype)
    return SlabState(torch.as_tensor(ids[mine], device=device, dtype=torch.int64), p,
                     p.clone(), torch.as_tensor(types[mine], device=device))


class SlabRunner:
    """Steps one rank's slab.  ``backend`` provides the local compute:

      forces(pos, types, ids) -> (n, 2) float64 forces of every given row
      em(pos, types, force, xi, drift) -> proposals (n, 2)
      boundaries(next, anchor) -> (status, bad_i, bad_ax), in place
      deposit(pos, types) -> (rho_a, rho_b) full-grid arrays (n_c^2,)
      rhs(c_rows, ra_rows, rb_rows) -> rhs rows
      gradient(c_ext) -> (rows, n_c, 2) from c rows with one ghost row per side
      bilinear_grad(grad_ext, row0, pos, types) -> drift (n, 2)
    """

    def __init__(self, backend, layout: SlabLayout, geom: CellGeometry, rank: int, world: int,
                 periodic_y: bool, field=None, group=None):
        self.be, self.layout, self.geom = backend, layout, geom
        self.rank, self.world, self.per = rank, world, periodic_y
        self.group = group
        self.field = field          # dict(n_c, gb, solver) or None

    # ---- halo ------------------------------------------------------------
    def halo(self, st: SlabState) -> SlabState:
        b0, b1 = int(self.layout.bounds[self.rank]), int(self.layout.bounds[self.rank + 1])
        rows = self.geom.row_of(st.pos[:, 1])
        W = self.world
        up, dn = (self.rank - 1) % W, (self.rank + 1) % W
        sel_up = rows == b0            # my first row -> rank above (their lower ghost)
        sel_dn = rows == b1 - 1        # my last row -> rank below
        if not self.per:
            sel_up &= self.rank > 0
            sel_dn &= self.rank < W - 1
        dest = torch.full_like(st.ids, -1)
        parts_ids, parts_pos, parts_t, parts_dest = [], [], [], []
        for sel, d in ((sel_up, up), (sel_dn, dn)):
            if W == 1:
                break
            parts_ids.append(st.ids[sel])
            parts_pos.append(st.pos[sel])
            parts_t.append(st.types[sel])
            parts_dest.append(torch.full((int(sel.sum()),), d, dtype=torch.int64,
                                         device=st.ids.device))
        if W == 1:
            return SlabState(st.ids[:0], st.pos[:0], st.anchor[:0], st.types[:0])
        ids = torch.cat(parts_ids)
        pos = torch.cat(parts_pos)
        ty = torch.cat(parts_t)
        dest = torch.cat(parts_dest)
        r_ids, r_pos, r_t = exchange([ids, pos, ty], dest, W, self.group)
        # the same particle may arrive twice when world == 2 (periodic): keep one
        if r_ids.numel():
            u, inv = torch.unique(r_ids, return_inverse=True)
            first = torch.full_like(u, r_ids.numel())
            first.scatter_reduce_(0, inv, torch.arange(r_ids.numel(), device=u.device),
                                  reduce="amin")
            r_ids, r_pos, r_t = r_ids[first], r_pos[first], r_t[first]
        return SlabState(r_ids, r_pos, r_pos.clone(), r_t)

    # ---- migration -----------------------------------------------------
    def migrate(self, st: SlabState) -> SlabState:
        rows = self.geom.row_of(st.pos[:, 1])
        dest = self.layout.owner_of_row(rows).to(torch.int64)
        ids, pos, anc, ty = exchange([st.ids, st.pos, st.anchor, st.types], dest, self.world,
                                     self.group)
        return SlabState(ids, pos, anc, ty).sort_by_id()

    # ---- one step ------------------------------------------------------
    def step(self, st: SlabState, xi_own: torch.Tensor, c_rows=None):
        """Advance the owned particles (xi_own rows match st rows) and the
        local field rows; returns (state, c_rows, status key)."""
        be = self.be
        drift = torch.zeros_like(st.pos, dtype=torch.float64)
        if self.field is not None:
            f = self.field
            gb = f["gb"]
            g0, g1 = int(gb[self.rank]), int(gb[self.rank + 1])
            n_c = f["n_c"]
            ra, rb = be.deposit(st.pos, st.types)                   # full grid, owned particles
            ra = ra.view(n_c, n_c)
            rb = rb.view(n_c, n_c)
            # local rows + the ghost rows just outside the slab (periodic wrap)
            def rows_ext(a):
                above = a[(g0 - 1) % n_c:(g0 - 1) % n_c + 1]
                below = a[g1 % n_c:g1 % n_c + 1]
                return a[g0:g1].clone(), above, below
            ra_l, ra_up, ra_dn = rows_ext(ra)
            rb_l, rb_up, rb_dn = rows_ext(rb)
            top = torch.cat([ra_up, rb_up], 1)
            bot = torch.cat([ra_dn, rb_dn], 1)
            from_up, from_dn = reduce_ghost_rows(top, bot, self.rank, self.world, self.per,
                                                 self.group)
            ra_l[0] += from_up[0, :n_c]
            rb_l[0] += from_up[0, n_c:]
            ra_l[-1] += from_dn[0, :n_c]
            rb_l[-1] += from_dn[0, n_c:]
            rhs = be.rhs(c_rows, ra_l, rb_l)
            c_rows = f["solver"].solve(rhs).to(c_rows.dtype)
            up, dn = ghost_rows(c_rows, self.rank, self.world, self.per, self.group)
            c_ext = torch.cat([up, c_rows, dn], 0)
            grad = be.gradient(c_ext)                                # (rows, n_c, 2)
            gup, gdn = ghost_rows(grad.reshape(grad.shape[0], -1), self.rank, self.world,
                                  self.per, self.group)
            g_ext = torch.cat([gup, grad.reshape(grad.shape[0], -1), gdn], 0)
            drift = be.bilinear_grad(g_ext.reshape(-1, n_c, 2), g0 - 1, st.pos, st.types)
        ghosts = self.halo(st)
        all_ids = torch.cat([st.ids, ghosts.ids])
        all_pos = torch.cat([st.pos, ghosts.pos])
        all_t = torch.cat([st.types, ghosts.types])
        o = torch.argsort(all_ids)
        forces_sorted = be.forces(all_pos[o], all_t[o], all_ids[o])
        forces = torch.empty_like(forces_sorted)
        forces[o] = forces_sorted
        f_own = forces[: st.ids.numel()]
        nxt = be.em(st.pos, st.types, f_own, xi_own, drift)
        anc = st.anchor.clone()
        status, bad_i, bad_ax = be.boundaries(nxt, anc)
        key = torch.tensor([status * (1 << 40) + (int(st.ids[bad_i]) if status else 0)
                            if status else (1 << 62)], dtype=torch.int64, device=st.ids.device)
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=self.group)
        new = SlabState(st.ids, nxt, anc, st.types)
        return self.migrate(new), c_rows, int(key.item())


# ----------------------------------------------------------------------------
# device backend: the library's C-ABI ops on this rank's GPU
# ----------------------------------------------------------------------------
class DeviceSlabBackend:
    """Local compute of one rank on its GPU.  Pair forces, the EM proposal,
    boundaries and deposits run in libchemo_b200 (cs_soft_forces, cs_em_step,
    cs_apply_boundaries, cs_deposit) on the global geometry; the slab-local
    grid stencils (rhs, gradient rows, bilinear drift) are exact elementwise
    restatements of the reference arithmetic on the rank's rows."""

    def __init__(self, domain, motion, grid=None, fparams=None, chi=(0.0, 1.0),
                 chi_pinned=(True, False), secretes=(True, False), consumes=(False, True),
                 dt=1e-5):
        from . import _native as N
        self.N = N
        self.domain, self.motion, self.grid, self.fp = domain, motion, grid, fparams
        self.chi, self.chi_pinned = chi, chi_pinned
        self.secretes, self.consumes = secretes, consumes
        self.dt = float(dt)
        eps, cut, cell = motion.pair_table()
        self.pp = N.pair_struct(eps, cut, cell)
        self.dom = N.domain_struct(domain.lo, domain.hi, domain.periodic)
        self.D = torch.tensor([motion.d_alpha, motion.d_beta], dtype=torch.float64)

    def forces(self, pos, types, ids):
        import ctypes
        N = self.N
        n = pos.shape[0]
        out = torch.empty((n, 2), dtype=torch.float64, device=pos.device)
        if n:
            N.check(N.load_library().cs_soft_forces(
                N.context(), N.prec_code(pos.dtype), N.ptr(pos.contiguous()),
                N.ptr(types.contiguous()), n, ctypes.byref(self.dom), ctypes.byref(self.pp),
                N.ptr(out)), "cs_soft_forces")
        return out

    def em(self, pos, types, force, xi, drift):
        from .motion import em_step
        D = self.D.to(pos.device)[types.long()]
        return em_step(pos, D, drift, force, self.dt, xi=xi.to(pos.dtype))

    def boundaries(self, nxt, anchor):
        import ctypes
        N = self.N
        bi, ba = ctypes.c_int64(-1), ctypes.c_int32(-1)
        n = nxt.shape[0]
        if n == 0:
            return 0, -1, -1
        st = N.load_library().cs_apply_boundaries(
            N.context(), N.prec_code(nxt.dtype), N.ptr(nxt), N.ptr(anchor), N.C_p(0), n,
            ctypes.byref(self.dom), ctypes.byref(bi), ctypes.byref(ba))
        N.check(st, "cs_apply_boundaries")
        return st, bi.value, ba.value

    def deposit(self, pos, types):
        from .coupling import Kernel, deposit as dep
        from .particles import Population
        kern = Kernel(kind="cic")
        sec = torch.tensor(self.secretes, device=pos.device)[types.long()]
        con = torch.tensor(self.consumes, device=pos.device)[types.long()]
        n = pos.shape[0]
        z = torch.zeros((n, 2), dtype=torch.float64, device=pos.device)
        out = []
        for mask in (sec, con):
            sp = torch.where(mask, 0, 1).to(torch.uint8)
            pop = Population(ids=torch.arange(n, device=pos.device), positions=pos,
                             next_positions=pos, species=sp, drift=z,
                             local_concentration=z[:, 0], start_anchor=pos)
            out.append(dep(pop, self.grid, kern, 0).to(torch.float64))
        return out[0], out[1]

    def rhs(self, c, ra, rb):
        fp, dt = self.fp, self.dt
        r = c.double() * (1.0 - dt * fp.gamma) if fp.gamma else c.double().clone()
        if fp.k_alpha:
            r = r + (dt * fp.k_alpha) * ra
        if fp.k_beta:
            r = r - (rb * c.double()) * (dt * fp.k_beta)
        return r

    def gradient(self, c_ext):
        """(rows, n, 2) central differences (periodic grid, field.py:128-137)
        for the interior rows of c_ext (one ghost row above and below)."""
        hx, hy = (float(v) for v in self.grid.spacing)
        c = c_ext.double()
        m1x, p1x = -1.0 / (2.0 * hx), 1.0 / (2.0 * hx)
        m1y, p1y = -1.0 / (2.0 * hy), 1.0 / (2.0 * hy)
        mid = c[1:-1]
        gx = m1x * torch.roll(mid, 1, 1) + p1x * torch.roll(mid, -1, 1)
        gy = m1y * c[:-2] + p1y * c[2:]
        return torch.stack([gx, gy], -1)

    def bilinear_grad(self, g_ext, row0, pos, types):
        """Bilinear drift (coupling.py:216-262, periodic) from grad rows
        row0 .. row0 + len(g_ext) - 1 (global row indices, may be -1)."""
        n_c = self.grid.n_c
        lo = torch.as_tensor(self.grid.lo, device=pos.device)
        h = torch.as_tensor(self.grid.spacing, device=pos.device)
        u = (pos.double() - lo) / h
        f = torch.floor(u)
        fr = u - f
        b = f.long()
        bx = torch.remainder(b[:, 0], n_c)
        cx = torch.remainder(bx + 1, n_c)
        by = b[:, 1] - row0
        # global row b1 maps to local row b1 - row0; a wrap at the seam keeps
        # the local offset (ghost rows carry the wrapped neighbours)
        by = torch.where(by < 0, by + n_c, by)
        by = torch.where(by >= g_ext.shape[0], by - n_c, by)
        cy = by + 1
        f0, f1 = fr[:, 0], fr[:, 1]
        w00 = (1.0 - f0) * (1.0 - f1)
        w10 = f0 * (1.0 - f1)
        w01 = (1.0 - f0) * f1
        w11 = f0 * f1
        g = g_ext.double()
        v = (w00[:, None] * g[by, bx] + w10[:, None] * g[by, cx]) + w01[:, None] * g[cy, bx]
        v = v + w11[:, None] * g[cy, cx]
        chi = torch.tensor(self.chi, dtype=torch.float64, device=pos.device)[types.long()]
        pin = torch.tensor(self.chi_pinned, device=pos.device)[types.long()]
        v = torch.where((chi != 1.0)[:, None], v * chi[:, None], v)
        return torch.where(pin[:, None], torch.zeros_like(v), v)


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
    def step(self, xi, transport: NcclTransport):
        if self.field is not None:
            if not hasattr(self, "_nf"):
                self._nf = NcclField(self.field, transport.group)
            self._nf.step()
        self.local(xi)
        recs, dest = self.outbox()
        self.claim(transport.exchange(recs, dest))
        self.finish()

    def status(self):
        return self.sim.status()

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


def step_in_process(engines, hub: LoopbackHub, xi):
    """One step of every rank of one process (tests): the phases in
    lockstep, the exchange through the hub."""
    if engines[0].field is not None:
        field_in_process([e.field for e in engines], move_in_process)
    for e in engines:
        e.local(xi)
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

    def spec_rows(self, inverse: bool):
        e = self.eng
        e.N.check(e.sim._bind().cs_slab_field_rows(e.sim._h, ctypes_byref(e.sim._st),
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
        e.N.check(e.sim._bind().cs_slab_field_cols(
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
        e.N.check(e.sim._bind().cs_slab_field_grad(e.sim._h, ctypes_byref(e.sim._st)),
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
        f.spec_in_blocks(self._a2a(f.spec_out(), [kl * p.rp * 2] * W))
        f.cols()
        f.blocks_in_spec(self._a2a(f.blocks_out(),
                                   [int(p.kx[q + 1] - p.kx[q]) * p.rp * 2 for q in range(W)]))
        f.spec_rows(inverse=True)
        f.c_in(self._a2a(f.c_out(), [n * rows.numel() for rows in f.c_recv]))
        f.gradient()
