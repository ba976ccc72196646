"""y-slab decomposition on CPU: world sizes 2 and 3 over gloo,
the oracle as the per-rank compute backend, checked against the
single-domain oracle run.  Field off: bit-identical; field on (distributed
spectral solve): 1e-12."""

import os
import socket

import numpy as np
import pytest
import torch

import oracle
from oracle.sim import OracleSim
from paper_1805_11007_b200 import slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend(slabs.DeviceSlabBackend):
    """The oracle as the local compute of a rank (test infrastructure)."""

    def __init__(self, lo, hi, periodic, radii, diffusion, dt, grid=None, fparams=None,
                 chi=(0.0, 1.0), chi_pinned=(True, False)):
        self.lo, self.hi, self.per = np.asarray(lo), np.asarray(hi), periodic
        self.size = self.hi - self.lo
        self.tab = oracle.pair_table(radii=radii)
        self.diffusion = np.asarray(diffusion)
        self.dt = dt
        self.grid, self.fp = grid, fparams
        self.chi, self.chi_pinned = chi, chi_pinned
        self.secretes, self.consumes = (True, False), (False, True)

    def forces(self, pos, types, ids):
        e, c, cell = self.tab
        f = oracle.soft_forces(pos.numpy(), self.lo, self.size, self.per, e, c, cell,
                               types=types.numpy())
        return torch.from_numpy(f)

    def em(self, pos, types, force, xi, drift):
        out = oracle.em_step(pos.numpy(), self.diffusion[types.numpy()], drift.numpy(),
                             force.numpy(), xi.numpy(), self.dt)
        return torch.from_numpy(out)

    def boundaries(self, nxt, anchor):
        x = nxt.numpy()
        a = anchor.numpy()
        return oracle.apply_boundaries(x, a, self.lo, self.hi, self.per)

    def deposit(self, pos, types):
        g = self.grid
        t = types.numpy()
        sec = np.asarray(self.secretes)[t]
        con = np.asarray(self.consumes)[t]
        ra = oracle.cic_deposit(pos.numpy(), sec, g.n_c, g.lo, g.spacing, True)
        rb = oracle.cic_deposit(pos.numpy(), con, g.n_c, g.lo, g.spacing, True)
        return torch.from_numpy(ra), torch.from_numpy(rb)


def _problem(n, seed, field):
    rng = np.random.default_rng(seed)
    pos = -0.5 + rng.random((n, 2))
    types = (np.arange(n) >= n // 2).astype(np.uint8)
    steps = 5
    xi = rng.standard_normal((steps, n, 2))
    xi[2, :7] *= 40.0        # large kicks: migration across several slabs
    return pos, types, xi, steps


def _worker(rank, world, port, outdir, n, field, radii):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1805_11007_b200 as cs
        pos, types, xi, steps = _problem(n, 7, field)
        lo, hi = [-0.5, -0.5], [0.5, 0.5]
        e, c, cell = oracle.pair_table(radii=radii)
        geom = slabs.CellGeometry.make(-0.5, 0.5, cell)
        rows = geom.row_of(pos[:, 1])
        layout = slabs.SlabLayout.balanced(np.bincount(rows, minlength=geom.n), world)
        st = slabs.scatter_initial(np.arange(n), pos, types, layout, geom, rank, "cpu",
                                   torch.float64)
        fdict, c_rows = None, None
        grid = cs.Grid.square(32, 1.0, "periodic")
        fp = cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1)
        be = OracleBackend(lo, hi, (True, True), radii, (1.0, 0.5), 1e-5, grid=grid,
                           fparams=fp, chi=(1.0, -0.5), chi_pinned=(False, False))
        if field:
            gb = slabs.grid_row_bounds(layout, geom, 32, -0.5, grid.spacing[1])
            solver = slabs.DistributedSpectralSolver(32, grid.spacing, 1e-5, 1.0, gb, rank,
                                                     world, "cpu")
            fdict = dict(n_c=32, gb=gb, solver=solver)
            c_rows = torch.zeros((int(gb[rank + 1] - gb[rank]), 32), dtype=torch.float64)
        runner = slabs.SlabRunner(be, layout, geom, rank, world, True, field=fdict)
        for s in range(steps):
            xi_own = torch.from_numpy(xi[s][st.ids.numpy()])
            st, c_rows, key = runner.step(st, xi_own, c_rows)
            assert key == (1 << 62), key
        np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=st.ids.numpy(), pos=st.pos.numpy(),
                 anchor=st.anchor.numpy(),
                 c=(c_rows.numpy() if c_rows is not None else np.zeros(0)),
                 g0=(fdict["gb"][rank] if fdict else 0))
    finally:
        dist.destroy_process_group()


def _run(world, tmp_path, n, field, radii=(0.005, 0.01)):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path), n, field, radii), nprocs=world)
    parts = [dict(np.load(os.path.join(tmp_path, f"r{r}.npz"))) for r in range(world)]
    ids = np.concatenate([p["ids"] for p in parts])
    pos = np.concatenate([p["pos"] for p in parts])
    anc = np.concatenate([p["anchor"] for p in parts])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(n))
    c = None
    if field:
        c = np.concatenate([p["c"] for p in sorted(parts, key=lambda p: int(p["g0"]))], 0)
    return pos[o], anc[o], c


def _reference(n, field, radii=(0.005, 0.01)):
    pos, types, xi, steps = _problem(n, 7, field)
    e, c, cell = oracle.pair_table(radii=radii)
    fd = None
    if field:
        fd = dict(n_c=32, boundary="periodic", d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1,
                  kernel="cic", secretes=(True, False), consumes=(False, True),
                  c0=np.zeros(32 * 32), splu_max=0)
    sim = OracleSim(pos, types, lo=[-0.5] * 2, hi=[0.5] * 2, periodic=(True, True), dt=1e-5,
                    diffusion=(1.0, 0.5), eps_tab=e, cut_tab=c, cell_cutoff=cell,
                    chi=(1.0, -0.5), chi_pinned=(False, False), field=fd)
    for s in range(steps):
        sim.step(xi[s])
    return sim


@pytest.mark.parametrize("world", [2, 3])
def test_slabs_forces_only_bitwise(world, tmp_path):
    n = 4000
    pos, anc, _ = _run(world, tmp_path, n, field=False)
    ref = _reference(n, field=False)
    assert np.array_equal(pos, ref.pos)
    assert np.array_equal(anc, ref.anchor)


def test_slabs_with_field_distributed_solve(tmp_path):
    n = 3000
    pos, anc, c = _run(2, tmp_path, n, field=True)
    ref = _reference(n, field=True)
    assert np.allclose(c.ravel(), ref.c, rtol=0, atol=1e-12 * max(1.0, np.abs(ref.c).max()))
    assert np.allclose(pos, ref.pos, rtol=0, atol=1e-12)


def test_balanced_layout_and_grid_rows():
    counts = np.array([0, 0, 10, 50, 50, 10, 0, 0, 0, 0])
    lay = slabs.SlabLayout.balanced(counts, 2)
    assert lay.bounds[0] == 0 and lay.bounds[-1] == 10
    left = counts[: lay.bounds[1]].sum()
    assert abs(left - 60) <= 50
    geom = slabs.CellGeometry.make(-0.5, 0.5, 0.1)
    gb = slabs.grid_row_bounds(lay, geom, 20, -0.5, 0.05)
    assert gb[0] == 0 and gb[-1] == 20 and gb[1] == 2 * lay.bounds[1]
    assert list(lay.owner_of_row(np.arange(10))) == [0] * lay.bounds[1] + [1] * (10 - lay.bounds[1])
