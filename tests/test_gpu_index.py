"""The reference's CellIndex / Neighbor query API, accumulate_forces and
deposit_gather on the device, against golden vectors the reference produced
(tests/golden/make_index.py): index arrays and query ids exact, query
displacements / distances and index forces bitwise, the gather deposit
within 1e-13 (the reference's vectorised numpy exp differs from glibc's by
an ulp on a few % of inputs)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402


def _pop(pos, sp=None):
    n = pos.shape[0]
    sp = np.ones(n, np.uint8) if sp is None else sp
    return cs.Population(ids=np.arange(n), positions=pos.copy(), next_positions=pos.copy(),
                         species=sp, drift=np.zeros((n, 2)), local_concentration=np.zeros(n),
                         start_anchor=pos.copy())


def test_cell_index_build_and_queries_match_reference():
    g = load_golden("index.npz")
    for k in range(int(g["n_builds"])):
        side, per = g[f"b{k}_meta"]
        dom = cs.Domain.square(1.0, periodic=bool(per))
        idx = cs.CellIndex.build(g[f"b{k}_pos"], dom, float(side))
        assert np.array_equal(idx.n_cells, g[f"b{k}_n_cells"]), k
        assert np.array_equal(idx.order, g[f"b{k}_order"]), k
        assert np.array_equal(idx.starts, g[f"b{k}_starts"]), k
        assert np.array_equal(idx.cell_xy, g[f"b{k}_cell_xy"]), k
        for q in range(int(g["n_queries"])):
            nb = idx.query(g[f"b{k}_q{q}_pt"], float(g[f"b{k}_q{q}_rad"]))
            ids = np.array([x.id for x in nb], dtype=np.int64)
            assert np.array_equal(ids, g[f"b{k}_q{q}_ids"]), (k, q)
            if len(nb):
                assert np.array_equal(np.array([x.dx for x in nb]), g[f"b{k}_q{q}_dx"]), (k, q)
                assert np.array_equal(np.array([x.distance for x in nb]),
                                      g[f"b{k}_q{q}_dist"]), (k, q)
            assert all(isinstance(x, cs.Neighbor) for x in nb)


def test_cell_index_errors_and_buckets():
    dom = cs.Domain.square(1.0)
    with pytest.raises(ValueError, match="cell_side must be positive"):
        cs.CellIndex.build(np.zeros((3, 2)), dom, 0.0)
    with pytest.raises(ValueError, match="outside the domain"):
        cs.CellIndex.build(np.array([[0.0, 0.0], [0.7, 0.1]]), dom, 0.1)
    idx = cs.CellIndex.build(np.array([[0.5, 0.5], [0.49, 0.49], [-0.5, -0.5]]), dom, 0.25)
    assert list(idx.bucket(3, 3)) == [0, 1]  # closed upper edge, ascending id
    assert list(idx.bucket(0, 0)) == [2]
    with pytest.raises(ValueError, match="radius must be positive"):
        idx.query([0.0, 0.0], 0.0)


def test_accumulate_forces_bitwise_vs_reference():
    g = load_golden("index.npz")
    for k in range(int(g["n_forces"])):
        eps, cut, side, per = g[f"f{k}_meta"]
        pos = g[f"f{k}_pos"]
        dom = cs.Domain.square(1.0, periodic=bool(per))
        idx = cs.CellIndex.build(pos, dom, float(side))
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            params = cs.MotionParams(epsilon=float(eps), cutoff=float(cut), dt=1e-9)
        f = cs.accumulate_forces(_pop(pos), idx, params)
        assert np.array_equal(f, g[f"f{k}_force"]), k


def test_accumulate_forces_equals_soft_forces_at_cutoff_cells():
    """Built with cell_side = cutoff (reach 1, >= 3 cells per axis) the index
    path sums in the fused kernel's order: bitwise equal."""
    rng = np.random.default_rng(3)
    pos = rng.uniform(-0.5, 0.5, (5000, 2))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        params = cs.MotionParams(epsilon=0.005, cutoff=0.01, dt=1e-9)
    for per in (False, True):
        dom = cs.Domain.square(1.0, periodic=per)
        idx = cs.CellIndex.build(pos, dom, 0.01)
        assert np.array_equal(cs.accumulate_forces(_pop(pos), idx, params),
                              cs.soft_forces(_pop(pos), dom, params))


def test_deposit_gather_vs_reference_and_scatter():
    g = load_golden("index.npz")
    for k in range(int(g["n_gathers"])):
        nc, per, h = g[f"g{k}_meta"]
        grid = cs.Grid.square(int(nc), 1.0, "periodic" if per else "neumann")
        ker = cs.Kernel("gaussian", float(h), 3.0 * float(h))
        pop = _pop(g[f"g{k}_pos"], g[f"g{k}_sp"])
        for sp, key in ((cs.Species.ALPHA, "rho_a"), (cs.Species.BETA, "rho_b")):
            out = cs.deposit_gather(pop, grid, ker, sp)
            ref = g[f"g{k}_{key}"]
            assert np.allclose(out, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max()), (k, key)
            scat = cs.deposit(pop, grid, ker, sp)
            assert np.allclose(out, scat, rtol=1e-12, atol=1e-12 * np.abs(ref).max()), (k, key)
    with pytest.raises(ValueError, match="gaussian"):
        cs.deposit_gather(pop, grid, cs.Kernel("cic", 0.02, 0.06), cs.Species.ALPHA)
