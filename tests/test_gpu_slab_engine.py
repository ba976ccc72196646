"""The y-slab decomposition on the device: W ranks' sorted
engines in slab mode, stepped in lockstep in one process on one GPU with the
records exchanged through device copies (slabs.LoopbackHub; over NCCL the
same records go through slabs.NcclTransport).  With the field off the
decomposed system must equal the single-domain sorted engine bit for bit:
the ghost rows give every owned particle its whole reference ring, rows stay
in ascending id inside a cell, and the cell geometry is the global one."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_11007_b200 as cs  # noqa: E402
from paper_1805_11007_b200 import slabs  # noqa: E402


def _params(n, radii, periodic=True):
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = cs.MotionParams(d_alpha=1.0, d_beta=0.5, epsilon=radii[0], cutoff=2 * radii[0],
                             dt=1e-5, radius_alpha=radii[0], radius_beta=radii[1])
    dom = cs.Domain.square(1.0, periodic=periodic)
    grid = cs.Grid.square(8, 1.0, "periodic" if periodic else "neumann")
    params = cs.sim_params_struct(
        n=n, prec=1, domain=dom, motion=mp, dt=1e-5, field_active=False, refresh_active=False,
        grid=grid, fparams=cs.FieldParams(d_c=0.0, k_alpha=0.0, k_beta=0.0, gamma=0.0),
        kernel=cs.Kernel(kind="cic"), secretes=(False, False), consumes=(False, False),
        chi=(0.0, 0.0), chi_pinned=(True, True), store_samples=False, store_next=False,
        engine="sorted")
    return params, mp, dom


def _state(pos, sp):
    f32 = torch.float32
    return dict(pos=torch.as_tensor(pos, device="cuda").to(f32).contiguous(),
                anchor=torch.as_tensor(pos, device="cuda").to(f32).contiguous(),
                species=torch.as_tensor(sp, device="cuda"), next_pos=None,
                drift=torch.zeros((pos.shape[0], 2), dtype=torch.float64, device="cuda"),
                local_c=None, c=None, grad=None, rho_a=None, rho_b=None)


def _bounds(pos, mp, dom, world):
    e, c, cell = mp.pair_table()
    geom = slabs.CellGeometry.make(dom.lo[1], dom.hi[1], cell)
    counts = np.bincount(geom.row_of(pos[:, 1].astype(np.float64)), minlength=geom.n)
    return slabs.SlabLayout.balanced(counts, world).bounds


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("clustered", [False, True])
def test_slab_engine_equals_single_domain_bitwise(world, clustered):
    rng = np.random.default_rng(10 + world)
    n, steps = 200_000, 6
    if clustered:  # cfg4's initial condition at 1/400 scale
        centres = -0.5 + rng.random((64, 2))
        pos = centres[rng.integers(0, 64, n)] + 0.02 * rng.standard_normal((n, 2))
        pos = np.mod(pos + 0.5, 1.0) - 0.5
    else:
        pos = -0.5 + rng.random((n, 2))
    pos = pos.astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    radii = (4.9e-4, 9.8e-4)
    params, mp, dom = _params(n, radii)
    xi = torch.as_tensor(rng.standard_normal((steps, n, 2)).astype(np.float32), device="cuda")
    # single domain
    st1 = _state(pos, sp)
    one = cs.DeviceSim(params, st1)
    one.step(xi, steps)
    one.export_state()
    assert one.status().code == 0
    # W slabs sharing the caller's arrays (each exports its own particles)
    st = _state(pos, sp)
    bounds = _bounds(pos, mp, dom, world)
    engines = [slabs.SlabEngine(params, st, bounds, r, world) for r in range(world)]
    hub = slabs.LoopbackHub(world)
    owned0 = sum(hi - lo for lo, hi in (e.owned_range() for e in engines))
    assert owned0 == n
    for k in range(steps):
        slabs.step_in_process(engines, hub, xi[k])
    for e in engines:
        assert e.status().code == 0
    owned = sum(hi - lo for lo, hi in (e.owned_range() for e in engines))
    assert owned == n  # every particle owned by exactly one rank
    for e in engines:
        e.export()
    torch.cuda.synchronize()
    assert torch.equal(st["pos"], st1["pos"])
    assert torch.equal(st["anchor"], st1["anchor"])
    for e in engines:
        e.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("clustered", [False, True])
def test_packed_exchange_equals_single_domain_bitwise(world, clustered):
    """The exchange without a host round trip (a segment of outbox slots and a
    device counter per destination rank, claimed from the same layout): two
    counted steps size the segments, the rest run packed -- the single
    domain's positions and anchors bit for bit."""
    rng = np.random.default_rng(40 + world)
    n, steps = 200_000, 6
    if clustered:
        centres = -0.5 + rng.random((64, 2))
        pos = centres[rng.integers(0, 64, n)] + 0.02 * rng.standard_normal((n, 2))
        pos = np.mod(pos + 0.5, 1.0) - 0.5
    else:
        pos = -0.5 + rng.random((n, 2))
    pos = pos.astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    params, mp, dom = _params(n, (4.9e-4, 9.8e-4))
    xi = torch.as_tensor(rng.standard_normal((steps, n, 2)).astype(np.float32), device="cuda")
    st1 = _state(pos, sp)
    one = cs.DeviceSim(params, st1)
    one.step(xi, steps)
    one.export_state()
    st = _state(pos, sp)
    bounds = _bounds(pos, mp, dom, world)
    engines = [slabs.SlabEngine(params, st, bounds, r, world) for r in range(world)]
    hub = slabs.PackedLoopbackHub(world)
    peak = 0
    for k in range(2):  # counted steps: the largest per-destination traffic
        for e in engines:
            e.local(xi[k])
        outs = [e.outbox() for e in engines]
        for recs, dest in outs:
            if recs.shape[0]:
                peak = max(peak, int(torch.bincount((dest & 0x3FFFFFFF).long()).max()))
        for e, g in zip(engines, hub.exchange_all(outs)):
            e.claim(g)
        for e in engines:
            e.finish()
    assert peak > 0
    seg = (2 * peak + 255) // 256 * 256
    for e in engines:
        e.set_exchange_cap(seg)
    for k in range(2, steps):
        slabs.step_in_process(engines, hub, xi[k])
    for e in engines:
        assert e.status().code == 0
        e.export()
    torch.cuda.synchronize()
    assert torch.equal(st["pos"], st1["pos"])
    assert torch.equal(st["anchor"], st1["anchor"])
    for e in engines:
        e.close()


def test_packed_exchange_overflow_stops_the_run():
    """A destination that gets more records in a step than its segment holds
    stops the run (CS_SORT_OVERFLOW) instead of dropping records."""
    rng = np.random.default_rng(5)
    n, world = 100_000, 2
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    params, mp, dom = _params(n, (4.9e-4, 9.8e-4))
    xi = torch.as_tensor(rng.standard_normal((1, n, 2)).astype(np.float32), device="cuda")
    st = _state(pos, sp)
    bounds = _bounds(pos, mp, dom, world)
    engines = [slabs.SlabEngine(params, st, bounds, r, world) for r in range(world)]
    hub = slabs.PackedLoopbackHub(world)
    for e in engines:
        e.set_exchange_cap(8)
    slabs.step_in_process(engines, hub, xi[0])
    assert any(e.status().code == cs._native.CS_SORT_OVERFLOW for e in engines)
    for e in engines:
        e.close()


def _field_params(n, radii, n_c):
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = cs.MotionParams(d_alpha=1.0, d_beta=0.5, epsilon=radii[0], cutoff=2 * radii[0],
                             dt=1e-5, radius_alpha=radii[0], radius_beta=radii[1])
    dom = cs.Domain.square(1.0, periodic=True)
    grid = cs.Grid.square(n_c, 1.0, "periodic")
    params = cs.sim_params_struct(
        n=n, prec=1, domain=dom, motion=mp, dt=1e-5, field_active=True, refresh_active=True,
        grid=grid, fparams=cs.FieldParams(d_c=1.0, k_alpha=0.1, k_beta=0.03, gamma=0.1),
        kernel=cs.Kernel(kind="cic"), secretes=(True, False), consumes=(False, True),
        chi=(1.0, -0.5), chi_pinned=(False, False), store_samples=False, store_next=False,
        engine="sorted")
    return params, mp, dom


def _field_state(pos, sp, c0, n_c, shared=None):
    f32 = torch.float32
    st = _state(pos, sp) if shared is None else dict(shared)
    st.update(c=torch.as_tensor(c0, device="cuda").to(f32).contiguous(),
              grad=torch.zeros((n_c * n_c, 2), dtype=f32, device="cuda"),
              rho_a=torch.zeros(n_c * n_c, dtype=f32, device="cuda"),
              rho_b=torch.zeros(n_c * n_c, dtype=f32, device="cuda"))
    return st


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("clustered", [False, True])
def test_slab_engine_with_field_equals_single_domain_bitwise(world, clustered):
    """The distributed field (deposit windows added into their owners' rows
    in exact int32, the spectral solve split into own-row passes and
    own-column passes around two all-to-all transposes, gradient windows
    from fetched c rows) on top of the particle slabs: positions and every
    rank's own field rows equal the single-domain engine's bit for bit."""
    rng = np.random.default_rng(20 + world)
    n, n_c, steps = 100_000, 256, 5
    if clustered:
        centres = -0.5 + rng.random((16, 2))
        pos = centres[rng.integers(0, 16, n)] + 0.03 * rng.standard_normal((n, 2))
        pos = np.mod(pos + 0.5, 1.0) - 0.5
    else:
        pos = -0.5 + rng.random((n, 2))
    pos = pos.astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    radii = (7e-4, 1.4e-3)
    c0 = (0.5 + 0.1 * rng.standard_normal(n_c * n_c)).astype(np.float32)
    params, mp, dom = _field_params(n, radii, n_c)
    xi = torch.as_tensor(rng.standard_normal((steps, n, 2)).astype(np.float32), device="cuda")
    st1 = _field_state(pos, sp, c0, n_c)
    one = cs.DeviceSim(params, st1)
    one.step(xi, steps)
    one.export_state()
    assert one.status().code == 0
    shared = _state(pos, sp)
    bounds = _bounds(pos, mp, dom, world)
    e, c, cell = mp.pair_table()
    n1 = slabs.CellGeometry.make(dom.lo[1], dom.hi[1], cell).n
    plan = slabs.FieldPlan.make(bounds, n1, n_c, world)
    sts = [_field_state(pos, sp, c0, n_c, shared) for _ in range(world)]
    engines = [slabs.SlabEngine(params, sts[r], bounds, r, world, field_plan=plan)
               for r in range(world)]
    hub = slabs.LoopbackHub(world)
    for k in range(steps):
        slabs.step_in_process(engines, hub, xi[k])
    for eng in engines:
        assert eng.status().code == 0, eng.status().code
        eng.export()
    torch.cuda.synchronize()
    assert torch.equal(shared["pos"], st1["pos"])
    c1 = st1["c"].view(n_c, n_c)
    for r in range(world):
        rows = slice(int(plan.g0[r]), int(plan.g0[r]) + plan.rp)
        assert torch.equal(sts[r]["c"].view(n_c, n_c)[rows], c1[rows]), r
    for eng in engines:
        eng.close()


def test_slab_step_over_nccl_on_one_rank_equals_single_domain_bitwise():
    """The N > 1 step as bench.py drives it -- SlabEngine.step over real NCCL
    (NcclField's static exchanges and transposes, the counted record exchange
    for two steps, then the packed one, a re-balance in between) -- on a
    one-rank process group (one B200 per session): positions, anchors and the
    field equal the single-domain engine's bit for bit."""
    import os
    import socket
    import torch.distributed as dist
    rng = np.random.default_rng(77)
    n, n_c, steps = 100_000, 256, 6
    pos = (-0.5 + rng.random((n, 2))).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    c0 = (0.5 + 0.1 * rng.standard_normal(n_c * n_c)).astype(np.float32)
    params, mp, dom = _field_params(n, (7e-4, 1.4e-3), n_c)
    xi = torch.as_tensor(rng.standard_normal((steps, n, 2)).astype(np.float32), device="cuda")
    st1 = _field_state(pos, sp, c0, n_c)
    one = cs.DeviceSim(params, st1)
    one.step(xi, steps)
    one.export_state()
    assert one.status().code == 0
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        st = _field_state(pos, sp, c0, n_c)
        bounds = _bounds(pos, mp, dom, 1)
        e, c, cell = mp.pair_table()
        n1 = slabs.CellGeometry.make(dom.lo[1], dom.hi[1], cell).n
        plan = slabs.FieldPlan.make(bounds, n1, n_c, 1)
        eng = slabs.SlabEngine(params, st, bounds, 0, 1, field_plan=plan)
        tr = slabs.PackedNcclTransport(1)
        for k in range(steps):
            eng.step(xi[k], tr)
            if k == 1:
                assert tr.calibrate() >= 4096
            if k == 3:
                eng.rebalance(tr, n1, n_c)
        assert eng.status().code == 0
        eng.export()
        torch.cuda.synchronize()
        assert torch.equal(st["pos"], st1["pos"])
        assert torch.equal(st["anchor"], st1["anchor"])
        assert torch.equal(st["c"], st1["c"])
        eng.close()
    finally:
        dist.destroy_process_group()


def test_bench_slab_setup_in_process():
    """bench.py's N > 1 path (one system over W slabs): its setup (seeded
    state, count-balanced bounds, field plan) at cfg3's parameters and 1/50
    of its size, the W ranks emulated in one process: the single-domain
    engine's result bit for bit."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    cfg = dict(bench.CONFIGS["cfg3"], n=200_000, n_c=512)
    world, steps = 4, 3
    one, st1, _, _ = bench.make_state(cfg, 0)
    assert one.engine == "sorted"
    xi = torch.randn((steps, cfg["n"], 2), generator=torch.Generator(device="cuda")
                     .manual_seed(5), device="cuda")
    one.step(xi, steps)
    one.export_state()
    params, _, bounds, plan = bench.slab_setup(cfg, world)
    engines, states = [], []
    shared = None
    for r in range(world):
        _, st, _, _ = bench.make_state(cfg, 0, engine="sorted", build_sim=False)
        if shared is None:
            shared = st
        else:
            for key in ("pos", "anchor", "species"):
                st[key] = shared[key]
        states.append(st)
        engines.append(slabs.SlabEngine(params, st, bounds, r, world, field_plan=plan))
    hub = slabs.LoopbackHub(world)
    for k in range(steps):
        slabs.step_in_process(engines, hub, xi[k])
    for eng in engines:
        assert eng.status().code == 0
        eng.export()
    torch.cuda.synchronize()
    assert torch.equal(shared["pos"], st1["pos"])
    n_c = cfg["n_c"]
    for r in range(world):
        rows = slice(int(plan.g0[r]), int(plan.g0[r]) + plan.rp)
        assert torch.equal(states[r]["c"].view(n_c, n_c)[rows], st1["c"].view(n_c, n_c)[rows])


@pytest.mark.parametrize("field", [False, True])
def test_slab_rebalancing_keeps_the_single_domain_result(field):
    """Re-balancing every M steps: clustered particles on EVEN
    slabs (badly balanced), re-balanced to the count-balanced bounds after 2
    steps: the run still equals the single-domain engine bit for bit, and
    the re-balanced slabs hold within 5 % of N / W particles."""
    world, n, n_c, steps = 4, 100_000, 256, 5
    rng = np.random.default_rng(31)
    centres = -0.5 + rng.random((8, 2))
    pos = centres[rng.integers(0, 8, n)] + 0.03 * rng.standard_normal((n, 2))
    pos = (np.mod(pos + 0.5, 1.0) - 0.5).astype(np.float32)
    sp = (np.arange(n) >= n // 2).astype(np.uint8)
    radii = (7e-4, 1.4e-3)
    c0 = (0.5 + 0.1 * rng.standard_normal(n_c * n_c)).astype(np.float32)
    if field:
        params, mp, dom = _field_params(n, radii, n_c)
    else:
        params, mp, dom = _params(n, radii)
    xi = torch.as_tensor(rng.standard_normal((steps, n, 2)).astype(np.float32), device="cuda")
    st1 = _field_state(pos, sp, c0, n_c) if field else _state(pos, sp)
    one = cs.DeviceSim(params, st1)
    one.step(xi, steps)
    one.export_state()
    e, c, cell = mp.pair_table()
    n1 = slabs.CellGeometry.make(dom.lo[1], dom.hi[1], cell).n
    bounds = slabs.SlabLayout.even(n1, world).bounds
    plan = slabs.FieldPlan.make(bounds, n1, n_c, world) if field else None
    shared = _state(pos, sp)
    sts = [_field_state(pos, sp, c0, n_c, shared) if field else shared for _ in range(world)]
    engines = [slabs.SlabEngine(params, sts[r], bounds, r, world, field_plan=plan)
               for r in range(world)]
    hub = slabs.LoopbackHub(world)
    for k in range(2):
        slabs.step_in_process(engines, hub, xi[k])
    new = slabs.rebalance_in_process(engines, hub, n_c)
    assert not np.array_equal(new, bounds)
    owned = [hi - lo for lo, hi in (eng.owned_range() for eng in engines)]
    assert sum(owned) == n and max(owned) <= 1.05 * n / world, owned
    for k in range(2, steps):
        slabs.step_in_process(engines, hub, xi[k])
    for eng in engines:
        assert eng.status().code == 0
        eng.export()
    torch.cuda.synchronize()
    assert torch.equal(shared["pos"], st1["pos"])
    if field:
        new_plan = slabs.FieldPlan.make(new, n1, n_c, world)
        for r in range(world):
            rows = slice(int(new_plan.g0[r]), int(new_plan.g0[r]) + new_plan.rp)
            assert torch.equal(sts[r]["c"].view(n_c, n_c)[rows], st1["c"].view(n_c, n_c)[rows])
