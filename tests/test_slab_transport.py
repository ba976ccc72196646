"""The multi-rank pieces of the device slab engine on CPU, over
gloo at world sizes 2 and 3 (the GPU tests emulate the ranks in one process,
tests/test_gpu_slab_engine.py):

* NcclTransport.exchange routes every outbox record (16 bytes, destination
  rank | kind << 30) to its destination, exactly once;
* PackedNcclTransport.exchange_packed moves the per-destination segments and
  their counts with equal-split all-to-alls (no host round trip);
* NcclField's static all-to-all moves the deposit-window rows, the spectrum
  blocks and the c rows with the sizes the FieldPlan row lists give both
  sides, without a count exchange;
* the layout / plan bookkeeping (count-balanced rows, windows, row lists)."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_1805_11007_b200 import slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _records_worker(rank, world, port, outdir):
    dist = _init(rank, world, port)
    try:
        rng = np.random.default_rng(rank)
        m = 50 + 17 * rank
        ids = np.arange(m, dtype=np.int32) + 1000 * rank
        recs = np.zeros((m, 4), np.int32)
        recs[:, 0] = ids
        recs[:, 1] = rank
        dest = rng.integers(0, world, m).astype(np.int32)
        kind = rng.integers(0, 2, m).astype(np.int32)
        recs[:, 2] = dest
        t = slabs.NcclTransport(world)
        got = t.exchange(torch.from_numpy(recs), torch.from_numpy(dest | (kind << 30)))
        np.save(os.path.join(outdir, f"r{rank}.npy"), got.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_transport_routes_every_record_once(world, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_records_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world)
    seen = []
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"r{r}.npy"))
        assert np.all(got[:, 2] == r)  # every record at its destination
        seen.append(got[:, 0])
    seen = np.sort(np.concatenate(seen))
    expect = np.sort(np.concatenate([np.arange(50 + 17 * r) + 1000 * r for r in range(world)]))
    assert np.array_equal(seen, expect)  # exactly once


def _packed_worker(rank, world, port, outdir):
    dist = _init(rank, world, port)
    try:
        seg = 16
        out = torch.zeros((world, seg, 4), dtype=torch.int32)
        counts = torch.zeros(world, dtype=torch.int32)
        for d in range(world):
            c = 3 + rank + 2 * d  # records rank -> d
            counts[d] = c
            out[d, :c, 0] = torch.arange(c, dtype=torch.int32)
            out[d, :c, 1] = rank
            out[d, :c, 2] = d
        t = slabs.PackedNcclTransport(world)
        t.seg = seg
        inbox, in_counts = t.exchange_packed(out, counts)
        np.savez(os.path.join(outdir, f"p{rank}.npz"), inbox=inbox.numpy(),
                 counts=in_counts.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_packed_transport_moves_segments_and_counts(world, tmp_path):
    """PackedNcclTransport.exchange_packed: segment s of a rank's inbox is
    what rank s put into its segment for that rank, with its count -- two
    equal-split all-to-alls, no sizes read on the host."""
    import torch.multiprocessing as mp
    mp.spawn(_packed_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world)
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"p{r}.npz"))
        for s_ in range(world):
            c = 3 + s_ + 2 * r
            assert got["counts"][s_] == c
            seg = got["inbox"][s_]
            assert np.array_equal(seg[:c, 0], np.arange(c))
            assert np.all(seg[:c, 1] == s_) and np.all(seg[:c, 2] == r)
            assert np.all(seg[c:] == 0)


class _FakeEngine:
    def __init__(self, rank):
        self.rank = rank


class _FakeField:
    """The payload side of SlabField on CPU arrays: rho (2, n, n) int32,
    c (n, n), spec (nh, rp, 2) and blocks (world, kl, rp, 2) float32 filled
    with values that encode (array, rank, row, column)."""

    def __init__(self, plan, rank):
        self.plan, self.eng = plan, _FakeEngine(rank)
        n, W = plan.n, plan.world
        nh = n // 2 + 1
        kl = int(plan.kx[rank + 1] - plan.kx[rank])
        self.rho = torch.zeros((2, n, n), dtype=torch.int32)
        j0, k = plan.dep[rank]
        for j in np.arange(j0, j0 + k) % n:
            self.rho[:, j, :] = 1 + rank
        self.c = torch.full((n, n), -1.0)
        g0 = int(plan.g0[rank])
        for j in range(g0, g0 + plan.rp):
            self.c[j] = float(j)
        self.spec = torch.arange(nh * plan.rp * 2, dtype=torch.float32).view(nh, plan.rp, 2) \
            + 1e6 * rank
        self.blocks = torch.zeros((W, kl, plan.rp, 2))
        self.dep_send = [torch.as_tensor(plan.dep_rows(rank, d)) if d != rank
                         else torch.zeros(0, dtype=torch.long) for d in range(W)]
        self.dep_recv = [torch.as_tensor(plan.dep_rows(s, rank)) if s != rank
                         else torch.zeros(0, dtype=torch.long) for s in range(W)]
        self.c_send = [torch.as_tensor(plan.c_rows(d, rank)) if d != rank
                       else torch.zeros(0, dtype=torch.long) for d in range(W)]
        self.c_recv = [torch.as_tensor(plan.c_rows(rank, s)) if s != rank
                       else torch.zeros(0, dtype=torch.long) for s in range(W)]
        self.calls = []

    deposit_out = slabs.SlabField.deposit_out
    deposit_in = slabs.SlabField.deposit_in
    spec_out = slabs.SlabField.spec_out
    spec_in_blocks = slabs.SlabField.spec_in_blocks
    blocks_out = slabs.SlabField.blocks_out
    blocks_in_spec = slabs.SlabField.blocks_in_spec
    c_out = slabs.SlabField.c_out
    c_in = slabs.SlabField.c_in

    def spec_rows(self, inverse):
        self.calls.append(("rows", inverse))

    def cols(self):
        self.calls.append(("cols",))

    def gradient(self):
        self.calls.append(("grad",))


def _field_worker(rank, world, port, outdir, bounds, n1, n):
    dist = _init(rank, world, port)
    try:
        plan = slabs.FieldPlan.make(np.asarray(bounds), n1, n, world)
        f = _FakeField(plan, rank)
        spec0 = f.spec.clone()
        slabs.NcclField(f).step()
        np.savez(os.path.join(outdir, f"f{rank}.npz"), rho=f.rho.numpy(), c=f.c.numpy(),
                 spec=f.spec.numpy(), spec0=spec0.numpy(), blocks=f.blocks.numpy())
        assert f.calls == [("rows", False), ("cols",), ("rows", True), ("grad",)]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_field_exchanges_with_static_sizes(world, tmp_path):
    import torch.multiprocessing as mp
    n, n1 = 32, 50
    counts = np.random.default_rng(world).integers(0, 100, n1)
    bounds = slabs.SlabLayout.balanced(counts, world).bounds
    mp.spawn(_field_worker, args=(world, _free_port(), str(tmp_path), list(bounds), n1, n),
             nprocs=world)
    plan = slabs.FieldPlan.make(bounds, n1, n, world)
    res = [dict(np.load(os.path.join(tmp_path, f"f{r}.npz"))) for r in range(world)]
    for r in range(world):
        g0 = int(plan.g0[r])
        # own deposit rows = own contribution (if in the own window) + every window covering them
        for j in range(g0, g0 + plan.rp):
            expect = sum(1 + s for s in range(world)
                         if j in set(np.arange(plan.dep[s][0], plan.dep[s][0] + plan.dep[s][1])
                                     % n))
            assert np.all(res[r]["rho"][:, j, :] == expect), (r, j)
        # c rows of the gradient window (one wider) hold their owners' values
        j0, k = plan.grad[r]
        for j in np.unique(np.arange(j0 - 1, j0 + k + 1) % n):
            assert np.all(res[r]["c"][j] == float(j)), (r, j)
        # spectrum: the columns went out and came back unchanged (cols is mocked)
        assert np.array_equal(res[r]["spec"], res[r]["spec0"])
        # blocks: block q of rank r = rank q's rows of rank r's kx columns
        kx0, kx1 = int(plan.kx[r]), int(plan.kx[r + 1])
        for q in range(world):
            assert np.array_equal(res[r]["blocks"][q], res[q]["spec0"][kx0:kx1])


def test_layout_and_plan_bookkeeping():
    counts = np.array([0, 0, 10, 50, 50, 10, 0, 0, 0, 0])
    lay = slabs.SlabLayout.balanced(counts, 2)
    assert lay.bounds[0] == 0 and lay.bounds[-1] == 10
    assert abs(counts[: lay.bounds[1]].sum() - 60) <= 50
    plan = slabs.FieldPlan.make(np.array([0, 100, 250, 330, 400]), 400, 256, 4)
    assert plan.rp == 64 and list(plan.g0) == [0, 64, 128, 192]
    for r in range(4):  # deposit windows include the own rows
        j0, k = plan.dep[r]
        own = set(range(int(plan.g0[r]), int(plan.g0[r]) + plan.rp))
        assert own <= set(np.arange(j0, j0 + k) % 256)
    assert list(plan.dep_rows(0, 1)) == [64, 65] and list(plan.dep_rows(0, 3)) == [255]
    with pytest.raises(ValueError):
        slabs.FieldPlan.make(np.array([0, 1, 2, 3]), 3, 100, 3)
