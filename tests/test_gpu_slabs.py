"""The slab runner with the device backend (C-ABI ops) over NCCL on one
B200 (world size 1: every exchange is a self-exchange), against the
single-domain direct engine.  Multi-rank correctness is covered on CPU by
tests/test_slabs.py (gloo, world sizes 2-3)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_1805_11007_b200 as cs  # noqa: E402
from paper_1805_11007_b200 import slabs  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_device_slab_runner_matches_direct_engine(nccl_world1):
    import warnings
    n, steps = 20000, 4
    rng = np.random.default_rng(3)
    pos = -0.5 + rng.random((n, 2))
    types = (np.arange(n) >= n // 2).astype(np.uint8)
    xi = rng.standard_normal((steps, n, 2))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mp = cs.MotionParams(d_alpha=1.0, d_beta=0.5, epsilon=0.002, cutoff=0.004, dt=1e-5,
                             radius_alpha=0.002, radius_beta=0.004)
    dom = cs.Domain.square(1.0, periodic=True)
    eps, cut, cell = mp.pair_table()
    geom = slabs.CellGeometry.make(-0.5, 0.5, cell)
    layout = slabs.SlabLayout.even(geom.n, 1)
    st = slabs.scatter_initial(np.arange(n), pos, types, layout, geom, 0, "cuda",
                               torch.float64)
    be = slabs.DeviceSlabBackend(dom, mp, dt=1e-5, chi=(1.0, -0.5), chi_pinned=(False, False))
    runner = slabs.SlabRunner(be, layout, geom, 0, 1, True)
    for s in range(steps):
        xi_own = torch.as_tensor(xi[s], device="cuda")[st.ids]
        st, _, key = runner.step(st, xi_own)
        assert key == (1 << 62)
    # single-domain direct engine, field off
    state = dict(pos=torch.as_tensor(pos, device="cuda"), next_pos=None,
                 anchor=torch.as_tensor(pos, device="cuda"),
                 species=torch.as_tensor(types, device="cuda"),
                 drift=torch.zeros((n, 2), dtype=torch.float64, device="cuda"), local_c=None,
                 c=None, grad=None, rho_a=None, rho_b=None)
    params = cs.sim_params_struct(n=n, prec=0, domain=dom, motion=mp, dt=1e-5,
                                  field_active=False, refresh_active=False, grid=None,
                                  fparams=None, kernel=None, secretes=(1, 0), consumes=(0, 1),
                                  chi=(1.0, -0.5), chi_pinned=(0, 0), store_samples=False,
                                  store_next=False, engine="direct")
    sim = cs.DeviceSim(params, state)
    sim.step(torch.as_tensor(xi, device="cuda"), steps)
    assert sim.status().code == 0
    o = torch.argsort(st.ids)
    assert torch.equal(st.pos[o], state["pos"])
    assert torch.equal(st.anchor[o], state["anchor"])
