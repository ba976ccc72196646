"""numpy's Generator(PCG64) restated on the device (csrc/rng.cu) against
numpy itself on this host: standard_normal and random draws bit for bit,
and the glibc-exact log1p of the ziggurat's tail against the host libm.
oracle/rng.py (the scalar restatement) is pinned against numpy on the CPU
in tests/test_oracle_golden.py."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1805_11007_b200 import _native as N  # noqa: E402


def _words(gens):
    w = np.empty((len(gens), 4), np.uint64)
    for s, g in enumerate(gens):
        st = g.bit_generator.state["state"]
        for q, v in enumerate((st["state"] >> 64, st["state"], st["inc"] >> 64, st["inc"])):
            w[s, q] = v & 0xFFFFFFFFFFFFFFFF
    return torch.as_tensor(w.view(np.int64), device="cuda")


@pytest.mark.parametrize("kind", [0, 1])
def test_device_draws_equal_numpy_bitwise(kind):
    S, k, m = 64, 6, 3001
    seeds = [np.random.SeedSequence(1000 + s).spawn(3)[1 + kind] for s in range(S)]
    dev = _words([np.random.default_rng(q) for q in seeds])
    out = torch.empty((k, S, m), dtype=torch.float64, device="cuda")
    lib = N.load_library()
    for rep in range(2):  # the device states advance like numpy's
        N.check(lib.cs_rng_fill(N.context(), N.ptr(dev), S, kind, k, m, N.ptr(out)), "rng")
        got = out.cpu().numpy()
        for s in range(0, S, 7):
            g = np.random.default_rng(seeds[s])
            if rep:
                g.standard_normal(k * m) if kind == 0 else g.random(k * m)
            ref = (g.standard_normal((k, m)) if kind == 0 else g.random((k, m)))
            assert np.array_equal(got[:, s].view(np.uint64), ref.view(np.uint64)), (rep, s)


def test_device_log1p_matches_host_libm_bitwise():
    rng = np.random.default_rng(4)
    x = np.concatenate([-rng.random(400000), -rng.random(100000) * 1e-3,
                        -(1.0 - rng.random(100000) * 1e-6), rng.random(100000),
                        -rng.random(50000) * 1e-9, [0.0, -0.0, -1.0, 1e-300, np.inf]])
    xt = torch.as_tensor(x, device="cuda")
    yt = torch.empty_like(xt)
    N.check(N.load_library().cs_log1p_batch(N.context(), N.ptr(xt), N.ptr(yt), x.size), "l1p")
    y = yt.cpu().numpy()
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    host = np.array([libm.log1p(float(v)) for v in x[::3]])
    assert np.array_equal(y[::3].view(np.uint64), host.view(np.uint64))
