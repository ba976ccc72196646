"""Realisation observables on the device (csrc/observe.cu) against numpy's
own arithmetic: msd = mean of (0 + dx^2) + dy^2 in numpy's pairwise
reduction order (engine.py:230-235), bit for bit for every size class of
the pairwise sum; histogram2d counts / normalisation bit for bit, including
values on bin edges, on the closed last edge and outside the range."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1805_11007_b200 import _native as N  # noqa: E402


def _msd(pos, anchor):
    p = torch.as_tensor(pos, device="cuda")
    a = torch.as_tensor(anchor, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    N.check(N.load_library().cs_msd(N.context(), N.prec_code(p.dtype), N.ptr(p), N.ptr(a),
                                    p.shape[0], N.ptr(out)), "cs_msd")
    return float(out.item())


@pytest.mark.parametrize("n", [1, 7, 8, 9, 127, 128, 129, 1000, 4097, 1_000_003])
def test_msd_bitwise_numpy(n):
    rng = np.random.default_rng(n)
    pos = rng.uniform(-0.5, 0.5, (n, 2))
    anchor = pos + rng.normal(0.0, 0.01, (n, 2))
    d = pos - anchor
    assert _msd(pos, anchor) == float((d * d).sum(axis=1).mean())
    p32, a32 = pos.astype(np.float32), anchor.astype(np.float32)
    d = p32.astype(np.float64) - a32.astype(np.float64)
    assert _msd(p32, a32) == float((d * d).sum(axis=1).mean())


def test_hist2d_matches_numpy():
    rng = np.random.default_rng(4)
    b = 26
    edges = np.linspace(-0.5, 0.5, b + 1)
    pos = rng.uniform(-0.5, 0.5, (200_000, 2))
    pos[:b + 1, 0] = edges       # on every edge, including the closed last one
    pos[b + 1:2 * b + 2, 1] = edges
    pos[-3] = [0.5, 0.5]
    pos[-2] = [0.7, 0.1]         # outliers
    pos[-1] = [-0.2, -0.9]
    sp = (rng.random(len(pos)) < 0.4).astype(np.uint8)
    pt = torch.as_tensor(pos, device="cuda")
    st = torch.as_tensor(sp, device="cuda")
    ex = torch.as_tensor(edges, device="cuda")
    cnt = torch.empty((b, b), dtype=torch.int64, device="cuda")
    for s in (0, 1, -1):
        N.check(N.load_library().cs_hist2d(N.context(), N.prec_code(pt.dtype), N.ptr(pt),
                                           N.ptr(st), len(pos), s, N.ptr(ex), N.ptr(ex), b, 0,
                                           N.ptr(cnt)), "cs_hist2d")
        p = pos if s < 0 else pos[sp == s]
        h, _, _ = np.histogram2d(p[:, 0], p[:, 1], bins=b, range=[[-0.5, 0.5], [-0.5, 0.5]])
        assert np.array_equal(cnt.cpu().numpy(), h.T.astype(np.int64)), s
        assert np.array_equal(cnt.cpu().numpy().astype(np.float64) / p.shape[0],
                              h.T / p.shape[0])
