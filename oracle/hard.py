"""The hard-sphere sweep restated -- TEST INFRASTRUCTURE ONLY.

chemosim/motion.py:301-352 (resolve_hard_sphere): the pairs (i < j) whose
minimum-image squared distance ((-0 + dx^2) + dy^2, numpy's row sum) is below
eps^2 at the start, processed in ascending (i, j) order against the live
buffer: d = sqrt(dx . dx) (numpy evaluates the 2-vector dot through BLAS
ddot, fma(dy, dy, dx dx) on an FMA host -- math.fma is not in Python 3.12,
so the dot is taken with numpy as the reference does), skip if d >= eps,
else push apart by 2 (eps - d) split by the diffusivities.  Pinned against
the reference by tests/test_oracle_golden.py (tests/golden/hard.npz).
"""

from __future__ import annotations

import math

import numpy as np

_GOLDEN = 0.6180339887498949


def _wrap(d, size, periodic):
    d = np.array(d, dtype=float, copy=True)
    for ax in range(2):
        if periodic[ax]:
            d[..., ax] -= size[ax] * np.round(d[..., ax] / size[ax])
    return d


def resolve_hard_sphere(prop, species, size, periodic, eps, d_alpha, d_beta):
    prop = np.array(prop, dtype=float, copy=True)
    n = prop.shape[0]
    size = np.asarray(size, dtype=float)
    delta = _wrap(prop[None, :, :] - prop[:, None, :], size, periodic)
    d2 = (delta * delta).sum(axis=2)
    iu, ju = np.triu_indices(n, k=1)
    hit = d2[iu, ju] < eps * eps
    dcoef = np.where(np.asarray(species) == 0, d_alpha, d_beta)
    for i, j in zip(iu[hit], ju[hit]):
        dx = _wrap(prop[j] - prop[i], size, periodic)
        d = math.sqrt(float(dx @ dx))
        if d >= eps:
            continue
        if d == 0.0:
            th = 2.0 * math.pi * ((_GOLDEN * (i + 1) + _GOLDEN * _GOLDEN * (j + 1)) % 1.0)
            u = np.array([math.cos(th), math.sin(th)])
        else:
            u = dx / d
        d_p = eps - d
        total = dcoef[i] + dcoef[j]
        share_i = 0.5 if total == 0.0 else dcoef[i] / total
        prop[i] -= u * (2.0 * d_p * share_i)
        prop[j] += u * (2.0 * d_p * (1.0 - share_i))
    return prop
