"""CPU parity oracle for the chemosim hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  The
product package ``paper_1805_11007_b200`` never imports it, and its CUDA path
fails loudly instead of falling back here.

The particle/grid kernels are a C restatement (chemo_oracle.c, built by
oracle/Makefile into oracle/_build/); the implicit field solve is restated in
oracle/field.py on numpy/scipy exactly as the reference calls them
(field.py:162-201).  Parity with the reference is pinned by
tests/test_oracle_golden.py against fixtures generated from the reference
itself by tests/golden/make_golden.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libchemo_oracle.so")
_lib = None


def build() -> str:
    """Compile the C oracle (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, I64, I32, D, U8 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_double, ctypes.c_void_p)
        L.or_soft_forces.argtypes = [P, U8, I64, D, D, D, D, I32, I32, P, P, D,
                                     P, P, I64, P, I32]
        L.or_soft_forces.restype = I32
        L.or_bin_cells.argtypes = [P, I64, D, D, D, D, D, P, P, P, I64, P]
        L.or_bin_cells.restype = I32
        L.or_em_step.argtypes = [P, P, P, P, P, D, I64, P, I32]
        L.or_em_step.restype = None
        L.or_boundaries.argtypes = [P, P, I64, D, D, D, D, I32, I32, P, P]
        L.or_boundaries.restype = I32
        L.or_cic_scatter.argtypes = [P, U8, I64, I32, D, D, D, D, I32, P]
        L.or_cic_scatter.restype = I32
        L.or_gauss_scatter.argtypes = [P, U8, I64, I32, D, D, D, D, I32, D, D,
                                       P, P]
        L.or_gauss_scatter.restype = None
        L.or_bilinear.argtypes = [P, I64, P, I32, D, D, D, D, I32, I32, P]
        L.or_bilinear.restype = I64
        L.or_gradient.argtypes = [P, I32, D, D, I32, P]
        L.or_gradient.restype = None
        L.or_field_rhs.argtypes = [P, P, P, I64, D, D, D, D, P]
        L.or_field_rhs.restype = None
        L.or_exp.argtypes = [D]
        L.or_exp.restype = D
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _u8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint8)


# --------------------------------------------------------------------------
# pair tables
# --------------------------------------------------------------------------

def pair_table(epsilon=None, cutoff=None, radii=None, cutoff_factor=2.0):
    """(eps_tab[4], cut_tab[4], cell_cutoff) for the force kernels.

    Homogeneous (reference, motion.py:165): every entry is (epsilon, cutoff).
    Per-type radii (BASELINE configs 2-4): eps_ij = (r_i + r_j) / 2 and
    cut_ij = cutoff_factor * eps_ij; with cutoff_factor = 2 this is
    r_i + r_j, and with r_A == r_B == epsilon it reduces bitwise to the
    homogeneous table (2 * ((e + e) / 2) == e + e == 2.0 * e).
    """
    if radii is None:
        eps = np.full(4, float(epsilon))
        cut = np.full(4, float(cutoff))
    else:
        r = [float(radii[0]), float(radii[1])]
        eps = np.array([(r[a] + r[b]) / 2.0 for a in range(2) for b in range(2)])
        cut = np.array([cutoff_factor * e for e in eps])
    return eps, cut, float(cut.max())


# --------------------------------------------------------------------------
# particle kernels
# --------------------------------------------------------------------------

def soft_forces(pos, lo, size, periodic, eps_tab, cut_tab, cell_cutoff,
                types=None, nthreads=1):
    pos = _f64(pos, (-1, 2))
    n = pos.shape[0]
    out = np.empty((n, 2))
    t = _u8(types)
    rc = lib().or_soft_forces(_p(pos), _p(t), n, float(lo[0]), float(lo[1]),
                              float(size[0]), float(size[1]), int(periodic[0]),
                              int(periodic[1]), _p(_f64(eps_tab)),
                              _p(_f64(cut_tab)), float(cell_cutoff), _p(out),
                              None, 0, None, int(nthreads))
    if rc:
        raise MemoryError("oracle soft_forces failed")
    return out


def soft_force_pairs(pos, lo, size, periodic, eps_tab, cut_tab, cell_cutoff,
                     types=None):
    """(forces, pairs) where pairs is (P, 2) int64 (i, j) in accumulation
    order: the exact pair set of the reference kernel arithmetic."""
    pos = _f64(pos, (-1, 2))
    n = pos.shape[0]
    out = np.empty((n, 2))
    t = _u8(types)
    cap = max(16, 64 * n)
    while True:
        pairs = np.empty((cap, 2), dtype=np.int64)
        cnt = ctypes.c_int64(0)
        rc = lib().or_soft_forces(_p(pos), _p(t), n, float(lo[0]), float(lo[1]),
                                  float(size[0]), float(size[1]),
                                  int(periodic[0]), int(periodic[1]),
                                  _p(_f64(eps_tab)), _p(_f64(cut_tab)),
                                  float(cell_cutoff), _p(out), _p(pairs), cap,
                                  ctypes.byref(cnt), 1)
        if rc:
            raise MemoryError("oracle soft_forces failed")
        if cnt.value <= cap:
            return out, pairs[:cnt.value].copy()
        cap = cnt.value


def bin_cells(pos, lo, size, cell_cutoff):
    """(n0, n1, starts, order) of the reference binning (motion.py:170-199)."""
    pos = _f64(pos, (-1, 2))
    n = pos.shape[0]
    n0 = ctypes.c_int64()
    n1 = ctypes.c_int64()
    lib().or_bin_cells(_p(pos), n, float(lo[0]), float(lo[1]), float(size[0]),
                       float(size[1]), float(cell_cutoff), ctypes.byref(n0),
                       ctypes.byref(n1), None, 0, None)
    starts = np.empty(n0.value * n1.value + 1, dtype=np.int64)
    order = np.empty(n, dtype=np.int64)
    lib().or_bin_cells(_p(pos), n, float(lo[0]), float(lo[1]), float(size[0]),
                       float(size[1]), float(cell_cutoff), ctypes.byref(n0),
                       ctypes.byref(n1), _p(starts), starts.size, _p(order))
    return n0.value, n1.value, starts, order


def em_step(pos, diffusion, drift, force, xi, dt, nthreads=1):
    pos = _f64(pos, (-1, 2))
    n = pos.shape[0]
    d = _f64(np.broadcast_to(np.asarray(diffusion, dtype=float), (n,)))
    dr = _f64(np.broadcast_to(np.asarray(drift, dtype=float), (n, 2)))
    fo = _f64(np.broadcast_to(np.asarray(force, dtype=float), (n, 2)))
    x = _f64(xi, (n, 2))
    out = np.empty((n, 2))
    lib().or_em_step(_p(pos), _p(d), _p(dr), _p(fo), _p(x), float(dt), n,
                     _p(out), int(nthreads))
    return out


def apply_boundaries(x, anchor, lo, hi, periodic):
    """In place on x/anchor (float64 C-contiguous); returns (status, i, ax)."""
    assert x.dtype == np.float64 and x.flags.c_contiguous
    assert anchor.dtype == np.float64 and anchor.flags.c_contiguous
    bi = ctypes.c_int64()
    ba = ctypes.c_int32()
    st = lib().or_boundaries(_p(x), _p(anchor), x.shape[0], float(lo[0]),
                             float(lo[1]), float(hi[0]), float(hi[1]),
                             int(periodic[0]), int(periodic[1]),
                             ctypes.byref(bi), ctypes.byref(ba))
    return st, bi.value, ba.value


# --------------------------------------------------------------------------
# grid coupling
# --------------------------------------------------------------------------

def cic_deposit(pos, mask, nc, lo, spacing, periodic):
    pos = _f64(pos, (-1, 2))
    out = np.empty(nc * nc)
    lib().or_cic_scatter(_p(pos), _p(_u8(mask)), pos.shape[0], int(nc),
                         float(lo[0]), float(lo[1]), float(spacing[0]),
                         float(spacing[1]), int(periodic), _p(out))
    return out


def gauss_deposit(pos, route, nc, lo, spacing, periodic, h, cutoff):
    """route[p] = 0 -> rho_a, 1 -> rho_b, other -> skipped."""
    pos = _f64(pos, (-1, 2))
    a = np.zeros(nc * nc)
    b = np.zeros(nc * nc)
    lib().or_gauss_scatter(_p(pos), _p(_u8(route)), pos.shape[0], int(nc),
                           float(lo[0]), float(lo[1]), float(spacing[0]),
                           float(spacing[1]), int(periodic), float(h),
                           float(cutoff), _p(a), _p(b))
    return a, b


def bilinear(points, values, nc, lo, spacing, periodic):
    pts = _f64(points, (-1, 2))
    vals = np.asarray(values, dtype=float)
    squeeze = vals.ndim == 1
    vals = _f64(vals.reshape(nc * nc, -1))
    m = vals.shape[1]
    out = np.empty((pts.shape[0], m))
    clamped = lib().or_bilinear(_p(pts), pts.shape[0], _p(vals), m,
                                float(lo[0]), float(lo[1]), float(spacing[0]),
                                float(spacing[1]), int(nc), int(periodic),
                                _p(out))
    return (out[:, 0] if squeeze else out), int(clamped)


def gradient(c, nc, spacing, periodic):
    c = _f64(c)
    g = np.empty((nc * nc, 2))
    lib().or_gradient(_p(c), int(nc), float(spacing[0]), float(spacing[1]),
                      int(periodic), _p(g))
    return g


def field_rhs(c, rho_a, rho_b, dt, k_alpha, k_beta, gamma):
    c = _f64(c)
    out = np.empty_like(c)
    lib().or_field_rhs(_p(c), _p(_f64(rho_a)), _p(_f64(rho_b)), c.size,
                       float(dt), float(k_alpha), float(k_beta), float(gamma),
                       _p(out))
    return out


def host_exp(x: float) -> float:
    return lib().or_exp(float(x))


from .field import OracleOperators, build_operators  # noqa: E402
from .sim import OracleSim  # noqa: E402
