"""Chemical field on a node-centred grid -- device implementation.

Mirror of chemosim/field.py (same names, conventions and checks).  Flat
index l = j * n_c + i (x fastest); neumann spacing L/(n_c-1) with nodes on
the walls, periodic spacing L/n_c.  The semi-implicit step

    (I - dt d_c L) c_new = c + dt (k_alpha rho_alpha - k_beta rho_beta c - gamma c)

runs in the library (csrc/field.cu): the explicit part and the checks are
elementwise kernels; the implicit solve is the reference's DCT-I modal solve
as fp64 GEMM kernels (neumann) or a 2-D real FFT diagonalisation of the same
circulant system (periodic; the reference's SuperLU path, field.py:197-198,
cannot factor the BASELINE 4096^2 / 8192^2 grids at all).
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _arrays as A
from . import _native as N


@dataclass(frozen=True, eq=False)
class Grid:
    n_c: int
    lo: np.ndarray
    hi: np.ndarray
    boundary: str  # "neumann" | "periodic"

    def __post_init__(self):
        if self.n_c < 3:
            raise ValueError("n_c must be at least 3")
        if self.boundary not in ("neumann", "periodic"):
            raise ValueError(f"unknown boundary closure {self.boundary!r}")

    @classmethod
    def square(cls, n_c: int, size: float, boundary: str) -> "Grid":
        half = float(size) / 2.0
        return cls(n_c=int(n_c), lo=np.array([-half, -half]), hi=np.array([half, half]),
                   boundary=boundary)

    @property
    def spacing(self) -> np.ndarray:
        div = self.n_c - 1 if self.boundary == "neumann" else self.n_c
        return (self.hi - self.lo) / div

    def axis_nodes(self, ax: int) -> np.ndarray:
        return self.lo[ax] + self.spacing[ax] * np.arange(self.n_c)

    def node_positions(self) -> np.ndarray:
        xs = self.axis_nodes(0)
        ys = self.axis_nodes(1)
        return np.column_stack([np.tile(xs, self.n_c), np.repeat(ys, self.n_c)])

    def quadrature_weights(self) -> np.ndarray:
        dx, dy = self.spacing
        if self.boundary == "periodic":
            return np.full(self.n_c * self.n_c, dx * dy)
        w1 = np.ones(self.n_c)
        w1[0] = w1[-1] = 0.5
        return (np.repeat(w1, self.n_c) * np.tile(w1, self.n_c)) * (dx * dy)


@dataclass
class FieldParams:
    d_c: float = 1.0
    k_alpha: float = 0.1
    k_beta: float = 0.03
    gamma: float = 0.0

    def __post_init__(self):
        for name in ("d_c", "k_alpha", "k_beta", "gamma"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")


@dataclass
class Field:
    c: object          # (n_c^2,) nodal concentration (numpy or CUDA tensor)
    grad: object       # (n_c^2, 2)
    rho_alpha: object  # (n_c^2,)
    rho_beta: object   # (n_c^2,)

    @classmethod
    def zeros(cls, grid: Grid) -> "Field":
        m = grid.n_c * grid.n_c
        return cls(c=np.zeros(m), grad=np.zeros((m, 2)), rho_alpha=np.zeros(m),
                   rho_beta=np.zeros(m))


def _lap_1d(n, h, periodic):
    import scipy.sparse as sp
    main = np.full(n, -2.0)
    off = np.ones(n - 1)
    m = sp.diags([off, main, off], [-1, 0, 1], format="lil")
    if periodic:
        m[0, n - 1] = 1.0
        m[n - 1, 0] = 1.0
    else:
        m[0, 1] = 2.0
        m[n - 1, n - 2] = 2.0
    return sp.csr_matrix(m / (h * h))


def _d1_1d(n, h, periodic):
    import scipy.sparse as sp
    off = np.ones(n - 1)
    m = sp.diags([-off, off], [-1, 1], format="lil")
    if periodic:
        m[0, n - 1] = -1.0
        m[n - 1, 0] = 1.0
    else:
        m[0, 0], m[0, 1], m[0, 2] = -3.0, 4.0, -1.0
        m[n - 1, n - 3], m[n - 1, n - 2], m[n - 1, n - 1] = 1.0, -4.0, 3.0
    return sp.csr_matrix(m / (2.0 * h))


class Operators:
    """Prepared implicit solver (device) for one grid, d_c and dt.

    ``solve`` runs on the device.  The sparse ``laplacian``/``d1x``/``d1y``/
    ``system`` matrices of the reference (field.py:152-156) are assembled
    lazily on the host for inspection only; the hot path never uses them.
    """

    def __init__(self, grid: Grid, params: FieldParams, dt: float, precision: str = "fp64"):
        if not dt > 0:
            raise ValueError("dt must be positive")
        self.grid = grid
        self.d_c = float(params.d_c)
        self.dt = float(dt)
        self.precision = precision
        self.weights = grid.quadrature_weights()
        self._handle = None
        self._dtype = None

    # ---- device solver ----------------------------------------------------
    def handle(self, dtype):
        if self._handle is None or self._dtype != dtype:
            self.close()
            h = N.C_p()
            N.check(N.load_library().cs_field_ops_create(
                N.context(), N.prec_code(dtype), ctypes.byref(N.grid_struct(self.grid)),
                self.d_c, self.dt, ctypes.byref(h)), "cs_field_ops_create")
            self._handle, self._dtype = h, dtype
        return self._handle

    def close(self):
        if self._handle is not None:
            try:
                N.load_library().cs_field_ops_destroy(self._handle)
            except Exception:  # pragma: no cover
                pass
            self._handle = None

    def __del__(self):  # pragma: no cover
        self.close()

    def solve(self, rhs):
        host = not A.on_device(rhs)
        dt_ = A.float_dtype_of(rhs)
        r = A.dev(rhs, dt_)
        out = A.empty(r.shape, dt_)
        N.check(N.load_library().cs_field_solve(self.handle(dt_), N.ptr(r), N.ptr(out)),
                "cs_field_solve")
        return A.back(out, host)

    # ---- host-side sparse views (lazy) --------------------------------------
    def _sparse(self):
        import scipy.sparse as sp
        if not hasattr(self, "_sp"):
            n = self.grid.n_c
            hx, hy = self.grid.spacing
            per = self.grid.boundary == "periodic"
            eye = sp.identity(n, format="csr")
            lap = sp.csr_matrix(sp.kron(eye, _lap_1d(n, hx, per)) + sp.kron(_lap_1d(n, hy, per), eye))
            self._sp = dict(
                laplacian=lap,
                d1x=sp.csr_matrix(sp.kron(eye, _d1_1d(n, hx, per))),
                d1y=sp.csr_matrix(sp.kron(_d1_1d(n, hy, per), eye)),
                system=sp.csc_matrix(sp.identity(n * n) - self.dt * self.d_c * lap))
        return self._sp

    @property
    def laplacian(self):
        return self._sparse()["laplacian"]

    @property
    def d1x(self):
        return self._sparse()["d1x"]

    @property
    def d1y(self):
        return self._sparse()["d1y"]

    @property
    def system(self):
        return self._sparse()["system"]


def build_operators(grid: Grid, params: FieldParams, dt: float) -> Operators:
    return Operators(grid, params, dt)


def discrete_mass(values, grid: Grid) -> float:
    return float(grid.quadrature_weights() @ A.to_numpy(values))


def step_field(field: Field, ops: Operators, params: FieldParams, dt: float) -> None:
    """Advance c by one semi-implicit step (field.py:209-239); rebinds
    field.c, raises FloatingPointError on a non-finite result and warns on a
    negative weighted mass below -1e-12."""
    if float(dt) != ops.dt:
        raise ValueError("step_field dt differs from the dt the operators were built with")
    host = not A.on_device(field.c)
    dt_ = A.float_dtype_of(field.c)
    c = A.dev(field.c, dt_).clone()
    ra = A.dev(field.rho_alpha, dt_)
    rb = A.dev(field.rho_beta, dt_)
    bad = ctypes.c_int32(0)
    neg = ctypes.c_double(0.0)
    N.check(N.load_library().cs_field_step(
        ops.handle(dt_), N.ptr(c), N.ptr(ra), N.ptr(rb), float(params.k_alpha),
        float(params.k_beta), float(params.gamma), ctypes.byref(bad), ctypes.byref(neg)),
        "cs_field_step")
    if bad.value:
        raise FloatingPointError("field update produced non-finite values")
    if neg.value < -1e-12:
        warnings.warn(f"concentration went negative (weighted mass {neg.value:.3e})",
                      stacklevel=2)
    field.c = A.back(c, host)


def gradient(field: Field, ops: Operators) -> None:
    """Refresh the nodal gradient from the current concentration
    (field.py:242-245), in place on field.grad."""
    host = not A.on_device(field.c)
    dt_ = A.float_dtype_of(field.c)
    c = A.dev(field.c, dt_)
    g = A.empty((c.shape[0], 2), dt_)
    N.check(N.load_library().cs_gradient(N.context(), N.prec_code(dt_), N.ptr(c),
                                         ctypes.byref(N.grid_struct(ops.grid)), N.ptr(g)),
            "cs_gradient")
    if host:
        field.grad[...] = g.cpu().numpy()
    elif A.is_tensor(field.grad) and field.grad.shape == g.shape:
        field.grad.copy_(g)
    else:
        field.grad = g
