"""Implicit field solve of the oracle -- TEST INFRASTRUCTURE ONLY.

Restates field.py:173-201 (build_operators) and field.py:162-170
(Operators.solve) of the reference with the same numpy/scipy calls:

* neumann: the DCT-I modal solve, ``modal = eig_inv * (F @ X @ F.T)`` and
  ``out = Finv @ modal @ Finv.T`` with F = scipy.fft.dct(eye, type=1, axis=0)
  (bitwise the reference's arithmetic when numpy links the same BLAS);
* periodic: scipy's SuperLU factorisation of ``I - dt d_c L`` for grids up to
  ``splu_max`` nodes per axis (the reference path), and above that a 2-D
  FFT diagonalisation of the same circulant system (the reference cannot
  factor 4096^2 / 8192^2 grids at all); both solve the identical
  linear system, so they agree to ~1e-13.
"""

from __future__ import annotations

import numpy as np
import scipy.fft
import scipy.sparse as sp
from scipy.sparse.linalg import splu


def _lap_1d(n: int, h: float, periodic: bool):
    # field.py:114-125
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


class OracleOperators:
    def __init__(self, n, spacing, periodic, d_c, dt, splu_max=256):
        self.n = n
        self.periodic = periodic
        hx, hy = float(spacing[0]), float(spacing[1])
        self.kind = "identity"
        if not dt > 0:
            raise ValueError("dt must be positive")
        if d_c * dt == 0.0:
            return
        if not periodic:
            self.kind = "dct"
            self.fwd = scipy.fft.dct(np.eye(n), type=1, axis=0)
            self.inv = scipy.fft.idct(np.eye(n), type=1, axis=0)
            lam_x = (2.0 * np.cos(np.pi * np.arange(n) / (n - 1)) - 2.0) / hx ** 2
            lam_y = (2.0 * np.cos(np.pi * np.arange(n) / (n - 1)) - 2.0) / hy ** 2
            self.eig_inv = 1.0 / (1.0 - dt * d_c
                                  * (lam_y[:, None] + lam_x[None, :]))
        elif n <= splu_max:
            self.kind = "splu"
            eye = sp.identity(n, format="csr")
            lap = sp.kron(eye, _lap_1d(n, hx, True)) + sp.kron(_lap_1d(n, hy, True), eye)
            system = sp.csc_matrix(sp.identity(n * n) - dt * d_c * sp.csr_matrix(lap))
            self.lu = splu(system)
        else:
            self.kind = "fft"
            k = np.arange(n)
            lam_x = (2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / hx ** 2
            lam_y = (2.0 * np.cos(2.0 * np.pi * k / n) - 2.0) / hy ** 2
            self.eig_inv = 1.0 / (1.0 - dt * d_c
                                  * (lam_y[:, None] + lam_x[None, :]))

    def solve(self, rhs):
        n = self.n
        if self.kind == "dct":
            x = rhs.reshape(n, n)
            modal = self.eig_inv * (self.fwd @ x @ self.fwd.T)
            return (self.inv @ modal @ self.inv.T).ravel()
        if self.kind == "splu":
            return self.lu.solve(rhs)
        if self.kind == "fft":
            x = rhs.reshape(n, n)
            return np.fft.ifft2(np.fft.fft2(x) * self.eig_inv).real.ravel()
        return rhs.copy()


def build_operators(n, spacing, periodic, d_c, dt, splu_max=256):
    return OracleOperators(n, spacing, periodic, d_c, dt, splu_max)


def quadrature_weights(n, spacing, periodic):
    # field.py:68-80
    dx, dy = float(spacing[0]), float(spacing[1])
    if periodic:
        return np.full(n * n, dx * dy)
    w1 = np.ones(n)
    w1[0] = w1[-1] = 0.5
    return (np.repeat(w1, n) * np.tile(w1, n)) * (dx * dy)
