"""Oracle: self-consistent field of a 2D+2V problem (N3): periodic 2D Poisson solve and the
cell-averaged E = (E_x, E_y).  TEST INFRASTRUCTURE ONLY.

The paper states the fourth-order discretisation for one configuration dimension:
    30 phi_i - 16 (phi_{i+1} + phi_{i-1}) + (phi_{i+2} + phi_{i-2}) = 12 dx^2 rho_i      (P:292,
        reading #2),   E_i = -[8 (phi_{i+1} - phi_{i-1}) - phi_{i+2} + phi_{i-2}] / (12 dx)   (reading #1)
and generalises every operator of the method dimension by dimension (the fluxes;
P:864-876, the interpolation).  Reading #32 (2D field): the same dimension-by-dimension
generalisation -- the cell average of phi_xx + phi_yy is the sum of the 1D fourth-order operators
applied along x and along y to the 2D cell averages (each is fourth order on 2D averages because
the operator along x commutes with the average along y), so
    [30 phi - 16 (phi_{i+1,k} + phi_{i-1,k}) + (phi_{i+2,k} + phi_{i-2,k})] / dx^2
  + [30 phi - 16 (phi_{i,k+1} + phi_{i,k-1}) + (phi_{i,k+2} + phi_{i,k-2})] / dy^2 = 12 rho_{ik},
with the periodic null space handled as in 1D (rho projected to mean zero, phi of mean zero,
P:304-311), and E_x, E_y the 1D fourth-order gradient along each axis with E = -grad phi.

Like the 1D oracle (field.py), the singular periodic matrix is bordered with sum(phi) = 0 and
LU-factorised once per (nx, ny, dx, dy).
"""
from __future__ import annotations

import functools

import numpy as np
import scipy.linalg as sla

from . import field


def poisson_matrix_2d(nx, ny, dx, dy):
    """The 2D operator above (row-major unknowns phi[i, k] -> i * ny + k), scaled so that
    A phi = 12 rho."""
    Ax = field.poisson_matrix(nx) / (dx * dx)
    Ay = field.poisson_matrix(ny) / (dy * dy)
    return np.kron(Ax, np.eye(ny)) + np.kron(np.eye(nx), Ay)


@functools.lru_cache(maxsize=8)
def _bordered_lu_2d(nx, ny, dx, dy):
    n = nx * ny
    B = np.zeros((n + 1, n + 1))
    B[:n, :n] = poisson_matrix_2d(nx, ny, dx, dy)
    B[:n, n] = 1.0
    B[n, :n] = 1.0
    return sla.lu_factor(B)


def solve_potential_2d(rho, dx, dy):
    """Mean-zero phi of the periodic 2D system with the projected rho."""
    rho = np.asarray(rho, dtype=np.float64)
    nx, ny = rho.shape
    rhs = np.concatenate([12.0 * (rho - rho.mean()).ravel(), [0.0]])
    sol = sla.lu_solve(_bordered_lu_2d(nx, ny, float(dx), float(dy)), rhs)
    return sol[:nx * ny].reshape(nx, ny)


def efield_from_potential_2d(phi, dx, dy):
    """(E_x, E_y) = -(D4_x phi, D4_y phi), periodic; shape (2, nx, ny)."""
    def d4(a, axis, h):
        p = lambda s: np.roll(a, -s, axis=axis)   # noqa: E731   p(s)[i] = a[i+s]
        return (8.0 * (p(1) - p(-1)) - p(2) + p(-2)) / (12.0 * h)
    return np.stack([-d4(phi, 0, dx), -d4(phi, 1, dy)])


def efield_from_rho_2d(rho, dx, dy):
    return efield_from_potential_2d(solve_potential_2d(rho, dx, dy), dx, dy)
